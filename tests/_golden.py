"""Golden-fixture loading and operator-tree deserialization for the tests.

Fixtures come from tests/golden/make_golden.py (run against the real
reference in the build container).  ``build_tree`` rebuilds an operator
expression with whichever constructor namespace it is given: the plain
CPU classes in tests/_exprs.py (oracle tests) or the product package's
``linop`` expression classes (GPU parity tests).
"""

from __future__ import annotations

import glob
import json
import os

import numpy as np
import scipy.sparse

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name: str):
    path = os.path.join(GOLDEN_DIR, name + ".npz")
    data = np.load(path, allow_pickle=False)
    meta = json.loads(str(data["meta"]))
    return data, meta


def scs_case_names() -> list[str]:
    names = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "scs_*.npz")))
    return names


def build_tree(t: dict, arrays, ns):
    """Rebuild an expression using classes from namespace ``ns``."""
    k = t["k"]
    if k == "DenseMatrix":
        return ns.DenseMatrix(np.array(arrays[t["values"]]))
    if k == "SparseMatrix":
        mat = scipy.sparse.csc_matrix(
            (arrays[t["data"]], arrays[t["indices"]], arrays[t["indptr"]]),
            shape=(t["m"], t["n"]))
        return ns.SparseMatrix(mat)
    if k == "Conv1D":
        return ns.Conv1D(np.array(arrays[t["kernel"]]), t["n"])
    if k == "Conv2D":
        return ns.Conv2D(np.array(arrays[t["kernel"]]), tuple(t["image_shape"]))
    if k == "Identity":
        return ns.Identity(t["n"])
    if k == "ZeroOp":
        return ns.ZeroOp(t["m"], t["n"])
    if k == "Scale":
        return ns.Scale(t["alpha"], build_tree(t["child"], arrays, ns))
    if k == "Sum":
        return ns.Sum(build_tree(t["left"], arrays, ns), build_tree(t["right"], arrays, ns))
    if k == "Compose":
        return ns.Compose(build_tree(t["left"], arrays, ns), build_tree(t["right"], arrays, ns))
    if k == "VStack":
        return ns.VStack([build_tree(c, arrays, ns) for c in t["children"]])
    if k == "AdjointOf":
        return ns.AdjointOf(build_tree(t["child"], arrays, ns))
    raise TypeError(k)


def build_cones(spec, ns):
    out = []
    for kind, dim in spec:
        out.append(getattr(ns, kind)(int(dim)))
    return out
