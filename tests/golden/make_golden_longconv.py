"""Golden vectors for LONG 1-d kernels, from the REAL reference (conegraph).

The reference's own deconvolution family uses kernel length n
(canon.py:166-179) and evaluates convolutions by FFT above 512 taps
(linop.py:35-50); the device splits such kernels into tiled tap blocks
(paper_1609_03488_b200/_plan.py, _emit_split_conv).  This script writes

  * long_conv_cases.npz -- Conv1D forward / adjoint applies of the
    reference (direct below 512 taps, FFT above) for kernel lengths 300 ..
    10001, Gaussian (the family's) and random kernels;
  * scs_deconv_300_0.npz -- the reference's solve of its own deconvolution
    problem with n = 300 (kernel length 300 > the tiled path's 240 taps),
    in the format of make_golden.gen_scs, so every golden SCS test picks it
    up.

Run in the build container:  python tests/golden/make_golden_longconv.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as G  # noqa: E402  (puts the reference on sys.path)
from conegraph import canon, linop  # noqa: E402
from conegraph.scs import ScsSettings  # noqa: E402


def gen_long_linop():
    arrays: dict = {}
    cases = []
    rng = np.random.default_rng(11)
    for n, k, kind in [(300, 300, "gauss"), (800, 600, "gauss"), (1000, 777, "random"),
                       (3000, 2001, "gauss"), (10001, 10001, "gauss")]:
        kern = canon.gaussian_kernel(k) if kind == "gauss" else rng.standard_normal(k)
        op = linop.conv1d(kern, n)
        x = rng.standard_normal(n)
        y = rng.standard_normal(op.rows)
        i = len(cases)
        t = G.ser(op.expr, arrays)
        keys = {}
        for nm, val in (("x", x), ("y", y), ("ax", op.forward(x)), ("aty", op.adjoint_apply(y))):
            keys[nm] = f"{nm}{i}"
            arrays[keys[nm]] = val
        cases.append({"tree": t, "rows": op.rows, "cols": op.cols, "n": n, "k": k, "kind": kind,
                      **keys})
    G.save("long_conv_cases", arrays, {"cases": cases})
    print(f"long_conv_cases: {len(cases)}")


def gen_long_deconv():
    n, seed = 300, 0
    c, b, _ = canon.gen_spike_data(n, seed)
    prob = canon.build_deconv(canon.DeconvProblem(c, b))
    cases = [(f"deconv_{n}_{seed}", prob, ScsSettings(eps=1e-3, max_iters=20000),
              {"n": n, "seed": seed, "kind": "deconv"})]
    orig = G.scs_cases
    G.scs_cases = lambda: cases
    try:
        G.gen_scs()
    finally:
        G.scs_cases = orig


if __name__ == "__main__":
    gen_long_linop()
    gen_long_deconv()
