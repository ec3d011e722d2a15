"""Rounding-sensitivity envelopes of the REAL reference's SCS solves.

The splitting solver with an inexact, warm-started CG subspace step is not
a nonexpansive map: CG's coefficients are ratios of inner products, so a
perturbation at the level of one rounding error grows (about 7% per
iteration on scs_feasible_lp_13) until the trajectory settles.  Any change
of floating-point summation order -- a different BLAS kernel, FFT instead
of direct convolution, or a GPU reduction tree -- therefore moves the
iteration at which the status latches on some instances.  The reference
itself is not reproducible at that level across machines.

This script measures that envelope with the reference itself: every
golden SCS case is re-solved by conegraph (/root/reference) with b and c
multiplied elementwise by (1 + d), |d| <= 4 ulp, for R seeds.  The GPU
parity test accepts an iteration count inside [min, max] of these runs
(widened by one check interval) or within 2% of the unperturbed count.

Run in the build container:  python tests/golden/make_envelopes.py
Writes tests/golden/scs_envelopes.json (committed).
"""

from __future__ import annotations

import glob
import json
import os
import sys
import time
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(HERE))

from conegraph import cones as rcones  # noqa: E402
from conegraph import linop as rlinop  # noqa: E402
from conegraph.scs import ConeProblem, ScsSettings, solve  # noqa: E402

from _golden import build_cones, build_tree, load  # noqa: E402

R = int(os.environ.get("ENVELOPE_SEEDS", "8"))
ULP = np.finfo(np.float64).eps


def ref_problem(data, meta, rng=None):
    ns = types.SimpleNamespace(**{k: getattr(rlinop, k) for k in dir(rlinop)})
    A = rlinop.Operator(build_tree(meta["tree"], data, ns))
    K = rcones.ConeProduct(build_cones(meta["cones"], rcones))
    b, c = np.array(data["b"]), np.array(data["c"])
    if rng is not None:
        b = b * (1.0 + 4 * ULP * rng.uniform(-1, 1, b.shape))
        c = c * (1.0 + 4 * ULP * rng.uniform(-1, 1, c.shape))
    return ConeProblem(A, b, c, K)


def main(names=None):
    out_path = os.path.join(HERE, "scs_envelopes.json")
    env = json.load(open(out_path)) if os.path.exists(out_path) else {}
    paths = sorted(glob.glob(os.path.join(HERE, "scs_*.npz")))
    for p in paths:
        name = os.path.basename(p)[:-4]
        if names and name not in names:
            continue
        data, meta = load(name)
        st = ScsSettings(**meta["settings"])
        t0 = time.time()
        its, pobjs, stats = [], [], []
        for seed in range(R):
            sol = solve(ref_problem(data, meta, np.random.default_rng(1000 + seed)), st)
            its.append(int(sol.iterations))
            pobjs.append(float(sol.pobj))
            stats.append(sol.status)
        env[name] = {"iterations": its, "pobj": pobjs, "status": stats,
                     "ref_iterations": meta["iterations"], "ref_pobj": meta.get("pobj"),
                     "seeds": R, "perturbation": "b, c *= 1 + U(-4, 4) ulp"}
        print(f"{name}: ref {meta['iterations']} perturbed {min(its)}..{max(its)} "
              f"statuses {sorted(set(stats))} ({time.time() - t0:.1f} s)", flush=True)
        with open(out_path, "w") as fh:
            json.dump(env, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or None)
