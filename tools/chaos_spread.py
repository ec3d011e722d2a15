"""Iteration-count spread of the bench solve under 4-ulp input perturbations
(development aid; evidence for DESIGN.md "Parity").

The splitting iteration with an inexact, warm-started CG amplifies rounding:
two runs whose data differ in the last bits reach eps = 1e-3 after different
iteration counts (tests/golden/make_envelopes.py measures this for the real
reference at test sizes).  This script measures the same spread for the
device solver on the full bench instance: b is perturbed by +-4 ulp per
entry (seeded), the solve is run to eps, and iterations / objective are
reported.  Seed 0 = the unperturbed bench instance.

usage: python tools/chaos_spread.py [n_perturbed]
"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1609_03488_b200 import canon, scs  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 12
n = bench.N_SIGNAL
c, b0, _ = bench._instance(n)
out = []
for s in range(K + 1):
    b = b0.copy()
    if s:
        rng = np.random.default_rng(1000 + s)
        steps = rng.integers(-4, 5, size=b.shape)
        for _ in range(4):
            up = steps > 0
            dn = steps < 0
            b[up] = np.nextafter(b[up], np.inf)
            b[dn] = np.nextafter(b[dn], -np.inf)
            steps = steps - np.sign(steps)
    prob = canon.build_deconv(canon.DeconvProblem(c, b, n=n))
    st_ = scs.ScsSettings(eps=bench.EPS, max_iters=100000)
    plan = scs.build_scs_graph(prob, st_)
    sol = scs.solve_built(prob, st_, plan)
    rec = {"seed": s, "iters": sol.iterations, "status": sol.status, "pobj": sol.pobj}
    out.append(rec)
    print(json.dumps(rec), flush=True)
its = [r["iters"] for r in out]
print(json.dumps({"n": n, "perturbed": K, "iters_min": min(its), "iters_max": max(its),
                  "iters_median": float(np.median(its)), "unperturbed": its[0]}))
