"""Lock-step oracle vs device iterates on a bench.py workload instance
(development aid): iterate distance and CG counts every few iterations,
then both full solves.
    python tools/diverge_bench.py lasso_dense [N]"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402
from oracle import scs_ref  # noqa: E402
from paper_1609_03488_b200 import scs  # noqa: E402


class A:
    workload = sys.argv[1]
    n = bench.N_SIGNAL


N = int(sys.argv[2]) if len(sys.argv) > 2 else 400
wl = bench.make_workload(A)
prob = wl.problem()
op = wl.oracle_problem()
st = scs.ScsSettings(eps=wl.eps, max_iters=100_000)
os_ = scs_ref.ScsOracleSettings(eps=wl.eps, max_iters=100_000)
g = scs.build_scs_graph(prob, st)
cached = scs_ref.prepare_subspace(op, os_.setup_cg_tol, os_.cg_max_iter)
out = {"denom": [g.cached.denom, cached.denom],
       "g_diff": float(np.abs(g.cached.g - cached.g).max() / np.abs(cached.g).max()), "trace": []}
pco = pcd = 0.0
for (k, so), (_, sd) in zip(scs_ref.iterate(op, os_, cached, N), scs.iterate_states(g, N)):
    du = float(np.linalg.norm(so.u - sd[0]) / (1 + np.linalg.norm(so.u)))
    cgo, cgd = so.cgt - pco, sd[6][0] - pcd
    pco, pcd = so.cgt, sd[6][0]
    if k <= 5 or k % 20 == 0 or cgo != cgd:
        out["trace"].append([k, du, int(cgo), int(cgd)])
sol = scs.solve(prob, st)
osol, _ = scs_ref.scs_solve(op, os_)
out["device"] = [sol.status, sol.iterations, sol.pobj]
out["oracle"] = [osol.status, osol.iterations, osol.pobj]
print(json.dumps(out))
