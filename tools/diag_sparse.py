"""Check the large sparse lasso pieces against the oracle (development aid)."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
from oracle import linop_ref, cones_ref, scs_ref  # noqa: E402
from paper_1609_03488_b200 import scs  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
wl = bench.LassoSparse(m, n, 1e-5 * 8e6 / m)
prob = wl.problem()
A = prob.A
rng = np.random.default_rng(0)
x = rng.standard_normal(A.cols)
y = rng.standard_normal(A.rows)
f = A.forward(x)
fr = linop_ref.forward(A.expr, x)
print("forward rel err", np.abs(f - fr).max() / np.abs(fr).max())
a = A.adjoint_apply(y)
ar = linop_ref.adjoint(A.expr, y)
print("adjoint rel err", np.abs(a - ar).max() / np.abs(ar).max())
Kd = prob.K.device()
v = torch.from_numpy(rng.standard_normal(A.rows)).cuda()
pd = Kd.project_device(v, dual=True).cpu().numpy()
pr = cones_ref.project_dual_product(prob.K.factors, v.cpu().numpy())
print("cone rel err", np.abs(pd - pr).max() / np.abs(pr).max())
# first iterations vs oracle
st = scs.ScsSettings(eps=1e-3, max_iters=100)
plan = scs.build_scs_graph(prob, st)


class P:
    pass


p = P()
p.A, p.b, p.c, p.K = prob.A.expr, prob.b, prob.c, prob.K
os_ = scs_ref.ScsOracleSettings(eps=1e-3, max_iters=100)
cached = scs_ref.prepare_subspace(p, os_.setup_cg_tol, os_.cg_max_iter)
print("denom dev/oracle", plan.cached.denom, cached.denom,
      "g diff", np.abs(plan.cached.g - cached.g).max() / np.abs(cached.g).max())
it = scs_ref.iterate(p, os_, cached, 25)
for (k, so), (k2, sd) in zip(it, scs.iterate_states(plan, 25)):
    du = np.linalg.norm(so.u - sd[0]) / (1 + np.linalg.norm(so.u))
    print(k, "du", du, "tau o/d", so.u[-1], sd[0][-1], "cg", so.cgt, sd[6][0], "st", so.status, sd[4][0])
