"""Lock-step oracle vs device iterates on a golden case (development aid)."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from _golden import load, build_tree, build_cones
import _exprs as E
from oracle import scs_ref
from paper_1609_03488_b200 import linop, cones, scs

name = sys.argv[1]; N = int(sys.argv[2])
data, meta = load(name)
A = linop.Operator(build_tree(meta["tree"], data, linop))
prob = scs.ConeProblem(A, np.array(data["b"]), np.array(data["c"]),
                       cones.ConeProduct(build_cones(meta["cones"], cones)))
st = scs.ScsSettings(**meta["settings"])
g = scs.build_scs_graph(prob, st)
op = E.Problem(build_tree(meta["tree"], data, E), np.array(data["b"]), np.array(data["c"]),
               E.ConeProduct(build_cones(meta["cones"], E)))
os_ = scs_ref.ScsOracleSettings(**meta["settings"])
cached = scs_ref.prepare_subspace(op, os_.setup_cg_tol, os_.cg_max_iter)
print("denom", g.cached.denom, cached.denom, "g diff", np.abs(g.cached.g - cached.g).max())
it_o = scs_ref.iterate(op, os_, cached, N)
prev_cg_o = prev_cg_d = 0
shown = 0
for (k, so), (k2, sd) in zip(it_o, scs.iterate_states(g, N)):
    du = np.linalg.norm(so.u - sd[0]) / (1 + np.linalg.norm(so.u))
    dv = np.linalg.norm(so.v - sd[1]) / (1 + np.linalg.norm(so.v))
    cgo, cgd = so.cgt - prev_cg_o, sd[6][0] - prev_cg_d
    prev_cg_o, prev_cg_d = so.cgt, sd[6][0]
    if cgo != cgd or k % 50 == 0 or (du > 1e-10 and shown < 30):
        shown += 1
        print(f"k={k} du={du:.2e} dv={dv:.2e} cg o/d {cgo}/{cgd} resid o {so.resid} d {sd[7]}")
