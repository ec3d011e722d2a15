import sys, json
sys.path.insert(0, ".")
import numpy as np, torch
import bench
from paper_1609_03488_b200 import scs, _lib
class A: workload = sys.argv[1]; n = bench.N_SIGNAL
wl = bench.make_workload(A)
prob = wl.problem()
st = scs.ScsSettings(eps=1e-3, max_iters=100000)
out = []
for i in range(3):
    sol = scs.solve(prob, st)
    out.append(("solve", sol.iterations, sol.pobj.hex()))
plan = scs.build_scs_graph(prob, st)
for i in range(3):
    plan.reset(); plan.run(st.max_iters); torch.cuda.synchronize()
    s_ = plan.state(); out.append(("plan", int(s_[_lib.ST_K]), float(plan.buf["u"][-1].item()).hex()))
plan.reset(); plan.run(5); plan.reset(); plan.run(st.max_iters); torch.cuda.synchronize()
out.append(("plan_after5", int(plan.state()[_lib.ST_K])))
print(json.dumps(out))
