"""Where the end-to-end step of bench.py's e2e leg goes (development aid):
host problem build, compile (plans, cones, setup solve), the bounded
iterations, classification and result copies.
    python tools/e2e_breakdown.py [workload] [iters]"""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1609_03488_b200 import _lib, scs  # noqa: E402


class A:
    workload = sys.argv[1] if len(sys.argv) > 1 else "deconv2d"
    n = bench.N_SIGNAL


iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
wl = bench.make_workload(A)
wl.data()
out = {}
for rep in range(2):
    t = {}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prob = wl.problem()
    t["problem_build"] = time.perf_counter() - t0
    st = scs.ScsSettings(eps=wl.eps, max_iters=iters)
    t0 = time.perf_counter()
    g = scs.build_scs_graph(prob, st)
    torch.cuda.synchronize()
    t["build_scs_graph"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    g.reset()
    g.run(st.max_iters)
    torch.cuda.synchronize()
    t["iterations"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    stt = g.state()
    u, v = g.host_uv()
    t["d2h_uv"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    resid = (float(stt[_lib.ST_PR]), float(stt[_lib.ST_DR]), float(stt[_lib.ST_GAP]),
             float(stt[_lib.ST_RES_U]), float(stt[_lib.ST_RES_I]))
    sol = scs._classify(prob, st, u, v, int(stt[_lib.ST_K]), float(stt[_lib.ST_CGT]), resid)
    t["classify"] = time.perf_counter() - t0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sol = scs.solve(wl.problem(), st)
    torch.cuda.synchronize()
    t["scs_solve_total"] = time.perf_counter() - t0
    out[f"rep{rep}"] = t
# finer: inside build_scs_graph
t0 = time.perf_counter()
prob = wl.problem()
dev = scs._own_device_op(prob.A)
torch.cuda.synchronize()
t1 = time.perf_counter()
cones = prob.K.device()
torch.cuda.synchronize()
t2 = time.perf_counter()
cached = scs.prepare_subspace(prob, 1e-12, None)
torch.cuda.synchronize()
t3 = time.perf_counter()
out["build_parts"] = {"device_op": t1 - t0, "cones": t2 - t1, "prepare_subspace": t3 - t2}
print(json.dumps(out, indent=1))
