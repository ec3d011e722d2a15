"""Iteration rate and time-to-eps of a bench.py workload (development aid).

usage: python tools/workload_probe.py <workload> [iters] [max_iters]
"""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1609_03488_b200 import _lib, scs  # noqa: E402


class A:
    workload = sys.argv[1]
    n = bench.N_SIGNAL


iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 100000
wl = bench.make_workload(A)
t0 = time.time()
prob = wl.problem()
t1 = time.time()
plan = scs.build_scs_graph(prob, scs.ScsSettings(eps=wl.eps, max_iters=cap))
torch.cuda.synchronize()
t2 = time.time()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
plan.reset()
plan.run(5)
prof = "--profile" in sys.argv
if prof:
    plan.enable_profile(True)
e0.record()
plan.run(iters)
e1.record()
torch.cuda.synchronize()
st = plan.state()
if prof:
    ph = plan.profile()
    print(json.dumps({k: (1e6 * v / iters if not isinstance(v, dict) else v)
                      for k, v in ph.items()}))
    plan.enable_profile(False)
out = {"workload": wl.name, "data_s": t1 - t0, "build_s": t2 - t1,
       "setup_cg_iters": plan.cached.setup_cg_iters,
       "us_per_iter": 1e3 * e0.elapsed_time(e1) / iters, "cg_per_iter": float(st[_lib.ST_CGT]) / max(1, st[_lib.ST_K])}
plan.reset()
e0.record()
plan.run(cap)
e1.record()
torch.cuda.synchronize()
st = plan.state()
out.update({"to_eps_s": e0.elapsed_time(e1) / 1e3, "iters": int(st[_lib.ST_K]),
            "cg_total": int(st[_lib.ST_CGT]), "status": float(st[_lib.ST_STATUS]),
            "pr_dr_gap": [float(st[_lib.ST_PR]), float(st[_lib.ST_DR]), float(st[_lib.ST_GAP])]})
print(json.dumps(out))
