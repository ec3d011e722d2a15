"""Per-phase device time of the splitting loop (k_scs phase profiler).

usage: python tools/phase_prof.py [n] [iters]   (deconv1d, kernel 101)
"""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1609_03488_b200 import _lib, canon, scs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 400
c, b, _ = bench._instance(n)
prob = canon.build_deconv(canon.DeconvProblem(c, b, n=n))
plan = scs.build_scs_graph(prob, scs.ScsSettings(eps=1e-3, max_iters=100000))
plan.reset()
plan.run(20)
torch.cuda.synchronize()
plan.enable_profile(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
plan.run(iters)
e1.record()
torch.cuda.synchronize()
st = plan.state()
ms = e0.elapsed_time(e1)
done = int(st[_lib.ST_K]) - 20
prof = plan.profile()
out = {"n": n, "iters": done, "cg_iters": int(st[_lib.ST_CGT]), "ms": ms,
       "us_per_iter": 1e3 * ms / max(done, 1),
       "phase_us_per_iter": {k: 1e6 * v / max(done, 1) for k, v in prof.items()
                             if not isinstance(v, dict)},
       "rhs_warp0_timeline_us_per_iter": {k: (v if k == "tiles" else 1e6 * v) / max(done, 1)
                                          for k, v in prof["rhs_warp0_timeline"].items()}}
print(json.dumps(out, indent=1))
plan.enable_profile(False)
plan.reset()
e0.record()
plan.run(100000)
e1.record()
torch.cuda.synchronize()
st = plan.state()
print(json.dumps({"to_eps_ms": e0.elapsed_time(e1), "iters": int(st[_lib.ST_K]),
                  "cg_total": int(st[_lib.ST_CGT]), "status": float(st[_lib.ST_STATUS])}))
