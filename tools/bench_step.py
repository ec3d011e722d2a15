"""One bench step (setup solve + splitting loop to eps) of bench.py's workload,
for ncu captures: `ncu ... python tools/bench_step.py [n]`."""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1609_03488_b200 import _lib, canon, scs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else bench.N_SIGNAL
c, b, _ = bench._instance(n)
prob = canon.build_deconv(canon.DeconvProblem(c, b, n=n))
settings = scs.ScsSettings(eps=bench.EPS, max_iters=bench.MAX_ITERS)
plan = scs.build_scs_graph(prob, settings)
plan.resetup()
plan.reset()
plan.run(settings.max_iters)
torch.cuda.synchronize()
st = plan.state()
it, cg = int(st[_lib.ST_K]), int(st[_lib.ST_CGT])
print(json.dumps({"iterations": it, "cg_total": cg, "status": float(st[_lib.ST_STATUS]),
                  "algorithmic_bytes": plan.launch_bytes(it, cg)}))
