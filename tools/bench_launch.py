"""The bench.py step of a workload as ONE standalone k_scs launch (for ncu):
setup solve, reset, `steps` splitting iterations from cold.
    python tools/bench_launch.py deconv2d 2000"""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1609_03488_b200 import _lib, scs  # noqa: E402


class A:
    workload = sys.argv[1] if len(sys.argv) > 1 else "deconv2d"
    n = bench.N_SIGNAL


steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
wl = bench.make_workload(A)
plan = scs.build_scs_graph(wl.problem(), scs.ScsSettings(eps=wl.eps, max_iters=bench.MAX_ITERS))
plan.resetup()
plan.reset()
plan.run(steps)
torch.cuda.synchronize()
st = plan.state()
print(json.dumps({"workload": wl.name, "iterations": int(st[_lib.ST_K]),
                  "cg_total": int(st[_lib.ST_CGT]),
                  "algorithmic_bytes": plan.launch_bytes(int(st[_lib.ST_K]), int(st[_lib.ST_CGT])),
                  "algorithmic_flops": plan.launch_flops(int(st[_lib.ST_K]), int(st[_lib.ST_CGT]))}))
