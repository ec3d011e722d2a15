"""Standalone k_apply timing of a bench workload's stuffed operator,
forward and adjoint (development aid).
    python tools/apply_bench.py soc_ls [reps]"""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402


class A:
    workload = sys.argv[1] if len(sys.argv) > 1 else "soc_ls"
    n = bench.N_SIGNAL


reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
wl = bench.make_workload(A)
prob = wl.problem()
dev = prob.A.device_op()[0]
x = torch.randn(prob.A.cols, dtype=torch.float64, device="cuda")
y = torch.randn(prob.A.rows, dtype=torch.float64, device="cuda")
out = {"workload": wl.name, "shape": [prob.A.rows, prob.A.cols]}
for name, adj, vin in (("forward", False, x), ("adjoint", True, y)):
    dst = torch.empty(prob.A.cols if adj else prob.A.rows, dtype=torch.float64, device="cuda")
    for _ in range(2):
        dev.apply(vin, dst, adjoint=adj)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        dev.apply(vin, dst, adjoint=adj)
    e1.record()
    torch.cuda.synchronize()
    us = 1e3 * e0.elapsed_time(e1) / reps
    nbytes = dev.algo_bytes(adj)
    out[name] = {"us": us, "algo_GBps": nbytes / us / 1e3}
print(json.dumps(out))
