"""Standalone 2-d convolution apply timing (k_apply) on the configs[2]
operator: 4096 x 4096 image, 15 x 15 Gaussian, forward (full conv) and
adjoint (valid corr).  Env A/B: CGB_STRIP=0 (per-warp tiles),
CGB_NO_SEPARABLE=1 (direct kh x kw sum).
    python tools/conv2d_bench.py [h] [k] [reps]"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_1609_03488_b200 import canon, linop
    h = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 15
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    K = canon.gaussian_kernel2d(k, k)
    op = linop.conv2d(K, (h, h))
    dev = op.device_op()[0]
    x = torch.randn(op.cols, dtype=torch.float64, device="cuda")
    y = torch.randn(op.rows, dtype=torch.float64, device="cuda")
    out = {"h": h, "k": k, "strip": os.environ.get("CGB_STRIP", "1"),
           "separable": not os.environ.get("CGB_NO_SEPARABLE")}
    for name, adj, vin in (("forward", False, x), ("adjoint", True, y)):
        dst = torch.empty(op.cols if adj else op.rows, dtype=torch.float64, device="cuda")
        for _ in range(3):
            dev.apply(vin, dst, adjoint=adj)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            dev.apply(vin, dst, adjoint=adj)
        e1.record()
        torch.cuda.synchronize()
        us = 1e3 * e0.elapsed_time(e1) / reps
        nbytes = 8 * (op.rows + op.cols)
        out[name] = {"us": us, "GBps_in_out": nbytes / us / 1e3}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
