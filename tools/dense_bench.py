"""Standalone dense GEMV timing (forward tall 2e5 x 2e3 and its split-K adjoint)."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1609_03488_b200 import linop  # noqa: E402

m, n = 200_000, 2_000
A = np.random.default_rng(0).standard_normal((m, n))
op = linop.dense(A)
x = torch.randn(n, dtype=torch.float64, device="cuda")
y = torch.randn(m, dtype=torch.float64, device="cuda")
ox = torch.empty(m, dtype=torch.float64, device="cuda")
oy = torch.empty(n, dtype=torch.float64, device="cuda")


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


us = timeit(lambda: op.apply_device(x, ox))
print(f"dense A x   : {us:9.1f} us {8 * m * n / us / 1e3:7.0f} GB/s")
us = timeit(lambda: op.apply_device(y, oy, adjoint=True))
print(f"dense A^T y : {us:9.1f} us {8 * m * n / us / 1e3:7.0f} GB/s")
