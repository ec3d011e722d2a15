"""Time the individual persistent kernels on the bench instance (development aid).

k_apply forward/adjoint of the stuffed deconvolution operator and of the bare
Conv1D, and k_cones on the cone product -- each launched back to back with
CUDA events; reports us/launch and the algorithmic GB/s.
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1609_03488_b200 import canon, linop  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
c, b, _ = bench._instance(n)
prob = canon.build_deconv(canon.DeconvProblem(c, b, n=n))
A = prob.A
m = A.rows


def timeit(fn, reps=50):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


x = torch.randn(n + 1, dtype=torch.float64, device="cuda")
y = torch.randn(m, dtype=torch.float64, device="cuda")
ox = torch.empty(m, dtype=torch.float64, device="cuda")
oy = torch.empty(n + 1, dtype=torch.float64, device="cuda")
us = timeit(lambda: A.apply_device(x, ox))
print(f"stuffed A x    : {us:8.2f} us  {8 * (n + 1 + m) / us / 1e3:7.0f} GB/s")
us = timeit(lambda: A.apply_device(y, oy, adjoint=True))
print(f"stuffed A^T y  : {us:8.2f} us  {8 * (n + 1 + m) / us / 1e3:7.0f} GB/s")
C = linop.conv1d(c, n)
xc = torch.randn(n, dtype=torch.float64, device="cuda")
yc = torch.empty(C.rows, dtype=torch.float64, device="cuda")
us = timeit(lambda: C.apply_device(xc, yc))
flops = 2 * 101 * n
print(f"conv C x       : {us:8.2f} us  {8 * (n + C.rows) / us / 1e3:7.0f} GB/s  {flops / us / 1e6:6.2f} TF/s")
us = timeit(lambda: C.apply_device(yc, xc, adjoint=True))
print(f"corr C^T y     : {us:8.2f} us  {8 * (n + C.rows) / us / 1e3:7.0f} GB/s  {flops / us / 1e6:6.2f} TF/s")
K = prob.K.device()
v = torch.randn(m, dtype=torch.float64, device="cuda")
o = torch.empty_like(v)
us = timeit(lambda: K.project_device(v, o, dual=True))
print(f"cones Pi_K* v  : {us:8.2f} us  {16 * m / us / 1e3:7.0f} GB/s")
from paper_1609_03488_b200 import _lib  # noqa: E402
lib = _lib.load_library()
ctx = _lib.device_context()
for mode, nm in ((0, "barrier"), (1, "reduce1"), (2, "reduce4"), (3, "reduce8"),
                 (4, "barrier_acqrel"), (5, "barrier_relacq")):
    us = timeit(lambda: _lib.check(lib.cgb_debug_barrier(ctx.handle, 1000, mode,
                                                         _lib.stream_handle())), reps=5)
    print(f"{nm} x1000 : {us / 1000:8.3f} us each")
I1 = linop.identity(64)
xi = torch.randn(64, dtype=torch.float64, device="cuda")
yi = torch.empty(64, dtype=torch.float64, device="cuda")
us = timeit(lambda: I1.apply_device(xi, yi))
print(f"identity(64)   : {us:8.2f} us  (cooperative launch + memset overhead)")
