"""Cost of one grid barrier / grid reduction inside the persistent kernels."""
import sys
sys.path.insert(0, ".")
import torch
from paper_1609_03488_b200 import _lib
ctx = _lib.device_context()
lib = _lib.load_library()
print("geometry", ctx.geometry())
for mode in (0, 1):
    for iters in (1000, 20000):
        _lib.check(lib.cgb_debug_barrier(ctx.handle, 10, mode, _lib.stream_handle()))
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(lib.cgb_debug_barrier(ctx.handle, iters, mode, _lib.stream_handle()))
        e1.record(); torch.cuda.synchronize()
        print(f"mode {mode} ({'sync' if mode == 0 else 'reduce'}): {iters} -> "
              f"{e0.elapsed_time(e1) * 1e3 / iters:.3f} us each")
