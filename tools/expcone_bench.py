"""Time the device exp-cone projection (k_cones) on 4e5 cones (development aid)."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1609_03488_b200 import cones  # noqa: E402

nc = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000
K = cones.ConeProduct([cones.ExpCone() for _ in range(nc)])
Kd = K.device()
v = torch.from_numpy(np.random.default_rng(0).standard_normal(3 * nc)).cuda()
o = torch.empty_like(v)
for dual in (False, True):
    Kd.project_device(v, o, dual=dual)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        Kd.project_device(v, o, dual=dual)
    e1.record()
    torch.cuda.synchronize()
    print(f"{nc} exp cones dual={dual}: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us")
