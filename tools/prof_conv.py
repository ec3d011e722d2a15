"""A few k_apply launches of the bare Conv1D (n=1e6, k=101) for ncu."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
import bench  # noqa: E402
from paper_1609_03488_b200 import linop  # noqa: E402
n = 1_000_000
c, _, _ = bench._instance(n)
C = linop.conv1d(c, n)
x = torch.randn(n, dtype=torch.float64, device="cuda")
y = torch.empty(C.rows, dtype=torch.float64, device="cuda")
for _ in range(3):
    C.apply_device(x, y)
torch.cuda.synchronize()
