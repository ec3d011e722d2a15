import sys, faulthandler; faulthandler.enable()
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1609_03488_b200 import _lib, linop
print("lib", _lib.load_library(), flush=True)
ctx = _lib.device_context(); print("ctx ok", ctx.geometry(), flush=True)
op = linop.conv1d([1.0, 1.0], 2)
print(op.forward(np.array([1.0, 2.0])), flush=True)
print(op.adjoint_apply(np.array([1.0, 3.0, 2.0])), flush=True)
d = linop.dense([[1.0, 2.0], [3.0, 4.0], [5.0, 6.0]])
print(d.forward(np.array([1.0, 1.0])), d.adjoint_apply(np.array([1.0, 1.0, 1.0])), flush=True)
