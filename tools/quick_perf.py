"""Quick on-GPU timing of the deconvolution path (development aid)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1609_03488_b200 import canon, scs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
k = 101
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
c, b, _ = canon.gen_deconv1d(n, k, seed=0)
prob = canon.build_deconv(canon.DeconvProblem(c, b, n=n))
st = scs.ScsSettings(eps=1e-3, max_iters=100000)
t0 = time.time(); g = scs.build_scs_graph(prob, st); torch.cuda.synchronize()
print("build+setup", time.time() - t0, "setup cg iters", g.cached.setup_cg_iters, flush=True)
print("geometry", g.dev.ctx.geometry(), g.dev.plan_info(False), g.dev.plan_info(True))
g.reset(); g.run(5); torch.cuda.synchronize()
for steps in (iters, iters):
    g.reset()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); g.run(steps); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    s = g.state()
    print(f"{steps} iters: {ms:.2f} ms -> {steps/ms*1e3:.1f} iter/s, cg total {s[3]}, status {s[2]}", flush=True)
g.reset()
e0.record(); g.run(100000); e1.record(); torch.cuda.synchronize()
s = g.state()
print(f"to eps=1e-3: {e0.elapsed_time(e1):.1f} ms, iters {s[0]}, cg {s[3]}, status {s[2]}")
