"""One k_scs launch of `steps` iterations on the n=1e6, k=101 deconvolution (for ncu)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_1609_03488_b200 import canon, scs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
c, b, _ = canon.gen_deconv1d(n, 101, seed=0)
prob = canon.build_deconv(canon.DeconvProblem(c, b, n=n))
g = scs.build_scs_graph(prob, scs.ScsSettings(eps=1e-3, max_iters=100000))
g.reset(); g.run(steps); torch.cuda.synchronize()
print("state", g.state()[:8])
