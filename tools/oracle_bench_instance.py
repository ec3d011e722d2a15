"""Full CPU-oracle solve of bench.py's default instance (n=1e6, k=101) to eps=1e-3:
the reference algorithm's own iteration count / objective for comparison with
the device solve.  Took 9304 s (~6 OpenBLAS threads) in the build container;
result in profiles/oracle_bench_instance.json."""
import sys, time, json
sys.path.insert(0, "/root/repo")
import numpy as np
import bench
from oracle import scs_ref
p = bench._cpu_problem(1_000_000)
s = scs_ref.ScsOracleSettings(eps=1e-3, max_iters=100000)
t0 = time.time()
sol, last = scs_ref.scs_solve(p, s)
out = {"status": sol.status, "iterations": int(sol.iterations), "pobj": float(sol.pobj),
       "avg_cg": float(sol.avg_cg_iterations), "pr": float(sol.primal_residual),
       "dr": float(sol.dual_residual), "gap": float(sol.gap), "seconds": time.time() - t0}
print(json.dumps(out), flush=True)
np.save("/tmp/oracle_bench_x.npy", sol.x)
