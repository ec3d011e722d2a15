"""Iteration count of one instance under different reduction orders on the
device: single-GPU solver at several grid sizes (CGB_GRID) and the sharded
solver at several world sizes (development aid).
    python tools/grid_spread.py lasso_dense"""
import json
import os
import subprocess
import sys

sys.path.insert(0, ".")

if len(sys.argv) > 2 and sys.argv[2] == "child":
    import bench
    from paper_1609_03488_b200 import scs, shard

    class A:
        workload = sys.argv[1]
        n = bench.N_SIGNAL
    wl = bench.make_workload(A)
    prob = wl.problem()
    st = scs.ScsSettings(eps=1e-3, max_iters=100000)
    world = int(sys.argv[3])
    if world == 0:
        sol = scs.solve(prob, st)
    else:
        g = shard.ShardGroup(prob, st, world=world)
        sol = g.solve()
        g.close()
    print(json.dumps([sol.status, sol.iterations, sol.pobj]))
    sys.exit(0)

out = {}
for grid in (148, 128, 100, 74, 37):
    env = dict(os.environ, CGB_GRID=str(grid))
    r = subprocess.run([sys.executable, __file__, sys.argv[1], "child", "0"], env=env,
                       capture_output=True, text=True)
    out[f"single_grid{grid}"] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-300:]
for world in (1, 2, 3, 4):
    r = subprocess.run([sys.executable, __file__, sys.argv[1], "child", str(world)],
                       capture_output=True, text=True)
    out[f"shard_world{world}"] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-300:]
print(json.dumps(out, indent=1))
