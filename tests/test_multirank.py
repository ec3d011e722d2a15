"""N > 1 host logic on CPU (gloo, world size 2): bench.py's whole-job
aggregation (time = max over ranks, work summed) and the replica
workload's identical per-rank instance."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        # rank r "ran" (r + 1) * 1.5 s doing 1000 + r iterations
        t, it = bench.aggregate((rank + 1) * 1.5, 1000 + rank)
        wl = bench.Deconv1D(5000)
        c, b, _ = wl.data()
        digest = torch.tensor([float(b.sum()), float(c.sum())], dtype=torch.float64)
        gathered = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, digest)
        out[rank] = (t, it, bench._dist(), [g.tolist() for g in gathered])
    finally:
        dist.destroy_process_group()


def test_bench_aggregation_two_ranks():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for rank in range(world):
        t, it, (w, r, lr), gathered = res[rank]
        assert t == pytest.approx(3.0)           # max over ranks
        assert it == 2001                        # summed
        assert (w, r, lr) == (world, rank, rank)
        assert gathered[0] == gathered[1]        # every replica solves the same instance


def test_aggregate_single_process_is_identity():
    import bench
    assert bench.aggregate(2.5, 7) == (2.5, 7)


def _shard_worker(rank, world, port, name, steps, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as np
        import _exprs as E
        from _golden import build_cones, build_tree, load
        from oracle import scs_ref, shard_ref
        data, meta = load(name)
        prob = E.Problem(build_tree(meta["tree"], data, E), np.array(data["b"]),
                         np.array(data["c"]), E.ConeProduct(build_cones(meta["cones"], E)))
        s = scs_ref.ScsOracleSettings(**meta["settings"])
        comm = shard_ref.TorchComm()
        st, sh = shard_ref.solve(prob, comm, s, max_steps=steps)
        out[rank] = (st.ux.tolist(), st.uy.tolist(), st.utau, st.vy.tolist(), st.kappa,
                     st.k, st.cgt, st.status, (sh.r0, sh.r1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,steps", [("scs_lasso_dense_30_7", 12), ("scs_deconv_100_0", 40),
                                        ("scs_soc_ball", 30)])
def test_row_sharded_iteration_matches_single_process(name, steps):
    """§8e decomposition: the splitting iteration with y-space rows split over
    2 gloo ranks (A^T y and y-space dots all-reduced, straddling SOC norms
    reduced) reproduces the single-process oracle's iterates."""
    import numpy as np
    import _exprs as E
    from _golden import build_cones, build_tree, load
    from oracle import scs_ref
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_shard_worker, args=(world, port, name, steps, out), nprocs=world, join=True)
        res = dict(out)
    data, meta = load(name)
    prob = E.Problem(build_tree(meta["tree"], data, E), np.array(data["b"]),
                     np.array(data["c"]), E.ConeProduct(build_cones(meta["cones"], E)))
    s = scs_ref.ScsOracleSettings(**meta["settings"])
    ref = None
    for _, st in scs_ref.iterate(prob, s, scs_ref.prepare_subspace(prob, s.setup_cg_tol,
                                                                   s.cg_max_iter), steps):
        ref = st
    n, m = prob.A.cols, prob.A.rows
    uy = np.concatenate([np.array(res[r][1]) for r in range(world)])
    vy = np.concatenate([np.array(res[r][3]) for r in range(world)])
    assert res[0][8][1] == res[1][8][0] and res[1][8][1] == m   # a row partition
    np.testing.assert_allclose(res[0][0], res[1][0])             # x replicated, identical
    u = np.concatenate([res[0][0], uy, [res[0][2]]])
    v = np.concatenate([np.zeros(n), vy, [res[0][4]]])
    scale = 1.0 + np.linalg.norm(ref.u)
    assert np.linalg.norm(u - ref.u) <= 1e-8 * scale
    assert np.linalg.norm(v - ref.v) <= 1e-8 * scale
    assert res[0][5] == ref.k and res[0][6] == ref.cgt
