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
