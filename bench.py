#!/usr/bin/env python
"""Benchmark of the B200 conegraph solver path (driver contract).

Workload (BASELINE.json configs[1]): 1-D nonnegative deconvolution, signal
n = 1e6, Gaussian kernel length 101, stuffed exactly like the reference's
build_deconv (variables n+1, constraints 2n+k), solved to eps = 1e-3.

A *step* is one complete solve to eps = 1e-3 from a cold start: the
one-time setup solve g = (I+Q_z)^{-1} h followed by the splitting
iterations until the device-latched status says solved.  ``value`` is
ADMM (splitting) iterations per second over the K timed steps with the
problem data resident in HBM (all ranks summed); ``time_to_eps_s`` is the
mean step time.  ``e2e`` is the same metric through the public API
(``scs.solve`` on numpy inputs: host->device copies of b, c and the
kernel, operator/cone compilation, setup, solve, device->host copy of
x, y, s) per step.

``--impl reference`` times the reference algorithm's CPU implementation
(the numpy restatement in oracle/, pinned to the real reference's golden
vectors) on the host cores: rank 0 only, a bounded sample of splitting
iterations of the same instance per step, same metric and unit.

Multi-GPU: this workload is a small structured operator, which the north
star keeps on one GPU, so N > 1 runs N independent replicas (one solve per
rank, no data-path collective; "scaling": "weak"); time is the max over
ranks of the per-rank device time.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_SIGNAL = 1_000_000
K_KERNEL = 101
EPS = 1e-3
MAX_ITERS = 100_000
SEED = 0
WORKLOAD = "deconv1d_nonneg"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=N_SIGNAL)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=0,
                    help="splitting iterations per CPU sample (0 = size for ~20 s)")
    return ap.parse_args()


def _config(n: int, n_gpus: int) -> dict:
    return {"workload": WORKLOAD, "signal_n": n, "kernel_k": K_KERNEL, "eps": EPS,
            "stuffed_n": n + 1, "stuffed_m": 2 * n + K_KERNEL, "seed": SEED,
            "step": "one full solve to eps (setup solve + splitting iterations, cold start)",
            "l2": "flushed between timed steps (256 MiB write)",
            "parallelism": f"replicas{n_gpus}" if n_gpus > 1 else "single"}


def _instance(n: int):
    """Synthetic instance (canon.gen_deconv1d's recipe: Gaussian kernel, 50
    nonnegative spikes, noise 0.01), generated on the host so both arms see
    bit-identical data."""
    import numpy as np
    from paper_1609_03488_b200 import canon
    rng = np.random.default_rng(SEED)
    c = canon.gaussian_kernel(K_KERNEL)
    x_hat = np.zeros(n)
    pos = rng.choice(n, size=min(50, n), replace=False)
    x_hat[pos] = rng.uniform(0.0, 10.0, size=len(pos))
    b = np.convolve(c, x_hat) + canon.NOISE_SIGMA * rng.standard_normal(n + K_KERNEL - 1)
    return c, b, x_hat


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._thr = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:  # noqa: BLE001 - sampling is best effort
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._thr.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._thr.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# reference arm: the CPU implementation of the path (oracle port)
# ---------------------------------------------------------------------------

def _cpu_problem(n: int):
    """The stuffed deconvolution as a duck-typed tree the oracle walks."""
    from paper_1609_03488_b200 import canon
    c, b, _ = _instance(n)
    prob = canon.build_deconv(canon.DeconvProblem(c, b, n=n))

    class P:
        pass
    p = P()
    p.A, p.b, p.c, p.K = prob.A.expr, prob.b, prob.c, prob.K
    return p


def cpu_sample(n: int, iters: int, warmup_iters: int = 1):
    """Time the oracle's splitting iterations on the host (setup excluded
    from the rate, reported separately).  Returns a dict."""
    from oracle import scs_ref
    p = _cpu_problem(n)
    s = scs_ref.ScsOracleSettings(eps=EPS, max_iters=MAX_ITERS)
    t0 = time.perf_counter()
    cached = scs_ref.prepare_subspace(p, s.setup_cg_tol, s.cg_max_iter)
    setup_s = time.perf_counter() - t0
    it = scs_ref.iterate(p, s, cached, warmup_iters + iters)
    for _ in range(warmup_iters):
        next(it)
    t0 = time.perf_counter()
    done = 0
    for _k, _st in it:
        done += 1
    dt = time.perf_counter() - t0
    return {"setup_s": setup_s, "iters": done, "seconds": dt, "iters_per_s": done / dt}


def _cpu_cores_used() -> int:
    """Host threads the oracle can use: numpy's FFTs are single-threaded, its
    dot products / norms run in OpenBLAS with this many threads."""
    try:
        from threadpoolctl import threadpool_info
        blas = [i["num_threads"] for i in threadpool_info() if i.get("user_api") == "blas"]
        if blas:
            return int(max(blas))
    except Exception:  # noqa: BLE001 - reporting only
        pass
    return os.cpu_count() or 1


def run_reference(args) -> None:
    world, rank, _ = _dist()
    if rank != 0:
        return
    n = args.n
    iters = args.cpu_iters or 10
    from oracle import scs_ref
    p = _cpu_problem(n)
    s = scs_ref.ScsOracleSettings(eps=EPS, max_iters=MAX_ITERS)
    t0 = time.perf_counter()
    cached = scs_ref.prepare_subspace(p, s.setup_cg_tol, s.cg_max_iter)
    setup_s = time.perf_counter() - t0
    state_it = scs_ref.iterate(p, s, cached, MAX_ITERS)
    times = []
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        for _ in range(iters):
            next(state_it)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
    total = sum(times)
    value = iters * len(times) / total
    line = {
        "impl": "reference", "metric": "ADMM iterations/s (time-to-eps=1e-3 in time_to_eps_s)",
        "value": value, "unit": "iter/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": _config(n, 1),
        "setup_s": setup_s,
        "cpu_baseline": {"value": value, "unit": "iter/s", "cores": _cpu_cores_used(),
                         "kind": "port",
                         "sample": f"{iters} splitting iterations per step of the n={n} "
                                   f"deconvolution after the oracle's own setup solve "
                                   f"({setup_s:.1f} s, untimed); numpy restatement of "
                                   f"conegraph scs.py (FFT convolution as linop.py)"},
        "e2e": {"value": value, "unit": "iter/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def run_b200(args) -> None:
    import numpy as np
    import torch

    world, rank, local = _dist()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the B200 path has no CPU fallback)")
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1609_03488_b200 import _lib, canon, scs

    n = args.n
    c, b, _ = _instance(n)
    settings = scs.ScsSettings(eps=EPS, max_iters=MAX_ITERS)

    # resident-data arm: compile once (graph build), then time setup + solve
    prob = canon.build_deconv(canon.DeconvProblem(c, b, n=n))
    t0 = time.perf_counter()
    plan = scs.build_scs_graph(prob, settings)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def one_step():
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(stream)
        plan.resetup()
        plan.reset()
        ev[1].record(stream)
        plan.run(settings.max_iters)
        ev[2].record(stream)
        torch.cuda.synchronize()
        st = plan.state()
        return (ev[0].elapsed_time(ev[2]) / 1e3, ev[1].elapsed_time(ev[2]) / 1e3,
                int(st[_lib.ST_K]), int(st[_lib.ST_CGT]), float(st[_lib.ST_STATUS]))

    for _ in range(args.warmup):
        flush.zero_()
        one_step()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    results = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            results.append(one_step())
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    step_s = [r[0] for r in results]
    kern_s = [r[1] for r in results]
    iters = [r[2] for r in results]
    cgs = [r[3] for r in results]
    statuses = {r[4] for r in results}
    total_s = sum(step_s)
    total_iters = sum(iters)
    if world > 1:
        t = torch.tensor([total_s], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_s = float(t.item())
        it = torch.tensor([float(total_iters)], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(it)
        total_iters = int(it.item())
    value = total_iters / total_s

    # roofline of the dominant kernel (k_scs: the splitting loop)
    launch_bytes = [plan.launch_bytes(i, c_) for i, c_ in zip(iters, cgs)]
    achieved = sum(launch_bytes) / sum(kern_s) / 1e9
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(peaks_path):
        peak = float(json.load(open(peaks_path))["hbm_gbs"])
        peak_src = "measured"
    else:
        peak, peak_src = 6650.0, "fallback"
    traffic = None
    tp = os.path.join(ROOT, "profiles", "k_scs_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("bytes_per_launch_at_bench")
        except Exception:  # noqa: BLE001
            traffic = None

    # end-to-end arm: public API on host (numpy) buffers, per step
    e2e_times = []
    h2d = 8 * (len(c) + len(b)) + 8 * (2 * n + K_KERNEL + n + 1)  # kernel, b; b_cone, c_obj
    d2h = 0
    e2e_status = None
    for step in range(1 + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        p2 = canon.build_deconv(canon.DeconvProblem(c, b, n=n))
        sol = scs.solve(p2, settings)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        d2h = 8 * (len(sol.x) + len(sol.y) + len(sol.s))
        e2e_status = sol.status
        if step >= 1:
            e2e_times.append((dt, sol.iterations))
    e2e_s = sum(t for t, _ in e2e_times)
    e2e_it = sum(i for _, i in e2e_times)
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
        it = torch.tensor([float(e2e_it)], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(it)
        e2e_it = int(it.item())

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        iters_cpu = args.cpu_iters or 20
        cs = cpu_sample(n, iters_cpu)
        per_it = cs["seconds"] / cs["iters"]
        cpu = {"value": cs["iters_per_s"], "unit": "iter/s", "cores": _cpu_cores_used(),
               "kind": "port",
               "sample": f"{cs['iters']} splitting iterations of the same n={n} instance "
                         f"after the oracle's setup solve ({cs['setup_s']:.1f} s); numpy "
                         f"restatement of conegraph scs.py (FFT convolutions single-threaded, "
                         f"dot products in OpenBLAS threads; host has {os.cpu_count()} cpus)",
               "setup_s": cs["setup_s"],
               "time_to_eps_s_extrapolated": cs["setup_s"] + per_it * statistics.mean(iters)}

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    line = {
        "metric": "ADMM iterations/s (time-to-eps=1e-3 in time_to_eps_s)",
        "value": value, "unit": "iter/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(step_s),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": _config(n, world),
        "time_to_eps_s": statistics.mean(step_s),
        "iterations_to_eps": iters[0], "avg_cg_iterations": cgs[0] / max(1, iters[0]),
        "status": sorted(statuses), "graph_build_s": build_s,
        "e2e": {"value": e2e_it / e2e_s, "unit": "iter/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "time_to_eps_s": e2e_s / len(e2e_times),
                "status": e2e_status},
        "roofline": {"bound": "hbm", "kernel": "k_scs", "achieved": achieved, "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic,
                     "algorithmic_bytes_per_launch": statistics.mean(launch_bytes),
                     "launch_ms": 1e3 * statistics.mean(kern_s)},
        "cpu_baseline": cpu,
        "gpu_launches": 2 * args.steps,  # k_inner (setup) + k_scs (loop) per step
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = _args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
