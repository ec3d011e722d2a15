#!/usr/bin/env python
"""Benchmark of the B200 conegraph solver path (driver contract).

Default workload (BASELINE.json configs[1]): 1-D nonnegative deconvolution,
signal n = 1e6, Gaussian kernel length 101, stuffed exactly like the
reference's build_deconv (variables n+1, constraints 2n+k), solved to
eps = 1e-3.  ``--workload`` selects the other BASELINE configs (their lines
are evidence for DESIGN.md; the driver runs the default):
  lasso_dense   configs[0]  dense lasso A 1000 x 500, lam = 0.1
  deconv1d      configs[1]  (default)
  deconv2d      configs[2]  2-d nonneg deconvolution 4096 x 4096, 15 x 15 blur
  lasso_sparse  configs[3]  sparse lasso A 8e6 x 1e6 CSR, density 1e-5 (1 GPU)
  logreg        configs[4]  l1 logistic regression, 2 exp cones per sample, A 2e5 x 2e3
  soc_ls        configs[4]  SOC-constrained least squares, dense A 2e5 x 2e3

A *step* is one complete solve to eps from a cold start: the one-time
setup solve g = (I+Q_z)^{-1} h followed by the splitting iterations until
the device-latched status says solved.  ``value`` is ADMM (splitting)
iterations per second over the K timed steps with the problem data
resident in HBM (all ranks summed); ``time_to_eps_s`` is the mean step
time.  ``e2e`` is the same metric through the public API (``scs.solve`` on
numpy inputs: host->device copies, operator / cone compilation, setup,
solve, device->host copy of x, y, s) per step.

``--impl reference`` times the reference algorithm's CPU implementation
(the numpy restatement in oracle/, pinned to the real reference's golden
vectors) on the host cores: rank 0 only, a bounded sample of splitting
iterations of the same instance per step, same metric and unit.

Multi-GPU: these workloads are single structured operators, which the
north star keeps on one GPU, so N > 1 runs N independent replicas (one
solve per rank, no data-path collective; "scaling": "weak"); time is the
max over ranks of the per-rank device time.
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
METRIC = "ADMM iterations/s (time-to-eps=1e-3 in time_to_eps_s)"


# ---------------------------------------------------------------------------
# workloads (host-generated, bit-identical for both arms)
# ---------------------------------------------------------------------------

def _instance(n: int):
    """deconv1d instance (canon.gen_deconv1d's recipe: Gaussian kernel, 50
    nonnegative spikes, noise 0.01), generated on the host."""
    import numpy as np
    from paper_1609_03488_b200 import canon
    rng = np.random.default_rng(SEED)
    c = canon.gaussian_kernel(K_KERNEL)
    x_hat = np.zeros(n)
    pos = rng.choice(n, size=min(50, n), replace=False)
    x_hat[pos] = rng.uniform(0.0, 10.0, size=len(pos))
    b = np.convolve(c, x_hat) + canon.NOISE_SIGMA * rng.standard_normal(n + K_KERNEL - 1)
    return c, b, x_hat


class Workload:
    name = ""
    eps = EPS

    def config(self) -> dict:
        raise NotImplementedError

    def problem(self):
        """The stuffed cone problem through the public API, from host data."""
        raise NotImplementedError

    def h2d_bytes(self) -> int:
        raise NotImplementedError


class Deconv1D(Workload):
    name = "deconv1d_nonneg"

    def __init__(self, n: int):
        self.n = n
        self._d = None

    def data(self):
        if self._d is None:
            self._d = _instance(self.n)
        return self._d

    def config(self):
        return {"workload": self.name, "baseline_config": 1, "signal_n": self.n,
                "kernel_k": K_KERNEL, "eps": self.eps, "stuffed_n": self.n + 1,
                "stuffed_m": 2 * self.n + K_KERNEL, "seed": SEED}

    def problem(self):
        from paper_1609_03488_b200 import canon
        c, b, _ = self.data()
        return canon.build_deconv(canon.DeconvProblem(c, b, n=self.n))

    def h2d_bytes(self):
        n = self.n
        return 8 * (K_KERNEL + (n + K_KERNEL - 1)) + 8 * ((2 * n + K_KERNEL) + (n + 1))


class Deconv2D(Workload):
    name = "deconv2d_nonneg"

    def __init__(self, h: int = 4096, w: int = 4096, k: int = 15):
        self.h, self.w, self.k = h, w, k
        self._d = None

    def data(self):
        if self._d is None:
            import numpy as np
            import scipy.signal
            from paper_1609_03488_b200 import canon
            rng = np.random.default_rng(SEED)
            K = canon.gaussian_kernel2d(self.k, self.k)
            x = np.zeros(self.h * self.w)
            pos = rng.choice(self.h * self.w, size=200, replace=False)
            x[pos] = rng.uniform(0.0, 10.0, size=200)
            full = scipy.signal.fftconvolve(x.reshape(self.h, self.w), K, mode="full")
            b = full.reshape(-1) + canon.NOISE_SIGMA * rng.standard_normal(full.size)
            self._d = (K, b, x)
        return self._d

    def config(self):
        N = self.h * self.w
        M = (self.h + self.k - 1) * (self.w + self.k - 1)
        return {"workload": self.name, "baseline_config": 2, "image": [self.h, self.w],
                "kernel": [self.k, self.k], "eps": self.eps, "stuffed_n": N + 1,
                "stuffed_m": N + 1 + M, "seed": SEED}

    def problem(self):
        from paper_1609_03488_b200 import canon
        K, b, _ = self.data()
        return canon.build_deconv2d(canon.Deconv2DProblem(K, b, (self.h, self.w)))

    def h2d_bytes(self):
        N = self.h * self.w
        M = (self.h + self.k - 1) * (self.w + self.k - 1)
        return 8 * (self.k * self.k + M) + 8 * ((N + 1 + M) + (N + 1))


class LassoDense(Workload):
    name = "lasso_dense"

    def __init__(self, m: int = 1000, n: int = 500, lam: float = 0.1):
        self.m, self.n, self.lam = m, n, lam
        self._d = None

    def data(self):
        if self._d is None:
            import numpy as np
            rng = np.random.default_rng(SEED)
            A = rng.standard_normal((self.m, self.n))
            x = rng.standard_normal(self.n) * (rng.uniform(size=self.n) < 0.1)
            b = A @ x + 0.01 * rng.standard_normal(self.m)
            self._d = (A, b)
        return self._d

    def config(self):
        return {"workload": self.name, "baseline_config": 0, "A": [self.m, self.n],
                "lam": self.lam, "eps": self.eps, "stuffed_n": 2 * self.n + 1,
                "stuffed_m": 2 * self.n + self.m + 2, "seed": SEED}

    def problem(self):
        from paper_1609_03488_b200 import canon, linop
        A, b = self.data()
        return canon.build_lasso(canon.LassoProblem(linop.dense(A), b, self.lam))

    def h2d_bytes(self):
        return 8 * (self.m * self.n * 2 + self.m + 2 * self.n + self.m + 2)


class LassoSparse(Workload):
    name = "lasso_sparse"

    def __init__(self, m: int = 8_000_000, n: int = 1_000_000, density: float = 1e-5):
        self.m, self.n, self.density = m, n, density
        self._d = None

    def data(self):
        if self._d is None:
            import numpy as np
            import scipy.sparse
            rng = np.random.default_rng(SEED)
            nnz = int(self.m * self.n * self.density)
            rows = rng.integers(0, self.m, nnz)
            cols = rng.integers(0, self.n, nnz)
            # columns of unit expected norm, 1 % of x nonzero
            vals = rng.standard_normal(nnz) / np.sqrt(self.m * self.density)
            A = scipy.sparse.csc_matrix((vals, (rows, cols)), shape=(self.m, self.n))
            A.sum_duplicates()
            x = rng.standard_normal(self.n) * (rng.uniform(size=self.n) < 0.01)
            b = A @ x + 0.01 * rng.standard_normal(self.m) / np.sqrt(self.m * self.density)
            # the splitting method has no equilibration (scs.py design note):
            # scale the data to ||b|| = 10 so tau does not collapse at once
            # (the lasso solution is invariant under A, b -> sA, sb with
            # lam -> s^2 lam)
            sc = 10.0 / float(np.linalg.norm(b))
            A = A * sc
            b = b * sc
            lam = 0.1 * float(np.max(np.abs(A.T @ b)))
            self._d = (A.tocsc(), b, lam)
        return self._d

    def config(self):
        A, _, lam = self.data()
        return {"workload": self.name, "baseline_config": 3, "A": [self.m, self.n],
                "nnz": int(A.nnz), "lam": lam, "eps": self.eps,
                "stuffed_n": 2 * self.n + 1, "stuffed_m": 2 * self.n + self.m + 2,
                "seed": SEED, "sharding": "1 GPU (row-sharded multi-GPU path: DESIGN.md §8e)"}

    def problem(self):
        from paper_1609_03488_b200 import canon, linop
        A, b, lam = self.data()
        return canon.build_lasso(canon.LassoProblem(linop.sparse_csc(A), b, lam))

    def h2d_bytes(self):
        A, _, _ = self.data()
        return 12 * A.nnz + 8 * (self.n + 1) + 8 * (2 * self.m + 4 * self.n)


class LogReg(Workload):
    name = "logreg_exp"

    def __init__(self, m: int = 200_000, n: int = 2_000, lam: float = 0.01):
        self.m, self.n, self.lam = m, n, lam
        self._d = None

    def data(self):
        if self._d is None:
            from paper_1609_03488_b200 import canon
            A, y, _ = canon.gen_logreg(self.m, self.n, seed=SEED)
            self._d = (A, y)
        return self._d

    def config(self):
        from paper_1609_03488_b200 import canon
        ns, ms = canon.logreg_dims(self.m, self.n)
        return {"workload": self.name, "baseline_config": 4, "A": [self.m, self.n],
                "lam": self.lam, "exp_cones": 2 * self.m, "eps": self.eps, "stuffed_n": ns,
                "stuffed_m": ms, "seed": SEED}

    def problem(self):
        from paper_1609_03488_b200 import canon
        A, y = self.data()
        return canon.build_logreg(canon.LogRegProblem(A, y, self.lam))

    def h2d_bytes(self):
        from paper_1609_03488_b200 import canon
        ns, ms = canon.logreg_dims(self.m, self.n)
        return 8 * (2 * self.m * self.n) + 12 * 6 * self.m + 8 * (ns + ms)


class SocLs(Workload):
    name = "soc_ls"

    def __init__(self, m: int = 200_000, n: int = 2_000, radius: float = 1.0):
        self.m, self.n, self.radius = m, n, radius
        self._d = None

    def data(self):
        if self._d is None:
            import numpy as np
            rng = np.random.default_rng(SEED)
            A = rng.standard_normal((self.m, self.n)) / np.sqrt(self.m)
            b = A @ rng.standard_normal(self.n) + 0.1 * rng.standard_normal(self.m) / np.sqrt(self.m)
            self._d = (A, b)
        return self._d

    def config(self):
        return {"workload": self.name, "baseline_config": 4, "A": [self.m, self.n],
                "radius": self.radius, "eps": self.eps, "stuffed_n": self.n + 1,
                "stuffed_m": self.m + self.n + 2, "seed": SEED}

    def problem(self):
        from paper_1609_03488_b200 import canon, linop
        A, b = self.data()
        return canon.build_soc_ls(canon.SocLsProblem(linop.dense(A), b, self.radius))

    def h2d_bytes(self):
        return 8 * (2 * self.m * self.n + 2 * (self.m + self.n + 2) + self.n + 1)


def make_workload(args) -> Workload:
    if args.workload == "deconv1d":
        return Deconv1D(args.n)
    if args.workload == "deconv2d":
        return Deconv2D()
    if args.workload == "lasso_dense":
        return LassoDense()
    if args.workload == "lasso_sparse":
        return LassoSparse()
    if args.workload == "logreg":
        return LogReg()
    if args.workload == "soc_ls":
        return SocLs()
    raise SystemExit(f"unknown workload {args.workload}")


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="deconv1d",
                    choices=["deconv1d", "deconv2d", "lasso_dense", "lasso_sparse", "logreg",
                             "soc_ls"])
    ap.add_argument("--n", type=int, default=N_SIGNAL, help="deconv1d signal length")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=0,
                    help="splitting iterations per CPU sample (0 = workload default)")
    return ap.parse_args()


def _config(wl: Workload, n_gpus: int) -> dict:
    cfg = wl.config()
    cfg.update({"step": "one full solve to eps (setup solve + splitting iterations, cold start)",
                "l2": "flushed between timed steps (256 MiB write)",
                "parallelism": f"replicas{n_gpus}" if n_gpus > 1 else "single"})
    return cfg


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


def aggregate(total_s: float, total_iters: int, device=None) -> tuple[float, int]:
    """Whole-job numbers over the ranks of the default process group: the
    time is the max over ranks (per-rank device time), the work is summed."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return total_s, total_iters
    t = torch.tensor([float(total_s)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    it = torch.tensor([float(total_iters)], dtype=torch.float64, device=device)
    dist.all_reduce(it)
    return float(t.item()), int(it.item())


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# reference arm: the CPU implementation of the path (oracle port)
# ---------------------------------------------------------------------------

class _Tree:
    """The stuffed problem as a duck-typed tree the oracle walks."""

    def __init__(self, prob):
        self.A, self.b, self.c, self.K = prob.A.expr, prob.b, prob.c, prob.K


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


def _default_cpu_iters(wl: Workload) -> int:
    return {"deconv1d_nonneg": 20, "deconv2d_nonneg": 2, "lasso_dense": 200,
            "lasso_sparse": 3, "logreg_exp": 2, "soc_ls": 3}.get(wl.name, 10)


def _oracle_cached(wl: Workload, own_setup: bool):
    """The oracle's setup (its own solve when affordable, else the device's
    cached g -- the per-iteration work does not depend on it)."""
    import numpy as np
    from oracle import scs_ref
    p = _Tree(wl.problem())
    s = scs_ref.ScsOracleSettings(eps=wl.eps, max_iters=MAX_ITERS)
    if own_setup:
        t0 = time.perf_counter()
        cached = scs_ref.prepare_subspace(p, s.setup_cg_tol, s.cg_max_iter)
        return p, s, cached, time.perf_counter() - t0
    from paper_1609_03488_b200 import scs
    pc = scs.prepare_subspace(wl.problem(), s.setup_cg_tol, s.cg_max_iter)
    cached = scs_ref.Cached(np.asarray(pc.h), np.asarray(pc.g), float(pc.denom),
                            s.setup_cg_tol, s.cg_max_iter, int(pc.setup_cg_iters))
    return p, s, cached, None


def cpu_sample(wl: Workload, iters: int, warmup_iters: int = 1):
    """Time the oracle's splitting iterations on the host (setup excluded
    from the rate; reported separately when the oracle ran it)."""
    from oracle import scs_ref
    own = wl.name in ("deconv1d_nonneg", "lasso_dense")
    p, s, cached, setup_s = _oracle_cached(wl, own)
    it = scs_ref.iterate(p, s, cached, warmup_iters + iters)
    for _ in range(warmup_iters):
        next(it)
    t0 = time.perf_counter()
    done = 0
    for _k, _st in it:
        done += 1
    dt = time.perf_counter() - t0
    return {"setup_s": setup_s, "iters": done, "seconds": dt, "iters_per_s": done / dt}


def run_reference(args) -> None:
    world, rank, _ = _dist()
    if rank != 0:
        return
    wl = make_workload(args)
    iters = args.cpu_iters or max(1, _default_cpu_iters(wl) // 2)
    from oracle import scs_ref
    own = wl.name in ("deconv1d_nonneg", "lasso_dense")
    p, s, cached, setup_s = _oracle_cached(wl, own)
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
    setup_note = (f"after the oracle's own setup solve ({setup_s:.1f} s, untimed)"
                  if setup_s is not None else "from the device's cached setup solution")
    line = {
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "iter/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": _config(wl, 1),
        "setup_s": setup_s,
        "cpu_baseline": {"value": value, "unit": "iter/s", "cores": _cpu_cores_used(),
                         "kind": "port",
                         "sample": f"{iters} splitting iterations per step of the "
                                   f"{wl.name} instance {setup_note}; numpy restatement of "
                                   f"conegraph scs.py (FFT convolution as linop.py)"},
        "e2e": {"value": value, "unit": "iter/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def run_b200(args) -> None:
    import torch

    world, rank, local = _dist()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the B200 path has no CPU fallback)")
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1609_03488_b200 import _lib, scs

    wl = make_workload(args)
    settings = scs.ScsSettings(eps=wl.eps, max_iters=MAX_ITERS)

    # resident-data arm: compile once (graph build), then time setup + solve
    prob = wl.problem()
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
    total_s, total_iters = aggregate(sum(step_s), sum(iters), "cuda")
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
    tp = os.path.join(ROOT, "profiles", f"k_scs_traffic_{args.workload}.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            # the capture belongs to this build's launch only if the
            # trajectory (iteration and CG counts) is the same
            if tj.get("iterations") == iters[0] and tj.get("cg_total") == cgs[0]:
                traffic = tj.get("bytes_per_launch_at_bench")
        except Exception:  # noqa: BLE001
            traffic = None

    # end-to-end arm: public API on host (numpy) buffers, per step
    e2e = None
    if not args.no_e2e:
        e2e_times = []
        d2h = 0
        e2e_status = None
        pobj = None
        for step in range(1 + args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            if world > 1:
                torch.distributed.barrier()
            t0 = time.perf_counter()
            sol = scs.solve(wl.problem(), settings)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            d2h = 8 * (len(sol.x) + len(sol.y) + len(sol.s))
            e2e_status = sol.status
            pobj = sol.pobj
            if step >= 1:
                e2e_times.append((dt, sol.iterations))
        e2e_s, e2e_it = aggregate(sum(t for t, _ in e2e_times),
                                  sum(i for _, i in e2e_times), "cuda")
        e2e = {"value": e2e_it / e2e_s, "unit": "iter/s", "h2d_bytes_per_step": wl.h2d_bytes(),
               "d2h_bytes_per_step": d2h, "time_to_eps_s": e2e_s / len(e2e_times),
               "status": e2e_status, "pobj": pobj}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        iters_cpu = args.cpu_iters or _default_cpu_iters(wl)
        cs = cpu_sample(wl, iters_cpu)
        per_it = cs["seconds"] / cs["iters"]
        setup_note = (f"after the oracle's own setup solve ({cs['setup_s']:.1f} s)"
                      if cs["setup_s"] is not None else
                      "from the device's cached setup solution (the oracle's own setup "
                      "solve is outside the bounded sample)")
        cpu = {"value": cs["iters_per_s"], "unit": "iter/s", "cores": _cpu_cores_used(),
               "kind": "port",
               "sample": f"{cs['iters']} splitting iterations of the same {wl.name} instance "
                         f"{setup_note}; numpy restatement of conegraph scs.py (FFT "
                         f"convolutions single-threaded, dot products in OpenBLAS threads; "
                         f"host has {os.cpu_count()} cpus)",
               "setup_s": cs["setup_s"],
               "time_to_eps_s_extrapolated": (cs["setup_s"] or 0.0)
               + per_it * statistics.mean(iters)}

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": "iter/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(step_s),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": _config(wl, world),
        "time_to_eps_s": statistics.mean(step_s),
        "iterations_to_eps": iters[0], "avg_cg_iterations": cgs[0] / max(1, iters[0]),
        "status": sorted(statuses), "graph_build_s": build_s,
        "e2e": e2e,
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
