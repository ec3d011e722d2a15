#!/usr/bin/env python
"""Benchmark of the B200 conegraph solver path (driver contract).

Default workload (BASELINE.json configs[2], the config the north star's
>= 50x time-to-eps target is quoted on): 2-D nonnegative image
deconvolution, 4096 x 4096 image, 15 x 15 Gaussian blur, stuffed like the
reference's build_deconv (variables N+1, constraints N+1+(4110^2)), eps =
1e-3.  ``--workload`` selects the other BASELINE configs:
  deconv2d      configs[2]  (default)
  lasso_dense   configs[0]  dense lasso A 1000 x 500, lam = 0.1
  deconv1d      configs[1]  1-d nonneg deconvolution, n = 1e6, kernel 101
  lasso_sparse  configs[3]  sparse lasso A 8e6 x 1e6 CSR, density 1e-5;
                            with --gpus N the rows of A are sharded over N ranks
  logreg        configs[4]  l1 logistic regression, 2 exp cones per sample, A 2e5 x 2e3
  soc_ls        configs[4]  SOC-constrained least squares, dense A 2e5 x 2e3

A *step* is one cold start of the solver with the problem data resident in
HBM: the one-time setup solve g = (I+Q_z)^{-1} h, then the splitting
iterations from u = v = (0, 0, 1) -- either to eps (small workloads) or a
bounded block of ``step_iters`` iterations (deconv2d: 2000 of the ~9e4 to
eps, so K steps fit the driver's step limit).  ``value`` is ADMM
(splitting) iterations per second over the K timed steps (all ranks
summed, time = max over ranks).  ``time_to_eps_s`` is measured once, by one
full cold solve to eps after the timed steps.  ``e2e`` is the same metric
through the public API (``scs.solve`` on numpy inputs: host->device copies,
operator / cone compilation, setup, the same bounded iterations, and the
device->host copy of x, y, s) per step.

``--impl reference`` times the reference algorithm's CPU implementation
(the numpy restatement in oracle/, pinned to the real reference's golden
vectors; the problem is stuffed by oracle/canon_ref.py, nothing of the
product is imported) on the host cores: rank 0 only, after the oracle's
own setup solve (untimed), each step a bounded block of splitting
iterations of the same instance, same metric and unit.

Multi-GPU: lasso_sparse is row-sharded over the ranks;
the single-operator workloads are kept on one GPU by the north star, so
N > 1 runs N independent replicas of them (no data-path collective).
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

EPS = 1e-3
MAX_ITERS = 200_000
SEED = 0
NOISE_SIGMA = 0.01
METRIC = "ADMM iterations/s (time-to-eps=1e-3 in time_to_eps_s)"
N_SIGNAL = 1_000_000
K_KERNEL = 101


# ---------------------------------------------------------------------------
# data generators (numpy only; the same arithmetic as canon.gaussian_kernel,
# canon.gaussian_kernel2d and canon.gen_logreg -- tests/test_host.py checks
# they agree -- so the reference arm needs nothing from the product)
# ---------------------------------------------------------------------------

def gaussian_kernel(n: int) -> np.ndarray:
    """Centered Gaussian kernel of length n, std n/10, unit sum (canon.py:135-139)."""
    i = np.arange(n, dtype=np.float64)
    k = np.exp(-((i - n / 2.0) ** 2) / (2.0 * (n / 10.0) ** 2))
    return k / k.sum()


def gaussian_kernel2d(kh: int, kw: int) -> np.ndarray:
    """Separable centered Gaussian blur (std k/6 per axis), unit sum."""
    def axis(k):
        i = np.arange(k, dtype=np.float64)
        return np.exp(-((i - (k - 1) / 2.0) ** 2) / (2.0 * (k / 6.0) ** 2))
    K = np.outer(axis(kh), axis(kw))
    return K / K.sum()


def gen_logreg(m: int, n: int, seed: int, density: float = 0.1):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, n)) / np.sqrt(n)
    w = rng.standard_normal(n) * (rng.uniform(size=n) < density) * 3.0
    pr = 1.0 / (1.0 + np.exp(-(A @ w)))
    y = np.where(rng.uniform(size=m) < pr, 1.0, -1.0)
    return A, y, w


def _instance(n: int):
    """deconv1d instance: Gaussian kernel 101, 50 nonnegative spikes, noise 0.01."""
    rng = np.random.default_rng(SEED)
    c = gaussian_kernel(K_KERNEL)
    x_hat = np.zeros(n)
    pos = rng.choice(n, size=min(50, n), replace=False)
    x_hat[pos] = rng.uniform(0.0, 10.0, size=len(pos))
    b = np.convolve(c, x_hat) + NOISE_SIGMA * rng.standard_normal(n + K_KERNEL - 1)
    return c, b, x_hat


# ---------------------------------------------------------------------------
# workloads (host-generated, bit-identical for both arms)
# ---------------------------------------------------------------------------

class Workload:
    name = ""
    baseline_config = -1
    eps = EPS
    step_iters = 0   # 0: a step runs to eps; else a bounded block of iterations
    cpu_iters = 2    # splitting iterations of the bench's cpu_baseline sample
    ref_iters = 1    # splitting iterations per --impl reference step

    def config(self) -> dict:
        raise NotImplementedError

    def problem(self):
        """The stuffed cone problem through the product's public API."""
        raise NotImplementedError

    def oracle_problem(self):
        """The same stuffed problem built by oracle/canon_ref.py."""
        raise NotImplementedError

    def h2d_bytes(self) -> int:
        raise NotImplementedError


class Deconv1D(Workload):
    name = "deconv1d_nonneg"
    baseline_config = 1
    cpu_iters = 20
    ref_iters = 10

    def __init__(self, n: int = N_SIGNAL):
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

    def oracle_problem(self):
        from oracle import canon_ref
        c, b, _ = self.data()
        return canon_ref.build_deconv(c, b, self.n)

    def h2d_bytes(self):
        n = self.n
        return 8 * (K_KERNEL + (n + K_KERNEL - 1)) + 8 * ((2 * n + K_KERNEL) + (n + 1))


class Deconv2D(Workload):
    name = "deconv2d_nonneg"
    baseline_config = 2
    step_iters = 2000
    cpu_iters = 2
    ref_iters = 1

    def __init__(self, h: int = 4096, w: int = 4096, k: int = 15):
        self.h, self.w, self.k = h, w, k
        self._d = None

    def data(self):
        if self._d is None:
            import scipy.signal
            rng = np.random.default_rng(SEED)
            K = gaussian_kernel2d(self.k, self.k)
            x = np.zeros(self.h * self.w)
            pos = rng.choice(self.h * self.w, size=200, replace=False)
            x[pos] = rng.uniform(0.0, 10.0, size=200)
            full = scipy.signal.fftconvolve(x.reshape(self.h, self.w), K, mode="full")
            b = full.reshape(-1) + NOISE_SIGMA * rng.standard_normal(full.size)
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

    def oracle_problem(self):
        from oracle import canon_ref
        K, b, _ = self.data()
        return canon_ref.build_deconv2d(K, b, (self.h, self.w))

    def h2d_bytes(self):
        N = self.h * self.w
        M = (self.h + self.k - 1) * (self.w + self.k - 1)
        return 8 * (self.k * self.k + M) + 8 * ((N + 1 + M) + (N + 1))


class LassoDense(Workload):
    name = "lasso_dense"
    baseline_config = 0
    cpu_iters = 200
    ref_iters = 50

    def __init__(self, m: int = 1000, n: int = 500, lam: float = 0.1):
        self.m, self.n, self.lam = m, n, lam
        self._d = None

    def data(self):
        if self._d is None:
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

    def oracle_problem(self):
        from oracle import canon_ref
        from oracle.exprs_ref import DenseMatrix
        A, b = self.data()
        return canon_ref.build_lasso(DenseMatrix(A), b, self.lam)

    def h2d_bytes(self):
        return 8 * (self.m * self.n * 2 + self.m + 2 * self.n + self.m + 2)


class LassoSparse(Workload):
    name = "lasso_sparse"
    baseline_config = 3
    cpu_iters = 3
    ref_iters = 1

    def __init__(self, m: int = 8_000_000, n: int = 1_000_000, density: float = 1e-5):
        self.m, self.n, self.density = m, n, density
        self._d = None

    def data(self):
        if self._d is None:
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
                "seed": SEED}

    def problem(self):
        from paper_1609_03488_b200 import canon, linop
        A, b, lam = self.data()
        return canon.build_lasso(canon.LassoProblem(linop.sparse_csc(A), b, lam))

    def oracle_problem(self):
        from oracle import canon_ref
        from oracle.exprs_ref import SparseMatrix
        A, b, lam = self.data()
        return canon_ref.build_lasso(SparseMatrix(A), b, lam)

    def h2d_bytes(self):
        A, _, _ = self.data()
        return 12 * A.nnz + 8 * (self.n + 1) + 8 * (2 * self.m + 4 * self.n)


class LogReg(Workload):
    name = "logreg_exp"
    baseline_config = 4
    cpu_iters = 2
    ref_iters = 1

    def __init__(self, m: int = 200_000, n: int = 2_000, lam: float = 0.01):
        self.m, self.n, self.lam = m, n, lam
        self._d = None

    def data(self):
        if self._d is None:
            A, y, _ = gen_logreg(self.m, self.n, seed=SEED)
            self._d = (A, y)
        return self._d

    def dims(self):
        return 2 * self.n + 3 * self.m, 2 * self.n + self.m + 6 * self.m

    def config(self):
        ns, ms = self.dims()
        return {"workload": self.name, "baseline_config": 4, "A": [self.m, self.n],
                "lam": self.lam, "exp_cones": 2 * self.m, "eps": self.eps, "stuffed_n": ns,
                "stuffed_m": ms, "seed": SEED}

    def problem(self):
        from paper_1609_03488_b200 import canon
        A, y = self.data()
        return canon.build_logreg(canon.LogRegProblem(A, y, self.lam))

    def oracle_problem(self):
        from oracle import canon_ref
        A, y = self.data()
        return canon_ref.build_logreg(A, y, self.lam)

    def h2d_bytes(self):
        ns, ms = self.dims()
        return 8 * (2 * self.m * self.n) + 12 * 6 * self.m + 8 * (ns + ms)


class SocLs(Workload):
    name = "soc_ls"
    baseline_config = 4
    cpu_iters = 3
    ref_iters = 2

    def __init__(self, m: int = 200_000, n: int = 2_000, radius: float = 1.0):
        self.m, self.n, self.radius = m, n, radius
        self._d = None

    def data(self):
        if self._d is None:
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

    def oracle_problem(self):
        from oracle import canon_ref
        from oracle.exprs_ref import DenseMatrix
        A, b = self.data()
        return canon_ref.build_soc_ls(DenseMatrix(A), b, self.radius)

    def h2d_bytes(self):
        return 8 * (2 * self.m * self.n + 2 * (self.m + self.n + 2) + self.n + 1)


WORKLOADS = {"deconv2d": Deconv2D, "deconv1d": Deconv1D, "lasso_dense": LassoDense,
             "lasso_sparse": LassoSparse, "logreg": LogReg, "soc_ls": SocLs}


def make_workload(args) -> Workload:
    if args.workload == "deconv1d":
        return Deconv1D(args.n)
    if args.workload in WORKLOADS:
        return WORKLOADS[args.workload]()
    raise SystemExit(f"unknown workload {args.workload}")


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="deconv2d", choices=sorted(WORKLOADS))
    ap.add_argument("--n", type=int, default=N_SIGNAL, help="deconv1d signal length")
    ap.add_argument("--step-iters", type=int, default=-1,
                    help="splitting iterations per step (0 = to eps; default per workload)")
    ap.add_argument("--shards", type=int, default=1,
                    help="lasso_sparse on one GPU: ranks of the sharded solver sharing it")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-full-solve", action="store_true",
                    help="skip the one full solve that measures time_to_eps_s")
    ap.add_argument("--cpu-iters", type=int, default=0,
                    help="splitting iterations per CPU sample (0 = workload default)")
    return ap.parse_args()


def _step_iters(args, wl: Workload) -> int:
    return wl.step_iters if args.step_iters < 0 else args.step_iters


def _config(wl: Workload, n_gpus: int, step_iters: int, parallelism: str | None = None) -> dict:
    cfg = wl.config()
    if step_iters > 0:
        step = (f"one cold start: setup solve + {step_iters} splitting iterations "
                f"(bounded; time to eps from one full solve, time_to_eps_s)")
    else:
        step = "one full solve to eps (setup solve + splitting iterations, cold start)"
    cfg.update({"step": step, "step_iters": step_iters,
                "l2": "flushed between timed steps (256 MiB write); every iterate vector "
                      "exceeds L2 as well" if step_iters else
                      "flushed between timed steps (256 MiB write)",
                "parallelism": parallelism or (f"replicas{n_gpus} (independent solves, no "
                                               f"data-path collective)" if n_gpus > 1
                                               else "single")})
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


def _peaks() -> dict:
    """HBM peak from the driver's MEASURED_PEAKS.json and the measured FP64
    DFMA peak (profiles/fp64_peak.json, tools/fp64_peak.cu), with fallbacks."""
    out = {"hbm_gbs": 6650.0, "hbm_src": "fallback (B200_PROFILING.md)",
           "fp64_tflops": 37.0, "fp64_src": "fallback (nominal B200 FP64 vector)"}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            out["hbm_gbs"] = float(json.load(open(p))["hbm_gbs"])
            out["hbm_src"] = "measured (MEASURED_PEAKS.json)"
        except Exception:  # noqa: BLE001
            pass
    p = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(p):
        try:
            out["fp64_tflops"] = float(json.load(open(p))["dfma_tflops"])
            out["fp64_src"] = "measured (profiles/fp64_peak.json)"
        except Exception:  # noqa: BLE001
            pass
    return out


# ---------------------------------------------------------------------------
# reference arm: the CPU implementation of the path (oracle port)
# ---------------------------------------------------------------------------

def _cpu_threads() -> int:
    return os.cpu_count() or 1


class _OracleRun:
    """The oracle's own setup solve and splitting loop on one workload
    (problem stuffed by oracle/canon_ref.py: no product code involved)."""

    def __init__(self, wl: Workload):
        import scipy.fft
        from oracle import scs_ref
        self.scs_ref = scs_ref
        self.workers = scipy.fft.set_workers(_cpu_threads())
        self.workers.__enter__()   # scipy FFTs (2-d convolutions) on every host core
        self.p = wl.oracle_problem()
        self.s = scs_ref.ScsOracleSettings(eps=wl.eps, max_iters=MAX_ITERS)
        t0 = time.perf_counter()
        self.cached = scs_ref.prepare_subspace(self.p, self.s.setup_cg_tol, self.s.cg_max_iter)
        self.setup_s = time.perf_counter() - t0
        self.it = scs_ref.iterate(self.p, self.s, self.cached, MAX_ITERS)

    def run(self, iters: int) -> float:
        t0 = time.perf_counter()
        for _ in range(iters):
            next(self.it)
        return time.perf_counter() - t0


def _oracle_full_solve_record(wl: Workload) -> dict | None:
    """The oracle's own full solve of this exact instance, when one was run
    (profiles/oracle_full_solves.json)."""
    p = os.path.join(ROOT, "profiles", "oracle_full_solves.json")
    if not os.path.exists(p):
        return None
    try:
        return json.load(open(p)).get(wl.name)
    except Exception:  # noqa: BLE001
        return None


def run_reference(args) -> None:
    world, rank, _ = _dist()
    if rank != 0:
        return
    wl = make_workload(args)
    iters = args.cpu_iters or wl.ref_iters
    orc = _OracleRun(wl)
    for _ in range(args.warmup):
        orc.run(iters)
    times = [orc.run(iters) for _ in range(args.steps)]
    total = sum(times)
    value = iters * len(times) / total
    line = {
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "iter/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": _config(wl, 1, _step_iters(args, wl)),
        "setup_s": orc.setup_s,
        "cpu_baseline": {"value": value, "unit": "iter/s", "cores": _cpu_threads(),
                         "kind": "port",
                         "sample": f"{iters} splitting iteration(s) per step of the {wl.name} "
                                   f"instance after the oracle's own setup solve "
                                   f"({orc.setup_s:.1f} s, untimed); numpy restatement of "
                                   f"conegraph scs.py (oracle/scs_ref.py), problem stuffed by "
                                   f"oracle/canon_ref.py; BLAS and scipy FFTs on "
                                   f"{_cpu_threads()} host threads"},
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
    if args.workload == "lasso_sparse" and (world > 1 or args.shards > 1):
        return run_b200_sharded(args)
    from paper_1609_03488_b200 import _lib, scs

    wl = make_workload(args)
    S = _step_iters(args, wl)
    cap = S if S > 0 else MAX_ITERS
    settings = scs.ScsSettings(eps=wl.eps, max_iters=MAX_ITERS)

    # resident-data arm: compile once (graph build), then time setup + loop
    prob = wl.problem()
    t0 = time.perf_counter()
    plan = scs.build_scs_graph(prob, settings)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def one_step(max_steps: int):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(stream)
        plan.resetup()
        plan.reset()
        ev[1].record(stream)
        plan.run(max_steps)
        ev[2].record(stream)
        torch.cuda.synchronize()
        st = plan.state()
        return (ev[0].elapsed_time(ev[2]) / 1e3, ev[1].elapsed_time(ev[2]) / 1e3,
                int(st[_lib.ST_K]), int(st[_lib.ST_CGT]), float(st[_lib.ST_STATUS]))

    for _ in range(args.warmup):
        flush.zero_()
        one_step(cap)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    results = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            results.append(one_step(cap))
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

    # time to eps: one full cold solve (outside the timed steps when bounded)
    if S > 0 and not args.no_full_solve:
        flush.zero_()
        torch.cuda.synchronize()
        full = one_step(MAX_ITERS)
    else:
        full = results[0] if S == 0 else None
    tte = None
    if full is not None:
        tte = {"time_to_eps_s": full[0] if S > 0 else statistics.mean(step_s),
               "iterations_to_eps": full[2], "cg_iterations": full[3],
               "status": {1.0: "solved", 2.0: "infeasible", 3.0: "unbounded"}.get(
                   full[4], "not converged"),
               "loop_s": full[1]}

    # roofline of the dominant kernel (k_scs: the splitting loop)
    peaks = _peaks()
    launch_bytes = [plan.launch_bytes(i, c_) for i, c_ in zip(iters, cgs)]
    launch_flops = [plan.launch_flops(i, c_) for i, c_ in zip(iters, cgs)]
    achieved = sum(launch_bytes) / sum(kern_s) / 1e9
    fp64_tflops = sum(launch_flops) / sum(kern_s) / 1e12
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
        e2e_settings = scs.ScsSettings(eps=wl.eps, max_iters=cap)
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
            sol = scs.solve(wl.problem(), e2e_settings)
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
               "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * e2e_s / len(e2e_times),
               "iterations_per_step": e2e_times[0][1], "status": e2e_status,
               "pobj": pobj}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        iters_cpu = args.cpu_iters or wl.cpu_iters
        orc = _OracleRun(wl)
        orc.run(1)
        dt = orc.run(iters_cpu)
        per_it = dt / iters_cpu
        rec = _oracle_full_solve_record(wl)
        cpu = {"value": iters_cpu / dt, "unit": "iter/s", "cores": _cpu_threads(),
               "kind": "port",
               "sample": f"{iters_cpu} splitting iterations (after 1 untimed) of the same "
                         f"{wl.name} instance after the oracle's own setup solve "
                         f"({orc.setup_s:.1f} s); numpy restatement of conegraph scs.py "
                         f"(oracle/scs_ref.py), problem stuffed by oracle/canon_ref.py; BLAS "
                         f"and scipy FFTs on {_cpu_threads()} host threads",
               "setup_s": orc.setup_s}
        if rec is not None:
            cpu["time_to_eps_s_measured"] = rec.get("seconds")
            cpu["iterations_to_eps_oracle"] = rec.get("iterations")
            cpu["measured_where"] = rec.get("where")
        if tte is not None:
            basis = rec.get("iterations") if rec else tte["iterations_to_eps"]
            cpu["time_to_eps_s_extrapolated"] = orc.setup_s + per_it * basis
            cpu["extrapolation_basis"] = ("the oracle's own iteration count to eps "
                                          "(profiles/oracle_full_solves.json)" if rec else
                                          "the device's iteration count (the oracle's own "
                                          "full solve is infeasible at this size)")

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": "iter/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(step_s),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": _config(wl, world, S),
        "time_to_eps_s": tte["time_to_eps_s"] if tte else None,
        "iterations_to_eps": tte["iterations_to_eps"] if tte else None,
        "full_solve": tte,
        "iterations_per_step": iters[0], "avg_cg_iterations": cgs[0] / max(1, iters[0]),
        "status": sorted(statuses), "graph_build_s": build_s,
        "e2e": e2e,
        "roofline": {"bound": "hbm", "kernel": "k_scs", "achieved": achieved,
                     "peak": peaks["hbm_gbs"], "peak_source": peaks["hbm_src"],
                     "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                     "traffic": traffic,
                     "algorithmic_bytes_per_launch": statistics.mean(launch_bytes),
                     "launch_ms": 1e3 * statistics.mean(kern_s),
                     "fp64": {"achieved": fp64_tflops, "peak": peaks["fp64_tflops"],
                              "peak_source": peaks["fp64_src"], "unit": "TFLOP/s",
                              "frac": fp64_tflops / peaks["fp64_tflops"],
                              "algorithmic_flops_per_launch": statistics.mean(launch_flops)}},
        "cpu_baseline": cpu,
        "gpu_launches": 2 * args.steps,  # k_inner (setup) + k_scs (loop) per step
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_b200_sharded(args) -> None:
    """configs[3] row-sharded (paper_1609_03488_b200/shard.py).

    Under torchrun: one rank per GPU, peer buffers mapped by CUDA IPC, the
    whole job is ONE solve (strong scaling): value = iterations / max over
    ranks of the device time.  With --shards R on a single process: R ranks
    sharing this GPU (each 1/R of the SMs) -- the sharded kernel's cost,
    not a scaling number."""
    import torch
    from paper_1609_03488_b200 import _lib, scs, shard

    world, rank, local = _dist()
    wl = make_workload(args)
    S = _step_iters(args, wl)
    cap = S if S > 0 else MAX_ITERS
    settings = scs.ScsSettings(eps=wl.eps, max_iters=MAX_ITERS)
    prob = wl.problem()
    stream = torch.cuda.current_stream()
    t0 = time.perf_counter()
    if world > 1:
        lay = shard.layout_for(prob, world, rank)
        rs = shard.RankSolver(prob, settings, lay, local, ipc=True)
        shard.connect_ipc(rs)
        ranks = [rs]
        parallelism = f"row-sharded over {world} GPUs (NVLink peer memory)"

        def launch(mode, steps):
            rs.launch(mode, steps, stream)
    else:
        grp = shard.ShardGroup(prob, settings, world=args.shards)
        ranks = grp.ranks
        parallelism = (f"row-sharded: {args.shards} ranks sharing one GPU "
                       f"({grp.ranks[0].ctx.geometry()[0] // args.shards} SMs each)")

        def launch(mode, steps):
            grp._all(mode, steps)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def one_step(max_steps):
        for r in ranks:
            r.reset()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        ev[0].record(stream)
        launch(0, 0)
        launch(1, max_steps)
        ev[1].record(stream)
        torch.cuda.synchronize()
        st = ranks[0].state()
        return ev[0].elapsed_time(ev[1]) / 1e3, int(st[_lib.ST_K]), int(st[_lib.ST_CGT]), \
            float(st[_lib.ST_STATUS])

    for _ in range(args.warmup):
        flush.zero_()
        one_step(cap)
    results = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            results.append(one_step(cap))
    tot = sum(r[0] for r in results)
    if world > 1:
        t = torch.tensor([tot], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        tot = float(t.item())
    iters = sum(r[1] for r in results)     # one solve for the whole job: not summed
    value = iters / tot
    e2e = None
    if not args.no_e2e and world > 1:
        e2e_t = []
        for step in range(1 + args.steps):
            torch.cuda.synchronize()
            torch.distributed.barrier()
            t1 = time.perf_counter()
            sol, rsx = shard.solve_sharded(wl.problem(), scs.ScsSettings(eps=wl.eps,
                                                                         max_iters=cap))
            torch.cuda.synchronize()
            dt = torch.tensor([time.perf_counter() - t1], dtype=torch.float64, device="cuda")
            torch.distributed.all_reduce(dt, op=torch.distributed.ReduceOp.MAX)
            it = int(rsx.state()[_lib.ST_K])
            rsx.close()
            if step >= 1:
                e2e_t.append((float(dt.item()), it))
        e2e = {"value": sum(i for _, i in e2e_t) / sum(t for t, _ in e2e_t), "unit": "iter/s",
               "h2d_bytes_per_step": wl.h2d_bytes(),
               "d2h_bytes_per_step": 8 * (2 * prob.A.rows + prob.A.cols),
               "ms_per_step": 1e3 * sum(t for t, _ in e2e_t) / len(e2e_t)}
    if rank != 0:
        torch.distributed.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": "iter/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(results),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": _config(wl, world, S, parallelism),
        "iterations_per_step": results[0][1],
        "avg_cg_iterations": results[0][2] / max(1, results[0][1]),
        "status": sorted({r[3] for r in results}), "graph_build_s": build_s,
        "ranks": [{"rows": [r.lay.y0, r.lay.y1], "x_slice": [r.lay.x0, r.lay.x1]}
                  for r in ranks] if world == 1 else None,
        "e2e": e2e, "cpu_baseline": None,
        "gpu_launches": 2 * args.steps * (args.shards if world == 1 else 1),
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
