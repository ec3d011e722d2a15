"""Homogeneous self-dual embedding splitting solver on the B200.

Mirrors conegraph.scs (scs.py:1-576): ConeProblem, ScsSettings,
ScsIterate, ScsSolution, prepare_subspace, subspace_project, residuals,
build_scs_graph, iterate_states, solve_built, solve -- same arithmetic,
same statuses, same iteration semantics (status latched every
``check_interval`` iterations, CG warm-started from the previous p1 with
the graph's tolerance schedule).

Execution: ``build_scs_graph`` compiles the operator plans and cones and
runs the one-time setup solve g = (I+Q_z)^{-1} h on device; the splitting
loop then runs inside ONE persistent cooperative kernel (``cgb_scs_run``)
that keeps every iterate in HBM and takes all loop decisions on device:
the host does not synchronise per iteration, or per CG step, at all.
Final classification (scs.py:497-538) reads u, v back once and evaluates
the residuals with device operator applications.
"""

from __future__ import annotations

import ctypes
import json
import warnings
from dataclasses import dataclass
from typing import Iterator

import numpy as np

from . import _lib
from .cones import ConeProduct
from .linop import Operator

SOLVED = "solved"
INACCURATE = "inaccurate"
MAX_ITERS = "max-iters"
INFEASIBLE = "infeasible"
UNBOUNDED = "unbounded"

_STATUS_RUNNING = 0.0
_STATUS_SOLVED = 1.0
_STATUS_INFEASIBLE = 2.0
_STATUS_UNBOUNDED = 3.0

SMALL_TAU = 1e-12

# loop-variable order of iterate_states (matches the reference graph)
_IU, _IV, _IK, _ISINCE, _ISTATUS, _ICGW, _ICGT, _IRESID = range(8)


@dataclass
class ConeProblem:
    """Cone program data in the equality convention A x + s = b, s in K."""

    A: Operator
    b: np.ndarray
    c: np.ndarray
    K: ConeProduct

    def __post_init__(self) -> None:
        self.b = np.asarray(self.b, dtype=np.float64)
        self.c = np.asarray(self.c, dtype=np.float64)
        m, n = self.A.shape
        if self.b.shape != (m,):
            raise ValueError(f"b has shape {self.b.shape}, expected ({m},)")
        if self.c.shape != (n,):
            raise ValueError(f"c has shape {self.c.shape}, expected ({n},)")
        if self.K.total_dim != m:
            raise ValueError(f"cone product has dim {self.K.total_dim}, expected {m}")

    @property
    def dims(self) -> tuple[int, int]:
        return (self.A.cols, self.A.rows)


@dataclass
class ScsSettings:
    """Solver knobs (scs.py:84-118), same fields, defaults and validation."""

    eps: float = 1e-3
    max_iters: int = 5000
    check_interval: int = 20
    cg_base_tol: float = 1e-9
    cg_tol_cap: float = 0.1
    cg_tol_power: float = 1.25
    cg_eps_factor: float = 0.1
    cg_max_iter: int | None = None
    setup_cg_tol: float = 1e-12
    cert_tau_ratio: float = 1e-6

    def __post_init__(self) -> None:
        if self.eps <= 0:
            raise ValueError("eps must be positive")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.cg_tol_power not in (0.5, 1.0, 1.25, 1.5, 2.0):
            raise ValueError("cg_tol_power must be one of 0.5, 1.0, 1.25, 1.5, 2.0")

    def cg_tolerance(self, k: int) -> float:
        raw = max(1.0 / (k + 1) ** self.cg_tol_power, self.cg_eps_factor * self.eps)
        return max(self.cg_base_tol, min(self.cg_tol_cap, raw))

    def to_c(self, n: int) -> _lib.ScsSettingsC:
        cg_max = self.cg_max_iter if self.cg_max_iter is not None else 10 * n
        return _lib.ScsSettingsC(
            eps=self.eps, max_iters=int(self.max_iters), check_interval=int(self.check_interval),
            cg_base_tol=self.cg_base_tol, cg_tol_cap=self.cg_tol_cap,
            cg_tol_power=self.cg_tol_power, cg_eps_factor=self.cg_eps_factor,
            cg_max_iter=int(cg_max), cert_tau_ratio=self.cert_tau_ratio)


@dataclass
class ScsIterate:
    """Embedding iterates u = (x, y, tau), v = (0, s, kappa)."""

    u: np.ndarray
    v: np.ndarray


@dataclass
class ScsSolution:
    status: str
    x: np.ndarray
    y: np.ndarray
    s: np.ndarray
    pobj: float
    dobj: float
    primal_residual: float
    dual_residual: float
    gap: float
    iterations: int
    avg_cg_iterations: float


@dataclass
class TraceRecord:
    iteration: int
    primal: float
    dual: float
    gap: float
    cg_iters: int
    u: np.ndarray
    v: np.ndarray


def _own_device_op(op: Operator):
    """A DeviceOp whose forward plan is ``op``'s forward (never flipped)."""
    dev, flip = op.device_op()
    if flip:
        from ._plan import DeviceOp
        dev = DeviceOp(op.expr)
    return dev


def _cuda(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda")


# -- subspace projection (scs.py:155-214) -------------------------------------

@dataclass
class PrecomputedSolve:
    """Cached pieces of the (I+Q) solve: h = (c, b), g = (I+Q_z)^{-1} h.
    ``h`` and ``g`` are host copies made on first access (the solver uses
    the device copies; a solve never pays for the transfers)."""

    A: Operator
    _h: object
    _g: object
    denom: float
    cg_tol: float
    cg_max_iter: int | None
    setup_cg_iters: int = 0
    g_device: object = None
    c_device: object = None
    b_device: object = None

    @property
    def h(self) -> np.ndarray:
        if callable(self._h):
            self._h = self._h()
        return self._h

    @property
    def g(self) -> np.ndarray:
        if self._g is None:
            self._g = self.g_device.cpu().numpy()
        return self._g


def _inner_solve(dev, d1, d2, tol, max_iter, c_dev=None, b_dev=None):
    """Device [[I, A^T], [-A, I]] z = (d1, d2) (scs.py:170-187)."""
    import torch
    n, m = dev.cols, dev.rows
    z = torch.zeros(n + m, dtype=torch.float64, device="cuda")
    scratch = torch.empty(4 * n + 2 * m + 1, dtype=torch.float64, device="cuda")
    res = _lib.CgResult()
    hdot = ctypes.c_double(0.0)
    if max_iter is None:
        max_iter = 10 * n
    _lib.check(_lib.load_library().cgb_inner_solve(
        dev.ctx.handle, dev.handle, _lib.ptr(d1), _lib.ptr(d2), _lib.ptr(z), float(tol),
        int(max_iter), _lib.ptr(c_dev), _lib.ptr(b_dev), _lib.ptr(scratch), ctypes.byref(res),
        ctypes.byref(hdot), _lib.stream_handle()))
    if not res.converged:
        warnings.warn(
            f"inner CG stopped at residual {res.final_residual_norm:.3e} after "
            f"{res.iterations} iterations without reaching tolerance {tol:g}; the subspace "
            f"step is inaccurate", RuntimeWarning, stacklevel=3)
    return z, res, hdot.value


def prepare_subspace(problem: ConeProblem, cg_tol: float = 1e-12,
                     cg_max_iter: int | None = None) -> PrecomputedSolve:
    """One-time high-accuracy solve used by every later subspace step (scs.py:190-196)."""
    dev = _own_device_op(problem.A)
    c_d, b_d = _cuda(problem.c), _cuda(problem.b)
    z, res, hdot = _inner_solve(dev, c_d, b_d, cg_tol, cg_max_iter, c_d, b_d)
    c, b = problem.c, problem.b
    denom = 1.0 + hdot
    return PrecomputedSolve(problem.A, lambda: np.concatenate([c, b]), None, denom, cg_tol,
                            cg_max_iter, int(res.iterations), z, c_d, b_d)


def subspace_project(w, cached: PrecomputedSolve) -> np.ndarray:
    """Solve (I + Q) out = w with the cached rank-one reduction (scs.py:199-214)."""
    A = cached.A
    n, m = A.cols, A.rows
    w = np.asarray(w, dtype=np.float64)
    if w.shape != (n + m + 1,):
        raise ValueError(f"w has shape {w.shape}, expected ({n + m + 1},)")
    dev = _own_device_op(A)
    wd = _cuda(w)
    c_d = cached.c_device if cached.c_device is not None else _cuda(cached.h[:n])
    b_d = cached.b_device if cached.b_device is not None else _cuda(cached.h[n:])
    p, _, hdot = _inner_solve(dev, wd[:n], wd[n:n + m], cached.cg_tol, cached.cg_max_iter,
                              c_d, b_d)
    tau = (w[-1] + hdot) / cached.denom
    z = p.cpu().numpy() - tau * cached.g
    return np.concatenate([z, [tau]])


def residuals(iterate: ScsIterate, problem: ConeProblem) -> tuple[float, float, float]:
    """Relative primal/dual residuals and gap (scs.py:217-244), device applies."""
    A, b, c = problem.A, problem.b, problem.c
    n, m = A.cols, A.rows
    u, v = np.asarray(iterate.u), np.asarray(iterate.v)
    ux, uy, tau = u[:n], u[n:n + m], u[-1]
    vs = v[n:n + m]
    if tau > SMALL_TAU:
        x, y, s = ux / tau, uy / tau, vs / tau
        pr = np.linalg.norm(A.forward(x) + s - b) / (1.0 + np.linalg.norm(b))
        dr = np.linalg.norm(A.adjoint_apply(y) + c) / (1.0 + np.linalg.norm(c))
        ct, bt = float(c @ x), float(b @ y)
        gap = abs(ct + bt) / (1.0 + abs(ct) + abs(bt))
        return float(pr), float(dr), float(gap)
    den_u = -float(c @ ux)
    den_i = -float(b @ uy)
    pr = np.linalg.norm(A.forward(ux) + vs) / den_u if den_u > 0 else np.inf
    dr = np.linalg.norm(A.adjoint_apply(uy)) / den_i if den_i > 0 else np.inf
    return float(pr), float(dr), np.inf


def _nonzero_range(v: np.ndarray) -> tuple[int, int]:
    """[first, last + 1) of v's nonzeros ((0, 0) when v == 0)."""
    nz = np.flatnonzero(v)
    return (int(nz[0]), int(nz[-1]) + 1) if len(nz) else (0, 0)


# -- the compiled solver ("graph") ---------------------------------------------------

class SolverPlan:
    """What build_scs_graph returns: compiled plans, cones, setup solve and
    the device work buffers of the persistent splitting kernel."""

    def __init__(self, problem: ConeProblem, settings: ScsSettings):
        import torch
        self.problem = problem
        self.settings = settings
        self.n, self.m = problem.A.cols, problem.A.rows
        self.dev = _own_device_op(problem.A)
        self.cones = problem.K.device()
        self.cached = prepare_subspace(problem, settings.setup_cg_tol, settings.cg_max_iter)
        n, m = self.n, self.m
        N = n + m + 1
        f64 = dict(dtype=torch.float64, device="cuda")
        self.buf = {nm: torch.zeros(N, **f64) for nm in ("u", "v", "w")}
        for nm in ("cgx", "gx", "r", "p0", "p1", "q"):
            self.buf[nm] = torch.zeros(n, **f64)
        for nm in ("tax", "t"):
            self.buf[nm] = torch.zeros(m, **f64)
        self.buf["state"] = torch.zeros(_lib.STATE_LEN, **f64)
        self.work = _lib.ScsWorkC(**{nm: t.data_ptr() for nm, t in self.buf.items()})
        ca = self.cached
        self.cprob = _lib.ScsProblemC(
            n=n, m=m, A=self.dev.handle.value, K=self.cones.handle.value,
            b=ca.b_device.data_ptr(), c=ca.c_device.data_ptr(), g=ca.g_device.data_ptr(),
            denom=ca.denom, pr_scale=1.0 / (1.0 + float(np.linalg.norm(problem.b))),
            dr_scale=1.0 / (1.0 + float(np.linalg.norm(problem.c))))
        self.csettings = settings.to_c(n)
        self.reset()

    # the loop skips the loads of b and c outside their nonzero ranges (it
    # measures them itself); these host ranges are for bytes_model only
    @property
    def b_nz(self) -> tuple[int, int]:
        if getattr(self, "_b_nz", None) is None:
            self._b_nz = _nonzero_range(self.problem.b)
        return self._b_nz

    @property
    def c_nz(self) -> tuple[int, int]:
        if getattr(self, "_c_nz", None) is None:
            self._c_nz = _nonzero_range(self.problem.c)
        return self._c_nz

    def resetup(self) -> int:
        """Re-run the one-time setup solve g = (I+Q_z)^{-1} h on device into
        the resident g buffer (no host copy of g; one 8-byte read-back for
        denom).  Used by bench.py to time setup + solve with inputs resident.
        Returns the setup CG iteration count."""
        ca = self.cached
        z, res, hdot = _inner_solve(self.dev, ca.c_device, ca.b_device, self.settings.setup_cg_tol,
                                    self.settings.cg_max_iter, ca.c_device, ca.b_device)
        ca.g_device.copy_(z)
        ca.denom = 1.0 + hdot
        self.cprob.denom = ca.denom
        return int(res.iterations)

    def reset(self) -> None:
        """u = v = (0, 0, 1), w = u + v, warm start 0 (scs.py:448-458)."""
        for t in self.buf.values():
            t.zero_()
        self.buf["u"][-1] = 1.0
        self.buf["v"][-1] = 1.0
        self.buf["w"][-1] = 2.0

    def run(self, max_steps: int, resid_every_iter: bool = False) -> None:
        """Asynchronous: enqueue up to max_steps splitting iterations."""
        _lib.check(_lib.load_library().cgb_scs_run(
            self.dev.ctx.handle, ctypes.byref(self.cprob), ctypes.byref(self.csettings),
            ctypes.byref(self.work), int(max_steps), int(bool(resid_every_iter)),
            _lib.stream_handle()))

    def state(self) -> np.ndarray:
        return self.buf["state"].cpu().numpy()

    def host_uv(self) -> tuple[np.ndarray, np.ndarray]:
        """u, v on the host: one DMA each into page-locked buffers from
        torch's caching host allocator, handed out as numpy views (the
        buffers live as long as the arrays)."""
        import torch
        N = self.n + self.m + 1
        hu = torch.empty(N, dtype=torch.float64, pin_memory=True)
        hv = torch.empty(N, dtype=torch.float64, pin_memory=True)
        hu.copy_(self.buf["u"], non_blocking=True)
        hv.copy_(self.buf["v"], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return hu.numpy(), hv.numpy()

    PROFILE_PHASES = ("rhs", "cg_forward", "cg_adjoint_update", "cone_x", "cone_elem",
                      "cone_soc_a", "cone_soc_b", "check", "launch_setup", "cone_soc_a_reduce")

    def enable_profile(self, on: bool = True) -> None:
        """Accumulate per-phase device time of later run() calls (ns)."""
        import torch
        if on:
            self._prof = torch.zeros(48, dtype=torch.float64, device="cuda")
            ptr = _lib.ptr(self._prof)
        else:
            self._prof = None
            ptr = _lib.ptr(None)
        _lib.check(_lib.load_library().cgb_scs_profile(self.dev.ctx.handle, ptr))

    def profile(self) -> dict:
        """Seconds spent per phase since enable_profile()."""
        vals = self._prof.cpu().numpy() * 1e-9
        out = {nm: float(vals[i]) for i, nm in enumerate(self.PROFILE_PHASES)}
        tl = vals[16:24]
        out["rhs_warp0_timeline"] = {"tiles": float(tl[0] * 1e9), "tma_wait": float(tl[1]),
                                     "conv": float(tl[2]), "other_terms": float(tl[3]),
                                     "epilogue": float(tl[4]), "level_total": float(tl[5])}
        sv = vals[24:32]
        out["rhs_strip_timeline"] = {"batch_wait": float(sv[0]), "colpass": float(sv[1]),
                                     "colpass_barrier": float(sv[2]),
                                     "rowpass_terms_epilogue": float(sv[3]),
                                     "step_barrier_issue": float(sv[4]),
                                     "steps": float(sv[5] * 1e9), "tasks": float(sv[6] * 1e9)}
        return out

    def loop_vars(self) -> list:
        st = self.state()
        return [self.buf["u"].cpu().numpy(), self.buf["v"].cpu().numpy(),
                np.array([st[_lib.ST_K]]), np.array([st[_lib.ST_SINCE]]),
                np.array([st[_lib.ST_STATUS]]), self.buf["cgx"].cpu().numpy(),
                np.array([st[_lib.ST_CGT]]),
                np.array([st[_lib.ST_PR], st[_lib.ST_DR], st[_lib.ST_GAP]])]

    # algorithmic traffic model used by bench.py for the roofline (DESIGN.md
    # "Algorithmic bytes"): every array a phase needs is read once and every
    # array it produces is written once; operator applies count their
    # operand reads (input vector, matrix / CSR / kernel data, temporaries)
    # but not their raw output, which the fused epilogues consume in place.
    def bytes_model(self) -> dict:
        n, m, W = self.n, self.m, 8
        fr = self.dev.algo_bytes(False) - W * m   # forward operand reads
        ar = self.dev.algo_bytes(True) - W * n    # adjoint operand reads
        per_iter = (ar + W * (7 * n + 3 * m)      # rhs = w_x - A^T w_y, r0, h-dots
                    + W * 7 * m                   # cone step: 4 reads, 3 writes
                    + W * 6 * n)                  # free block: 3 reads, 3 writes
        per_cg = (fr + W * (2 * n + m)            # p = r + beta p fused into A p -> t
                  + ar + W * 2 * n                # q = p + A^T t, p.q
                  + W * (9 * n + 5 * m))          # x, r, A^T A x, A x updates + dots
        per_check = fr + ar + W * (3 * n + 4 * m)  # A u_x, A^T u_y, c.u_x, b.u_y
        # the loop skips b / c where they are zero (cgb_scs_problem.*_nz_*):
        # the rhs c read and the tracked c.p / b.t dots stream only the range
        skip = not (self.cprob.flags & _lib.SCS_NO_ZERO_SKIP)
        cz = n - (self.c_nz[1] - self.c_nz[0]) if skip else 0
        bz = m - (self.b_nz[1] - self.b_nz[0]) if skip else 0
        per_iter -= W * cz
        per_cg -= W * (cz + bz)
        return {"per_iter": per_iter, "per_cg_iter": per_cg, "per_check": per_check}

    def launch_flops(self, iterations: int, cg_total: int) -> int:
        """Algorithmic operator flops of one k_scs launch: one adjoint apply
        per iteration (rhs), a forward and an adjoint per CG step, both per
        residual check (the FP64 side of the roofline; the stream passes'
        few flops per element are not counted)."""
        ff, fa = self.dev.algo_flops(False), self.dev.algo_flops(True)
        checks = iterations // max(1, self.settings.check_interval)
        return iterations * fa + cg_total * (ff + fa) + checks * (ff + fa)

    def launch_bytes(self, iterations: int, cg_total: int) -> int:
        """Algorithmic bytes of one k_scs launch that ran ``iterations``
        splitting iterations and ``cg_total`` inner CG iterations from k=0."""
        bm = self.bytes_model()
        checks = iterations // max(1, self.settings.check_interval)
        return (iterations * bm["per_iter"] + cg_total * bm["per_cg_iter"]
                + checks * bm["per_check"])


def build_scs_graph(problem: ConeProblem, settings: ScsSettings | None = None) -> SolverPlan:
    """Compile the solver for ``problem`` (setup solve included; scs.py:433-469)."""
    settings = settings or ScsSettings()
    return SolverPlan(problem, settings)


def iterate_states(graph: SolverPlan, max_iters: int) -> Iterator[tuple[int, list]]:
    """Step the solver one splitting iteration at a time (scs.py:482-494).

    Yields (iteration, loop-variable list [u, v, k, since, status, cgw, cgt,
    resid]) after each iteration; every step is one device launch running
    exactly one iteration with the residual triple evaluated.
    """
    graph.reset()
    k = 0
    state = graph.loop_vars()
    while k < max_iters and state[_ISTATUS][0] == _STATUS_RUNNING:
        graph.run(1, resid_every_iter=True)
        k += 1
        state = graph.loop_vars()
        yield k, state


def _classify(problem: ConeProblem, settings: ScsSettings, u: np.ndarray, v: np.ndarray,
              iterations: int, cg_total: float, device_resid=None) -> ScsSolution:
    """scs.py:497-538.  ``device_resid`` = (pr, dr, gap, res_u, res_i) the
    loop evaluated on exactly this iterate (its last check), used instead
    of recomputing the residuals / certificate residuals with operator
    applies on host copies."""
    A, b, c = problem.A, problem.b, problem.c
    n, m = A.cols, A.rows
    tau, kappa = float(u[-1]), float(v[-1])
    ux, uy, vs = u[:n], u[n:n + m], v[n:n + m]
    avg_cg = cg_total / iterations if iterations > 0 else 0.0
    nan_n, nan_m = np.full(n, np.nan), np.full(m, np.nan)
    eps = settings.eps
    if tau > SMALL_TAU:
        x, y, s = ux / tau, uy / tau, vs / tau
        pr, dr, gap = (device_resid[:3] if device_resid is not None
                       else residuals(ScsIterate(u, v), problem))
        pobj, dobj = float(c @ x), -float(b @ y)
        if max(pr, dr, gap) <= eps:
            return ScsSolution(SOLVED, x, y, s, pobj, dobj, pr, dr, gap, iterations, avg_cg)
    else:
        pr = dr = gap = np.inf
        x = y = s = None
    den_i = -float(b @ uy)
    if den_i > 0:
        res_i = (device_resid[4] if device_resid is not None
                 else float(np.linalg.norm(A.adjoint_apply(uy))) / den_i)
        if tau < settings.cert_tau_ratio * max(kappa, 1.0) and res_i <= eps:
            return ScsSolution(INFEASIBLE, nan_n, uy / den_i, nan_m, np.nan, np.nan,
                               np.inf, res_i, np.inf, iterations, avg_cg)
    den_u = -float(c @ ux)
    if den_u > 0:
        res_u = (device_resid[3] if device_resid is not None
                 else float(np.linalg.norm(A.forward(ux) + vs)) / den_u)
        if tau < settings.cert_tau_ratio * max(kappa, 1.0) and res_u <= eps:
            return ScsSolution(UNBOUNDED, ux / den_u, nan_m, vs / den_u, np.nan, np.nan,
                               res_u, np.inf, np.inf, iterations, avg_cg)
    if x is None:
        return ScsSolution(MAX_ITERS, nan_n, nan_m, nan_m, np.nan, np.nan, pr, dr, gap,
                           iterations, avg_cg)
    status = INACCURATE if max(pr, dr, gap) <= 10.0 * eps else MAX_ITERS
    return ScsSolution(status, x, y, s, float(c @ x), -float(b @ y), pr, dr, gap,
                       iterations, avg_cg)


def solve_built(problem: ConeProblem, settings: ScsSettings, graph: SolverPlan,
                trace_path=None) -> ScsSolution:
    """Run a compiled solver to termination (scs.py:541-568)."""
    if trace_path is None:
        graph.reset()
        graph.run(settings.max_iters)
        st = graph.state()
        u, v = graph.host_uv()
        k = int(st[_lib.ST_K])
        # the loop's residual triple belongs to this iterate when its last
        # iteration was a check (k a multiple of check_interval; a latched
        # status always is one)
        fresh = k > 0 and k % settings.check_interval == 0
        resid = (float(st[_lib.ST_PR]), float(st[_lib.ST_DR]), float(st[_lib.ST_GAP]),
                 float(st[_lib.ST_RES_U]), float(st[_lib.ST_RES_I])) if fresh else None
        return _classify(problem, settings, u, v, k, float(st[_lib.ST_CGT]), resid)
    prev_cg = 0.0
    state = graph.loop_vars()
    with open(trace_path, "w") as fh:
        for k, state in iterate_states(graph, settings.max_iters):
            cg_now = float(state[_ICGT][0])
            pr, dr, gp = state[_IRESID]
            fh.write(json.dumps({"iteration": k, "primal": float(pr), "dual": float(dr),
                                 "gap": float(gp), "cg_iters": int(cg_now - prev_cg)}) + "\n")
            prev_cg = cg_now
    u, v = state[_IU], state[_IV]
    return _classify(problem, settings, u, v, int(state[_IK][0]), float(state[_ICGT][0]))


def solve(problem: ConeProblem, settings: ScsSettings | None = None,
          trace_path=None) -> ScsSolution:
    """Build the solver for ``problem`` and run it to termination (scs.py:571-576)."""
    settings = settings or ScsSettings()
    graph = build_scs_graph(problem, settings)
    return solve_built(problem, settings, graph, trace_path)
