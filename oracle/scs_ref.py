"""numpy restatement of the reference SCS solver path (TEST ORACLE ONLY).

The reference emits the iteration as a computation graph and evaluates
it node by node; this file restates the SAME arithmetic as a direct loop
so it can serve as the parity checker and the CPU baseline:

  ScsOracleSettings.cg_tolerance   scs.py:116-118 (host form)
  _cg_tolerance_graph              scs.py:290-311 (graph form, used in-loop)
  prepare_subspace                 scs.py:170-196
  subspace_project                 scs.py:199-214
  residuals                        scs.py:217-244
  _body                            scs.py:314-413 (_emit_body)
  loop condition                   scs.py:416-430 (_emit_cond)
  classify                         scs.py:497-538 (_classify)
  scs_solve                        scs.py:433-469 + 541-576

``problem`` is duck-typed: .A (expression tree), .b, .c, .K.factors.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .cg_ref import cg, normal_apply
from .cones_ref import project_dual_product
from .linop_ref import adjoint, forward

SMALL_TAU = 1e-12  # scs.py:51


@dataclass
class ScsOracleSettings:
    """scs.py:84-118 (same fields and defaults as ScsSettings)."""

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

    def cg_tolerance(self, k: int) -> float:
        raw = max(1.0 / (k + 1) ** self.cg_tol_power, self.cg_eps_factor * self.eps)
        return max(self.cg_base_tol, min(self.cg_tol_cap, raw))


def _cg_tolerance_graph(k: float, s: ScsOracleSettings) -> float:
    """scs.py:290-311 -- the tolerance exactly as the graph computes it."""
    kp1 = k + 1.0
    pw = s.cg_tol_power
    if pw == 0.5:
        den = np.sqrt(kp1)
    elif pw == 1.0:
        den = kp1
    elif pw == 1.25:
        den = kp1 * np.sqrt(np.sqrt(kp1))
    elif pw == 1.5:
        den = kp1 * np.sqrt(kp1)
    else:
        den = kp1 * kp1
    tol_raw = 1.0 / den
    sat = s.cg_eps_factor * s.eps
    cap = s.cg_tol_cap
    base = s.cg_base_tol
    tol_sat = sat + max(tol_raw - sat, 0.0)
    tol_capped = cap - max(cap - tol_sat, 0.0)
    return base + max(tol_capped - base, 0.0)


@dataclass
class Cached:
    """scs.py:158-167 (PrecomputedSolve)."""

    h: np.ndarray
    g: np.ndarray
    denom: float
    cg_tol: float
    cg_max_iter: int | None
    setup_cg_iters: int = 0


def _solve_inner_block(A, d1, d2, tol, max_iter, x0=None):
    """scs.py:170-187 -- [[I, A^T], [-A, I]] z = (d1, d2) via CG on I + A^T A."""
    n = A.cols
    rhs = d1 - adjoint(A, d2)
    if x0 is None:
        x0 = np.zeros(n)
    if max_iter is None:
        max_iter = 10 * len(rhs)
    delta = tol * float(np.linalg.norm(rhs))
    z1, k, rns = cg(normal_apply(A, 1.0), rhs, x0, delta, max_iter)
    z2 = d2 + forward(A, z1)
    return np.concatenate([z1, z2]), k, float(np.sqrt(rns)) <= delta


def prepare_subspace(problem, cg_tol: float = 1e-12, cg_max_iter=None) -> Cached:
    """scs.py:190-196."""
    h = np.concatenate([problem.c, problem.b])
    g, k, _ = _solve_inner_block(problem.A, problem.c, problem.b, cg_tol, cg_max_iter)
    denom = 1.0 + float(h @ g)
    return Cached(h, g, denom, cg_tol, cg_max_iter, k)


def subspace_project(w: np.ndarray, cached: Cached, A) -> np.ndarray:
    """scs.py:199-214."""
    n, m = A.cols, A.rows
    p, _, _ = _solve_inner_block(A, w[:n], w[n:n + m], cached.cg_tol, cached.cg_max_iter)
    tau = (w[-1] + float(cached.h @ p)) / cached.denom
    z = p - tau * cached.g
    return np.concatenate([z, [tau]])


def residuals(u, v, problem):
    """scs.py:217-244."""
    A, b, c = problem.A, problem.b, problem.c
    n, m = A.cols, A.rows
    ux, uy, tau = u[:n], u[n:n + m], u[-1]
    vs = v[n:n + m]
    if tau > SMALL_TAU:
        x, y, s = ux / tau, uy / tau, vs / tau
        pr = np.linalg.norm(forward(A, x) + s - b) / (1.0 + np.linalg.norm(b))
        dr = np.linalg.norm(adjoint(A, y) + c) / (1.0 + np.linalg.norm(c))
        ct, bt = float(c @ x), float(b @ y)
        gap = abs(ct + bt) / (1.0 + abs(ct) + abs(bt))
        return float(pr), float(dr), float(gap)
    den_u = -float(c @ ux)
    den_i = -float(b @ uy)
    pr = np.linalg.norm(forward(A, ux) + vs) / den_u if den_u > 0 else np.inf
    dr = np.linalg.norm(adjoint(A, uy)) / den_i if den_i > 0 else np.inf
    return float(pr), float(dr), np.inf


@dataclass
class LoopState:
    """Loop variables of the reference solver graph (scs.py:54, 449-459)."""

    u: np.ndarray
    v: np.ndarray
    k: int = 0
    since: int = 0
    status: float = 0.0
    cgw: np.ndarray | None = None
    cgt: float = 0.0
    resid: np.ndarray = field(default_factory=lambda: np.array([np.inf] * 3))


def _body(st: LoopState, problem, s: ScsOracleSettings, cached: Cached,
          pr_scale: float, dr_scale: float) -> LoopState:
    """scs.py:314-413 -- one splitting iteration, same op order as the graph."""
    A, b, c = problem.A, problem.b, problem.c
    n, m = A.cols, A.rows
    N = n + m + 1
    cg_max = s.cg_max_iter if s.cg_max_iter is not None else 10 * n
    u, v = st.u, st.v

    # subspace step
    w = u + v
    wz1, wz2, wtau = w[:n], w[n:n + m], w[N - 1]
    rhs = wz1 - adjoint(A, wz2)
    tol_k = _cg_tolerance_graph(float(st.k), s)
    delta = tol_k * float(np.linalg.norm(rhs))
    p1, cg_k, _ = cg(normal_apply(A, 1.0), rhs, st.cgw, delta, cg_max)
    p2 = wz2 + forward(A, p1)
    p = np.concatenate([p1, p2])
    tau_t = (wtau + float(np.dot(cached.h, p))) / cached.denom
    u_t = np.concatenate([p - tau_t * cached.g, [tau_t]])

    # cone step onto R^n x K* x R+
    w2 = u_t - v
    ux = w2[:n]
    uy = project_dual_product(problem.K.factors, w2[n:n + m])
    utau = max(w2[N - 1], 0.0)
    u2 = np.concatenate([ux, uy, [utau]])
    v2 = (v - u_t) + u2

    # termination measures
    s2 = v2[n:n + m]
    kappa = v2[N - 1]
    raw_p = (forward(A, ux) + s2) - utau * b
    raw_d = adjoint(A, uy) + utau * c
    ctx = float(np.dot(c, ux))
    bty = float(np.dot(b, uy))
    pos = 1.0 if utau > 0.0 else 0.0
    tinv = pos / (utau + (1.0 - pos))
    pr = pr_scale * (float(np.linalg.norm(raw_p)) * tinv)
    dr = dr_scale * (float(np.linalg.norm(raw_d)) * tinv)
    sc = ctx * tinv
    sb = bty * tinv
    gap = np.sqrt((sc + sb) * (sc + sb)) / (1.0 + (np.sqrt(sc * sc) + np.sqrt(sb * sb)))
    eps = s.eps
    solved = float(eps > pr) * float(eps > dr) * (float(eps > gap) * pos)

    max_k1 = max(kappa - 1.0, 0.0) + 1.0
    tau_small = float(s.cert_tau_ratio * max_k1 > utau)
    den_u = max(-1.0 * ctx, 0.0)
    pos_u = float(den_u > 0.0)
    unb_num = float(np.linalg.norm(raw_p + utau * b))
    res_u = unb_num / (den_u + (1.0 - pos_u))
    unb_ok = pos_u * float(eps > res_u)
    den_i = max(-1.0 * bty, 0.0)
    pos_i = float(den_i > 0.0)
    inf_num = float(np.linalg.norm(raw_d - utau * c))
    res_i = inf_num / (den_i + (1.0 - pos_i))
    inf_ok = pos_i * float(eps > res_i)
    cert = tau_small * (2.0 * inf_ok + (1.0 - inf_ok) * (3.0 * unb_ok))
    cand = solved + (1.0 - solved) * cert

    since2 = st.since + 1
    is_check = 1.0 if since2 > s.check_interval - 0.5 else 0.0
    not_set = 1.0 - (1.0 if st.status > 0.5 else 0.0)
    status2 = st.status + (not_set * is_check) * cand
    since3 = int(since2 * (1.0 - is_check))
    return LoopState(u2, v2, st.k + 1, since3, status2, p1, st.cgt + cg_k,
                     np.array([pr, dr, gap]))


def init_state(problem) -> LoopState:
    """scs.py:448-458 -- u = v = (0, 0, 1), cg warm start 0."""
    n, m = problem.A.cols, problem.A.rows
    N = n + m + 1
    start = np.zeros(N)
    start[-1] = 1.0
    return LoopState(start.copy(), start.copy(), cgw=np.zeros(n))


def iterate(problem, s: ScsOracleSettings, cached: Cached, max_steps: int):
    """scs.py:482-494 (iterate_states) -- yields (k, LoopState)."""
    pr_scale = 1.0 / (1.0 + np.linalg.norm(problem.b))
    dr_scale = 1.0 / (1.0 + np.linalg.norm(problem.c))
    st = init_state(problem)
    while st.k < max_steps and st.status == 0.0:
        st = _body(st, problem, s, cached, pr_scale, dr_scale)
        yield st.k, st


@dataclass
class OracleSolution:
    """scs.py:129-141 (ScsSolution) field-for-field."""

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


def classify(problem, s: ScsOracleSettings, u, v, iterations, cg_total) -> OracleSolution:
    """scs.py:497-538."""
    A, b, c = problem.A, problem.b, problem.c
    n, m = A.cols, A.rows
    tau, kappa = float(u[-1]), float(v[-1])
    ux, uy, vs = u[:n], u[n:n + m], v[n:n + m]
    avg_cg = cg_total / iterations if iterations > 0 else 0.0
    nan_n, nan_m = np.full(n, np.nan), np.full(m, np.nan)
    eps = s.eps
    if tau > SMALL_TAU:
        x, y, sv = ux / tau, uy / tau, vs / tau
        pr, dr, gap = residuals(u, v, problem)
        pobj, dobj = float(c @ x), -float(b @ y)
        if max(pr, dr, gap) <= eps:
            return OracleSolution("solved", x, y, sv, pobj, dobj, pr, dr, gap,
                                  iterations, avg_cg)
    else:
        pr = dr = gap = np.inf
        x = y = sv = None
    den_i = -float(b @ uy)
    if den_i > 0:
        res_i = float(np.linalg.norm(adjoint(A, uy))) / den_i
        if tau < s.cert_tau_ratio * max(kappa, 1.0) and res_i <= eps:
            return OracleSolution("infeasible", nan_n, uy / den_i, nan_m, np.nan,
                                  np.nan, np.inf, res_i, np.inf, iterations, avg_cg)
    den_u = -float(c @ ux)
    if den_u > 0:
        res_u = float(np.linalg.norm(forward(A, ux) + vs)) / den_u
        if tau < s.cert_tau_ratio * max(kappa, 1.0) and res_u <= eps:
            return OracleSolution("unbounded", ux / den_u, nan_m, vs / den_u, np.nan,
                                  np.nan, res_u, np.inf, np.inf, iterations, avg_cg)
    if x is None:
        return OracleSolution("max-iters", nan_n, nan_m, nan_m, np.nan, np.nan,
                              pr, dr, gap, iterations, avg_cg)
    status = "inaccurate" if max(pr, dr, gap) <= 10.0 * eps else "max-iters"
    return OracleSolution(status, x, y, sv, float(c @ x), -float(b @ y),
                          pr, dr, gap, iterations, avg_cg)


def scs_solve(problem, s: ScsOracleSettings | None = None, max_steps: int | None = None):
    """scs.py:571-576 -- setup solve, loop to termination, classify.

    ``max_steps`` bounds the loop (for timing samples) without changing
    the arithmetic of the iterations that do run.
    """
    s = s or ScsOracleSettings()
    cached = prepare_subspace(problem, s.setup_cg_tol, s.cg_max_iter)
    last = init_state(problem)
    cap = min(s.max_iters, max_steps) if max_steps is not None else s.max_iters
    for _, st in iterate(problem, s, cached, cap):
        last = st
    return classify(problem, s, last.u, last.v, last.k, last.cgt), last
