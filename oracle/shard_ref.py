"""Row-sharded splitting iteration (TEST ORACLE ONLY; north-star §8e design).

The north star shards a large row-partitioned A over the GPUs of a box,
with collectives carrying only the dot-product all-reduces and the A^T y
reduction.  This module restates the reference iteration (scs.py:314-413,
as restated in scs_ref._body) for that decomposition so the communication
pattern can be checked on CPU with torch.distributed (gloo) before it is
built into the persistent kernel:

  * the stuffed problem's y-space rows [0, m) are split into contiguous
    per-rank ranges; x-space vectors (length n) are replicated;
  * A x is local (each rank owns its rows), A^T y = sum_r A_r^T y_r is one
    all-reduce of an n-vector (the rhs step and every CG step);
  * dot products / norms over y-space are local partials + all-reduce,
    over x-space they are computed redundantly (bitwise identical);
  * a second-order cone whose rows straddle ranks gets its tail norm as an
    all-reduced partial sum of squares and its head from the owning rank.

Operators are materialized densely per rank (test sizes only).  Every
function cites the single-process restatement it mirrors.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .cg_ref import cg
from .linop_ref import materialize
from .scs_ref import SMALL_TAU, ScsOracleSettings, _cg_tolerance_graph  # noqa: F401


class LocalComm:
    """Single process: every all-reduce is the identity."""

    rank, world = 0, 1

    def allreduce(self, x: np.ndarray) -> np.ndarray:
        return np.asarray(x, dtype=np.float64)


class TorchComm:
    """torch.distributed (gloo on CPU) all-reduce of float64 arrays."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()

    def allreduce(self, x: np.ndarray) -> np.ndarray:
        import torch
        t = torch.from_numpy(np.array(x, dtype=np.float64, copy=True))
        self.dist.all_reduce(t)
        return t.numpy()


def row_ranges(m: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, balanced y-row ranges."""
    cuts = [round(r * m / world) for r in range(world + 1)]
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


@dataclass
class Shard:
    """One rank's part of a stuffed cone problem (A x + s = b, s in K)."""

    A_loc: np.ndarray      # (r1 - r0) x n rows of the materialized operator
    b_loc: np.ndarray
    c: np.ndarray          # replicated
    r0: int
    r1: int
    m: int
    n: int
    factors: list          # (kind, begin, end) of the cone product, global rows


def make_shard(problem, comm) -> Shard:
    A = materialize(problem.A)
    m, n = A.shape
    r0, r1 = row_ranges(m, comm.world)[comm.rank]
    factors, off = [], 0
    for f in problem.K.factors:
        factors.append((type(f).__name__, off, off + f.dim))
        off += f.dim
    return Shard(A[r0:r1].copy(), np.asarray(problem.b[r0:r1], dtype=np.float64),
                 np.asarray(problem.c, dtype=np.float64), r0, r1, m, n, factors)


def _adj(sh: Shard, comm, y_loc: np.ndarray) -> np.ndarray:
    """A^T y: local partial, then the n-vector all-reduce."""
    return comm.allreduce(sh.A_loc.T @ y_loc)


def _ydot(comm, a: np.ndarray, b: np.ndarray) -> float:
    return float(comm.allreduce(np.array([float(np.dot(a, b))]))[0])


def _normal(sh: Shard, comm):
    """cg_ref.normal_apply(A, 1): x + A^T (A x) with the sharded A."""
    return lambda x: x + _adj(sh, comm, sh.A_loc @ x)


def _project_dual(sh: Shard, comm, z_loc: np.ndarray) -> np.ndarray:
    """cones_ref.project_dual_product on the rank's rows; SOCs that straddle
    ranks reduce (tail^2, head) across ranks (scs.py:250-283)."""
    out = z_loc.copy()
    socs = [(b, e) for k, b, e in sh.factors if k == "SecondOrderCone"]
    part = np.zeros(2 * len(socs))
    for j, (b, e) in enumerate(socs):
        lo, hi = max(b + 1, sh.r0), min(e, sh.r1)
        if hi > lo:
            t = z_loc[lo - sh.r0:hi - sh.r0]
            part[2 * j] = float(np.dot(t, t))
        if sh.r0 <= b < sh.r1:
            part[2 * j + 1] = z_loc[b - sh.r0]
    red = comm.allreduce(part)
    for kind, b, e in sh.factors:
        lo, hi = max(b, sh.r0), min(e, sh.r1)
        if hi <= lo:
            continue
        seg = slice(lo - sh.r0, hi - sh.r0)
        if kind == "ZeroCone":
            continue
        if kind == "NonNegCone":
            out[seg] = np.maximum(z_loc[seg], 0.0)
            continue
        if kind != "SecondOrderCone":
            raise TypeError(f"shard oracle: cone {kind} not supported")
        j = socs.index((b, e))
        t, nu = red[2 * j + 1], np.sqrt(red[2 * j])
        inside = 1.0 - float(nu > t)
        in_polar = 1.0 - float(nu > -1.0 * t)
        p_else = (1.0 - inside) * (1.0 - in_polar)
        coef = 0.5 * (t + nu)
        safe = nu + (1.0 - float(nu > 0.0))
        for i in range(lo, hi):
            zi = z_loc[i - sh.r0]
            cand = coef if i == b else coef * (zi / safe)
            out[i - sh.r0] = inside * zi + p_else * cand
    return out


@dataclass
class ShardCached:
    g_x: np.ndarray
    g_y: np.ndarray   # this rank's rows
    denom: float


def prepare(sh: Shard, comm, s: ScsOracleSettings) -> ShardCached:
    """scs_ref.prepare_subspace with sharded applies (scs.py:170-196)."""
    rhs = sh.c - _adj(sh, comm, sh.b_loc)
    delta = s.setup_cg_tol * float(np.linalg.norm(rhs))
    cg_max = s.cg_max_iter if s.cg_max_iter is not None else 10 * sh.n
    z1, _, _ = cg(_normal(sh, comm), rhs, np.zeros(sh.n), delta, cg_max)
    z2 = sh.b_loc + sh.A_loc @ z1
    denom = 1.0 + float(np.dot(sh.c, z1)) + _ydot(comm, sh.b_loc, z2)
    return ShardCached(z1, z2, denom)


@dataclass
class ShardState:
    ux: np.ndarray
    uy: np.ndarray
    utau: float
    vy: np.ndarray      # v_x == 0 (embedding invariant)
    kappa: float
    cgw: np.ndarray
    k: int = 0
    since: int = 0
    status: float = 0.0
    cgt: float = 0.0


def init(sh: Shard) -> ShardState:
    """scs.py:448-458 (u = v = (0, 0, 1))."""
    ny = sh.r1 - sh.r0
    return ShardState(np.zeros(sh.n), np.zeros(ny), 1.0, np.zeros(ny), 1.0, np.zeros(sh.n))


def step(sh: Shard, comm, s: ScsOracleSettings, ca: ShardCached, st: ShardState,
         pr_scale: float, dr_scale: float) -> ShardState:
    """scs_ref._body with the y-space split (scs.py:314-413)."""
    cg_max = s.cg_max_iter if s.cg_max_iter is not None else 10 * sh.n
    wz1, wz2, wtau = st.ux, st.uy + st.vy, st.utau + st.kappa
    rhs = wz1 - _adj(sh, comm, wz2)
    delta = _cg_tolerance_graph(float(st.k), s) * float(np.linalg.norm(rhs))
    p1, cg_k, _ = cg(_normal(sh, comm), rhs, st.cgw, delta, cg_max)
    p2 = wz2 + sh.A_loc @ p1
    hp = float(np.dot(sh.c, p1)) + _ydot(comm, sh.b_loc, p2)
    tau_t = (wtau + hp) / ca.denom
    ut_x, ut_y = p1 - tau_t * ca.g_x, p2 - tau_t * ca.g_y
    w2y = ut_y - st.vy
    uy = _project_dual(sh, comm, w2y)
    ux = ut_x                     # free block (v_x == 0)
    utau = max(tau_t - st.kappa, 0.0)
    vy = (st.vy - ut_y) + uy
    kappa = (st.kappa - tau_t) + utau
    # termination measures, the reference's arithmetic with y-space sums reduced
    raw_p = (sh.A_loc @ ux + vy) - utau * sh.b_loc
    raw_d = _adj(sh, comm, uy) + utau * sh.c
    ctx = float(np.dot(sh.c, ux))
    q = comm.allreduce(np.array([float(np.dot(raw_p, raw_p)), float(np.dot(sh.b_loc, uy)),
                                 float(np.dot(raw_p + utau * sh.b_loc,
                                              raw_p + utau * sh.b_loc))]))
    bty = float(q[1])
    pos = 1.0 if utau > 0.0 else 0.0
    tinv = pos / (utau + (1.0 - pos))
    pr = pr_scale * (float(np.sqrt(q[0])) * tinv)
    dr = dr_scale * (float(np.linalg.norm(raw_d)) * tinv)
    sc, sb = ctx * tinv, bty * tinv
    gap = np.sqrt((sc + sb) * (sc + sb)) / (1.0 + (np.sqrt(sc * sc) + np.sqrt(sb * sb)))
    eps = s.eps
    solved = float(eps > pr) * float(eps > dr) * (float(eps > gap) * pos)
    max_k1 = max(kappa - 1.0, 0.0) + 1.0
    tau_small = float(s.cert_tau_ratio * max_k1 > utau)
    den_u = max(-1.0 * ctx, 0.0)
    pos_u = float(den_u > 0.0)
    res_u = float(np.sqrt(q[2])) / (den_u + (1.0 - pos_u))
    unb_ok = pos_u * float(eps > res_u)
    den_i = max(-1.0 * bty, 0.0)
    pos_i = float(den_i > 0.0)
    res_i = float(np.linalg.norm(raw_d - utau * sh.c)) / (den_i + (1.0 - pos_i))
    inf_ok = pos_i * float(eps > res_i)
    cert = tau_small * (2.0 * inf_ok + (1.0 - inf_ok) * (3.0 * unb_ok))
    cand = solved + (1.0 - solved) * cert
    since2 = st.since + 1
    is_check = 1.0 if since2 > s.check_interval - 0.5 else 0.0
    not_set = 1.0 - (1.0 if st.status > 0.5 else 0.0)
    return ShardState(ux, uy, utau, vy, kappa, p1, st.k + 1, int(since2 * (1.0 - is_check)),
                      st.status + (not_set * is_check) * cand, st.cgt + cg_k)


def solve(problem, comm, s: ScsOracleSettings, max_steps: int | None = None):
    """Run the sharded iteration; returns (state, shard)."""
    sh = make_shard(problem, comm)
    pr_scale = 1.0 / (1.0 + float(np.sqrt(_ydot(comm, sh.b_loc, sh.b_loc))))
    dr_scale = 1.0 / (1.0 + float(np.linalg.norm(sh.c)))
    ca = prepare(sh, comm, s)
    st = init(sh)
    cap = s.max_iters if max_steps is None else min(s.max_iters, max_steps)
    while st.k < cap and st.status == 0.0:
        st = step(sh, comm, s, ca, st, pr_scale, dr_scale)
    return st, sh
