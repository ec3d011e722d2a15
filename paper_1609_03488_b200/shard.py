"""Row-sharded splitting solver: one rank per GPU.

The north star shards a large row-partitioned A over the GPUs of one box
with communication only for the dot products and the A^T y reduction.  The
reference solver has no sharding; its iteration (scs.py:314-413) is run
unchanged, with the stuffed problem split as follows (oracle/shard_ref.py
restates the same decomposition on the host and is the parity oracle):

* rows of the stuffed operator A (the y-space: cone pieces, b, w_y, v_y,
  u_y, A x) are cut into contiguous per-rank ranges, balanced by an
  estimate of their apply cost (``plan_cuts``); each rank's operator is
  ``row_slice(A, y0, y1)``, lowered to an ordinary device plan;
* x-space vectors (CG iterate, direction, A^T A x, w_x, g_x) are cut into
  contiguous slices; a full-length copy of the vector A is applied to next
  (the CG residual, or u_x on check iterations) lives on every rank;
* the per-rank persistent kernel (k_shard) reduce-scatters A^T y inside the
  adjoint's epilogue (peer stores into the inbox of the rank owning each
  column), all-gathers the CG residual by peer stores into every rank's
  copy, and reduces every dot product over the world in rank order, so all
  loop decisions are bitwise identical on every rank.

Two ways to run it:
  * ``ShardGroup(problem, settings, world)`` -- every rank in this process
    on one device (each rank a private cgb_ctx with 1/world of the SMs,
    launched concurrently on its own stream): the single-GPU test rig;
  * ``solve_sharded(problem, settings)`` under torch.distributed with one
    process per GPU: peer buffers are cudaMalloc'd by the library and
    exchanged as CUDA IPC handles (``cgb_ipc_*``).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import linop as L
from .cones import ExpCone, NonNegCone, SecondOrderCone, ZeroCone
from .scs import (INACCURATE, INFEASIBLE, MAX_ITERS, SMALL_TAU, SOLVED, UNBOUNDED,
                  ConeProblem, ScsSettings, ScsSolution)

SMALL_SOC_MAX = 4096       # SOCs up to this size are projected whole by one warp
ROW_BASE_COST = 10.0       # per-row y-space stream traffic (doubles)
NNZ_COST = 2.5             # per nonzero: value + index + gather (doubles)


# ---------------------------------------------------------------------------
# expression slicing
# ---------------------------------------------------------------------------

def _hstack_expr(blocks):
    """hstack of expressions, in linop.hstack's form adjoint(vstack(adjoints))."""
    blocks = [b for b in blocks if b.cols > 0]
    if len(blocks) == 1:
        return blocks[0]
    return L.AdjointOf(L.VStack([L.derive_adjoint(b) for b in blocks]))


def _vstack_expr(blocks):
    blocks = [b for b in blocks if b.rows > 0]
    return blocks[0] if len(blocks) == 1 else L.VStack(blocks)


def row_slice(e: L.LinOpExpr, r0: int, r1: int) -> L.LinOpExpr:
    """Rows [r0, r1) of the operator expression e, as an expression."""
    if not 0 <= r0 <= r1 <= e.rows:
        raise L.LinOpError(f"row slice [{r0}, {r1}) of an operator with {e.rows} rows")
    if r0 == 0 and r1 == e.rows:
        return e
    k = r1 - r0
    if k == 0:
        return L.ZeroOp(0, e.cols)
    if isinstance(e, L.Scale):
        return L.Scale(e.alpha, row_slice(e.child, r0, r1))
    if isinstance(e, L.Sum):
        return L.Sum(row_slice(e.left, r0, r1), row_slice(e.right, r0, r1))
    if isinstance(e, L.Compose):
        return L.Compose(row_slice(e.left, r0, r1), e.right)
    if isinstance(e, L.AdjointOf):
        return L.AdjointOf(col_slice(e.child, r0, r1))
    if isinstance(e, L.VStack):
        pieces, off = [], 0
        for c in e.children:
            a, b = max(r0, off), min(r1, off + c.rows)
            if b > a:
                pieces.append(row_slice(c, a - off, b - off))
            off += c.rows
        return _vstack_expr(pieces)
    if isinstance(e, L.ZeroOp):
        return L.ZeroOp(k, e.cols)
    if isinstance(e, L.Identity):
        return _hstack_expr([L.ZeroOp(k, r0), L.Identity(k), L.ZeroOp(k, e.cols - r1)])
    if isinstance(e, L.DenseMatrix):
        return L.DenseMatrix(e.values[r0:r1])
    if isinstance(e, L.SparseMatrix):
        return L.SparseMatrix(e.matrix[r0:r1])
    raise L.LinOpError(f"cannot cut through a {type(e).__name__} leaf; structured operators "
                       f"stay whole on one rank")


def col_slice(e: L.LinOpExpr, c0: int, c1: int) -> L.LinOpExpr:
    """Columns [c0, c1) of e (the row slice of its adjoint, transposed)."""
    if not 0 <= c0 <= c1 <= e.cols:
        raise L.LinOpError(f"column slice [{c0}, {c1}) of an operator with {e.cols} columns")
    if c0 == 0 and c1 == e.cols:
        return e
    k = c1 - c0
    if isinstance(e, L.Scale):
        return L.Scale(e.alpha, col_slice(e.child, c0, c1))
    if isinstance(e, L.Sum):
        return L.Sum(col_slice(e.left, c0, c1), col_slice(e.right, c0, c1))
    if isinstance(e, L.Compose):
        return L.Compose(e.left, col_slice(e.right, c0, c1))
    if isinstance(e, L.AdjointOf):
        return L.AdjointOf(row_slice(e.child, c0, c1))
    if isinstance(e, L.VStack):
        return L.VStack([col_slice(c, c0, c1) for c in e.children])
    if isinstance(e, L.ZeroOp):
        return L.ZeroOp(e.rows, k)
    if isinstance(e, L.Identity):
        return _vstack_expr([L.ZeroOp(c0, k), L.Identity(k), L.ZeroOp(e.rows - c1, k)])
    if isinstance(e, L.DenseMatrix):
        return L.DenseMatrix(e.values[:, c0:c1])
    if isinstance(e, L.SparseMatrix):
        return L.SparseMatrix(e.matrix[:, c0:c1])
    raise L.LinOpError(f"cannot cut through a {type(e).__name__} leaf; structured operators "
                       f"stay whole on one rank")


def _row_cuttable(e) -> bool:
    """row_slice can cut e at any row."""
    if isinstance(e, (L.DenseMatrix, L.SparseMatrix, L.Identity, L.ZeroOp)):
        return True
    if isinstance(e, L.Scale):
        return _row_cuttable(e.child)
    if isinstance(e, L.Sum):
        return _row_cuttable(e.left) and _row_cuttable(e.right)
    if isinstance(e, L.Compose):
        return _row_cuttable(e.left)
    if isinstance(e, L.AdjointOf):
        return _col_cuttable(e.child)
    if isinstance(e, L.VStack):
        return all(_row_cuttable(c) for c in e.children)
    return False


def _col_cuttable(e) -> bool:
    if isinstance(e, (L.DenseMatrix, L.SparseMatrix, L.Identity, L.ZeroOp)):
        return True
    if isinstance(e, L.Scale):
        return _col_cuttable(e.child)
    if isinstance(e, L.Sum):
        return _col_cuttable(e.left) and _col_cuttable(e.right)
    if isinstance(e, L.Compose):
        return _col_cuttable(e.right)
    if isinstance(e, L.AdjointOf):
        return _row_cuttable(e.child)
    if isinstance(e, L.VStack):
        return all(_col_cuttable(c) for c in e.children)
    return False


def whole_spans(e: L.LinOpExpr, off: int = 0) -> list[tuple[int, int]]:
    """Row spans no cut may enter (blocks holding a convolution / Kronecker
    leaf); stacked blocks are examined one by one."""
    if isinstance(e, L.VStack):
        out, o = [], off
        for c in e.children:
            out.extend(whole_spans(c, o))
            o += c.rows
        return out
    if isinstance(e, L.Scale):
        return whole_spans(e.child, off)
    return [] if _row_cuttable(e) else [(off, off + e.rows)]


def row_nnz(e: L.LinOpExpr) -> np.ndarray:
    """Estimated nonzeros of every row of e (exact for sparse / dense /
    identity blocks; structured leaves count their taps)."""
    if isinstance(e, L.Scale):
        return row_nnz(e.child)
    if isinstance(e, L.Sum):
        return row_nnz(e.left) + row_nnz(e.right)
    if isinstance(e, L.VStack):
        return np.concatenate([row_nnz(c) for c in e.children])
    if isinstance(e, L.AdjointOf):
        return col_nnz(e.child)
    if isinstance(e, L.ZeroOp):
        return np.zeros(e.rows)
    if isinstance(e, L.Identity):
        return np.ones(e.rows)
    if isinstance(e, L.DenseMatrix):
        return np.full(e.rows, float(e.cols))
    if isinstance(e, L.SparseMatrix):
        return np.bincount(e.matrix.indices, minlength=e.rows).astype(np.float64)
    if isinstance(e, L.Compose):
        return row_nnz(e.left) + float(np.mean(row_nnz(e.right)) if e.right.rows else 0.0)
    return np.full(e.rows, float(L.nnz_estimate(L.Operator(e))) / max(1, e.rows))


def col_nnz(e: L.LinOpExpr) -> np.ndarray:
    if isinstance(e, L.Scale):
        return col_nnz(e.child)
    if isinstance(e, L.Sum):
        return col_nnz(e.left) + col_nnz(e.right)
    if isinstance(e, L.VStack):
        return sum(col_nnz(c) for c in e.children)
    if isinstance(e, L.AdjointOf):
        return row_nnz(e.child)
    if isinstance(e, L.ZeroOp):
        return np.zeros(e.cols)
    if isinstance(e, L.Identity):
        return np.ones(e.cols)
    if isinstance(e, L.DenseMatrix):
        return np.full(e.cols, float(e.rows))
    if isinstance(e, L.SparseMatrix):
        return np.diff(e.matrix.indptr).astype(np.float64)
    return np.full(e.cols, float(L.nnz_estimate(L.Operator(e))) / max(1, e.cols))


# ---------------------------------------------------------------------------
# partition
# ---------------------------------------------------------------------------

def _cone_spans(K):
    off = 0
    for f in K.factors:
        yield f, off, off + f.dim
        off += f.dim


def _world_socs(K, cuts) -> list[int]:
    """Start rows of the SOCs reduced across the world: longer than one
    warp's block, or cut by a rank boundary."""
    inner = {c for c in cuts[1:-1]}
    out = []
    for f, b, e in _cone_spans(K):
        if isinstance(f, SecondOrderCone) and (f.dim > SMALL_SOC_MAX or
                                               any(b < c < e for c in inner)):
            out.append(b)
    return out


MAX_WORLD_SOCS = 4         # CGB_MAX_LARGE_SOC


def plan_cuts(problem: ConeProblem, world: int) -> list[int]:
    """Row cuts [0, c1, ..., m] balancing ROW_BASE_COST + NNZ_COST * nnz per
    row.  A cut never splits an exponential cone; it splits a small SOC
    (which then becomes world-reduced) only while at most MAX_WORLD_SOCS
    SOCs are world-reduced, else it moves to the SOC's nearer end."""
    m = problem.A.rows
    if world == 1:
        return [0, m]
    w = ROW_BASE_COST + NNZ_COST * row_nnz(problem.A.expr)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    whole = whole_spans(problem.A.expr)

    def snap(c: int, lo: int, snap_soc: bool) -> int:
        spans = list(whole)
        for f, b, e in _cone_spans(problem.K):
            if isinstance(f, ExpCone) or (snap_soc and isinstance(f, SecondOrderCone) and
                                          f.dim <= SMALL_SOC_MAX):
                spans.append((b, e))
        for _ in range(len(spans) + 1):
            hit = [(b, e) for b, e in spans if b < c < e]
            if not hit:
                break
            b, e = hit[0]
            c = b if (c - b <= e - c and b > lo) or e >= m else e
        return c

    def cuts_for(snap_soc: bool):
        cuts = [0]
        for q in range(1, world):
            c = snap(int(np.searchsorted(cum, cum[-1] * q / world)), cuts[-1], snap_soc)
            cuts.append(min(max(c, cuts[-1]), m))
        cuts.append(m)
        if any(b >= e for b, e in zip(cuts, cuts[1:])):
            raise L.LinOpError(f"cannot cut the operator's rows into {world} nonempty ranks "
                               f"(convolution / Kronecker blocks stay whole): {cuts}")
        return cuts

    cuts = cuts_for(False)
    if len(_world_socs(problem.K, cuts)) > MAX_WORLD_SOCS:
        cuts = cuts_for(True)
    if len(_world_socs(problem.K, cuts)) > MAX_WORLD_SOCS:
        raise L.LinOpError(f"more than {MAX_WORLD_SOCS} second-order cones longer than "
                           f"{SMALL_SOC_MAX}: not supported by the sharded solver")
    return cuts


def x_slices(n: int, world: int) -> list[int]:
    """Even x-space slices, boundaries on 16-byte multiples."""
    cuts = [0]
    for q in range(1, world):
        cuts.append(min(n, max(cuts[-1], (round(n * q / world) + 1) // 2 * 2)))
    cuts.append(n)
    return cuts


def cone_pieces(K, y0: int, y1: int, world_socs: list[int]):
    """This rank's pieces of the cone product: (kinds, begins, ends, soc_id,
    has_head) in local row coordinates."""
    kinds, begins, ends, sid, head = [], [], [], [], []
    code = {ZeroCone: _lib.CONE_ZERO, NonNegCone: _lib.CONE_NONNEG,
            SecondOrderCone: _lib.CONE_SOC, ExpCone: _lib.CONE_EXP}
    for f, b, e in _cone_spans(K):
        a, z = max(b, y0), min(e, y1)
        if z <= a:
            continue
        kinds.append(code[type(f)])
        begins.append(a - y0)
        ends.append(z - y0)
        if isinstance(f, SecondOrderCone) and b in world_socs:
            sid.append(world_socs.index(b))
        else:
            sid.append(-1)
        head.append(1 if a == b else 0)
    return kinds, begins, ends, sid, head


# ---------------------------------------------------------------------------
# one rank
# ---------------------------------------------------------------------------

class _Peer:
    """This rank's peer-visible buffers (inbox, full-length x copy, mailbox)."""

    def __init__(self, device: int, nl_world: int, n: int, ipc: bool):
        import torch
        self.ipc = ipc
        self.sizes = {"inbox": max(1, nl_world), "xfull": max(1, n),
                      "mbox": 2 * _lib.MAX_RANKS * _lib.MBOX_STRIDE}
        self.ptrs, self.handles, self._keep = {}, {}, {}
        lib = _lib.load_library()
        for nm, cnt in self.sizes.items():
            if ipc:
                p = ctypes.c_void_p()
                h = ctypes.create_string_buffer(64)
                _lib.check(lib.cgb_ipc_alloc(device, 8 * cnt, ctypes.byref(p), h))
                self.ptrs[nm] = p.value
                self.handles[nm] = h.raw
            else:
                t = torch.zeros(cnt, dtype=torch.float64, device=f"cuda:{device}")
                self._keep[nm] = t
                self.ptrs[nm] = t.data_ptr()
        self.opened: list[int] = []

    def free(self):
        lib = _lib.load_library()
        for p in self.opened:
            lib.cgb_ipc_close(ctypes.c_void_p(p))
        self.opened = []
        if self.ipc:
            for p in self.ptrs.values():
                lib.cgb_ipc_free(ctypes.c_void_p(p))
        self.ptrs = {}
        self._keep = {}


@dataclass
class RankLayout:
    world: int
    rank: int
    cuts: list[int]       # y rows
    xb: list[int]         # x slices
    world_socs: list[int]

    @property
    def y0(self):
        return self.cuts[self.rank]

    @property
    def y1(self):
        return self.cuts[self.rank + 1]

    @property
    def x0(self):
        return self.xb[self.rank]

    @property
    def x1(self):
        return self.xb[self.rank + 1]


class RankSolver:
    """One rank's compiled share of the problem and its device buffers."""

    def __init__(self, problem: ConeProblem, settings: ScsSettings, layout: RankLayout,
                 device: int, ctx=None, ipc: bool = False):
        import torch
        from ._plan import DeviceOp
        self.problem, self.settings, self.lay = problem, settings, layout
        self.device = device
        self.ctx = ctx if ctx is not None else _lib.device_context()
        lay = layout
        n = problem.A.cols
        self.n, self.m = n, lay.y1 - lay.y0
        self.nl = lay.x1 - lay.x0
        with torch.cuda.device(device):
            self.expr = row_slice(problem.A.expr, lay.y0, lay.y1)
            self.op = DeviceOp(self.expr, self.ctx)
            kinds, bg, en, sid, hd = cone_pieces(problem.K, lay.y0, lay.y1, lay.world_socs)
            arr = lambda t, v: (t * max(1, len(v)))(*v)  # noqa: E731
            h = ctypes.c_void_p()
            lib = _lib.load_library()
            _lib.check(lib.cgb_shard_cones_create(
                self.ctx.handle, arr(ctypes.c_int32, kinds), arr(ctypes.c_int64, bg),
                arr(ctypes.c_int64, en), arr(ctypes.c_int32, sid), arr(ctypes.c_int32, hd),
                len(kinds), self.m, len(lay.world_socs), ctypes.byref(h)))
            self.cones = h
            f64 = dict(dtype=torch.float64, device=f"cuda:{device}")
            # (one element of padding: an empty slice still needs a pointer)
            self.b = torch.zeros(self.m + 1, **f64)
            self.b[:self.m] = torch.from_numpy(np.ascontiguousarray(problem.b[lay.y0:lay.y1]))
            self.c = torch.zeros(self.nl + 1, **f64)
            self.c[:self.nl] = torch.from_numpy(np.ascontiguousarray(problem.c[lay.x0:lay.x1]))
            self.buf = {nm: torch.zeros(max(1, self.nl), **f64)
                        for nm in ("cgx", "gx", "p", "wx", "gxs")}
            for nm in ("wy", "vy", "uy", "tax", "t", "gy"):
                self.buf[nm] = torch.zeros(max(1, self.m), **f64)
            self.buf["state"] = torch.zeros(_lib.STATE_LEN, **f64)
            self.peer = _Peer(device, lay.world * self.nl, n, ipc)
        self.work = _lib.ShardWorkC(**{nm: t.data_ptr() for nm, t in self.buf.items()})
        self.cprob = _lib.ShardProblemC(
            n=n, m=self.m, A=self.op.handle.value, K=self.cones.value, b=self.b.data_ptr(),
            c=self.c.data_ptr(),
            pr_scale=1.0 / (1.0 + float(np.linalg.norm(problem.b))),
            dr_scale=1.0 / (1.0 + float(np.linalg.norm(problem.c))),
            setup_tol=settings.setup_cg_tol)
        self.csettings = settings.to_c(n)
        self.comm = None
        self.reset()

    def connect(self, peers: list[dict]) -> None:
        """peers[q] = {"inbox", "xfull", "mbox"} device pointers valid here."""
        lay = self.lay
        cm = _lib.ShardCommC(world=lay.world, rank=lay.rank)
        for q in range(lay.world + 1):
            cm.x_begin[q] = lay.xb[q]
        for q in range(lay.world):
            cm.inbox[q] = peers[q]["inbox"]
            cm.xfull[q] = peers[q]["xfull"]
            cm.mbox[q] = peers[q]["mbox"]
        self.comm = cm

    def reset(self) -> None:
        """u = v = (0, 0, 1), warm start 0 (scs.py:448-458); the world
        synchronisation count survives (the mailboxes are monotonic)."""
        st = self.buf["state"]
        keep = {i: float(st[i].item()) for i in (_lib.ST_EPOCH, _lib.ST_DENOM,
                                                  _lib.ST_SETUP_CG)}
        for nm, t in self.buf.items():
            if nm not in ("gxs", "gy"):
                t.zero_()
        st[_lib.ST_TAU] = 1.0
        st[_lib.ST_KAPPA] = 1.0
        for i, v in keep.items():
            st[i] = v

    def validate(self, mode: int) -> None:
        """Check this rank's launch arguments without launching."""
        _lib.check(_lib.load_library().cgb_shard_run(
            self.ctx.handle, ctypes.byref(self.cprob), ctypes.byref(self.csettings),
            ctypes.byref(self.comm), ctypes.byref(self.work), int(mode), -1, None))

    def launch(self, mode: int, max_steps: int, stream) -> None:
        import torch
        with torch.cuda.device(self.device):
            _lib.check(_lib.load_library().cgb_shard_run(
                self.ctx.handle, ctypes.byref(self.cprob), ctypes.byref(self.csettings),
                ctypes.byref(self.comm), ctypes.byref(self.work), int(mode), int(max_steps),
                ctypes.c_void_p(stream.cuda_stream)))

    def state(self) -> np.ndarray:
        return self.buf["state"].cpu().numpy()

    def close(self) -> None:
        lib = _lib.load_library()
        if getattr(self, "cones", None) is not None and self.cones.value:
            lib.cgb_cones_destroy(self.cones)
            self.cones = None
        if getattr(self, "peer", None) is not None:
            self.peer.free()
            self.peer = None


def layout_for(problem: ConeProblem, world: int, rank: int) -> RankLayout:
    cuts = plan_cuts(problem, world)
    return RankLayout(world, rank, cuts, x_slices(problem.A.cols, world),
                      _world_socs(problem.K, cuts))


def _solution(problem: ConeProblem, settings: ScsSettings, ux, uy, vy, st) -> ScsSolution:
    """Classification from the latched device residuals (scs.py:497-538;
    the status arithmetic already ran on device every check_interval)."""
    n, m = problem.A.cols, problem.A.rows
    tau, status = float(st[_lib.ST_TAU]), float(st[_lib.ST_STATUS])
    k, cgt = int(st[_lib.ST_K]), float(st[_lib.ST_CGT])
    pr, dr, gap = float(st[_lib.ST_PR]), float(st[_lib.ST_DR]), float(st[_lib.ST_GAP])
    avg = cgt / k if k else 0.0
    nan_n, nan_m = np.full(n, np.nan), np.full(m, np.nan)
    if status == 2.0:
        den = -float(problem.b @ uy)
        return ScsSolution(INFEASIBLE, nan_n, uy / den, nan_m, np.nan, np.nan, np.inf, dr,
                           np.inf, k, avg)
    if status == 3.0:
        den = -float(problem.c @ ux)
        return ScsSolution(UNBOUNDED, ux / den, nan_m, vy / den, np.nan, np.nan, pr, np.inf,
                           np.inf, k, avg)
    if tau <= SMALL_TAU:
        return ScsSolution(MAX_ITERS, nan_n, nan_m, nan_m, np.nan, np.nan, pr, dr, gap, k, avg)
    x, y, s = ux / tau, uy / tau, vy / tau
    pobj, dobj = float(problem.c @ x), -float(problem.b @ y)
    if status == 1.0:
        return ScsSolution(SOLVED, x, y, s, pobj, dobj, pr, dr, gap, k, avg)
    stat = INACCURATE if max(pr, dr, gap) <= 10.0 * settings.eps else MAX_ITERS
    return ScsSolution(stat, x, y, s, pobj, dobj, pr, dr, gap, k, avg)


class ShardGroup:
    """Every rank in this process on one device: rank q gets a private
    cgb_ctx of grid/world CTAs and its own stream; launches of one phase go
    out back to back so the ranks' persistent kernels run concurrently."""

    def __init__(self, problem: ConeProblem, settings: ScsSettings | None = None,
                 world: int = 2, device: int = 0, grid: int | None = None):
        import torch
        self.problem = problem
        self.settings = settings or ScsSettings()
        self.world = world
        sms = torch.cuda.get_device_properties(device).multi_processor_count
        g = grid or max(1, sms // world)
        self.ranks = []
        for q in range(world):
            lay = layout_for(problem, world, q)
            ctx = _lib.new_context(device, g)
            self.ranks.append(RankSolver(problem, self.settings, lay, device, ctx))
        peers = [dict(r.peer.ptrs) for r in self.ranks]
        for r in self.ranks:
            r.connect(peers)
        self.streams = [torch.cuda.Stream(device=device) for _ in range(world)]
        self.setup()

    def _all(self, mode: int, max_steps: int) -> None:
        import torch
        for r in self.ranks:          # all arguments first: no rank launches alone
            r.validate(mode)
        cur = torch.cuda.current_stream()
        for s in self.streams:
            s.wait_stream(cur)
        for r, s in zip(self.ranks, self.streams):
            r.launch(mode, max_steps, s)
        for s in self.streams:
            cur.wait_stream(s)

    def setup(self) -> None:
        self._all(0, 0)

    def reset(self) -> None:
        import torch
        torch.cuda.synchronize()
        for r in self.ranks:
            r.reset()

    def run(self, max_steps: int) -> None:
        self._all(1, max_steps)

    def states(self) -> list[np.ndarray]:
        return [r.state() for r in self.ranks]

    def gather(self):
        ux = np.concatenate([r.buf["wx"][:r.nl].cpu().numpy() for r in self.ranks])
        uy = np.concatenate([r.buf["uy"][:r.m].cpu().numpy() for r in self.ranks])
        vy = np.concatenate([r.buf["vy"][:r.m].cpu().numpy() for r in self.ranks])
        gx = np.concatenate([r.buf["gxs"][:r.nl].cpu().numpy() for r in self.ranks])
        gy = np.concatenate([r.buf["gy"][:r.m].cpu().numpy() for r in self.ranks])
        return ux, uy, vy, gx, gy

    def solve(self) -> ScsSolution:
        self.reset()
        self.run(self.settings.max_iters)
        import torch
        torch.cuda.synchronize()
        st = self.ranks[0].state()
        ux, uy, vy, _, _ = self.gather()
        return _solution(self.problem, self.settings, ux, uy, vy, st)

    def close(self) -> None:
        for r in self.ranks:
            r.close()


def solve_sharded(problem: ConeProblem, settings: ScsSettings | None = None,
                  max_steps: int | None = None):
    """One rank per GPU under torch.distributed (already initialised): this
    rank's share on torch's current device, peer buffers exchanged as CUDA
    IPC handles.  Returns (solution on rank 0 else None, RankSolver)."""
    import torch
    import torch.distributed as dist
    settings = settings or ScsSettings()
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = torch.cuda.current_device()
    lay = layout_for(problem, world, rank)
    rs = RankSolver(problem, settings, lay, dev, ipc=world > 1)
    connect_ipc(rs)
    stream = torch.cuda.current_stream()
    rs.validate(0)
    dist.barrier()
    rs.launch(0, 0, stream)
    rs.launch(1, settings.max_iters if max_steps is None else max_steps, stream)
    torch.cuda.synchronize()
    sol = gather_solution(rs)
    return sol, rs


def connect_ipc(rs: RankSolver) -> None:
    """Exchange the peer buffers' IPC handles over torch.distributed and map
    every other rank's buffers on this device."""
    import torch.distributed as dist
    world = rs.lay.world
    if world == 1:
        rs.connect([dict(rs.peer.ptrs)])
        return
    mine = {nm: rs.peer.handles[nm] for nm in ("inbox", "xfull", "mbox")}
    allh: list = [None] * world
    dist.all_gather_object(allh, mine)
    lib = _lib.load_library()
    peers = []
    for q in range(world):
        if q == rs.lay.rank:
            peers.append(dict(rs.peer.ptrs))
            continue
        d = {}
        for nm in ("inbox", "xfull", "mbox"):
            p = ctypes.c_void_p()
            _lib.check(lib.cgb_ipc_open(rs.device, allh[q][nm], ctypes.byref(p)))
            rs.peer.opened.append(p.value)
            d[nm] = p.value
        peers.append(d)
    dist.barrier()
    rs.connect(peers)


def gather_solution(rs: RankSolver) -> ScsSolution | None:
    """Rank 0 assembles u, v from every rank's share (torch.distributed)."""
    import torch.distributed as dist
    part = (rs.buf["wx"][:rs.nl].cpu().numpy(), rs.buf["uy"][:rs.m].cpu().numpy(),
            rs.buf["vy"][:rs.m].cpu().numpy())
    st = rs.state()
    if rs.lay.world == 1:
        return _solution(rs.problem, rs.settings, *part, st)
    parts: list = [None] * rs.lay.world
    dist.all_gather_object(parts, part)
    if rs.lay.rank != 0:
        return None
    ux = np.concatenate([p[0] for p in parts])
    uy = np.concatenate([p[1] for p in parts])
    vy = np.concatenate([p[2] for p in parts])
    return _solution(rs.problem, rs.settings, ux, uy, vy, st)
