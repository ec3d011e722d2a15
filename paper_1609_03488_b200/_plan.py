"""Lowering of operator expressions to flat device plans.

A plan is what one persistent kernel executes for y = A x: every leaf
(dense / CSR / 1-d conv / 2-d conv / identity) becomes a *term*
``out[row_origin + i] += alpha * leaf(in[in_off:])[i]``; the output rows
are cut into *row blocks* that see a fixed term list, so each output
element is produced by exactly one warp lane summing its terms -- no
atomics, no zero-fill pass, deterministic.  Scale and VStack/HStack
(adjoint-of-VStack) structure folds into alpha / offsets; Sum adds terms
to the same rows; Compose of two non-trivial operators introduces a plan
temporary produced one *level* earlier (a grid barrier apart).  The
adjoint plan is lowered from the same tree with the adjoint flag pushed
to the leaves (linop.py:187-207 rules), so Conv1D's adjoint is a valid
correlation leaf, Dense's is the row-major transpose, CSC's is the CSR
of the transpose.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from . import linop as L


def _scaled_identity(e) -> float | None:
    """alpha if e is alpha * Identity (through Scale/AdjointOf), else None."""
    if isinstance(e, L.Identity):
        return 1.0
    if isinstance(e, L.Scale):
        s = _scaled_identity(e.child)
        return None if s is None else e.alpha * s
    if isinstance(e, L.AdjointOf):
        return _scaled_identity(e.child)
    return None


SEPARABLE_KMAX = 63   # CGB_SEP_KMAX
CONV_KMAX = 240       # CGB_CONV_KMAX: longest 1-d kernel of the tiled conv path


def separable(kernel: np.ndarray) -> bool:
    """A 2-d kernel of numerical rank one (sigma_2 <= 1e-13 sigma_1) is
    applied as a column pass and a row pass (kh + kw instead of kh * kw
    multiply-adds per output; the library re-verifies the factorization
    entrywise).  CGB_NO_SEPARABLE=1 forces the direct 2-d sum."""
    import os
    if os.environ.get("CGB_NO_SEPARABLE"):
        return False
    k = np.asarray(kernel, dtype=np.float64)
    if k.ndim != 2 or k.shape[1] > SEPARABLE_KMAX or not np.any(k):
        return False
    s = np.linalg.svd(k, compute_uv=False)
    return len(s) < 2 or s[1] <= 1e-13 * s[0]


def _cuda(a: np.ndarray, dtype=None):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a if dtype is None else a.astype(dtype)))
    return t.to("cuda")


def _leaf_buffers(e) -> dict:
    """Device copies of a leaf's data, cached on the expression object."""
    cache = getattr(e, "_cgb_dev", None)
    if cache is None:
        cache = {}
        e._cgb_dev = cache
    return cache


def _perm(rows_of_cols: np.ndarray) -> "L.SparseMatrix":
    """Permutation matrix P with P[rows_of_cols[c], c] = 1."""
    import scipy.sparse
    k = len(rows_of_cols)
    return L.SparseMatrix(scipy.sparse.csc_matrix(
        (np.ones(k), (rows_of_cols, np.arange(k))), shape=(k, k)))


def _block_diag(e, copies: int):
    """I_copies (x) e as an expression (zero blocks lower to nothing)."""
    r, c = e.rows, e.cols
    blocks = []
    for j in range(copies):
        parts = []
        if j:
            parts.append(L.ZeroOp(r, j * c))
        parts.append(e)
        if copies - 1 - j:
            parts.append(L.ZeroOp(r, (copies - 1 - j) * c))
        blocks.append(parts[0] if len(parts) == 1 else
                      L.AdjointOf(L.VStack([L.derive_adjoint(pp) for pp in parts])))
    return blocks[0] if copies == 1 else L.VStack(blocks)


def _kron_tree(e, adj: bool):
    """Kron(Lk, Rk) (np.kron convention; adjoint = Kron(Lk^T, Rk^T)) as
    plan-lowerable structure: with x viewed as X (q x s) row-major,
        T1 = (I_q (x) R) x              Z = X R^T, rows of X
        T2 = P1 T1                       Z^T (r x q)
        T3 = (I_r (x) L) T2              (L Z)^T
        y  = P2 T3                       L Z = L X R^T, row-major (p x r)
    so the device runs R and L as ordinary leaves and two sparse
    permutations.  Cached on the expression per direction."""
    cache = e.__dict__.setdefault("_cgb_kron", {})
    if adj in cache:
        return cache[adj]
    Lk = L.AdjointOf(e.left) if adj else e.left
    Rk = L.AdjointOf(e.right) if adj else e.right
    p, q = Lk.rows, Lk.cols
    r, s = Rk.rows, Rk.cols
    j = np.repeat(np.arange(q), r)
    kk = np.tile(np.arange(r), q)
    p1 = _perm(kk * q + j)                        # T1[j*r + kk] -> T2[kk*q + j]
    kk2 = np.repeat(np.arange(r), p)
    i2 = np.tile(np.arange(p), r)
    p2 = _perm(i2 * r + kk2)                      # T3[kk*p + i] -> y[i*r + kk]
    tree = L.Compose(p2, L.Compose(_block_diag(Lk, r), L.Compose(p1, _block_diag(Rk, q))))
    cache[adj] = tree
    return tree


class _Builder:
    def __init__(self):
        self.leaves: list[_lib.Leaf] = []
        self.leaf_key: dict = {}
        self.terms: list[tuple] = []  # (leaf, in_buf, row_origin, in_off, alpha, out_buf)
        self.temp_len: list[int] = []
        self.temp_level: list[int] = []
        self.keep: list = []
        self.leaf_nnz: dict[int, int] = {}  # CSR leaf index -> nnz (roofline bytes)

    # -- leaves -------------------------------------------------------------
    def _add_leaf(self, key, make):
        idx = self.leaf_key.get(key)
        if idx is None:
            leaf, nbytes = make()
            idx = len(self.leaves)
            self.leaves.append(leaf)
            self.leaf_key[key] = idx
        return idx

    def leaf(self, e, adj: bool) -> int:
        if isinstance(e, (L.DenseMatrix, L.SparseMatrix)) and e._transpose_of is not None:
            e, adj = e._transpose_of, not adj
        if isinstance(e, L.Identity):
            n = e.rows
            return self._add_leaf(("I", n), lambda: (_lib.Leaf(kind=_lib.LEAF_IDENTITY, rows=n,
                                                               cols=n), 0))
        if isinstance(e, L.DenseMatrix):
            def make():
                buf = _leaf_buffers(e)
                key = "adj" if adj else "fwd"
                if key not in buf:
                    buf[key] = _cuda(e.values.T if adj else e.values)
                t = buf[key]
                self.keep.append(t)
                rows, cols = (e.cols, e.rows) if adj else (e.rows, e.cols)
                return _lib.Leaf(kind=_lib.LEAF_DENSE, rows=rows, cols=cols,
                                 val=t.data_ptr(), ld=cols), 0
            return self._add_leaf((id(e), adj), make)
        if isinstance(e, L.SparseMatrix):
            def make():
                buf = _leaf_buffers(e)
                key = "adj" if adj else "fwd"
                if key not in buf:
                    csc = e.matrix
                    if adj:  # CSC of A == CSR of A^T
                        ptr, idx, val = csc.indptr, csc.indices, csc.data
                    else:
                        csr = csc.tocsr()
                        csr.sort_indices()
                        ptr, idx, val = csr.indptr, csr.indices, csr.data
                    buf[key] = (_cuda(ptr, np.int64), _cuda(idx, np.int32),
                                _cuda(val, np.float64))
                p, i, v = buf[key]
                self.keep.extend((p, i, v))
                rows, cols = (e.cols, e.rows) if adj else (e.rows, e.cols)
                self.leaf_nnz[len(self.leaves)] = int(e.matrix.nnz)
                return _lib.Leaf(kind=_lib.LEAF_CSR, rows=rows, cols=cols, val=v.data_ptr(),
                                 rowptr=p.data_ptr(), colidx=i.data_ptr()), 0
            return self._add_leaf((id(e), adj), make)
        if isinstance(e, L.Conv1D):
            def make():
                buf = _leaf_buffers(e)
                if "kernel" not in buf:
                    buf["kernel"] = _cuda(e.kernel)
                t = buf["kernel"]
                self.keep.append(t)
                k, n = len(e.kernel), e.n
                if adj:
                    return _lib.Leaf(kind=_lib.LEAF_CORR1D, rows=n, cols=n + k - 1,
                                     val=t.data_ptr(), k0=k, n0=n), 0
                return _lib.Leaf(kind=_lib.LEAF_CONV1D, rows=n + k - 1, cols=n,
                                 val=t.data_ptr(), k0=k, n0=n), 0
            return self._add_leaf((id(e), adj), make)
        if isinstance(e, L.Conv2D):
            def make():
                buf = _leaf_buffers(e)
                if "kernel" not in buf:
                    buf["kernel"] = _cuda(e.kernel)
                t = buf["kernel"]
                self.keep.append(t)
                kh, kw = e.kernel.shape
                h, w = e.image_shape
                kind = _lib.LEAF_CORR2D if adj else _lib.LEAF_CONV2D
                rows, cols = (e.cols, e.rows) if adj else (e.rows, e.cols)
                return _lib.Leaf(kind=kind, rows=rows, cols=cols, val=t.data_ptr(), k0=kh,
                                 k1=kw, n0=h, n1=w,
                                 reserved=_lib.LEAF_FLAG_SEPARABLE if separable(e.kernel)
                                 else 0), 0
            return self._add_leaf((id(e), adj), make)
        raise L.LinOpError(f"no device leaf for {type(e).__name__}")

    # -- lowering -------------------------------------------------------------
    def new_temp(self, length: int, level: int) -> int:
        self.temp_len.append(int(length))
        self.temp_level.append(level)
        return len(self.temp_len)  # buffer id (t+1)

    def emit(self, e, adj, in_buf, in_off, out_buf, out_row, alpha, level):
        if alpha == 0.0:
            return
        if isinstance(e, L.ZeroOp):
            return
        if isinstance(e, L.Scale):
            self.emit(e.child, adj, in_buf, in_off, out_buf, out_row, alpha * e.alpha, level)
            return
        if isinstance(e, L.Sum):
            self.emit(e.left, adj, in_buf, in_off, out_buf, out_row, alpha, level)
            self.emit(e.right, adj, in_buf, in_off, out_buf, out_row, alpha, level)
            return
        if isinstance(e, L.AdjointOf):
            self.emit(e.child, not adj, in_buf, in_off, out_buf, out_row, alpha, level)
            return
        if isinstance(e, L.VStack):
            off = 0
            for c in e.children:
                if adj:   # sum_i child_i^T y[block i]
                    self.emit(c, True, in_buf, in_off + off, out_buf, out_row, alpha, level)
                else:     # stacked outputs
                    self.emit(c, False, in_buf, in_off, out_buf, out_row + off, alpha, level)
                off += c.rows
            return
        if isinstance(e, L.Compose):
            first, second = (e.left, e.right) if adj else (e.right, e.left)
            s1, s2 = _scaled_identity(first), _scaled_identity(second)
            if s1 is not None:
                self.emit(second, adj, in_buf, in_off, out_buf, out_row, alpha * s1, level)
                return
            if s2 is not None:
                self.emit(first, adj, in_buf, in_off, out_buf, out_row, alpha * s2, level)
                return
            inner = e.right.rows
            t = self.new_temp(inner, level + 1)
            self.emit(first, adj, in_buf, in_off, t, 0, 1.0, level + 1)
            self.emit(second, adj, t, 0, out_buf, out_row, alpha, level)
            return
        if isinstance(e, L.Kron):
            self.emit(_kron_tree(e, adj), False, in_buf, in_off, out_buf, out_row, alpha, level)
            return
        rows = e.cols if adj else e.rows
        if rows == 0 or (e.rows if adj else e.cols) == 0:
            return
        if isinstance(e, L.DenseMatrix) and self._emit_split_dense(e, adj, in_buf, in_off,
                                                                   out_buf, out_row, alpha, level):
            return
        if isinstance(e, L.Conv1D) and len(e.kernel) > CONV_KMAX:
            self._emit_split_conv(e, adj, in_buf, in_off, out_buf, out_row, alpha, level)
            return
        li = self.leaf(e, adj)
        self.terms.append((li, in_buf, out_row, in_off, float(alpha), out_buf))

    # short-wide GEMV (e.g. A^T of a tall A): a warp per row block would put
    # a handful of warps on the whole matrix, so the columns are split into
    # P slices whose partial products land in a temporary one level deeper,
    # summed by P identity terms -- a deterministic split-K.
    SPLIT_MIN_COLS = 8192

    def _emit_split_dense(self, e, adj, in_buf, in_off, out_buf, out_row, alpha, level) -> bool:
        base, badj = (e._transpose_of, not adj) if e._transpose_of is not None else (e, adj)
        rows, cols = (base.cols, base.rows) if badj else (base.rows, base.cols)
        if cols < self.SPLIT_MIN_COLS or cols < 16 * rows:
            return False
        nsplit = int(min(32, -(-cols // 4096)))
        chunk = -(-cols // nsplit)
        nsplit = -(-cols // chunk)
        t = self.new_temp(nsplit * rows, level + 1)
        for k in range(nsplit):
            c0 = k * chunk
            cw = min(chunk, cols - c0)

            def make(c0=c0, cw=cw):
                buf = _leaf_buffers(base)
                key = "adj" if badj else "fwd"
                if key not in buf:
                    buf[key] = _cuda(base.values.T if badj else base.values)
                tt = buf[key]
                self.keep.append(tt)
                return _lib.Leaf(kind=_lib.LEAF_DENSE, rows=rows, cols=cw,
                                 val=tt.data_ptr() + 8 * c0, ld=cols), 0
            li = self._add_leaf((id(base), badj, "split", k, nsplit), make)
            self.terms.append((li, in_buf, k * rows, in_off + c0, 1.0, t))
        ident = self._add_leaf(("I", rows), lambda: (_lib.Leaf(kind=_lib.LEAF_IDENTITY,
                                                               rows=rows, cols=rows), 0))
        for k in range(nsplit):
            self.terms.append((ident, t, out_row, k * rows, float(alpha), out_buf))
        return True

    # long 1-d kernels (the reference's own deconvolution family uses
    # kernel length n; it switches to FFT above 512 taps, linop.py:35-50):
    # the taps are cut into blocks of <= CONV_KMAX, each an ordinary tiled
    # conv leaf, and the blocks' contributions are summed by the row block's
    # term list (deterministic order, no atomics):
    #   full conv   y[i]  = sum_b conv(c_b, x)[i - j_b]      (output shift j_b)
    #   valid corr  y[i]  = sum_b corr(c_b, x[j_b:])[i]       (input shift j_b)
    def _emit_split_conv(self, e, adj, in_buf, in_off, out_buf, out_row, alpha, level):
        k, n = len(e.kernel), e.n
        nblk = -(-k // CONV_KMAX)
        blk = -(-k // nblk)
        parts = e.__dict__.setdefault("_cgb_tap_blocks", {})
        for j0 in range(0, k, blk):
            sub = parts.get(j0)
            if sub is None:
                sub = parts[j0] = L.Conv1D(e.kernel[j0:j0 + blk], n)
            if adj:
                self.emit(sub, True, in_buf, in_off + j0, out_buf, out_row, alpha, level)
            else:
                self.emit(sub, False, in_buf, in_off, out_buf, out_row + j0, alpha, level)

    def finish(self, in_len: int, out_len: int):
        buf_len = [out_len] + self.temp_len
        # stage of a buffer = 1 + max stage of the buffers its terms read
        # (input = stage 0); every term runs at its output buffer's stage.
        writers: dict[int, list] = {b: [] for b in range(len(buf_len))}
        for t in self.terms:
            writers[t[5]].append(t)
        stage: dict[int, int] = {}

        def stage_of(buf: int) -> int:  # buffer id; -1 is the apply input
            if buf == -1:
                return 0
            if buf not in stage:
                srcs = [(-1 if t[1] == 0 else t[1]) for t in writers[buf]]
                stage[buf] = 1 + max((stage_of(s) for s in srcs), default=0)
            return stage[buf]

        # temporaries that never reach the output (e.g. composed with a zero
        # operator) are dropped: length 0, no terms
        live = {0}
        frontier = [0]
        while frontier:
            b = frontier.pop()
            for t in writers[b]:
                if t[1] != 0 and t[1] not in live:
                    live.add(t[1])
                    frontier.append(t[1])
        for b in range(1, len(buf_len)):
            if b not in live:
                buf_len[b] = 0
                writers[b] = []
        self.terms = [t for t in self.terms if t[5] in live]
        self.temp_len = buf_len[1:]
        top = stage_of(0)
        buf_level = [top - stage_of(b) if b in live else 1 for b in range(len(buf_len))]
        if any(lv < 0 for lv in buf_level):
            raise L.LinOpError("plan lowering produced an inconsistent stage order")
        self.temp_level = buf_level[1:]
        terms_c: list[_lib.Term] = []
        rbs: list[_lib.RowBlock] = []
        by_buf: dict[int, list] = {b: [] for b in range(len(buf_len))}
        for t in self.terms:
            by_buf[t[5]].append(t)
        for b, length in enumerate(buf_len):
            if length == 0:
                continue
            ts = by_buf[b]
            cuts = {0, length}
            for (li, _, r0, _, _, _) in ts:
                cuts.add(r0)
                cuts.add(r0 + self.leaves[li].rows)
            cuts = sorted(c for c in cuts if 0 <= c <= length)
            for a, z in zip(cuts[:-1], cuts[1:]):
                if z <= a:
                    continue
                begin = len(terms_c)
                for (li, ib, r0, io, al, _) in ts:
                    if r0 <= a and z <= r0 + self.leaves[li].rows:
                        terms_c.append(_lib.Term(leaf=li, in_buf=ib, row_origin=r0, in_off=io,
                                                 alpha=al))
                rbs.append(_lib.RowBlock(row_begin=a, row_end=z, out_buf=b, level=buf_level[b],
                                         term_begin=begin, term_end=len(terms_c)))
        arr_leaves = (_lib.Leaf * max(1, len(self.leaves)))(*self.leaves)
        arr_terms = (_lib.Term * max(1, len(terms_c)))(*terms_c)
        arr_rbs = (_lib.RowBlock * max(1, len(rbs)))(*rbs)
        arr_tl = (ctypes.c_int64 * max(1, len(self.temp_len)))(*self.temp_len)
        desc = _lib.PlanDesc(in_len=in_len, out_len=out_len, nleaves=len(self.leaves),
                             nterms=len(terms_c), nrowblocks=len(rbs),
                             ntemps=len(self.temp_len), leaves=arr_leaves, terms=arr_terms,
                             rowblocks=arr_rbs, temp_len=arr_tl)
        self.keep_c = (arr_leaves, arr_terms, arr_rbs, arr_tl)
        self.nlevels = 1 + max(self.temp_level, default=0)
        self.nrowblocks = len(rbs)
        self.nterms = len(terms_c)
        return desc


def _leaf_data_bytes(leaf: _lib.Leaf, nnz: int) -> int:
    """Compulsory HBM bytes of a leaf's own data (matrix values / indices)."""
    k = leaf.kind
    if k == _lib.LEAF_DENSE:
        return 8 * leaf.rows * leaf.cols
    if k == _lib.LEAF_CSR:
        return 12 * nnz + 8 * (leaf.rows + 1)
    if k in (_lib.LEAF_CONV1D, _lib.LEAF_CORR1D):
        return 8 * leaf.k0
    if k in (_lib.LEAF_CONV2D, _lib.LEAF_CORR2D):
        return 8 * leaf.k0 * leaf.k1
    return 0


def _leaf_flops(leaf: _lib.Leaf, nnz: int) -> int:
    """Algorithmic float64 flops (2 per multiply-add) of one leaf application."""
    k = leaf.kind
    if k == _lib.LEAF_DENSE:
        return 2 * leaf.rows * leaf.cols
    if k == _lib.LEAF_CSR:
        return 2 * nnz
    if k in (_lib.LEAF_CONV1D, _lib.LEAF_CORR1D):
        return 2 * leaf.n0 * leaf.k0          # every signal sample meets every tap once
    if k in (_lib.LEAF_CONV2D, _lib.LEAF_CORR2D):
        if leaf.reserved & _lib.LEAF_FLAG_SEPARABLE:   # column pass + row pass per output
            return 2 * leaf.rows * (leaf.k0 + leaf.k1)
        return 2 * leaf.n0 * leaf.n1 * leaf.k0 * leaf.k1
    return 0


class DeviceOp:
    """Compiled forward + adjoint plans of one expression (a cgb_op)."""

    def __init__(self, expr, ctx=None):
        self.ctx = ctx if ctx is not None else _lib.device_context()
        self.rows, self.cols = expr.rows, expr.cols
        self.fwd = _Builder()
        self.fwd.emit(expr, False, 0, 0, 0, 0, 1.0, 0)
        self.adj = _Builder()
        self.adj.emit(expr, True, 0, 0, 0, 0, 1.0, 0)
        self.handle = None
        self._empty = self.rows == 0 or self.cols == 0
        if self._empty:
            return
        fdesc = self.fwd.finish(self.cols, self.rows)
        adesc = self.adj.finish(self.rows, self.cols)
        h = ctypes.c_void_p()
        lib = _lib.load_library()
        _lib.check(lib.cgb_op_create(self.ctx.handle, ctypes.byref(fdesc), ctypes.byref(adesc),
                                     ctypes.byref(h)))
        self.handle = h
        self._lib = lib

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.cgb_op_destroy(h)
            except Exception:  # noqa: BLE001 - interpreter shutdown
                pass

    def apply(self, x, out=None, adjoint: bool = False):
        import torch
        n_out = self.cols if adjoint else self.rows
        if out is None:
            out = torch.empty(n_out, dtype=torch.float64, device=x.device)
        if self._empty:
            out.zero_()
            return out
        _lib.check(self._lib.cgb_op_apply(self.ctx.handle, self.handle, int(adjoint),
                                          _lib.ptr(x), _lib.ptr(out), _lib.stream_handle()))
        return out

    def plan_info(self, adjoint: bool = False) -> dict:
        b = self.adj if adjoint else self.fwd
        return {"leaves": len(b.leaves), "terms": getattr(b, "nterms", 0),
                "rowblocks": getattr(b, "nrowblocks", 0), "levels": getattr(b, "nlevels", 1),
                "temps": len(b.temp_len)}

    def algo_flops(self, adjoint: bool = False) -> int:
        """Algorithmic flops of one application (leaf multiply-adds; the
        alpha-scaled term sums are not counted)."""
        b = self.adj if adjoint else self.fwd
        return sum(_leaf_flops(leaf, b.leaf_nnz.get(i, 0)) for i, leaf in enumerate(b.leaves))

    def algo_bytes(self, adjoint: bool = False) -> int:
        """Compulsory bytes of one application: operand reads + output write."""
        b = self.adj if adjoint else self.fwd
        total = sum(_leaf_data_bytes(leaf, b.leaf_nnz.get(i, 0))
                    for i, leaf in enumerate(b.leaves))
        n_in, n_out = (self.rows, self.cols) if adjoint else (self.cols, self.rows)
        return total + 8 * n_in + 8 * n_out + 16 * sum(b.temp_len)
