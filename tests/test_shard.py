"""Row-sharded solver: host partitioning on CPU (row /
column slicing of expressions, row cuts, cone pieces, and the partition
agreeing across two gloo ranks), and on the GPU the per-rank persistent
kernels -- two ranks sharing one device -- against the oracle: the setup
solve, the first iterates (before rounding chaos sets in) and full solves."""

import os
import socket

import numpy as np
import pytest
import scipy.sparse

from oracle import linop_ref


def _lasso(m, n, density, seed, lam_frac=0.1):
    from paper_1609_03488_b200 import canon, linop
    rng = np.random.default_rng(seed)
    A = scipy.sparse.random(m, n, density=density, random_state=rng, format="csc")
    A.data = rng.standard_normal(A.nnz)
    x = rng.standard_normal(n) * (rng.uniform(size=n) < 0.1)
    b = A @ x + 0.01 * rng.standard_normal(m)
    lam = lam_frac * float(np.max(np.abs(A.T @ b)))
    return canon.build_lasso(canon.LassoProblem(linop.sparse_csc(A), b, lam))


def _mixed_expr(seed=0):
    """A stacked operator with every sliceable leaf kind."""
    from paper_1609_03488_b200 import linop as L
    rng = np.random.default_rng(seed)
    S = L.SparseMatrix(scipy.sparse.random(7, 5, density=0.4, random_state=rng, format="csc"))
    D = L.DenseMatrix(rng.standard_normal((4, 5)))
    top = L.AdjointOf(L.VStack([L.derive_adjoint(L.Scale(2.0, S)),
                                L.derive_adjoint(L.Identity(7))]))          # [2S | I] 7 x 12
    mid = L.AdjointOf(L.VStack([L.derive_adjoint(D), L.ZeroOp(7, 4)]))      # [D | 0]  4 x 12
    low = L.Sum(L.Identity(12), L.Scale(-0.5, L.Identity(12)))              # 12 x 12
    comp = L.Compose(L.DenseMatrix(rng.standard_normal((3, 6))),
                     L.AdjointOf(L.VStack([L.Identity(6), L.ZeroOp(6, 6)])))  # 3 x 12
    return L.VStack([top, mid, low, comp])


@pytest.mark.parametrize("r0,r1", [(0, 26), (0, 1), (3, 9), (6, 14), (10, 23), (25, 26),
                                   (22, 26), (0, 11)])
def test_row_slice_matches_materialized(r0, r1):
    from paper_1609_03488_b200 import shard
    e = _mixed_expr()
    full = linop_ref.materialize(e)
    part = shard.row_slice(e, r0, r1)
    assert part.shape == (r1 - r0, e.cols)
    np.testing.assert_array_equal(linop_ref.materialize(part), full[r0:r1])


@pytest.mark.parametrize("c0,c1", [(0, 12), (0, 5), (5, 12), (2, 9), (11, 12)])
def test_col_slice_matches_materialized(c0, c1):
    from paper_1609_03488_b200 import shard
    e = _mixed_expr(1)
    full = linop_ref.materialize(e)
    np.testing.assert_array_equal(linop_ref.materialize(shard.col_slice(e, c0, c1)),
                                  full[:, c0:c1])


def test_slice_refuses_to_cut_a_convolution():
    from paper_1609_03488_b200 import linop as L
    from paper_1609_03488_b200 import shard
    C = L.Conv1D(np.ones(3), 10)
    with pytest.raises(L.LinOpError):
        shard.row_slice(C, 2, 5)
    v = L.VStack([L.Identity(10), C])
    assert shard.row_slice(v, 0, 10).shape == (10, 10)       # a cut beside it is fine
    assert shard.row_nnz(v).shape == (22,)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_lasso_partition(world):
    from paper_1609_03488_b200 import shard
    prob = _lasso(300, 60, 0.05, 3)
    n, m = prob.A.cols, prob.A.rows
    cuts = shard.plan_cuts(prob, world)
    assert cuts[0] == 0 and cuts[-1] == m and all(a <= b for a, b in zip(cuts, cuts[1:]))
    xb = shard.x_slices(n, world)
    assert xb[0] == 0 and xb[-1] == n and all(x % 2 == 0 for x in xb[:-1])
    socs = shard._world_socs(prob.K, cuts)
    full = linop_ref.materialize(prob.A.expr)
    rows, pieces_dim = [], 0
    for q in range(world):
        part = shard.row_slice(prob.A.expr, cuts[q], cuts[q + 1])
        rows.append(linop_ref.materialize(part))
        kinds, bg, en, sid, hd = shard.cone_pieces(prob.K, cuts[q], cuts[q + 1], socs)
        assert bg == sorted(bg) and (not bg or bg[0] == 0)
        assert (en[-1] if en else 0) == cuts[q + 1] - cuts[q]
        pieces_dim += sum(e - b for b, e in zip(bg, en))
        # the big SOC (rows 2n' .. m) has its head on the rank holding row 2n'
        head_row = 2 * ((n - 1) // 2)
        soc_heads = [hd[i] for i in range(len(kinds)) if kinds[i] == 2]
        assert sum(soc_heads) == int(cuts[q] <= head_row < cuts[q + 1])
    np.testing.assert_array_equal(np.vstack(rows), full)
    assert pieces_dim == m
    if world > 1:
        assert socs == [2 * ((n - 1) // 2)]            # the (m+2)-SOC is world-reduced
    # balance: every rank's estimated cost within 2x of the mean
    w = shard.ROW_BASE_COST + shard.NNZ_COST * shard.row_nnz(prob.A.expr)
    cost = [w[cuts[q]:cuts[q + 1]].sum() for q in range(world)]
    assert max(cost) <= 2.0 * np.mean(cost) + w.max()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1609_03488_b200 import shard
        prob = _lasso(400, 80, 0.04, 11)
        lay = shard.layout_for(prob, world, rank)
        part = shard.row_slice(prob.A.expr, lay.y0, lay.y1)
        mat = torch.from_numpy(linop_ref.materialize(part))
        sizes = [None] * world
        dist.all_gather_object(sizes, (lay.y0, lay.y1, lay.x0, lay.x1, tuple(lay.world_socs)))
        rows = [None] * world
        dist.all_gather_object(rows, mat.numpy())
        out[rank] = (sizes, rows, shard.cone_pieces(prob.K, lay.y0, lay.y1, lay.world_socs))
    finally:
        dist.destroy_process_group()


def test_partition_agrees_across_gloo_ranks():
    """Every rank derives the same cuts and slices independently (no
    coordination beyond the problem itself); the ranks' row blocks stack to
    the full operator and their x slices tile [0, n)."""
    import torch.multiprocessing as mp
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_gloo_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    prob = _lasso(400, 80, 0.04, 11)
    assert res[0][0] == res[1][0]
    sizes = res[0][0]
    assert sizes[0][1] == sizes[1][0] and sizes[1][1] == prob.A.rows
    assert sizes[0][3] == sizes[1][2] and sizes[1][3] == prob.A.cols
    np.testing.assert_array_equal(np.vstack(res[0][1]), linop_ref.materialize(prob.A.expr))
    heads = sum(h for r in range(world) for h, s in zip(res[r][2][4], res[r][2][3]) if s >= 0)
    assert heads == 1


# ---------------------------------------------------------------------------
# GPU: two ranks on one device
# ---------------------------------------------------------------------------

def _oracle_problem(prob):
    class P:
        pass
    p = P()
    p.A, p.b, p.c, p.K = prob.A.expr, prob.b, prob.c, prob.K
    return p


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3])
def test_shard_setup_matches_oracle(world):
    from oracle import scs_ref
    from paper_1609_03488_b200 import scs, shard
    prob = _lasso(2000, 300, 0.01, 5)
    st = scs.ScsSettings(eps=1e-3, max_iters=5000)
    grp = shard.ShardGroup(prob, st, world=world)
    try:
        import torch
        torch.cuda.synchronize()
        _, _, _, gx, gy = grp.gather()
        ref = scs_ref.prepare_subspace(_oracle_problem(prob), st.setup_cg_tol, st.cg_max_iter)
        n = prob.A.cols
        g = np.concatenate([gx, gy])
        assert np.linalg.norm(g - ref.g) <= 1e-9 * np.linalg.norm(ref.g)
        denom = grp.ranks[0].state()[10]
        assert abs(denom - ref.denom) <= 1e-10 * abs(ref.denom)
        for r in grp.ranks[1:]:   # identical on every rank
            assert r.state()[10] == denom
        assert n == len(gx)
    finally:
        grp.close()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2])
def test_shard_first_iterates_match_oracle(world):
    """Iterates 1..12 of the sharded kernel vs the oracle's (scs_ref.iterate)
    at 1e-8 relative: the splitting map is still contractive there, so the
    decomposition's different summation order stays at rounding level."""
    from oracle import scs_ref
    from paper_1609_03488_b200 import scs, shard
    import torch
    prob = _lasso(2000, 300, 0.01, 5)
    st = scs.ScsSettings(eps=1e-3, max_iters=5000)
    grp = shard.ShardGroup(prob, st, world=world)
    try:
        op = _oracle_problem(prob)
        s = scs_ref.ScsOracleSettings(eps=1e-3, max_iters=5000)
        cached = scs_ref.prepare_subspace(op, s.setup_cg_tol, s.cg_max_iter)
        ref = {k: stt for k, stt in scs_ref.iterate(op, s, cached, 12)}
        grp.reset()
        done = 0
        for k in (1, 5, 12):
            grp.run(k - done)
            done = k
            torch.cuda.synchronize()
            sts = grp.states()
            assert all(x[0] == k for x in sts)
            ux, uy, vy, _, _ = grp.gather()
            r = ref[k]
            n = prob.A.cols
            # u_y is written on check / last iterations: the last of each call
            u = np.concatenate([ux, uy, [sts[0][8]]])
            v = np.concatenate([np.zeros(n), vy, [sts[0][9]]])
            scale = 1.0 + np.linalg.norm(r.u)
            assert np.linalg.norm(u - r.u) <= 1e-8 * scale, k
            assert np.linalg.norm(v - r.v) <= 1e-8 * scale, k
            assert sts[0][3] == r.cgt
    finally:
        grp.close()


@pytest.mark.gpu
@pytest.mark.parametrize("world,m,n,seed", [(2, 2000, 300, 5), (2, 6000, 1000, 8),
                                            (3, 6000, 1000, 8)])
def test_shard_solve_matches_oracle(world, m, n, seed):
    """Full solves: status, residual certificate recomputed with the oracle's
    applies, iteration count within 2 % or one check interval, objective
    within eps of the oracle's (1e-6 when the counts agree)."""
    from oracle import scs_ref
    from paper_1609_03488_b200 import scs, shard
    prob = _lasso(m, n, 0.01, seed)
    st = scs.ScsSettings(eps=1e-3, max_iters=20000)
    grp = shard.ShardGroup(prob, st, world=world)
    try:
        sol = grp.solve()
    finally:
        grp.close()
    osol, _ = scs_ref.scs_solve(_oracle_problem(prob),
                                scs_ref.ScsOracleSettings(eps=1e-3, max_iters=20000))
    assert sol.status == osol.status == "solved"
    A = prob.A.expr
    pr = np.linalg.norm(linop_ref.forward(A, sol.x) + sol.s - prob.b) / (1 + np.linalg.norm(prob.b))
    dr = np.linalg.norm(linop_ref.adjoint(A, sol.y) + prob.c) / (1 + np.linalg.norm(prob.c))
    assert max(pr, dr) <= st.eps * (1 + 1e-6)
    assert abs(sol.iterations - osol.iterations) <= max(0.02 * osol.iterations,
                                                        st.check_interval)
    # lasso instances are rounding-chaotic (the reference's own 4-ulp
    # envelopes of the golden lasso cases span 1360-3080 iterations, and the
    # single-GPU solver departs from the oracle the same way:
    # tools/shard_diag.py), so the objective is held to the eps-level rule
    # of the single-GPU golden test (10 eps relative; the gap alone allows
    # eps (1 + |c.x| + |b.y|))
    rel = abs(sol.pobj - osol.pobj) / abs(osol.pobj)
    assert rel <= 10 * st.eps, rel


def test_cuts_keep_convolution_blocks_whole():
    from paper_1609_03488_b200 import canon, shard
    c = canon.gaussian_kernel(11)
    prob = canon.build_deconv(canon.DeconvProblem(c, np.ones(60 + 10), n=60))
    cuts = shard.plan_cuts(prob, 2)
    assert cuts == [0, 61, prob.A.rows]            # identity rows | the conv block
    assert shard.whole_spans(prob.A.expr) == [(61, prob.A.rows)]
    with pytest.raises(Exception):
        shard.plan_cuts(prob, 3)                    # only one admissible cut


# ---------------------------------------------------------------------------
# GPU: golden reference cases, sharded over ranks sharing one device
# ---------------------------------------------------------------------------

def _golden_problem(name):
    from _golden import build_cones, build_tree, load
    from paper_1609_03488_b200 import cones, linop, scs
    data, meta = load(name)
    A = linop.Operator(build_tree(meta["tree"], data, linop))
    K = cones.ConeProduct(build_cones(meta["cones"], cones))
    return scs.ConeProblem(A, np.array(data["b"]), np.array(data["c"]), K), data, meta


def _golden_names():
    from _golden import scs_case_names
    return scs_case_names()


def _group_or_skip(prob, st, world):
    from paper_1609_03488_b200 import linop, shard
    try:
        shard.plan_cuts(prob, world)
    except linop.LinOpError as exc:
        pytest.skip(str(exc))
    return shard.ShardGroup(prob, st, world=world)


@pytest.mark.gpu
@pytest.mark.parametrize("name", _golden_names())
def test_shard_trace_matches_reference(name):
    """First 10 iterates of the 2-rank sharded kernel vs the REAL reference's
    trace (tests/golden, make_golden.py) at 1e-7, like the single-GPU test."""
    import torch
    from paper_1609_03488_b200 import scs
    prob, data, meta = _golden_problem(name)
    grp = _group_or_skip(prob, scs.ScsSettings(**meta["settings"]), 2)
    try:
        assert abs(grp.ranks[0].state()[10] - meta["denom"]) <= 1e-9 * abs(meta["denom"])
        tu, tv, tcg = data["trace_u"], data["trace_v"], data["trace_cgt"]
        grp.reset()
        n = prob.A.cols
        for k in range(1, min(len(tu), 10) + 1):
            grp.run(1)
            torch.cuda.synchronize()
            st = grp.states()
            ux, uy, vy, _, _ = grp.gather()
            u = np.concatenate([ux, uy, [st[0][8]]])
            v = np.concatenate([np.zeros(n), vy, [st[0][9]]])
            assert np.linalg.norm(u - tu[k - 1]) <= 1e-7 * (1 + np.linalg.norm(tu[k - 1])), k
            assert np.linalg.norm(v - tv[k - 1]) <= 1e-7 * (1 + np.linalg.norm(tv[k - 1])), k
            assert abs(st[0][3] - tcg[k - 1]) <= 1
    finally:
        grp.close()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", _golden_names())
def test_shard_solve_matches_reference(name, world):
    """Full sharded solves of the golden cases under the single-GPU parity
    rule: status identical; zero-spread reference envelope -> the exact
    iteration count and the objective to 1e-6; chaotic instances -> inside
    the reference's own 4-ulp envelope (+- one check interval) or 2 %, the
    objective within the envelope's spread."""
    import json
    from paper_1609_03488_b200 import scs
    prob, data, meta = _golden_problem(name)
    st = scs.ScsSettings(**meta["settings"])
    grp = _group_or_skip(prob, st, world)
    try:
        sol = grp.solve()
    finally:
        grp.close()
    assert sol.status == meta["status"], (sol.status, sol.iterations, meta["iterations"])
    env = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                                      "scs_envelopes.json"))).get(name)
    it_ref = meta["iterations"]
    its = [it_ref] + (env["iterations"] if env else [])
    zero_spread = min(its) == max(its)
    if zero_spread:
        assert sol.iterations == it_ref, (sol.iterations, it_ref)
    else:
        in_env = min(its) - st.check_interval <= sol.iterations <= max(its) + st.check_interval
        assert abs(sol.iterations - it_ref) <= 0.02 * it_ref or in_env, (sol.iterations, its)
    if sol.status == "solved":
        ref = meta["pobj"]
        if sol.iterations == it_ref and zero_spread:
            tol = 1e-6 * max(1.0, abs(ref))
        else:
            pobjs = [p for p, s_ in zip(env["pobj"], env["status"]) if s_ == "solved"]
            spread = max([abs(p - ref) for p in pobjs] + [0.0])
            tol = 2.0 * spread + 10 * st.eps * max(1.0, abs(ref))
        assert abs(sol.pobj - ref) <= tol, (sol.pobj, ref, tol)


def _ipc_worker(rank, world, port, name, out):
    """One rank of a 2-process sharded solve on ONE GPU: the IPC handle
    exchange, cudaIpcOpenMemHandle'd peer buffers, rank-0 gather."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), CGB_GRID="16")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1609_03488_b200 import scs, shard
        prob, _, meta = _golden_problem(name)
        sol, rs = shard.solve_sharded(prob, scs.ScsSettings(**meta["settings"]))
        st = rs.state()
        out[rank] = (None if sol is None else (sol.status, sol.iterations, float(sol.pobj)),
                     float(st[0]), float(st[11]))
        rs.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["scs_lp_equality", "scs_soc_ball"])
def test_multiprocess_ipc_sharded_solve(name):
    """shard.solve_sharded as a 2-process torch.distributed job sharing one
    GPU (the transport of a one-rank-per-GPU run: peer buffers allocated by
    cgb_ipc_alloc, handles exchanged with all_gather_object, mapped with
    cgb_ipc_open).  Without MPS the two contexts time-slice the GPU, so the
    case is tiny; the result must equal the reference's exactly."""
    import torch.multiprocessing as mp
    _, _, meta = _golden_problem(name)
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_ipc_worker, args=(world, port, name, out), nprocs=world, join=True)
        res = dict(out)
    sol0 = res[0][0]
    assert sol0 is not None and res[1][0] is None          # gathered on rank 0
    assert res[0][1] == res[1][1] and res[0][2] == res[1][2]  # same k, same epoch
    assert sol0[0] == meta["status"] and sol0[1] == meta["iterations"], (sol0, meta["iterations"])
    if sol0[0] == "solved":
        assert abs(sol0[2] - meta["pobj"]) <= 1e-6 * max(1.0, abs(meta["pobj"]))
