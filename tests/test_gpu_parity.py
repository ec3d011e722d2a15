"""GPU parity: the CUDA path vs the reference's golden vectors and the oracle.

Every test here calls through the C ABI (libcgb200.so via ctypes) on a
B200.  Tolerances (north star): operator applies and cone projections to
1e-12 relative (only summation order differs), CG iteration counts within
one step, SCS status identical, iteration counts within +-2% (or one
check interval for short runs), objective within 1e-6 relative at
convergence, residuals <= eps.
"""

import ctypes
import json

import numpy as np
import pytest

import paper_1609_03488_b200 as pkg
from paper_1609_03488_b200 import cg, cones, linop, scs
from _golden import build_cones, build_tree, load, scs_case_names

pytestmark = pytest.mark.gpu


def _lib_loaded():
    from paper_1609_03488_b200 import _lib
    return _lib.load_library()


def test_library_is_the_native_path():
    from paper_1609_03488_b200 import _lib
    lib = _lib_loaded()
    assert lib.cgb_abi_version() == _lib.ABI_VERSION
    ctx = _lib.device_context()
    sms, per_sm, threads = ctx.geometry()
    assert sms >= 100 and per_sm >= 1 and threads >= 128


def test_linop_cases_match_reference():
    data, meta = load("linop_cases")
    for i, case in enumerate(meta["cases"]):
        op = linop.Operator(build_tree(case["tree"], data, linop))
        ax = op.forward(data[case["x"]])
        aty = op.adjoint_apply(data[case["y"]])
        sx = 1.0 + np.abs(data[case["ax"]]).max(initial=0)
        sy = 1.0 + np.abs(data[case["aty"]]).max(initial=0)
        np.testing.assert_allclose(ax, data[case["ax"]], rtol=1e-11, atol=1e-11 * sx,
                                   err_msg=f"case {i} forward")
        np.testing.assert_allclose(aty, data[case["aty"]], rtol=1e-11, atol=1e-11 * sy,
                                   err_msg=f"case {i} adjoint")
        assert linop.nnz_estimate(op) == case["nnz"]


def test_adjoint_identity_random():
    rng = np.random.default_rng(5)
    data, meta = load("linop_cases")
    for case in meta["cases"]:
        op = linop.Operator(build_tree(case["tree"], data, linop))
        x = rng.standard_normal(op.cols)
        y = rng.standard_normal(op.rows)
        ax, aty = op.forward(x), op.adjoint_apply(y)
        assert abs(ax @ y - x @ aty) <= 1e-10 * (1.0 + np.linalg.norm(ax) * np.linalg.norm(y))


def test_conv_by_hand_and_large():
    op = linop.conv1d([1.0, 1.0], 2)
    np.testing.assert_allclose(op.forward(np.array([1.0, 2.0])), [1.0, 3.0, 2.0])
    np.testing.assert_allclose(op.adjoint_apply(np.array([1.0, 3.0, 2.0])), [4.0, 5.0])
    from oracle import linop_ref
    rng = np.random.default_rng(1)
    for k, n in [(101, 100_000), (7, 33), (600, 550)]:
        c = rng.standard_normal(k)
        x = rng.standard_normal(n)
        y = rng.standard_normal(n + k - 1)
        op = linop.conv1d(c, n)
        f = op.forward(x)
        np.testing.assert_allclose(f, linop_ref.conv_full(c, x, "direct"), rtol=1e-10,
                                   atol=1e-11 * np.abs(f).max())
        a = op.adjoint_apply(y)
        np.testing.assert_allclose(a, linop_ref.corr_valid(c, y, "direct"), rtol=1e-10,
                                   atol=1e-11 * np.abs(a).max())


def test_conv2d_against_oracle():
    from oracle import linop_ref
    import _exprs as E
    rng = np.random.default_rng(2)
    for (h, w, kh, kw) in [(7, 5, 3, 3), (40, 33, 15, 15), (64, 64, 1, 5)]:
        K = rng.standard_normal((kh, kw))
        op = linop.conv2d(K, (h, w))
        ref = E.Conv2D(K, (h, w))
        x = rng.standard_normal(h * w)
        y = rng.standard_normal(op.rows)
        np.testing.assert_allclose(op.forward(x), linop_ref.forward(ref, x), rtol=1e-10,
                                   atol=1e-10)
        np.testing.assert_allclose(op.adjoint_apply(y), linop_ref.adjoint(ref, y), rtol=1e-10,
                                   atol=1e-10)


def test_cone_cases_match_reference():
    data, meta = load("cone_cases")
    for j, (kind, dim) in enumerate(meta["cones"]):
        cone = getattr(cones, kind)(dim)
        V, P = data[f"v{j}"], data[f"p{j}"]
        K = cones.ConeProduct([cone] * len(V))
        out = cones.project_product(K, V.reshape(-1)).reshape(V.shape)
        np.testing.assert_allclose(out, P, rtol=1e-13, atol=1e-13)
        if kind != "ZeroCone":
            outd = cones.project_product_dual(K, V.reshape(-1)).reshape(V.shape)
            np.testing.assert_allclose(outd, P, rtol=1e-13, atol=1e-13)
        else:
            np.testing.assert_array_equal(cones.project_product_dual(K, V.reshape(-1)),
                                          V.reshape(-1))


def test_large_soc_grid_reduction():
    from oracle import cones_ref
    import _exprs as E
    rng = np.random.default_rng(3)
    for dim in (5000, 300_001):
        v = rng.standard_normal(dim)
        for t0 in (0.0, 1e4, -1e4, np.linalg.norm(v[1:])):
            v[0] = t0
            got = cones.project(cones.SecondOrderCone(dim), v)
            want = cones_ref.project_cone(E.SecondOrderCone(dim), v)
            np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)


def test_cg_cases_match_reference():
    data, meta = load("cg_cases")
    for case in meta["cases"]:
        A = linop.Operator(build_tree(case["tree"], data, linop))
        b = data[case["b"]]
        rec = cg.operator_recipe(A) if case["recipe"] == "direct" else \
            cg.make_normal_operator(A, case["lam"])
        res = cg.cg_solve(cg.CgSpec(rec, b, np.zeros(len(b)), tol=case["tol"]))
        assert res.converged == case["converged"]
        assert abs(res.iterations - case["iters"]) <= 1
        ref = data[case["x"]]
        assert np.linalg.norm(res.x - ref) <= 1e-7 * np.linalg.norm(ref)


def test_cg_edge_cases():
    res = cg.cg_solve(cg.CgSpec(cg.operator_recipe(linop.identity(4)), np.zeros(4), np.zeros(4)))
    assert res.iterations == 0 and res.converged and res.final_residual_norm == 0.0
    b = np.array([3.0, -1.0, 2.0])
    res = cg.cg_solve(cg.CgSpec(cg.operator_recipe(linop.identity(3)), b, np.zeros(3)))
    np.testing.assert_allclose(res.x, b, atol=1e-14)
    assert res.iterations == 1
    rng = np.random.default_rng(6)
    M = rng.standard_normal((40, 40))
    Ad = M.T @ M + np.eye(40)
    res = cg.cg_solve(cg.CgSpec(cg.operator_recipe(linop.dense(Ad)), rng.standard_normal(40),
                                np.zeros(40), max_iter=2))
    assert not res.converged and res.iterations == 2


def test_subspace_cases_match_reference():
    data, meta = load("subspace_cases")
    for i, case in enumerate(meta["cases"]):
        A = linop.dense(data[f"A{i}"])
        prob = scs.ConeProblem(A, data[f"b{i}"], data[f"c{i}"],
                               cones.ConeProduct([cones.NonNegCone(case["m"])]))
        cached = scs.prepare_subspace(prob)
        np.testing.assert_allclose(cached.g, data[f"g{i}"], rtol=1e-9, atol=1e-11)
        out = scs.subspace_project(data[f"w{i}"], cached)
        np.testing.assert_allclose(out, data[f"out{i}"], rtol=1e-8, atol=1e-10)


def _problem(data, meta):
    A = linop.Operator(build_tree(meta["tree"], data, linop))
    K = cones.ConeProduct(build_cones(meta["cones"], cones))
    return scs.ConeProblem(A, np.array(data["b"]), np.array(data["c"]), K)


def _settings(meta):
    return scs.ScsSettings(**meta["settings"])


@pytest.mark.parametrize("name", scs_case_names())
def test_scs_trace_matches_reference(name):
    data, meta = load(name)
    prob = _problem(data, meta)
    graph = scs.build_scs_graph(prob, _settings(meta))
    assert abs(graph.cached.denom - meta["denom"]) <= 1e-9 * abs(meta["denom"])
    tu, tv, tcg = data["trace_u"], data["trace_v"], data["trace_cgt"]
    for k, state in scs.iterate_states(graph, min(len(tu), 10)):
        su = 1.0 + np.linalg.norm(tu[k - 1])
        assert np.linalg.norm(state[0] - tu[k - 1]) <= 1e-7 * su, f"u at iteration {k}"
        sv = 1.0 + np.linalg.norm(tv[k - 1])
        assert np.linalg.norm(state[1] - tv[k - 1]) <= 1e-7 * sv, f"v at iteration {k}"
        assert abs(state[6][0] - tcg[k - 1]) <= 1


def _envelope(name):
    """Iteration counts / objectives of the REAL reference re-solving this
    case with b, c perturbed by <= 4 ulp (tests/golden/make_envelopes.py)."""
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                        "scs_envelopes.json")
    with open(path) as fh:
        return json.load(fh).get(name)


@pytest.mark.parametrize("name", scs_case_names())
def test_scs_solve_matches_reference(name):
    """Status identical; iteration count within 2% of the reference or
    inside the reference's own rounding envelope (+- one check interval):
    the inexact-CG splitting map amplifies rounding differences on some
    instances, so the reference itself moves by more than 2% under a 4-ulp
    input perturbation (scs_envelopes.json).  Objective to 1e-6 relative
    when the trajectories agree, to the envelope's spread otherwise."""
    data, meta = load(name)
    prob = _problem(data, meta)
    st = _settings(meta)
    sol = scs.solve(prob, st)
    assert sol.status == meta["status"], (sol.status, sol.iterations, meta["iterations"])
    it_ref = meta["iterations"]
    env = _envelope(name)
    its = [it_ref] + (env["iterations"] if env else [])
    in_env = min(its) - st.check_interval <= sol.iterations <= max(its) + st.check_interval
    assert abs(sol.iterations - it_ref) <= 0.02 * it_ref or in_env, (sol.iterations, its)
    if sol.status == "solved":
        assert max(sol.primal_residual, sol.dual_residual, sol.gap) <= st.eps
        ref = meta["pobj"]
        if sol.iterations == it_ref:
            tol = 1e-6 * max(1.0, abs(ref))
        else:
            pobjs = [p for p, s_ in zip(env["pobj"], env["status"]) if s_ == "solved"]
            spread = max([abs(p - ref) for p in pobjs] + [0.0])
            tol = 2.0 * spread + 10 * st.eps * max(1.0, abs(ref))
        assert abs(sol.pobj - ref) <= tol, (sol.pobj, ref, tol)
    if sol.status == "infeasible":
        y = sol.y
        assert np.all(y >= -1e-8)
        np.testing.assert_allclose(prob.b @ y, -1.0, atol=1e-9)
    if sol.status == "unbounded":
        np.testing.assert_allclose(prob.c @ sol.x, -1.0, atol=1e-9)


@pytest.mark.parametrize("name", ["scs_deconv1d_n1000_k101", "scs_deconv_100_0"])
def test_scs_matches_oracle_exactly_on_stable_cases(name):
    """On instances whose reference trajectory is rounding-stable (its
    envelope has zero spread) the device solve takes EXACTLY the
    reference's iteration count and lands on its objective to 1e-6."""
    from oracle import scs_ref
    import _exprs as E
    data, meta = load(name)
    env = _envelope(name)
    assert env and min(env["iterations"]) == max(env["iterations"]) == meta["iterations"]
    prob = _problem(data, meta)
    st = _settings(meta)
    sol = scs.solve(prob, st)
    oprob = E.Problem(build_tree(meta["tree"], data, E), np.array(data["b"]),
                      np.array(data["c"]), E.ConeProduct(build_cones(meta["cones"], E)))
    osol, _ = scs_ref.scs_solve(oprob, scs_ref.ScsOracleSettings(**meta["settings"]))
    assert sol.iterations == osol.iterations == meta["iterations"]
    assert abs(sol.pobj - osol.pobj) <= 1e-6 * abs(osol.pobj)
    assert abs(sol.avg_cg_iterations - osol.avg_cg_iterations) <= 0.02 * osol.avg_cg_iterations


def test_trace_file_round_trip(tmp_path):
    prob = scs.ConeProblem(linop.dense([[-1.0]]), np.array([-1.0]), np.array([1.0]),
                           cones.ConeProduct([cones.NonNegCone(1)]))
    settings = scs.ScsSettings(eps=1e-6, max_iters=2000)
    path = tmp_path / "trace.jsonl"
    graph = scs.build_scs_graph(prob, settings)
    sol = scs.solve_built(prob, settings, graph, trace_path=path)
    records = [json.loads(line) for line in path.read_text().splitlines()]
    assert len(records) == sol.iterations
    sol2 = scs.solve_built(prob, settings, graph)
    assert sol2.iterations == sol.iterations
    np.testing.assert_array_equal(sol2.x, sol.x)


def test_cone_step_orthogonality():
    rng = np.random.default_rng(11)
    n, m = 4, 6
    Ad = rng.standard_normal((m, n))
    x0 = rng.standard_normal(n)
    s0 = np.abs(rng.standard_normal(m)) + 0.1
    y0 = np.abs(rng.standard_normal(m)) + 0.1
    prob = scs.ConeProblem(linop.dense(Ad), Ad @ x0 + s0, -Ad.T @ y0,
                           cones.ConeProduct([cones.NonNegCone(m)]))
    graph = scs.build_scs_graph(prob, scs.ScsSettings(eps=1e-9, max_iters=100))
    for _, state in scs.iterate_states(graph, 100):
        u, v = state[0], state[1]
        assert abs(u @ v) / (1.0 + np.linalg.norm(u) * np.linalg.norm(v)) <= 1e-9


@pytest.mark.parametrize("h,w,kh,kw", [(50, 700, 15, 15), (33, 611, 5, 7), (20, 300, 1, 15),
                                        (17, 1200, 15, 1), (9, 289, 3, 3)])
def test_conv2d_tiled_against_oracle(h, w, kh, kw):
    """The tiled 2-d path (periodic row blocks, TMA row windows for interior
    tiles, hand staging at the edges) vs scipy full convolution / valid
    correlation, forward and adjoint, 1e-12 relative."""
    from oracle import linop_ref
    import _exprs as E
    rng = np.random.default_rng(h * 1000 + w)
    K = rng.standard_normal((kh, kw))
    op = linop.conv2d(K, (h, w))
    ref = E.Conv2D(K, (h, w))
    x = rng.standard_normal(h * w)
    y = rng.standard_normal(op.rows)
    f = op.forward(x)
    np.testing.assert_allclose(f, linop_ref.forward(ref, x), rtol=1e-12,
                               atol=1e-12 * np.abs(f).max())
    a = op.adjoint_apply(y)
    np.testing.assert_allclose(a, linop_ref.adjoint(ref, y), rtol=1e-12,
                               atol=1e-12 * np.abs(a).max())


@pytest.mark.parametrize("h,w,kh,kw,kind", [(50, 700, 15, 15, "gauss"), (33, 611, 5, 7, "outer"),
                                             (20, 300, 1, 15, "outer"), (17, 1200, 15, 1, "outer"),
                                             (9, 289, 3, 3, "gauss"), (40, 2000, 31, 63, "outer")])
def test_conv2d_separable_against_oracle(h, w, kh, kw, kind):
    """Rank-one 2-d kernels take the column-pass + row-pass tile path
    (CGB_LEAF_FLAG_SEPARABLE): forward and adjoint vs the oracle's scipy
    convolution at 1e-12, and vs the direct kh x kw path (CGB_NO_SEPARABLE)
    at 1e-13."""
    import os
    from oracle import linop_ref
    from paper_1609_03488_b200 import _plan, canon
    import _exprs as E
    rng = np.random.default_rng(h * 7 + w)
    K = (canon.gaussian_kernel2d(kh, kw) if kind == "gauss" else
         np.outer(rng.standard_normal(kh), rng.standard_normal(kw)))
    assert _plan.separable(K)
    op = linop.conv2d(K, (h, w))
    ref = E.Conv2D(K, (h, w))
    x = rng.standard_normal(h * w)
    y = rng.standard_normal(op.rows)
    f, a = op.forward(x), op.adjoint_apply(y)
    np.testing.assert_allclose(f, linop_ref.forward(ref, x), rtol=1e-12,
                               atol=1e-12 * np.abs(f).max())
    np.testing.assert_allclose(a, linop_ref.adjoint(ref, y), rtol=1e-12,
                               atol=1e-12 * np.abs(a).max())
    os.environ["CGB_NO_SEPARABLE"] = "1"
    try:
        op2 = linop.conv2d(K, (h, w))
        f2, a2 = op2.forward(x), op2.adjoint_apply(y)
    finally:
        del os.environ["CGB_NO_SEPARABLE"]
    np.testing.assert_allclose(f, f2, rtol=1e-13, atol=1e-13 * np.abs(f).max())
    np.testing.assert_allclose(a, a2, rtol=1e-13, atol=1e-13 * np.abs(a).max())


def test_conv2d_rank_two_kernel_is_not_separable():
    from paper_1609_03488_b200 import _plan
    rng = np.random.default_rng(3)
    K = np.outer(rng.standard_normal(5), rng.standard_normal(5))
    K += 1e-6 * np.outer(rng.standard_normal(5), rng.standard_normal(5))
    assert not _plan.separable(K)
    assert _plan.separable(K[:1]) and _plan.separable(K[:, :1])


def test_exp_cone_projection_matches_oracle():
    """Device exp-cone projection (k_cones) vs the oracle restatement, primal
    and dual, on a product of many exp cones mixed with other factors."""
    from oracle import expcone_ref as X
    rng = np.random.default_rng(21)
    ncone = 3000
    K = cones.ConeProduct([cones.NonNegCone(5)] + [cones.ExpCone() for _ in range(ncone)] +
                          [cones.SecondOrderCone(4)])
    v = rng.standard_normal(K.total_dim) * np.exp(rng.uniform(-2, 2, K.total_dim))
    p = cones.project_product(K, v)
    pd = cones.project_product_dual(K, v)
    for c in range(ncone):
        blk = v[5 + 3 * c:8 + 3 * c]
        sc = 1e-10 * (1.0 + np.linalg.norm(blk))
        np.testing.assert_allclose(p[5 + 3 * c:8 + 3 * c], X.project_exp(blk), atol=sc)
        np.testing.assert_allclose(pd[5 + 3 * c:8 + 3 * c], X.project_exp_dual(blk), atol=sc)
    np.testing.assert_allclose(p[:5], np.maximum(v[:5], 0.0))


def _oracle_problem(prob):
    class _P:
        pass
    p = _P()
    p.A, p.b, p.c, p.K = prob.A.expr, prob.b, prob.c, prob.K
    return p


def test_short_wide_dense_split_matches_numpy():
    """A tall dense A (its adjoint is a short-wide GEMV, lowered as a
    column-split with a deterministic identity-sum level) and a wide A:
    forward / adjoint vs numpy, and the adjoint identity."""
    rng = np.random.default_rng(31)
    for m, n in [(20000, 300), (150, 30000), (9000, 9000 // 20)]:
        Ad = rng.standard_normal((m, n))
        op = linop.dense(Ad)
        x = rng.standard_normal(n)
        y = rng.standard_normal(m)
        np.testing.assert_allclose(op.forward(x), Ad @ x, rtol=1e-11, atol=1e-10)
        np.testing.assert_allclose(op.adjoint_apply(y), Ad.T @ y, rtol=1e-11, atol=1e-10)
        cop = linop.scale(-2.0, linop.vstack([op, linop.identity(n)]))
        yy = rng.standard_normal(m + n)
        np.testing.assert_allclose(cop.adjoint_apply(yy),
                                   -2.0 * (Ad.T @ yy[:m] + yy[m:]), rtol=1e-11, atol=1e-9)


def test_kron_lowering_matches_numpy():
    """Kron leaves (np.kron convention) lowered to block-diagonal leaves and
    two sparse permutations: forward / adjoint vs np.kron, including a
    structured factor."""
    rng = np.random.default_rng(41)
    A = rng.standard_normal((4, 3))
    B = rng.standard_normal((5, 6))
    op = linop.kron(linop.dense(A), linop.dense(B))
    M = np.kron(A, B)
    x = rng.standard_normal(M.shape[1])
    y = rng.standard_normal(M.shape[0])
    np.testing.assert_allclose(op.forward(x), M @ x, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(op.adjoint_apply(y), M.T @ y, rtol=1e-12, atol=1e-12)
    C = linop.conv1d([1.0, -2.0, 0.5], 7)        # 9 x 7
    op2 = linop.kron(linop.identity(3), C)
    M2 = np.kron(np.eye(3), linop.materialize_dense(C))
    x2 = rng.standard_normal(21)
    np.testing.assert_allclose(op2.forward(x2), M2 @ x2, rtol=1e-12, atol=1e-12)
    op3 = linop.scale(2.0, linop.kron(C, linop.dense(A)))
    M3 = 2.0 * np.kron(linop.materialize_dense(C), A)
    y3 = rng.standard_normal(M3.shape[0])
    np.testing.assert_allclose(op3.adjoint_apply(y3), M3.T @ y3, rtol=1e-12, atol=1e-11)


def test_zero_range_skipping_is_bitwise_neutral():
    """Skipping b / c loads over their zero ranges (measured on device once
    per launch) must not change a single bit of the trajectory: the same
    plan run with CGB_SCS_NO_ZERO_SKIP (stream everything) ends in the
    identical state; a wrong struct_size is rejected."""
    from paper_1609_03488_b200 import _lib, canon
    n, k = 20_000, 101
    c, b, _ = canon.gen_deconv1d(n, k, seed=5, spikes=20)
    prob = canon.build_deconv(canon.DeconvProblem(c, b, n=n))
    plan = scs.build_scs_graph(prob, scs.ScsSettings(eps=1e-3, max_iters=5000))
    cp = plan.cprob
    assert (plan.b_nz[0], plan.c_nz) == (n + 1, (n, n + 1))
    plan.reset()
    plan.run(300)
    skipped = plan.state().copy()
    u_skip = plan.buf["u"].cpu().numpy()
    cp.flags = _lib.SCS_NO_ZERO_SKIP
    plan.reset()
    plan.run(300)
    full = plan.state().copy()
    assert np.array_equal(skipped, full)
    assert np.array_equal(u_skip, plan.buf["u"].cpu().numpy())
    cp.flags = 0
    cp.struct_size = 8
    with pytest.raises(_lib.CgbError):
        plan.run(1)
    cp.struct_size = ctypes.sizeof(_lib.ScsProblemC)


def test_calls_on_two_streams_are_ordered():
    """one cgb_ctx (grid barrier, reduction banks, plan
    temporaries) serves every caller; launches on a second stream are
    ordered after the ctx's previous stream, so two solves issued back to
    back on different streams give the sequential results bit for bit."""
    import torch
    from paper_1609_03488_b200 import canon
    n, k = 20_000, 101
    c, b, _ = canon.gen_deconv1d(n, k, seed=3, spikes=20)
    prob = canon.build_deconv(canon.DeconvProblem(c, b, n=n))
    st = scs.ScsSettings(eps=1e-3, max_iters=400)
    p1 = scs.build_scs_graph(prob, st)
    p2 = scs.build_scs_graph(prob, st)
    p1.reset()
    p1.run(400)
    ref = p1.state().copy()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    p1.reset()
    p2.reset()
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        p1.run(400)
    with torch.cuda.stream(s2):
        p2.run(400)
    torch.cuda.synchronize()
    assert np.array_equal(p1.state(), ref)
    assert np.array_equal(p2.state(), ref)


def test_tracked_products_do_not_drift():
    """the loop never recomputes A cgx (tax) or A^T A cgx (gx);
    they follow cgx through every CG update.  After a long run they must
    still equal fresh operator applications to ~1e-12 relative."""
    from paper_1609_03488_b200 import canon
    n, k = 20_000, 101
    c, b, _ = canon.gen_deconv1d(n, k, seed=5, spikes=20)
    prob = canon.build_deconv(canon.DeconvProblem(c, b, n=n))
    plan = scs.build_scs_graph(prob, scs.ScsSettings(eps=1e-6, max_iters=6000))
    plan.reset()
    plan.run(6000)
    st = plan.state()
    assert st[3] > 500, "the run should take many CG steps"
    x = plan.buf["cgx"]
    ax = plan.dev.apply(x)
    gx = plan.dev.apply(ax, adjoint=True)
    tax, tgx = plan.buf["tax"], plan.buf["gx"]
    rel_a = float((ax - tax).norm() / ax.norm())
    rel_g = float((gx - tgx).norm() / gx.norm())
    assert rel_a < 1e-12 and rel_g < 1e-12, (rel_a, rel_g)


def test_long_kernel_conv_matches_reference():
    """Kernels longer than the tiled path's 240 taps (the reference's own
    deconvolution family uses kernel length n, evaluated by FFT above 512
    taps, linop.py:35-50) run as tap blocks of tiled conv leaves: forward
    and adjoint vs the REAL reference's applies (tests/golden/
    make_golden_longconv.py) up to n = k = 10001."""
    data, meta = load("long_conv_cases")
    for case in meta["cases"]:
        op = linop.Operator(build_tree(case["tree"], data, linop))
        ax = op.forward(np.array(data[case["x"]]))
        ref = np.array(data[case["ax"]])
        np.testing.assert_allclose(ax, ref, rtol=1e-9, atol=1e-12 * np.abs(ref).max(),
                                   err_msg=f"forward n={case['n']} k={case['k']}")
        aty = op.adjoint_apply(np.array(data[case["y"]]))
        ref = np.array(data[case["aty"]])
        np.testing.assert_allclose(aty, ref, rtol=1e-9, atol=1e-12 * np.abs(ref).max(),
                                   err_msg=f"adjoint n={case['n']} k={case['k']}")


@pytest.mark.parametrize("name", ["scs_soc_ball", "scs_lp_equality", "scs_deconv_100_0",
                                  "scs_feasible_lp_11", "scs_infeasible"])
def test_cluster_mode_matches_reference(name):
    """CGB_CLUSTER=16: the persistent kernels launched as one 16-CTA
    thread-block cluster (hardware cluster barrier instead of the grid
    barrier) on zero-spread golden cases: status and the exact reference
    iteration count."""
    import os
    data, meta = load(name)
    prob = _problem(data, meta)
    os.environ["CGB_CLUSTER"] = "16"
    try:
        sol = scs.solve(prob, _settings(meta))
    finally:
        del os.environ["CGB_CLUSTER"]
    assert sol.status == meta["status"]
    assert sol.iterations == meta["iterations"], (sol.iterations, meta["iterations"])
    if sol.status == "solved":
        assert abs(sol.pobj - meta["pobj"]) <= 1e-6 * max(1.0, abs(meta["pobj"]))
