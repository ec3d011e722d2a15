"""BASELINE configs at their FULL sizes: the device solve re-verified on the
host with the oracle's independent operator applies (the oracle cannot run
these solves to convergence in test time; their families' iteration-count
and objective parity is pinned by tests/test_gpu_envelopes.py):

  * primal / dual residual and gap <= eps, recomputed from x, y, s with
    oracle/linop_ref applies (scs.py:217-244 formulas);
  * s in K and y in K* (every factor, exponential cones included);
  * configs[3] also through the row-sharded solver (2 ranks sharing the
    GPU), whose certificate must hold the same way.
configs[0] (dense lasso 1000 x 500) runs at full size in the envelope test;
configs[1] in tests/test_gpu_fullsize.py.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

EPS = 1e-3


def _in_cone(kind, blk, dual, tol):
    """Distance-style membership of one factor block (tolerance tol)."""
    if kind == "ZeroCone":
        return True if dual else float(np.abs(blk).max(initial=0.0)) <= tol
    if kind == "NonNegCone":
        return float(blk.min(initial=0.0)) >= -tol
    if kind == "SecondOrderCone":
        return float(np.linalg.norm(blk[1:])) <= blk[0] + tol
    raise TypeError(kind)


def _exp_members(v, dual, tol):
    """v: (k, 3) rows (x, y, z).  K_exp = cl{y > 0, y e^{x/y} <= z};
    K_exp* = cl{u < 0, -u e^{v/u} <= e w}."""
    x, y, z = v[:, 0], v[:, 1], v[:, 2]
    scale = 1.0 + np.abs(v).max(axis=1)
    if not dual:
        pos = y > tol * scale
        with np.errstate(over="ignore", invalid="ignore"):
            lhs = np.where(pos, y * np.exp(np.minimum(x / np.where(pos, y, 1.0), 700.0)), 0.0)
        ok_pos = lhs <= z + tol * scale
        ok_face = (x <= tol * scale) & (z >= -tol * scale)
        return bool(np.all(np.where(pos, ok_pos, ok_face)))
    neg = x < -tol * scale
    with np.errstate(over="ignore", invalid="ignore"):
        lhs = np.where(neg, -x * np.exp(np.minimum(y / np.where(neg, x, -1.0), 700.0)), 0.0)
    ok_neg = lhs <= np.e * z + tol * scale
    ok_face = (y >= -tol * scale) & (z >= -tol * scale)
    return bool(np.all(np.where(neg, ok_neg, ok_face)))


def _certificate(prob, sol, eps=EPS):
    from oracle import linop_ref
    assert sol.status == "solved", sol.status
    A = prob.A.expr
    x, y, s = sol.x, sol.y, sol.s
    pr = np.linalg.norm(linop_ref.forward(A, x) + s - prob.b) / (1 + np.linalg.norm(prob.b))
    dr = np.linalg.norm(linop_ref.adjoint(A, y) + prob.c) / (1 + np.linalg.norm(prob.c))
    cx, by = float(prob.c @ x), float(prob.b @ y)
    gap = abs(cx + by) / (1 + abs(cx) + abs(by))
    assert max(pr, dr, gap) <= eps * (1 + 1e-6), (pr, dr, gap)
    off = 0
    exp_s, exp_y = [], []
    for f in prob.K.factors:
        kind = type(f).__name__
        sb, yb = s[off:off + f.dim], y[off:off + f.dim]
        tol = 1e-8 * (1.0 + float(np.abs(sb).max(initial=0.0)) + float(np.abs(yb).max(initial=0.0)))
        if kind == "ExpCone":
            exp_s.append(sb)
            exp_y.append(yb)
        else:
            assert _in_cone(kind, sb, False, tol), (kind, off)
            assert _in_cone(kind, yb, True, tol), (kind, off)
        off += f.dim
    if exp_s:
        S, Y = np.array(exp_s), np.array(exp_y)
        assert _exp_members(S, False, 1e-8)
        assert _exp_members(Y, True, 1e-8)
    return pr, dr, gap


def _solve(prob, max_iters=200_000):
    from paper_1609_03488_b200 import scs
    return scs.solve(prob, scs.ScsSettings(eps=EPS, max_iters=max_iters))


def test_configs2_deconv2d_4096_full_solve_certificate():
    """configs[2]: 4096 x 4096 image, 15 x 15 blur, solved to eps on the
    device (~9e4 iterations), verified with scipy FFT convolutions."""
    import bench
    prob = bench.Deconv2D().problem()
    sol = _solve(prob)
    _certificate(prob, sol)
    assert sol.x[:-1].min() >= -1e-6 * (1 + np.abs(sol.x).max())   # nonnegative image


@pytest.fixture(scope="module")
def lasso_sparse_full():
    import bench
    return bench.LassoSparse().problem()


def test_configs3_sparse_lasso_full_solve_certificate(lasso_sparse_full):
    """configs[3]: sparse lasso 8e6 x 1e6 (8e7 nonzeros) on one GPU."""
    sol = _solve(lasso_sparse_full)
    _certificate(lasso_sparse_full, sol)


def test_configs3_sparse_lasso_row_sharded_certificate(lasso_sparse_full):
    """configs[3] through the row-sharded solver: 2 ranks (74 SMs each) on
    this GPU exchanging A^T y, the CG residual and every dot product through
    peer memory -- the same kernel a 2-GPU run executes."""
    from paper_1609_03488_b200 import scs, shard
    st = scs.ScsSettings(eps=EPS, max_iters=200_000)
    grp = shard.ShardGroup(lasso_sparse_full, st, world=2)
    try:
        sol = grp.solve()
    finally:
        grp.close()
    _certificate(lasso_sparse_full, sol)


def test_configs4_soc_constrained_ls_full_solve_certificate():
    """configs[4a]: SOC-constrained least squares, dense A 2e5 x 2e3."""
    import bench
    prob = bench.SocLs().problem()
    sol = _solve(prob)
    _certificate(prob, sol)
    n = bench.SocLs().n
    assert np.linalg.norm(sol.x[:n]) <= bench.SocLs().radius * (1 + 1e-3)


def test_configs4_logreg_exp_cones_full_solve_certificate():
    """configs[4b]: l1 logistic regression, 4e5 exponential cones, dense A
    2e5 x 2e3."""
    import bench
    prob = bench.LogReg().problem()
    sol = _solve(prob)
    _certificate(prob, sol)
