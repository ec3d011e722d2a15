"""GPU parity at BASELINE.json's full sizes, through size-independent
properties (the oracle cannot run these solves to convergence in test time):

* the stuffed operators at full size against the oracle's FFT applies on
  random vectors, and the adjoint identity <Ax, y> = <x, A^T y>;
* cone projections of the full-size cone products: idempotence, Moreau
  decomposition v = Pi_K(v) - Pi_K*(-v) with orthogonal parts;
* the bench solve (configs[1], n = 1e6) re-verified on the host with the
  oracle's independent operator applies: primal / dual residual and gap
  <= eps, s in K, y in K*, and the objective against the oracle's own full
  solve of the same instance (profiles/oracle_bench_instance.json, 2.6 h
  of CPU: pobj 9.894003).  The two trajectories differ (rounding chaos, see
  DESIGN.md "Parity"), so the objectives agree to eps-level, not 1e-6.
  Its iteration count is held against the oracle's own envelope of the
  same instance in tests/test_gpu_envelopes.py (deconv1d_n1000000_k101).
"""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class _P:
    def __init__(self, prob):
        self.A, self.b, self.c, self.K = prob.A.expr, prob.b, prob.c, prob.K


@pytest.fixture(scope="module")
def deconv1d():
    import bench
    from paper_1609_03488_b200 import canon
    c, b, _ = bench._instance(bench.N_SIGNAL)
    return c, b, canon.build_deconv(canon.DeconvProblem(c, b, n=bench.N_SIGNAL))


def test_full_size_deconv1d_operator_vs_oracle(deconv1d):
    from oracle import linop_ref
    _, _, prob = deconv1d
    A = prob.A
    rng = np.random.default_rng(0)
    x = rng.standard_normal(A.cols)
    y = rng.standard_normal(A.rows)
    ax, aty = A.forward(x), A.adjoint_apply(y)
    np.testing.assert_allclose(ax, linop_ref.forward(A.expr, x), rtol=1e-9,
                               atol=1e-11 * np.abs(ax).max())
    np.testing.assert_allclose(aty, linop_ref.adjoint(A.expr, y), rtol=1e-9,
                               atol=1e-11 * np.abs(aty).max())
    assert abs(ax @ y - x @ aty) <= 1e-10 * (1 + np.linalg.norm(ax) * np.linalg.norm(y))


def test_full_size_deconv2d_operator_vs_oracle():
    import bench
    from oracle import linop_ref
    wl = bench.Deconv2D()
    prob = wl.problem()
    C = prob.A
    rng = np.random.default_rng(1)
    x = rng.standard_normal(C.cols)
    y = rng.standard_normal(C.rows)
    ax, aty = C.forward(x), C.adjoint_apply(y)
    np.testing.assert_allclose(ax, linop_ref.forward(C.expr, x), rtol=1e-9,
                               atol=1e-10 * np.abs(ax).max())
    np.testing.assert_allclose(aty, linop_ref.adjoint(C.expr, y), rtol=1e-9,
                               atol=1e-10 * np.abs(aty).max())


def test_full_size_cone_product_properties(deconv1d):
    import torch
    _, _, prob = deconv1d
    Kd = prob.K.device()
    rng = np.random.default_rng(2)
    v = torch.from_numpy(rng.standard_normal(prob.A.rows) * 3.0).cuda()
    p = Kd.project_device(v).cpu().numpy()
    pp = Kd.project_device(torch.from_numpy(p).cuda()).cpu().numpy()
    q = Kd.project_device(-v, dual=True).cpu().numpy()   # self-dual here
    vv = v.cpu().numpy()
    np.testing.assert_allclose(pp, p, atol=1e-12 * np.abs(vv).max())
    np.testing.assert_allclose(p - q, vv, atol=1e-12 * np.abs(vv).max())
    assert abs(p @ q) <= 1e-10 * (np.linalg.norm(p) * np.linalg.norm(q) + 1.0)


def test_full_size_bench_solve_certificate(deconv1d):
    from oracle import linop_ref
    from paper_1609_03488_b200 import scs
    c, b, prob = deconv1d
    st = scs.ScsSettings(eps=1e-3, max_iters=100_000)
    sol = scs.solve(prob, st)
    assert sol.status == "solved"
    A = prob.A.expr
    x, y, s = sol.x, sol.y, sol.s
    pr = np.linalg.norm(linop_ref.forward(A, x) + s - prob.b) / (1 + np.linalg.norm(prob.b))
    dr = np.linalg.norm(linop_ref.adjoint(A, y) + prob.c) / (1 + np.linalg.norm(prob.c))
    cx, by = float(prob.c @ x), float(prob.b @ y)
    gap = abs(cx + by) / (1 + abs(cx) + abs(by))
    assert max(pr, dr, gap) <= st.eps * (1 + 1e-6), (pr, dr, gap)
    n = prob.A.cols - 1
    # s, y in K = NonNeg(n) x SOC(m - n) (self-dual): tolerance at eps scale
    for vec in (s, y):
        assert vec[:n].min() >= -1e-6 * (1 + np.abs(vec).max())
        t, tail = vec[n], vec[n + 1:]
        assert np.linalg.norm(tail) <= t + 1e-6 * (1 + abs(t))
    ref = json.load(open(os.path.join(ROOT, "profiles", "oracle_bench_instance.json")))
    assert ref["status"] == "solved"
    assert abs(sol.pobj - ref["pobj"]) <= 10 * st.eps * abs(ref["pobj"])
