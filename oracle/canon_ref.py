"""Problem stuffing on the oracle side (TEST ORACLE / CPU BASELINE ONLY).

Restates the reference's matrix stuffing (conegraph canon.py) with the
plain expression classes of oracle/exprs_ref.py, so bench.py's reference
arm and cpu_baseline leg build and solve every workload without importing
the product package:

  build_lasso      canon.py:99-114   (lasso -> NonNeg(2n) x SOC(m+2))
  build_deconv     canon.py:117-129  (nonneg deconvolution; short-kernel
                                      form: signal n, kernel k, b of n+k-1)
  build_deconv2d   north-star 2-d analogue of build_deconv
  build_soc_ls     north-star SOC-constrained least squares
  build_logreg     north-star l1 logistic regression with exponential cones
  hstack           linop.py:360-362 (adjoint of the stacked adjoints)

The product's builders (paper_1609_03488_b200/canon.py) must produce the
same expression structure and vectors; tests/test_host.py checks that the
two agree entry for entry on small instances.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse

from .exprs_ref import (AdjointOf, Compose, ConeProduct, Conv1D, Conv2D, DenseMatrix, ExpCone,
                        Identity, NonNegCone, Problem, Scale, SecondOrderCone, SparseMatrix,
                        VStack, ZeroOp)


def hstack(children):
    """linop.py:360-362: hstack = adjoint(vstack(adjoints))."""
    return AdjointOf(VStack([AdjointOf(c) for c in children]))


def build_lasso(A, b: np.ndarray, lam: float) -> Problem:
    """canon.py:99-114."""
    m, n = A.rows, A.cols
    eye_n = Identity(n)
    stuffed = VStack([
        hstack([Scale(-1.0, eye_n), eye_n, ZeroOp(n, 1)]),
        hstack([eye_n, eye_n, ZeroOp(n, 1)]),
        hstack([ZeroOp(1, n), ZeroOp(1, n), Scale(2.0, Identity(1))]),
        hstack([Scale(2.0, A), ZeroOp(m, n), ZeroOp(m, 1)]),
        hstack([ZeroOp(1, n), ZeroOp(1, n), Scale(-2.0, Identity(1))]),
    ])
    b_cone = np.concatenate([np.zeros(2 * n), [1.0], -2.0 * np.asarray(b), [1.0]])
    c_obj = np.concatenate([np.zeros(n), lam * np.ones(n), [1.0]])
    K = ConeProduct([NonNegCone(2 * n), SecondOrderCone(m + 2)])
    return Problem(Scale(-1.0, stuffed), b_cone, c_obj, K)


def _deconv_like(C, n: int, b: np.ndarray) -> Problem:
    """canon.py:117-129 with the convolution operator C (rows mc, cols n)."""
    mc = C.rows
    stuffed = VStack([
        hstack([Identity(n), ZeroOp(n, 1)]),
        hstack([ZeroOp(1, n), Identity(1)]),
        hstack([C, ZeroOp(mc, 1)]),
    ])
    b_cone = np.concatenate([np.zeros(n), [0.0], -np.asarray(b)])
    c_obj = np.concatenate([np.zeros(n), [1.0]])
    K = ConeProduct([NonNegCone(n), SecondOrderCone(mc + 1)])
    return Problem(Scale(-1.0, stuffed), b_cone, c_obj, K)


def build_deconv(kernel: np.ndarray, b: np.ndarray, n: int) -> Problem:
    return _deconv_like(Conv1D(kernel, n), n, b)


def build_deconv2d(kernel: np.ndarray, b: np.ndarray, image_shape) -> Problem:
    h, w = image_shape
    return _deconv_like(Conv2D(kernel, (h, w)), h * w, b)


def build_soc_ls(A, b: np.ndarray, radius: float) -> Problem:
    """minimize ||A x - b|| s.t. ||x|| <= radius: (t, A x - b) in SOC(m+1),
    (radius, x) in SOC(n+1)."""
    m, n = A.rows, A.cols
    stuffed = VStack([
        hstack([ZeroOp(1, n), Identity(1)]),
        hstack([A, ZeroOp(m, 1)]),
        hstack([ZeroOp(1, n), ZeroOp(1, 1)]),
        hstack([Identity(n), ZeroOp(n, 1)]),
    ])
    b_cone = np.concatenate([[0.0], -np.asarray(b), [radius], np.zeros(n)])
    c_obj = np.concatenate([np.zeros(n), [1.0]])
    K = ConeProduct([SecondOrderCone(m + 1), SecondOrderCone(n + 1)])
    return Problem(Scale(-1.0, stuffed), b_cone, c_obj, K)


def build_logreg(A: np.ndarray, y: np.ndarray, lam: float) -> Problem:
    """l1 logistic regression: z = (x, w, t, u, v); (w -/+ x) >= 0,
    1 - u - v >= 0, (-t_i, 1, u_i), (z_i - t_i, 1, v_i) in K_exp with
    z_i = -y_i a_i^T x; exp rows interleaved by a permutation."""
    m, n = A.shape
    eye_n, eye_m = Identity(n), Identity(m)
    z_mn, z_mm, z_nm = ZeroOp(m, n), ZeroOp(m, m), ZeroOp(n, m)
    nonneg = VStack([
        hstack([Scale(-1.0, eye_n), eye_n, z_nm, z_nm, z_nm]),
        hstack([eye_n, eye_n, z_nm, z_nm, z_nm]),
        hstack([z_mn, z_mn, z_mm, Scale(-1.0, eye_m), Scale(-1.0, eye_m)]),
    ])
    ya = DenseMatrix(-np.asarray(y)[:, None] * np.asarray(A))
    blocks = VStack([
        hstack([z_mn, z_mn, Scale(-1.0, eye_m), z_mm, z_mm]),
        ZeroOp(m, 2 * n + 3 * m),
        hstack([z_mn, z_mn, z_mm, eye_m, z_mm]),
        hstack([ya, z_mn, Scale(-1.0, eye_m), z_mm, z_mm]),
        ZeroOp(m, 2 * n + 3 * m),
        hstack([z_mn, z_mn, z_mm, z_mm, eye_m]),
    ])
    k = np.repeat(np.arange(6), m)
    i = np.tile(np.arange(m), 6)
    dest = 3 * (i + m * (k // 3)) + (k % 3)
    perm = scipy.sparse.csc_matrix((np.ones(6 * m), (dest, np.arange(6 * m))),
                                   shape=(6 * m, 6 * m))
    stuffed = VStack([nonneg, Compose(SparseMatrix(perm), blocks)])
    b_exp = np.zeros(6 * m)
    b_exp[1::3] = 1.0
    b_cone = np.concatenate([np.zeros(2 * n), np.ones(m), b_exp])
    c_obj = np.concatenate([np.zeros(n), lam * np.ones(n), np.ones(m), np.zeros(2 * m)])
    K = ConeProduct([NonNegCone(2 * n + m)] + [ExpCone() for _ in range(2 * m)])
    return Problem(Scale(-1.0, stuffed), b_cone, c_obj, K)
