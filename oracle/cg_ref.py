"""numpy restatement of the reference CG loop (TEST ORACLE ONLY).

  cg        cg.py:87-137 (emit_cg_loop body/cond), cg.py:140-161
            (build_cg_graph: delta = tol*||b||; solve_built: converged rule)
  normal    cg.py:71-84  (make_normal_operator: lam*x + A^T(A x))
"""

from __future__ import annotations

from typing import Callable

import numpy as np

from .linop_ref import adjoint, forward


def normal_apply(A, lam: float) -> Callable[[np.ndarray], np.ndarray]:
    """cg.py:71-84 -- x -> lam*x + A^T(A x) (lam == 0 gives the bare Gram)."""
    def apply(x):
        gram = adjoint(A, forward(A, x))
        if lam == 0.0:
            return gram
        return lam * x + gram
    return apply


def direct_apply(A) -> Callable[[np.ndarray], np.ndarray]:
    """cg.py:64-68 (operator_recipe)."""
    return lambda x: forward(A, x)


def cg(apply, b: np.ndarray, x_init: np.ndarray, delta: float, max_iter: int):
    """cg.py:87-137 -- returns (x, k, r_norm_sq).

    Pre-test loop: continue while sqrt(rns) > delta, rns > floor and
    k < max_iter, with floor = eps^2 * max(n,1) * <b,b>.
    """
    n = len(b)
    eps_floor = np.finfo(np.float64).eps ** 2 * max(n, 1)
    r = b - apply(x_init)
    rns = float(np.dot(r, r))
    floor = eps_floor * float(np.dot(b, b))
    x = x_init.copy()
    p = r.copy()
    k = 0
    while np.sqrt(rns) > delta and rns > floor and max_iter > k:
        Ap = apply(p)
        alpha = rns / float(np.dot(p, Ap))
        x = x + alpha * p
        r = r - alpha * Ap
        rns2 = float(np.dot(r, r))
        beta = rns2 / rns
        p = r + beta * p
        rns = rns2
        k += 1
    return x, k, rns


def cg_solve(apply, b, x_init, tol: float = 1e-8, max_iter: int | None = None):
    """cg.py:140-165 -- (x, iterations, final_residual_norm, converged)."""
    b = np.asarray(b, dtype=np.float64)
    x_init = np.asarray(x_init, dtype=np.float64)
    if max_iter is None:
        max_iter = 10 * len(b)
    delta = tol * float(np.linalg.norm(b))
    x, k, rns = cg(apply, b, x_init, delta, max_iter)
    frn = float(np.sqrt(rns))
    return x, k, frn, frn <= tol * float(np.linalg.norm(b))
