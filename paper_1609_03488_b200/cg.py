"""Conjugate gradient on the B200 (mirrors conegraph.cg, cg.py:1-165).

The reference emits CG as a while-loop graph over an operator *recipe*.
Here a recipe is a small descriptor -- ``operator_recipe(A)`` (solve
A x = b) or ``make_normal_operator(A, lam)`` (solve (lam I + A^T A) x = b)
-- and the whole loop (direction update fused into the operator read,
fused axpy + dot passes, device-side convergence test) runs in one
persistent kernel (``cgb_cg_solve``).  Arbitrary Python graph-emitting
callables are not supported on the device path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .linop import Operator

DEFAULT_TOL = 1e-8


@dataclass(frozen=True)
class Recipe:
    """Operator-application recipe understood by the device CG."""

    kind: int          # _lib.RECIPE_DIRECT or _lib.RECIPE_NORMAL
    A: Operator
    lam: float = 0.0

    @property
    def n(self) -> int:
        return self.A.cols


def operator_recipe(A: Operator) -> Recipe:
    """Recipe applying an operator handle directly (cg.py:64-68)."""
    if A.rows != A.cols:
        raise ValueError(f"operator_recipe needs a square operator, got {A.shape}")
    return Recipe(_lib.RECIPE_DIRECT, A, 0.0)


def make_normal_operator(A: Operator, lam: float) -> Recipe:
    """x -> lam*x + A^T(A x) (cg.py:71-84); self-adjoint PSD."""
    if lam < 0:
        raise ValueError(f"lam must be nonnegative, got {lam}")
    return Recipe(_lib.RECIPE_NORMAL, A, float(lam))


@dataclass
class CgSpec:
    """A linear system solve over a self-adjoint PSD recipe (cg.py:32-53)."""

    apply_op: Recipe
    b: np.ndarray
    x_init: np.ndarray
    tol: float = DEFAULT_TOL
    max_iter: int | None = None

    def __post_init__(self) -> None:
        self.b = np.asarray(self.b, dtype=np.float64)
        self.x_init = np.asarray(self.x_init, dtype=np.float64)
        if self.b.shape != self.x_init.shape:
            raise ValueError(
                f"b has shape {self.b.shape} but x_init has shape {self.x_init.shape}")
        if self.max_iter is None:
            self.max_iter = 10 * len(self.b)
        if not isinstance(self.apply_op, Recipe):
            raise TypeError("apply_op must come from operator_recipe() or "
                            "make_normal_operator(); graph-emitting callables have no "
                            "device implementation")
        if self.apply_op.n != len(self.b):
            raise ValueError(f"recipe acts on length {self.apply_op.n}, b has {len(self.b)}")


@dataclass
class CgResult:
    x: np.ndarray
    iterations: int
    final_residual_norm: float
    converged: bool


@dataclass
class CgPlan:
    """What build_cg_graph returns: the spec bound to its compiled operator."""

    spec: CgSpec


def build_cg_graph(spec: CgSpec) -> CgPlan:
    """Compile the operator plans for ``spec`` (cg.py:140-149 counterpart)."""
    spec.apply_op.A.device_op()
    return CgPlan(spec)


def cg_solve_device(recipe: Recipe, b, x, tol: float, max_iter: int):
    """Run CG on CUDA float64 tensors; x is overwritten.  -> CgResult-like."""
    ctx = _lib.device_context()
    dev, flip = recipe.A.device_op()
    if flip:
        # an adjoint handle: compile the plans for its own expression instead
        from ._plan import DeviceOp
        dev = DeviceOp(recipe.A.expr)
    res = _lib.CgResult()
    _lib.check(_lib.load_library().cgb_cg_solve(
        ctx.handle, dev.handle, recipe.kind, recipe.lam, _lib.ptr(b), _lib.ptr(x), float(tol),
        int(max_iter), ctypes.byref(res), _lib.stream_handle()))
    return res


def solve_built(graph: CgPlan, spec: CgSpec) -> CgResult:
    """Evaluate a plan produced by build_cg_graph (cg.py:152-161)."""
    import torch
    b = torch.from_numpy(spec.b.copy()).to("cuda")
    x = torch.from_numpy(spec.x_init.copy()).to("cuda")
    res = cg_solve_device(spec.apply_op, b, x, spec.tol, spec.max_iter)
    frn = float(res.final_residual_norm)
    converged = frn <= spec.tol * float(np.linalg.norm(spec.b))
    return CgResult(x.cpu().numpy(), int(res.iterations), frn, converged)


def cg_solve(spec: CgSpec) -> CgResult:
    return solve_built(build_cg_graph(spec), spec)
