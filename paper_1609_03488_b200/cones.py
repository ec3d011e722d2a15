"""Cone types and Euclidean projections, executed on the B200.

Same API as the reference (conegraph.cones, cones.py:1-137): ZeroCone,
NonNegCone, SecondOrderCone, ConeProduct, project / project_dual /
project_product / project_product_dual, contains / contains_product.
Projections run in the library's cone kernel (``cgb_cones_project``):
elementwise segments stream, small SOC blocks get one warp each, large
SOC blocks (> 4096) reduce their norm across the whole grid.
``contains`` is a host predicate (test plumbing in the reference too).
The exponential cone is a north-star extension (``ExpCone``).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib


class ConeError(ValueError):
    pass


@dataclass(frozen=True)
class ZeroCone:
    dim: int


@dataclass(frozen=True)
class NonNegCone:
    dim: int


@dataclass(frozen=True)
class SecondOrderCone:
    dim: int


@dataclass(frozen=True)
class ExpCone:
    """K_exp = cl{(x, y, z) : y > 0, y exp(x / y) <= z} (dimension 3)."""

    dim: int = 3


Cone = ZeroCone | NonNegCone | SecondOrderCone | ExpCone

_KIND = {ZeroCone: _lib.CONE_ZERO, NonNegCone: _lib.CONE_NONNEG,
         SecondOrderCone: _lib.CONE_SOC, ExpCone: _lib.CONE_EXP}


def _check(cone, v) -> np.ndarray:
    if cone.dim < 1:
        raise ConeError(f"cone dimension must be >= 1, got {cone.dim}")
    if isinstance(cone, ExpCone) and cone.dim != 3:
        raise ConeError("exponential cone has dimension 3")
    v = np.asarray(v, dtype=np.float64)
    if v.shape != (cone.dim,):
        raise ConeError(f"vector of shape {v.shape} for cone of dim {cone.dim}")
    return v


class _DeviceCones:
    """A cgb_cones handle for an ordered list of factors."""

    def __init__(self, factors):
        self.ctx = _lib.device_context()
        lib = _lib.load_library()
        kinds = (ctypes.c_int32 * len(factors))(*[_KIND[type(f)] for f in factors])
        dims = (ctypes.c_int64 * len(factors))(*[int(f.dim) for f in factors])
        h = ctypes.c_void_p()
        _lib.check(lib.cgb_cones_create(self.ctx.handle, kinds, dims, len(factors),
                                        ctypes.byref(h)))
        self.handle = h
        self._lib = lib
        self.total = sum(int(f.dim) for f in factors)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.cgb_cones_destroy(h)
            except Exception:  # noqa: BLE001
                pass

    def project_device(self, v, out=None, dual: bool = False):
        import torch
        if out is None:
            out = torch.empty_like(v)
        _lib.check(self._lib.cgb_cones_project(self.ctx.handle, self.handle, int(dual),
                                               _lib.ptr(v), _lib.ptr(out),
                                               _lib.stream_handle()))
        return out

    def project_host(self, v: np.ndarray, dual: bool) -> np.ndarray:
        import torch
        vd = torch.from_numpy(np.ascontiguousarray(v)).to("cuda")
        return self.project_device(vd, dual=dual).cpu().numpy()


@dataclass(frozen=True)
class ConeProduct:
    """Ordered product of cone factors."""

    factors: tuple

    def __init__(self, factors) -> None:
        object.__setattr__(self, "factors", tuple(factors))
        for f in self.factors:
            if f.dim < 1:
                raise ConeError(f"cone dimension must be >= 1, got {f.dim}")
            if isinstance(f, ExpCone) and f.dim != 3:
                raise ConeError("exponential cone has dimension 3")

    @property
    def total_dim(self) -> int:
        return sum(f.dim for f in self.factors)

    def device(self) -> _DeviceCones:
        dev = self.__dict__.get("_dev")
        if dev is None:
            dev = _DeviceCones(self.factors)
            object.__setattr__(self, "_dev", dev)
        return dev


_single_cache: dict = {}


def _single(cone) -> _DeviceCones:
    key = (type(cone), cone.dim)
    dev = _single_cache.get(key)
    if dev is None:
        dev = _single_cache[key] = _DeviceCones([cone])
    return dev


def project(cone, v):
    """Euclidean projection onto the cone (cones.py:64-83), on the device."""
    v = _check(cone, v)
    return _single(cone).project_host(v, dual=False)


def project_dual(cone, v):
    """Projection onto the dual cone (free for the zero cone; cones.py:86-90)."""
    v = _check(cone, v)
    return _single(cone).project_host(v, dual=True)


def project_product(K: ConeProduct, v):
    v = np.asarray(v, dtype=np.float64)
    if v.shape != (K.total_dim,):
        raise ConeError(f"vector of shape {v.shape} for product of dim {K.total_dim}")
    return K.device().project_host(v, dual=False)


def project_product_dual(K: ConeProduct, v):
    v = np.asarray(v, dtype=np.float64)
    if v.shape != (K.total_dim,):
        raise ConeError(f"vector of shape {v.shape} for product of dim {K.total_dim}")
    return K.device().project_host(v, dual=True)


def contains(cone, v, tol: float = 0.0) -> bool:
    """Cone membership up to an additive tolerance (cones.py:118-127)."""
    v = _check(cone, v)
    if isinstance(cone, ZeroCone):
        return bool(np.max(np.abs(v), initial=0.0) <= tol)
    if isinstance(cone, NonNegCone):
        return bool(np.min(v, initial=0.0) >= -tol)
    if isinstance(cone, SecondOrderCone):
        return bool(np.linalg.norm(v[1:]) <= v[0] + tol)
    if isinstance(cone, ExpCone):
        x, y, z = v
        if y > 0:
            return bool(y * np.exp(x / y) <= z + tol)
        return bool(x <= tol and abs(y) <= tol and z >= -tol)
    raise ConeError(f"unknown cone type {type(cone).__name__}")


def contains_product(K: ConeProduct, v, tol: float = 0.0) -> bool:
    v = np.asarray(v, dtype=np.float64)
    off = 0
    for f in K.factors:
        if not contains(f, v[off:off + f.dim], tol):
            return False
        off += f.dim
    return True
