"""Minimal CPU expression / cone classes (TEST ORACLE ONLY).

Same class names and attribute names as the reference's LinOpExpr
variants (linop.py:81-184) and cones (cones.py:20-61), so the oracle's
duck-typed dispatch walks them; no product code is involved.  Used by the
oracle-side problem builders (oracle/canon_ref.py) and the oracle tests.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class DenseMatrix:
    def __init__(self, values):
        self.values = np.asarray(values, dtype=np.float64)
        self.rows, self.cols = self.values.shape


class SparseMatrix:
    def __init__(self, matrix):
        self.matrix = matrix.tocsc()
        self.rows, self.cols = matrix.shape


class Conv1D:
    def __init__(self, kernel, n):
        self.kernel = np.asarray(kernel, dtype=np.float64)
        self.n = int(n)
        self.rows, self.cols = len(self.kernel) + self.n - 1, self.n


class Conv2D:
    def __init__(self, kernel, image_shape):
        self.kernel = np.asarray(kernel, dtype=np.float64)
        self.image_shape = tuple(image_shape)
        h, w = self.image_shape
        kh, kw = self.kernel.shape
        self.rows, self.cols = (h + kh - 1) * (w + kw - 1), h * w


class Identity:
    def __init__(self, n):
        self.rows = self.cols = int(n)


class ZeroOp:
    def __init__(self, m, n):
        self.rows, self.cols = int(m), int(n)


class Scale:
    def __init__(self, alpha, child):
        self.alpha, self.child = float(alpha), child
        self.rows, self.cols = child.rows, child.cols


class Sum:
    def __init__(self, left, right):
        self.left, self.right = left, right
        self.rows, self.cols = left.rows, left.cols


class Compose:
    def __init__(self, left, right):
        self.left, self.right = left, right
        self.rows, self.cols = left.rows, right.cols


class VStack:
    def __init__(self, children):
        self.children = tuple(children)
        self.rows = sum(c.rows for c in self.children)
        self.cols = self.children[0].cols


class AdjointOf:
    def __init__(self, child):
        self.child = child
        self.rows, self.cols = child.cols, child.rows


class Kron:
    def __init__(self, left, right):
        self.left, self.right = left, right
        self.rows, self.cols = left.rows * right.rows, left.cols * right.cols


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
    dim: int = 3


class ConeProduct:
    def __init__(self, factors):
        self.factors = tuple(factors)
        self.total_dim = sum(f.dim for f in self.factors)


@dataclass
class Problem:
    A: object
    b: np.ndarray
    c: np.ndarray
    K: ConeProduct
