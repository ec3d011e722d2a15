"""Oracle-side expression classes (moved to oracle/exprs_ref.py)."""

from oracle.exprs_ref import *  # noqa: F401,F403
from oracle.exprs_ref import (AdjointOf, Compose, ConeProduct, Conv1D, Conv2D,  # noqa: F401
                              DenseMatrix, ExpCone, Identity, Kron, NonNegCone, Problem,
                              Scale, SecondOrderCone, SparseMatrix, Sum, VStack, ZeroCone,
                              ZeroOp)
