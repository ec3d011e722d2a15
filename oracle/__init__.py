"""CPU oracle for the conegraph SCS/CG hot path -- TEST INFRASTRUCTURE ONLY.

This package is a plain-numpy restatement of the reference solver path
(``/root/reference/pkg/src/conegraph``: linop.py, cones.py, cg.py, scs.py).
It exists to CHECK the CUDA product path, never to stand in for it:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  Nothing in
``paper_1609_03488_b200`` imports this package.

Parity pinning: the restatement is checked against golden vectors produced
by running the *real* reference in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``); see
``tests/test_oracle_golden.py``.  Every function cites the reference
file:line it restates.

Operators are duck-typed expression trees: any object whose class name is
one of the reference's LinOpExpr variants (DenseMatrix, SparseMatrix,
Conv1D, Identity, ZeroOp, Scale, Sum, Compose, VStack, AdjointOf) with the
reference's attribute names, plus the north-star extensions (Conv2D, Kron).
"""

from .linop_ref import adjoint, forward, materialize  # noqa: F401
from .cones_ref import project_cone, project_dual_product  # noqa: F401
from .cg_ref import cg  # noqa: F401
from .scs_ref import ScsOracleSettings, scs_solve  # noqa: F401
