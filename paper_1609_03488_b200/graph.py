"""conegraph's general computation-graph engine (graph.py) is OUT OF SCOPE
for the B200 path (the device kernels ARE the compiled solver
graph; there is no per-node evaluation).  The names the reference exports
from it (conegraph/__init__.py:3-4) exist here so that code importing them
keeps importing; using any of them raises GraphEngineUnavailable with a
pointer to the compiled entry points (scs.build_scs_graph / solve_built,
cg.build_cg_graph / solve_built)."""

from __future__ import annotations

NodeId = int


class GraphError(ValueError):
    """Base error of the graph engine (graph.py:37)."""


class GraphEngineUnavailable(GraphError, NotImplementedError):
    """The per-node graph engine is not part of the device path."""


_MSG = ("the conegraph node-by-node graph engine is not part of the B200 path: solvers are "
        "compiled to device plans by scs.build_scs_graph / cg.build_cg_graph and run by "
        "scs.solve_built / cg.solve_built (see DESIGN.md, out of scope)")


def _unavailable(*_args, **_kwargs):
    raise GraphEngineUnavailable(_MSG)


class _Unavailable:
    def __init__(self, *args, **kwargs):
        _unavailable()


class Graph(_Unavailable):
    """graph.py:120."""


class Node(_Unavailable):
    """graph.py:58."""


class LoopSpec(_Unavailable):
    """graph.py:69."""


evaluate = evaluate_args = while_loop = topological_order = debug_dump = _unavailable
