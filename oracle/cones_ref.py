"""numpy restatement of the reference cone projections (TEST ORACLE ONLY).

  project_cone          cones.py:64-83   (closed-form, branchy)
  project_dual_product  scs.py:250-283   (_emit_soc_projection /
                        _emit_dual_projection: the branch-free form the
                        solver graph actually evaluates each iteration;
                        zero-cone blocks are free in the dual)
Exponential cone (north-star extension) lives in expcone_ref.py.
"""

from __future__ import annotations

import numpy as np


def _name(c) -> str:
    return type(c).__name__


def project_cone(cone, v: np.ndarray) -> np.ndarray:
    """cones.py:64-83."""
    v = np.asarray(v, dtype=np.float64)
    k = _name(cone)
    if k == "ZeroCone":
        return np.zeros(cone.dim)
    if k == "NonNegCone":
        return np.maximum(v, 0.0)
    if k == "SecondOrderCone":
        t, u = v[0], v[1:]
        nu = np.linalg.norm(u)
        if nu <= t:
            return v.copy()
        if nu <= -t:
            return np.zeros(cone.dim)
        coef = 0.5 * (t + nu)
        out = np.empty(cone.dim)
        out[0] = coef
        out[1:] = coef * (u / nu)
        return out
    if k == "ExpCone":
        from .expcone_ref import project_exp
        return project_exp(v)
    raise TypeError(f"oracle: unknown cone {k}")


def _soc_graph_form(z: np.ndarray) -> np.ndarray:
    """scs.py:250-264 -- branch-free SOC projection as the graph computes it."""
    t = z[0:1]
    u = z[1:]
    nu = np.array([np.linalg.norm(u)])
    one = np.array([1.0])
    inside = one - (nu > t).astype(np.float64)
    in_polar = one - (nu > -1.0 * t).astype(np.float64)
    p_else = (one - inside) * (one - in_polar)
    coef = 0.5 * (t + nu)
    pos_nu = (nu > 0.0).astype(np.float64)
    safe = nu + (one - pos_nu)
    direction = u / safe[0]
    cand = np.concatenate([coef, coef[0] * direction])
    return inside[0] * z + p_else[0] * cand


def project_dual_product(factors, y: np.ndarray) -> np.ndarray:
    """scs.py:267-283 -- projection onto K* block by block."""
    parts = []
    off = 0
    for f in factors:
        blk = y[off:off + f.dim]
        k = _name(f)
        if k == "ZeroCone":
            parts.append(blk)
        elif k == "NonNegCone":
            parts.append(np.maximum(blk, 0.0))
        elif k == "SecondOrderCone":
            parts.append(_soc_graph_form(blk))
        elif k == "ExpCone":
            from .expcone_ref import project_exp_dual
            parts.append(project_exp_dual(blk))
        else:
            raise TypeError(f"oracle: unknown cone {k}")
        off += f.dim
    return parts[0] if len(parts) == 1 else np.concatenate(parts)
