"""Exponential-cone projection (TEST ORACLE ONLY; north-star extension).

The reference (conegraph) has no exponential cone -- its spec lists it as a
non-goal -- so this restatement is not pinned to reference outputs ("parity
unpinned" for the exp cone): it is validated against a
brute-force search over the cone's boundary rays in
tests/test_oracle_golden.py.

K_exp = cl{(x, y, z) : y > 0, y exp(x / y) <= z}
K_exp* = cl{(u, v, w) : u < 0, -u exp(v / u) <= e w}

Projection of v0 = (r, s, t):
  1. v0 in K_exp                      -> v0
  2. v0 in the polar cone -K_exp*     -> 0
  3. r < 0 and s < 0                  -> (r, 0, max(t, 0))   (the face y = 0)
  4. otherwise the projection is s_p (rho, 1, e^rho) on the curved boundary
     (or on the face y = 0).  Stationarity v0 = p + mu grad f(p),
     f = y e^{x/y} - z, eliminates s_p and mu and leaves one equation in
     rho = x / y, scaled by e^{-2 rho}:
        G(rho) = (r - s rho) e^{-2rho} + (r - r rho - s)
                 + t e^{-rho} (rho^2 - rho + 1) = 0.
     G has up to two roots; the projection's root is the one with
     s_p = <v0, d>/|d|^2 > 0 and mu = s_p e^rho - t >= 0, d = (rho, 1, e^rho).
     Roots are bracketed on a unit grid over [-60, 40] and bisected to
     machine precision; the result is compared with the face point.
Dual projection by Moreau: Pi_{K*}(v) = v + Pi_K(-v).
"""

from __future__ import annotations

import math

import numpy as np

RHO_LO, RHO_HI, RHO_STEP = -60.0, 40.0, 1.0
BISECT = 64


def in_exp(v, tol: float = 0.0) -> bool:
    r, s, t = (float(a) for a in v)
    if s > 0:
        return s * math.exp(r / s) <= t + tol if r / s < 700 else False
    return r <= tol and abs(s) <= tol and t >= -tol


def in_polar(v) -> bool:
    r, s, t = (float(a) for a in v)
    if r > 0:
        return (r * math.exp(s / r) + math.e * t <= 0.0) if s / r < 700 else False
    return r == 0.0 and s <= 0.0 and t <= 0.0


def _g(rho: float, r: float, s: float, t: float) -> float:
    e1 = math.exp(-rho)
    return (r - s * rho) * e1 * e1 + (r - r * rho - s) + t * e1 * (rho * rho - rho + 1.0)


def _ray_point(rho: float, r: float, s: float, t: float):
    e = math.exp(rho)
    dd = rho * rho + 1.0 + e * e
    sp = (r * rho + s + t * e) / dd
    return sp, e


def project_exp(v) -> np.ndarray:
    r, s, t = (float(a) for a in v)
    if in_exp((r, s, t)):
        return np.array([r, s, t])
    if in_polar((r, s, t)):
        return np.zeros(3)
    if r < 0 and s < 0:
        return np.array([r, 0.0, max(t, 0.0)])
    face = (min(r, 0.0), 0.0, max(t, 0.0))
    best = face
    best_d = (r - face[0]) ** 2 + s * s + (t - face[2]) ** 2
    lo = RHO_LO
    glo = _g(lo, r, s, t)
    while lo < RHO_HI:
        hi = lo + RHO_STEP
        ghi = _g(hi, r, s, t)
        if (glo < 0) != (ghi < 0) or ghi == 0.0:
            a, b, ga = lo, hi, glo
            for _ in range(BISECT):
                mid = 0.5 * (a + b)
                gm = _g(mid, r, s, t)
                if (gm < 0) == (ga < 0):
                    a, ga = mid, gm
                else:
                    b = mid
            rho = 0.5 * (a + b)
            sp, e = _ray_point(rho, r, s, t)
            mu = sp * e - t
            if sp > 0 and mu >= -1e-12 * (1.0 + abs(t)):
                p = (sp * rho, sp, sp * e)
                d = (r - p[0]) ** 2 + (s - p[1]) ** 2 + (t - p[2]) ** 2
                if d < best_d:
                    best, best_d = p, d
        lo, glo = hi, ghi
    return np.array(best)


def project_exp_dual(v) -> np.ndarray:
    v = np.asarray(v, dtype=np.float64)
    return v + project_exp(-v)


def brute_project(v, n: int = 400001) -> np.ndarray:
    """Check-only: best boundary ray on a fine rho grid, the face and 0."""
    r, s, t = (float(a) for a in v)
    if in_exp((r, s, t)):
        return np.array([r, s, t])
    rhos = np.linspace(RHO_LO, RHO_HI, n)
    e = np.exp(rhos)
    nd2 = rhos * rhos + 1.0 + e * e
    h = (r * rhos + s + t * e)
    sp = np.maximum(h / nd2, 0.0)
    pts = np.stack([sp * rhos, sp, sp * e], axis=1)
    cands = list(pts[np.argmin(np.sum((pts - np.array([r, s, t])) ** 2, axis=1))][None])
    cands += [np.zeros(3), np.array([min(r, 0.0), 0.0, max(t, 0.0)])]
    d = [np.sum((c - np.array([r, s, t])) ** 2) for c in cands]
    return np.asarray(cands[int(np.argmin(d))])
