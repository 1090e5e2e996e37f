"""Periodic cubic spline of a boundary density (test infrastructure only).

The paper only says "Interpolate Φ" (Alg. 2 step 4) and "compute corresponding jumps"
(P:718).  Reading R10: a periodic cubic spline on the uniform arc-length knots of each
component.  Knot second derivatives M_m solve the cyclic system
    M_{m−1} + 4 M_m + M_{m+1} = 6 (φ_{m+1} − 2 φ_m + φ_{m−1}) / Δ²,
solved here directly as a circulant system (library primitive).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg


def knots(phi: np.ndarray, delta: float) -> np.ndarray:
    m = phi.size
    rhs = 6.0 * (np.roll(phi, -1) - 2.0 * phi + np.roll(phi, 1)) / (delta * delta)
    col = np.zeros(m)
    col[0] = 4.0
    col[1] += 1.0
    col[-1] += 1.0
    return np.real(scipy.linalg.solve_circulant(col, rhs))


def evaluate(phi, Mk, delta, s):
    """g, g', g'' at arc length s ∈ [0, L)."""
    m_count = phi.size
    u = np.asarray(s, dtype=np.float64) / delta
    m = np.floor(u).astype(np.int64)
    t = u - m
    wrap = m >= m_count
    m = np.where(wrap, m - m_count, m)
    m1 = np.where(m + 1 >= m_count, m + 1 - m_count, m + 1)
    g0, g1 = phi[m], phi[m1]
    a, b = Mk[m], Mk[m1]
    w = 1.0 - t
    g = w * g0 + t * g1 + (delta * delta / 6.0) * ((w ** 3 - w) * a + (t ** 3 - t) * b)
    gp = (g1 - g0) / delta + (delta / 6.0) * (-(3.0 * w * w - 1.0) * a + (3.0 * t * t - 1.0) * b)
    gpp = w * a + t * b
    return g, gp, gpp
