"""2D/3D interface geometry for the oracle (test infrastructure only; see oracle/__init__).

Γ = ∂Ω is a union of closed components.  Ω = {ℓ_outer ≤ 0} ∩ {ℓ_hole ≥ 0}; points on
Γ count as Ω (reading R30).  2D curves are parametrised CCW by θ ∈ [0, 2π); the Ω-orientation
is CCW for the outer curve and CW for holes so that n = (τ2, −τ1) is the outward normal of Ω
(reading R8).
"""
from __future__ import annotations

import math

import numpy as np

from workloads import ELLIPSE, STAR, ELLIPSOID, TORUS, OUTER, HOLE

TWO_PI = 2.0 * math.pi
_GL_X, _GL_W = np.polynomial.legendre.leggauss(16)
_PANELS = 64


# ---------------------------------------------------------------- 2D curves ---------
def curve(comp, th):
    """γ(θ), γ'(θ), γ''(θ) for a 2D component (readings R25/R26)."""
    th = np.asarray(th, dtype=np.float64)
    cx, cy = comp.center[0], comp.center[1]
    if comp.kind == ELLIPSE:
        ra, rb = comp.p[0], comp.p[1]
        c, s = np.cos(th), np.sin(th)
        g = np.stack([cx + ra * c, cy + rb * s])
        g1 = np.stack([-ra * s, rb * c])
        g2 = np.stack([-ra * c, -rb * s])
        return g, g1, g2
    if comp.kind == STAR:
        r, eps, m, al = comp.p
        rho = r * (1.0 + eps * np.sin(m * (th - al)))
        rho1 = r * eps * m * np.cos(m * (th - al))
        rho2 = -r * eps * m * m * np.sin(m * (th - al))
        c, s = np.cos(th), np.sin(th)
        g = np.stack([cx + rho * c, cy + rho * s])
        g1 = np.stack([rho1 * c - rho * s, rho1 * s + rho * c])
        g2 = np.stack([rho2 * c - 2 * rho1 * s - rho * c, rho2 * s + 2 * rho1 * c - rho * s])
        return g, g1, g2
    raise ValueError("not a 2D curve kind")


def level_set(comp, *xs):
    """ℓ_c(x): negative inside the component's bounded region (reading R25-R28)."""
    if comp.kind == ELLIPSE:
        x, y = xs
        return ((x - comp.center[0]) / comp.p[0]) ** 2 + ((y - comp.center[1]) / comp.p[1]) ** 2 - 1.0
    if comp.kind == STAR:
        x, y = xs
        r, eps, m, al = comp.p
        dx, dy = x - comp.center[0], y - comp.center[1]
        return np.sqrt(dx * dx + dy * dy) - r * (1.0 + eps * np.sin(m * (np.arctan2(dy, dx) - al)))
    if comp.kind == ELLIPSOID:
        x, y, z = xs
        a, b, c = comp.p[:3]
        return (((x - comp.center[0]) / a) ** 2 + ((y - comp.center[1]) / b) ** 2
                + ((z - comp.center[2]) / c) ** 2 - 1.0)
    if comp.kind == TORUS:
        x, y, z = xs
        R, r = comp.p[:2]
        dx, dy, dz = x - comp.center[0], y - comp.center[1], z - comp.center[2]
        q = np.sqrt(dx * dx + dy * dy) - R
        return q * q + dz * dz - r * r
    raise ValueError(comp.kind)


def omega_side(comp, *xs):
    """True where x lies on the Ω side of this component (ℓ ≤ 0 outer, ℓ ≥ 0 hole), R30."""
    l = level_set(comp, *xs)
    return (l <= 0.0) if comp.role == OUTER else (l >= 0.0)


def in_omega(comps, *xs):
    ok = None
    for c in comps:
        s = omega_side(c, *xs)
        ok = s if ok is None else (ok & s)
    return ok


def arc_length_ccw(comp, th):
    """s_ccw(θ) = ∫_0^θ |γ'(t)| dt by composite 16-point Gauss–Legendre on 64 panels."""
    th = np.atleast_1d(np.asarray(th, dtype=np.float64))
    width = TWO_PI / _PANELS
    # full-panel prefix sums
    a = np.arange(_PANELS) * width
    tq = a[:, None] + 0.5 * width * (_GL_X[None, :] + 1.0)
    sp = np.linalg.norm(curve(comp, tq)[1], axis=0)
    panel = 0.5 * width * (sp * _GL_W[None, :]).sum(axis=1)
    prefix = np.concatenate([[0.0], np.cumsum(panel)])
    k = np.minimum((th // width).astype(np.int64), _PANELS - 1)
    a0 = k * width
    part = th - a0
    tq = a0[:, None] + 0.5 * part[:, None] * (_GL_X[None, :] + 1.0)
    sp = np.linalg.norm(curve(comp, tq)[1], axis=0)
    return prefix[k] + 0.5 * part * (sp * _GL_W[None, :]).sum(axis=1)


def perimeter(comp):
    return float(arc_length_ccw(comp, np.array([TWO_PI]))[0])


def theta_of_s_ccw(comp, s):
    """Invert s_ccw(θ) = s by Newton from θ = 2πs/L (|Δs| ≤ 1e-14 L)."""
    s = np.atleast_1d(np.asarray(s, dtype=np.float64))
    L = perimeter(comp)
    th = TWO_PI * s / L
    for _ in range(60):
        r = arc_length_ccw(comp, th) - s
        if np.all(np.abs(r) <= 1e-14 * L):
            break
        th = th - r / np.linalg.norm(curve(comp, th)[1], axis=0)
    return th


def orient(comp):
    return 1.0 if comp.role == OUTER else -1.0


def frame(comp, th):
    """Unit tangent τ in the Ω orientation, τ' = dτ/ds, normal n = (τ2, −τ1)."""
    g, g1, g2 = curve(comp, th)
    sp2 = (g1 * g1).sum(axis=0)
    sp = np.sqrt(sp2)
    tau = orient(comp) * g1 / sp
    dot = (g1 * g2).sum(axis=0)
    taup = (g2 * sp2 - g1 * dot) / (sp2 * sp2)
    n = np.stack([tau[1], -tau[0]])
    return g, tau, taup, n


def s_omega(comp, th, L):
    """Arc length measured in the Ω orientation (CW for holes)."""
    s = arc_length_ccw(comp, th)
    if comp.role == HOLE:
        s = np.mod(L - s, L)
    return s


def default_ctrl_count(L, h):
    """Reading R11: uniform arc-length spacing Δs ≈ 1.18 h."""
    return int(round(L / (1.18 * h)))
