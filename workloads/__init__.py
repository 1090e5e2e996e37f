"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the KFBI method (no jumps, corrections, transforms,
interpolation or Krylov steps).  It only describes *problems*: geometry descriptors, the
manufactured exact solutions with their right-hand sides, and seeded densities.  Both the
CPU oracle (``oracle/``) and the CUDA path (``paper_2404_15249_b200``) consume it; neither
imports the other.

Readings:
  R24  u*_2D = e^x cos y + e^y sin x + sin x sin y        (P:235 plus a non-harmonic term)
       u*_3D = e^x cos y + e^z sin x + sin x sin y sin z
       f = Δu* − κ u*                                    (PDE P:447-451)
  R25  star ρ(θ) = r (1 + ε sin(m(θ − α)))
  R26  C1 ellipse semi-axes (1.0, 0.8)                   (first two axes of P:330-333)
  R27  C3 = ellipse(1, 0.8) minus two disks             (not in the paper)
  R28  torus R = 0.7, r = 0.3                            (not in the paper)
  R29  κ = 1 for "modified Helmholtz"
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence

import numpy as np

# geometry kinds / roles (mirrors include/kfbi.h)
ELLIPSE = 1      # 2D ellipse / circle: p = (ra, rb)
STAR = 2         # 2D star: p = (r, eps, m, alpha)
ELLIPSOID = 3    # 3D ellipsoid / sphere: p = (a, b, c)
TORUS = 4        # 3D torus about the z axis: p = (R, r)
OUTER = 0
HOLE = 1


@dataclasses.dataclass(frozen=True)
class Component:
    kind: int
    center: tuple
    p: tuple
    role: int = OUTER
    n_ctrl: int = 0          # 2D only; 0 -> default spacing (reading R11)


@dataclasses.dataclass(frozen=True)
class Problem:
    name: str
    dim: int
    n: int                   # intervals per axis (power of two, reading R2)
    lo: float
    hi: float
    comps: tuple
    kappa: float
    bc: int = 0              # DIRICHLET (0) or NEUMANN (1)

    @property
    def h(self) -> float:
        return (self.hi - self.lo) / self.n

    @property
    def unknowns(self) -> int:
        return (self.n - 1) ** self.dim


def ellipse(ra, rb, center=(0.0, 0.0), role=OUTER, n_ctrl=0):
    return Component(ELLIPSE, tuple(float(c) for c in center), (float(ra), float(rb), 0.0, 0.0), role, n_ctrl)


def circle(r, center=(0.0, 0.0), role=OUTER, n_ctrl=0):
    return ellipse(r, r, center, role, n_ctrl)


def star(r, eps, m, alpha=0.0, center=(0.0, 0.0), role=OUTER, n_ctrl=0):
    return Component(STAR, tuple(float(c) for c in center), (float(r), float(eps), float(m), float(alpha)), role, n_ctrl)


def ellipsoid(a, b, c, center=(0.0, 0.0, 0.0)):
    return Component(ELLIPSOID, tuple(float(x) for x in center), (float(a), float(b), float(c), 0.0), OUTER, 0)


def torus(R, r, center=(0.0, 0.0, 0.0)):
    return Component(TORUS, tuple(float(x) for x in center), (float(R), float(r), 0.0, 0.0), OUTER, 0)


DIRICHLET, NEUMANN = 0, 1


def problem(name, dim, n, comps, kappa, lo=-1.2, hi=1.2, bc=DIRICHLET) -> Problem:
    return Problem(name, dim, int(n), float(lo), float(hi), tuple(comps), float(kappa), int(bc))


def neumann(prob: Problem) -> Problem:
    """The same geometry and κ with the Neumann boundary condition ∂_n u = g_N."""
    return dataclasses.replace(prob, name=prob.name + "-neumann", bc=NEUMANN)


# --- BASELINE.json configs -------------------------------------------
def C1(n=64):
    """2D Poisson, ellipse (1, 0.8), 64^2, 128 control points (M fixed; scales with N)."""
    return problem("C1-ellipse", 2, n, [ellipse(1.0, 0.8, n_ctrl=2 * n)], 0.0)


def C2(n=1024):
    """2D modified Helmholtz (κ=1) on the 4-fold star r=1, ε=0.2."""
    return problem("C2-star", 2, n, [star(1.0, 0.2, 4)], 1.0)


def C3(n=8192):
    """2D Poisson on ellipse(1,0.8) minus two disks (reading R27), hole completion."""
    return problem("C3-multiply-connected", 2, n,
                   [ellipse(1.0, 0.8),
                    circle(0.25, center=(-0.4, 0.05), role=HOLE),
                    circle(0.2, center=(0.45, -0.1), role=HOLE)], 0.0)


def C4(n=128):
    return problem("C4-ellipsoid", 3, n, [ellipsoid(1.0, 0.8, 0.6)], 0.0)


def C5(n=512):
    return problem("C5-torus", 3, n, [torus(0.7, 0.3)], 1.0)


CONFIGS = {"C1": C1, "C2": C2, "C3": C3, "C4": C4, "C5": C5}


# --- manufactured solutions (reading R24) ---------------------------------------------
def u_exact(x, y, z=None):
    if z is None:
        return np.exp(x) * np.cos(y) + np.exp(y) * np.sin(x) + np.sin(x) * np.sin(y)
    return np.exp(x) * np.cos(y) + np.exp(z) * np.sin(x) + np.sin(x) * np.sin(y) * np.sin(z)


def lap_u_exact(x, y, z=None):
    # e^x cos y and e^y sin x are harmonic (and e^z sin x); Δ(sin x sin y) = −2 sin x sin y
    if z is None:
        return -2.0 * np.sin(x) * np.sin(y)
    return -3.0 * np.sin(x) * np.sin(y) * np.sin(z)


def grad_u_exact(x, y, z=None):
    """∇u*, for the Neumann data g_N = n·∇u* (P:787)."""
    if z is None:
        ux = np.exp(x) * np.cos(y) + np.exp(y) * np.cos(x) + np.cos(x) * np.sin(y)
        uy = -np.exp(x) * np.sin(y) + np.exp(y) * np.sin(x) + np.sin(x) * np.cos(y)
        return ux, uy
    ux = np.exp(x) * np.cos(y) + np.exp(z) * np.cos(x) + np.cos(x) * np.sin(y) * np.sin(z)
    uy = -np.exp(x) * np.sin(y) + np.sin(x) * np.cos(y) * np.sin(z)
    uz = np.exp(z) * np.sin(x) + np.sin(x) * np.sin(y) * np.cos(z)
    return ux, uy, uz


def f_exact(kappa, x, y, z=None):
    """f = Δu* − κ u* (P:449)."""
    return lap_u_exact(x, y, z) - kappa * u_exact(x, y, z)


# --- densities ------------------------------------------------------------------------
def random_density(m: int, seed: int) -> np.ndarray:
    """U(−1, 1) density from numpy.random.default_rng(seed)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=m)


def smooth_density(comp_counts: Sequence[int]) -> np.ndarray:
    """cos(2π s/L) + 0.5 sin(6π s/L) per component, sampled at uniform knots m/M."""
    out = []
    for mc in comp_counts:
        u = np.arange(mc) / mc
        out.append(np.cos(2 * np.pi * u) + 0.5 * np.sin(6 * np.pi * u))
    return np.concatenate(out)


# --- Gray–Scott workload: parameters, initial data, problems ---
GS_PARAMS = dict(gamma=0.024, kr=0.06, eps0=0.01, eps1=0.008, eps2=0.004)


def gray_scott_initial(X, Y):
    """v = ¼ sin²(4πx) sin²(4πy) on |x|, |y| ≤ 0.25 (0 elsewhere), u = 1 − 2v."""
    sq = (np.abs(X) <= 0.25) & (np.abs(Y) <= 0.25)
    v = np.where(sq, 0.25 * np.sin(4 * np.pi * X) ** 2 * np.sin(4 * np.pi * Y) ** 2, 0.0)
    return 1.0 - 2.0 * v, v


def gray_scott_problem(n, eps, dt):
    """One species' diffusion substep: Neumann modified Helmholtz with κ = 2/(εΔt) on the disk r = 1.8
    in B = (−2, 2)²."""
    return problem(f"gray-scott-{eps:g}", 2, n, [circle(1.8)], 2.0 / (eps * dt), lo=-2.0, hi=2.0, bc=NEUMANN)
