"""Gray–Scott reaction–diffusion on an irregular domain with homogeneous Neumann BC (test infrastructure
only).

  u_t = ε₁Δu + (1/ε₀)[γ(1 − u) − uv²],   v_t = ε₂Δv + (1/ε₀)[uv² − (γ + κ_r)v],   ∂_n u = ∂_n v = 0
with γ = 0.024, κ_r = 0.06, ε₀ = 0.01, ε₁ = 0.008, ε₂ = 0.004, the disk r = 1.8 in B = (−2, 2)²,
v(x, y, 0) = ¼ sin²(4πx) sin²(4πy) on |x|, |y| ≤ 0.25 (0 elsewhere), u = 1 − 2v.

Readings (the paper names only "second-order Strang splitting"), R40:
  * step = R(Δt/2) ∘ D(Δt) ∘ R(Δt/2); R = explicit midpoint rule, pointwise at every grid node;
  * D = Crank–Nicolson per species, realised as ONE Neumann solve: with a = εΔt/2,
    (I − aΔ)^{-1}(I + aΔ)w = 2y − w where (Δ − κ_cn) y = −κ_cn w, ∂_n y = 0, κ_cn = 2/(εΔt)
    (the Neumann BVP of reading R38, κ_cn > 0 as it requires);
  * the source's boundary data ([F] = f at the intersection and control points) is the bilinear
    interpolant of the grid field w at those points (R41); w lives on the full node grid (the
    solve returns the interface solution outside Ω, continuous across Γ);
  * GMRES warm-started from the previous step's density of the same species.
"""
from __future__ import annotations

import numpy as np

import workloads as W
from .bie import Oracle2D

PARAMS = W.GS_PARAMS
initial = W.gray_scott_initial


def rates(u, v, p=PARAMS):
    uv2 = u * v * v
    return (p["gamma"] * (1.0 - u) - uv2) / p["eps0"], (uv2 - (p["gamma"] + p["kr"]) * v) / p["eps0"]


def reaction(u, v, dt, p=PARAMS):
    """Explicit midpoint rule for the pointwise reaction ODEs."""
    du, dv = rates(u, v, p)
    um, vm = u + 0.5 * dt * du, v + 0.5 * dt * dv
    du, dv = rates(um, vm, p)
    return u + dt * du, v + dt * dv


def bilinear(field, lo, h, px, py):
    """Bilinear interpolant of a full (N+1)² node field at the points (R41)."""
    sx, sy = (px - lo) / h, (py - lo) / h
    i, j = np.floor(sx).astype(int), np.floor(sy).astype(int)
    tx, ty = sx - i, sy - j
    return ((1 - tx) * (1 - ty) * field[i, j] + tx * (1 - ty) * field[i + 1, j]
            + (1 - tx) * ty * field[i, j + 1] + tx * ty * field[i + 1, j + 1])


problem = W.gray_scott_problem


class GrayScott:
    def __init__(self, n, dt, tol=1e-8, p=PARAMS):
        self.p, self.dt, self.tol = p, dt, tol
        self.ou = Oracle2D(problem(n, p["eps1"], dt))
        self.ov = Oracle2D(problem(n, p["eps2"], dt))
        o = self.ou
        self.u, self.v = initial(o.X, o.Y)
        self.psi = [None, None]
        self.iters = []

    def diffuse(self, o, w, k):
        n, st = o.st.n, o.st
        kap = o.kappa
        px, py = o.isect_points()
        zx, zy = o.ctrl_points()
        fg = -kap * w[1:n, 1:n]
        fq = -kap * bilinear(w, st.lo, st.h, px, py)
        fz = -kap * bilinear(w, st.lo, st.h, zx, zy)
        y, psi, stats = o.solve(np.zeros(o.M), fdata=(fg, fq, fz), tol=self.tol, phi0=self.psi[k])
        assert stats.converged
        self.psi[k] = psi
        self.iters.append(stats.iters)
        return 2.0 * y - w

    def step(self):
        h = 0.5 * self.dt
        self.u, self.v = reaction(self.u, self.v, h, self.p)
        self.u = self.diffuse(self.ou, self.u, 0)
        self.v = self.diffuse(self.ov, self.v, 1)
        self.u, self.v = reaction(self.u, self.v, h, self.p)
