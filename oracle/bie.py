"""KFBI operators and the Dirichlet BVP solve in 2D (test infrastructure only).

§2.1-2.2 of the paper: ½φ + Wφ + Yf = g_D on Γ, u = Wφ + Yf in Ω, and the
potentials are evaluated as interface problems Δv − κv = F, [v] = Φ, [∂_n v] = Ψ (P:515-534,
P:815-823 for Ψ).  One interface solve = Algorithm 1 steps 4-6:
jumps → correction (Alg. 2) → fast solve (Alg. 4) → interpolation (Alg. 3).

Reading R17: K_D φ = ½φ + Wφ is the interior one-sided value V⁺ of the interface solution
with Φ = φ (no explicit ½φ term).  Neumann (reading R38): K_N ψ = ½ψ − ∂_n(Sψ) is the
interior one-sided normal derivative ∂_n V⁺ of the interface solution with [v] = 0, [∂_n v] = ψ
(the interface problem of P:812-821, v = −Sψ), read off the local quadratic fit of Alg. 3 (its
gradient rows); ĝ_N = g_N − ∂_n(Yf)⁺ and u = Yf − Sψ = one interface solve with
Ψ = ψ and F = f.  κ > 0 only (κ = 0 has the constant null space).  Reading R27 (multiply connected, κ = 0): the completed
operator K̃φ = K_Dφ + Σ_h a_h(φ) w_h|Γ with a_h = ∫_{Γ_h} φ ds (periodic trapezoid) and
w_h the fast solve of (Δ_h − κ) w = b_h, b_h a smooth bump inside hole h.
"""
from __future__ import annotations

import numpy as np

from workloads import HOLE
from . import correction, fastsolve, geometry as geo, grid, interp, jumps, spline
from .gmres import gmres
from .krylov import bicgstab, richardson


def bump(comp, X, Y):
    """b_h(p) = exp(1 − 1/(1 − ρ²)), ρ = |p − c_h| / (r_h / 2) < 1."""
    rad = 0.5 * min(comp.p[0], comp.p[1])
    rho2 = ((X - comp.center[0]) ** 2 + (Y - comp.center[1]) ** 2) / (rad * rad)
    out = np.zeros_like(X)
    m = rho2 < 1.0
    out[m] = np.exp(1.0 - 1.0 / (1.0 - rho2[m]))
    return out


class Oracle2D:
    def __init__(self, prob):
        self.prob = prob
        self.kappa = prob.kappa
        self.st = grid.build(prob)
        st = self.st
        self.nodes = grid.stencil(st)
        self.M = st.M
        # frames at intersections and control points
        self.q_tau = np.empty((2, st.q_xi.size))
        self.q_taup = np.empty((2, st.q_xi.size))
        self.z_tau = np.empty((2, self.M))
        self.z_taup = np.empty((2, self.M))
        for k, c in enumerate(prob.comps):
            sel = st.q_comp == k
            _, t, tp, _ = geo.frame(c, st.q_theta[sel])
            self.q_tau[:, sel], self.q_taup[:, sel] = t, tp
            sel = st.z_comp == k
            _, t, tp, _ = geo.frame(c, st.z_theta[sel])
            self.z_tau[:, sel], self.z_taup[:, sel] = t, tp
        n = st.n
        X, Y = np.meshgrid(st.x, st.x, indexing="ij")
        self.X, self.Y = X, Y
        self.neumann = getattr(prob, "bc", 0) == 1
        if self.neumann and self.kappa <= 0.0:
            raise ValueError("Neumann BVP needs κ > 0 (S:555)")
        self.z_nrm = np.stack([self.z_tau[1], -self.z_tau[0]])       # outward normal n = (τ2, −τ1)
        self.holes = ([k for k, c in enumerate(prob.comps) if c.role == HOLE]
                      if self.kappa == 0.0 and not self.neumann else [])
        self.w_gamma = []
        for k in self.holes:
            b = bump(prob.comps[k], X, Y)[1:n, 1:n]
            w = np.zeros((n + 1, n + 1))
            w[1:n, 1:n] = fastsolve.solve2d(b, st.h, self.kappa)
            self.w_gamma.append(interp.interpolate2d(st, w, np.zeros((self.M, 6)), self.nodes))

    # ------------------------------------------------------------------ points
    def isect_points(self):
        st = self.st
        px = np.where(st.q_axis == 0, st.q_xi, st.x[st.q_i])
        py = np.where(st.q_axis == 1, st.q_xi, st.x[st.q_j])
        return px, py

    def ctrl_points(self):
        return self.st.z[0], self.st.z[1]

    # ------------------------------------------------------------------ jumps
    def density_derivs(self, phi):
        """Spline of φ per component → (Φ, Φ_s, Φ_ss) at intersections and control points."""
        st = self.st
        q = np.zeros((3, st.q_xi.size))
        z = np.zeros((3, self.M))
        for k in range(len(self.prob.comps)):
            o, m = st.comp_off[k], st.comp_M[k]
            ph = phi[o:o + m]
            delta = st.comp_L[k] / m
            Mk = spline.knots(ph, delta)
            sel = st.q_comp == k
            q[:, sel] = spline.evaluate(ph, Mk, delta, st.q_s[sel])
            z[:, o:o + m] = spline.evaluate(ph, Mk, delta, np.arange(m) * delta)
        return q, z

    def jumps_from(self, phi=None, psi=None, Fq=None, Fz=None):
        st = self.st
        nq, M = st.q_xi.size, self.M
        zq, zz = np.zeros((3, nq)), np.zeros((3, M))
        dq, dz = self.density_derivs(phi) if phi is not None else (zq, zz)
        pq, pz = self.density_derivs(psi) if psi is not None else (zq, zz)
        Fq = np.zeros(nq) if Fq is None else Fq
        Fz = np.zeros(M) if Fz is None else Fz
        jq = jumps.jumps2d(dq[0], dq[1], dq[2], pq[0], pq[1], Fq, self.kappa, self.q_tau, self.q_taup)
        jz = jumps.jumps2d(dz[0], dz[1], dz[2], pz[0], pz[1], Fz, self.kappa, self.z_tau, self.z_taup)
        return jq, jz

    # ------------------------------------------------------------------ interface solve
    def interface_solve(self, base, jq, jz, want_grad=False):
        """Alg. 1 steps 4-6: correction → fast solve → interpolation.  base: (N−1, N−1)."""
        st = self.st
        n = st.n
        f = correction.correct2d(st, base, jq)
        v = np.zeros((n + 1, n + 1))
        v[1:n, 1:n] = fastsolve.solve2d(f, st.h, self.kappa)
        return v, interp.interpolate2d(st, v, jz, self.nodes, want_grad)

    def hole_coeffs(self, phi):
        st = self.st
        return [st.comp_L[k] / st.comp_M[k] * phi[st.comp_off[k]:st.comp_off[k] + st.comp_M[k]].sum()
                for k in self.holes]

    def apply_KD(self, phi):
        """K_D φ = V⁺ of the interface problem with Φ = φ, F = 0 (R17) [+ R27]."""
        n = self.st.n
        jq, jz = self.jumps_from(phi=phi)
        _, out = self.interface_solve(np.zeros((n - 1, n - 1)), jq, jz)
        for a, wg in zip(self.hole_coeffs(phi), self.w_gamma):
            out = out + a * wg
        return out

    def normal_derivative(self, coef):
        """∂_n V⁺ = n·(V⁺_x, V⁺_y) from the local quadratic fit coefficients at the control points."""
        return coef[:, 1] * self.z_nrm[0] + coef[:, 2] * self.z_nrm[1]

    def apply_KN(self, psi):
        """K_N ψ = ∂_n V⁺ of the interface problem with Φ = 0, Ψ = ψ, F = 0 (R38)."""
        n = self.st.n
        jq, jz = self.jumps_from(psi=psi)
        _, coef = self.interface_solve(np.zeros((n - 1, n - 1)), jq, jz, want_grad=True)
        return self.normal_derivative(coef)

    def apply_K(self, x):
        return self.apply_KN(x) if self.neumann else self.apply_KD(x)

    def apply_Yn(self, f_grid, f_isect, f_ctrl):
        """∂_n(Yf)⁺ at the control points."""
        jq, jz = self.jumps_from(Fq=f_isect, Fz=f_ctrl)
        _, coef = self.interface_solve(self.base_rhs(f_grid), jq, jz, want_grad=True)
        return self.normal_derivative(coef)

    def base_rhs(self, f_grid):
        """Zero extension f̃ = f·1_Ω at the unknowns."""
        n = self.st.n
        return np.where(self.st.side[1:n, 1:n], f_grid, 0.0)

    def apply_Y(self, f_grid, f_isect, f_ctrl):
        """(Yf)⁺ at control points: F = f̃, Φ = 0; [F] = f on Γ."""
        jq, jz = self.jumps_from(Fq=f_isect, Fz=f_ctrl)
        _, out = self.interface_solve(self.base_rhs(f_grid), jq, jz)
        return out

    def final(self, phi, f_grid, f_isect, f_ctrl):
        """u_h = Wφ + Yf (+ Σ a_h w_h, R27) on the grid."""
        n = self.st.n
        base = self.base_rhs(f_grid) if f_grid is not None else np.zeros((n - 1, n - 1))
        for a, k in zip(self.hole_coeffs(phi), self.holes):
            base = base + a * bump(self.prob.comps[k], self.X, self.Y)[1:n, 1:n]
        jq, jz = self.jumps_from(phi=phi, Fq=f_isect, Fz=f_ctrl)
        v, _ = self.interface_solve(base, jq, jz)
        return v

    def _krylov(self, K, ghat, phi0, tol, restart, max_restarts, method, gamma):
        if method == "richardson":
            return richardson(K, ghat, gamma=gamma, x0=phi0, tol=tol, max_iter=restart * max_restarts)
        if method == "bicgstab":
            return bicgstab(K, ghat, x0=phi0, tol=tol, max_iter=restart * max_restarts)
        return gmres(K, ghat, x0=phi0, tol=tol, restart=restart, max_restarts=max_restarts)

    def solve(self, g, f=None, tol=1e-8, restart=30, max_restarts=50, phi0=None, method="gmres", gamma=1.0,
              fdata=None):
        """Procedures 2-3: ĝ = g − (Yf)⁺, GMRES on K φ = ĝ, final field.
        f: callable f(x, y), or fdata = (f at the interior nodes (N−1)², f at intersections, f at
        control points) when f is only known as data (e.g. the Gray–Scott diffusion substeps)."""
        n = self.st.n
        if f is not None or fdata is not None:
            if fdata is not None:
                fg, fq, fz = fdata
                f = True
            else:
                px, py = self.isect_points()
                zx, zy = self.ctrl_points()
                fg = f(self.X[1:n, 1:n], self.Y[1:n, 1:n])
                fq, fz = f(px, py), f(zx, zy)
            ghat = g - self.apply_Y(fg, fq, fz) if not self.neumann else None
        else:
            fg = fq = fz = None
            ghat = g.copy()
        if self.neumann:   # g = g_N = ∂_n u on Γ at the control points
            ghat = g - (self.apply_Yn(fg, fq, fz) if f is not None else 0.0)
            psi, stats = self._krylov(self.apply_KN, ghat, phi0, tol, restart, max_restarts, method, gamma)
            base = self.base_rhs(fg) if f is not None else np.zeros((n - 1, n - 1))
            jq, jz = self.jumps_from(psi=psi, Fq=fq, Fz=fz)
            u, _ = self.interface_solve(base, jq, jz)   # u = Yf − Sψ
            return u, psi, stats
        phi, stats = self._krylov(self.apply_KD, ghat, phi0, tol, restart, max_restarts, method, gamma)
        u = self.final(phi, fg, fq, fz)
        return u, phi, stats

    def errors(self, u, uex):
        m = self.st.side
        e = (u - uex)[m]
        return float(np.abs(e).max()), float(np.sqrt(np.mean(e * e)))
