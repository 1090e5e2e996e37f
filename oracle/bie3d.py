"""KFBI operators and the Dirichlet BVP solve in 3D (test infrastructure only).

Same pipeline as oracle/bie.py (Alg. 1-5) with the 3D readings R12-R14:
control points = intersection nodes, density derivatives from a tangent-plane LSQ fit, jumps from the
tangential/normal differentiation of [v] = Φ, [∂_n v] = Ψ plus the PDE trace, solved here as linear
systems (3×3 first order, 6×6 second order) rather than through the closed form; seven-point
correction; ten-point interpolation solved by LU.
"""
from __future__ import annotations

import numpy as np

from . import fastsolve, grid3d
from .gmres import gmres


def jumps3d(Phi, dPhi, d2Phi, Psi, dPsi, F, kappa, n, e1, e2, kab):
    """Columns: [v], [v_x], [v_y], [v_z], [v_xx], [v_yy], [v_zz], [v_xy], [v_xz], [v_yz]."""
    m = n.shape[0]
    A1 = np.stack([e1, e2, n], 1)                                    # rows e1, e2, n
    b1 = np.stack([dPhi[:, 0], dPhi[:, 1], Psi], -1)
    g = np.linalg.solve(A1, b1[..., None])[..., 0]
    # unknown H = (xx, yy, zz, xy, xz, yz); uᵀHw = Σ coefficients below
    def quad(u, w):
        return np.stack([u[:, 0] * w[:, 0], u[:, 1] * w[:, 1], u[:, 2] * w[:, 2],
                         u[:, 0] * w[:, 1] + u[:, 1] * w[:, 0], u[:, 0] * w[:, 2] + u[:, 2] * w[:, 0],
                         u[:, 1] * w[:, 2] + u[:, 2] * w[:, 1]], -1)
    A2 = np.stack([quad(e1, e1), quad(e1, e2), quad(e2, e2), quad(e1, n), quad(e2, n),
                   np.broadcast_to(np.array([1.0, 1.0, 1.0, 0, 0, 0]), (m, 6))], 1)
    b2 = np.stack([d2Phi[:, 0] - kab[:, 0, 0] * Psi,
                   d2Phi[:, 1] - kab[:, 0, 1] * Psi,
                   d2Phi[:, 2] - kab[:, 1, 1] * Psi,
                   dPsi[:, 0] + kab[:, 0, 0] * dPhi[:, 0] + kab[:, 0, 1] * dPhi[:, 1],
                   dPsi[:, 1] + kab[:, 1, 0] * dPhi[:, 0] + kab[:, 1, 1] * dPhi[:, 1],
                   F + kappa * Phi], -1)
    H = np.linalg.solve(A2, b2[..., None])[..., 0]
    return np.concatenate([Phi[:, None], g, H], -1)


def correct3d(st, base, jq):
    """Seven-point analogue of Alg. 2 (A.3 along each axis)."""
    h = st.h
    f = base.copy()
    ax = st.q_axis
    p0 = np.stack([st.q_i, st.q_j, st.q_k], -1)
    p1 = p0 + np.eye(3, dtype=np.int64)[ax]
    rows = np.arange(ax.size)
    va = jq[rows, 1 + ax]
    vaa = jq[rows, 4 + ax]
    for pa, pb in ((p0, p1), (p1, p0)):
        xbar = st.x[pb[rows, ax]]
        d = xbar - st.q_xi
        P = jq[:, 0] + va * d + 0.5 * vaa * d * d
        sgn = np.where(st.side[pa[:, 0], pa[:, 1], pa[:, 2]], -1.0, 1.0)
        np.add.at(f, (pa[:, 0] - 1, pa[:, 1] - 1, pa[:, 2] - 1), sgn * P / (h * h))
    return f


def interpolate3d(st, v_full, jz, nodes, want_grad=False):
    M = st.M
    d = st.x[nodes] - st.q_pos[:, None, :]                      # (M, 10, 3)
    dx, dy, dz = d[..., 0], d[..., 1], d[..., 2]
    A = np.stack([np.ones_like(dx), dx, dy, dz, 0.5 * dx * dx, 0.5 * dy * dy, 0.5 * dz * dz,
                  dx * dy, dx * dz, dy * dz], -1)
    J = (jz[:, 0:1] + jz[:, 1:2] * dx + jz[:, 2:3] * dy + jz[:, 3:4] * dz + 0.5 * jz[:, 4:5] * dx * dx
         + 0.5 * jz[:, 5:6] * dy * dy + 0.5 * jz[:, 6:7] * dz * dz + jz[:, 7:8] * dx * dy + jz[:, 8:9] * dx * dz
         + jz[:, 9:10] * dy * dz)
    inside = st.side[nodes[..., 0], nodes[..., 1], nodes[..., 2]]
    rhs = v_full[nodes[..., 0], nodes[..., 1], nodes[..., 2]] + np.where(inside, 0.0, J)
    coef = np.linalg.solve(A, rhs[..., None])[..., 0]
    return coef if want_grad else coef[:, 0]


class Oracle3D:
    def __init__(self, prob):
        self.prob = prob
        self.kappa = prob.kappa
        self.st = grid3d.build(prob)
        self.M = self.st.M
        self.nb = grid3d.lsq_neighbours(self.st)
        self.lsq_idx, self.lsq_pinv = grid3d.lsq_operator(self.st, self.nb)
        self.nodes = grid3d.stencil(self.st)
        self.neumann = getattr(prob, "bc", 0) == 1   # reading R38 in 3D: K_N ψ = ∂_n V⁺, [v] = 0, [∂_n v] = ψ
        if self.neumann and self.kappa <= 0.0:
            raise ValueError("Neumann BVP needs κ > 0 (S:555)")

    def points(self):
        return self.st.q_pos

    def jumps_from(self, phi=None, F=None, psi=None):
        """(Φ, Ψ, [F]) → jumps; Φ and Ψ tangential derivatives from the same LSQ fit (R12)."""
        st = self.st
        M = self.M
        zero5 = np.zeros((M, 5))
        d = grid3d.lsq_fit(self.lsq_idx, self.lsq_pinv, phi) if phi is not None else zero5
        dpsi = grid3d.lsq_fit(self.lsq_idx, self.lsq_pinv, psi) if psi is not None else zero5
        phi = np.zeros(M) if phi is None else phi
        psi = np.zeros(M) if psi is None else psi
        F = np.zeros(M) if F is None else F
        return jumps3d(phi, d[:, 0:2], d[:, 2:5], psi, dpsi[:, 0:2], F, self.kappa,
                       st.nrm, st.e1, st.e2, st.kab)

    def interface_solve(self, base, jq, want_grad=False):
        """Correction → fast solve → interpolation; control points = intersections, so the same
        jumps serve both (R12, R15)."""
        st = self.st
        n = st.n
        f = correct3d(st, base, jq)
        v = np.zeros((n + 1,) * 3)
        v[1:n, 1:n, 1:n] = fastsolve.solve3d(f, st.h, self.kappa)
        return v, interpolate3d(st, v, jq, self.nodes, want_grad)

    def apply_KD(self, phi):
        n = self.st.n
        _, out = self.interface_solve(np.zeros((n - 1,) * 3), self.jumps_from(phi=phi))
        return out

    def apply_KN(self, psi):
        """K_N ψ = ∂_n V⁺ of the interface problem [v] = 0, [∂_n v] = ψ (R38)."""
        n = self.st.n
        _, coef = self.interface_solve(np.zeros((n - 1,) * 3), self.jumps_from(psi=psi), want_grad=True)
        return np.sum(coef[:, 1:4] * self.st.nrm, -1)

    def apply_K(self, x):
        return self.apply_KN(x) if self.neumann else self.apply_KD(x)

    def base_rhs(self, f_grid):
        n = self.st.n
        return np.where(self.st.side[1:n, 1:n, 1:n], f_grid, 0.0)

    def solve(self, g, f=None, tol=1e-8, restart=30, max_restarts=50):
        n = self.st.n
        x = self.st.x
        if f is not None:
            X, Y, Z = np.meshgrid(x[1:n], x[1:n], x[1:n], indexing="ij")
            fg = f(X, Y, Z)
            fq = f(*self.st.q_pos.T)
            _, yf = self.interface_solve(self.base_rhs(fg), self.jumps_from(F=fq), want_grad=self.neumann)
            ghat = g - (np.sum(yf[:, 1:4] * self.st.nrm, -1) if self.neumann else yf)
        else:
            fg = fq = None
            ghat = g.copy()
        phi, stats = gmres(self.apply_K, ghat, tol=tol, restart=restart, max_restarts=max_restarts)
        base = self.base_rhs(fg) if fg is not None else np.zeros((n - 1,) * 3)
        jumps = self.jumps_from(psi=phi, F=fq) if self.neumann else self.jumps_from(phi=phi, F=fq)
        v, _ = self.interface_solve(base, jumps)
        return v, phi, stats

    def errors(self, u, uex):
        e = (u - uex)[self.st.side]
        return float(np.abs(e).max()), float(np.sqrt(np.mean(e * e)))
