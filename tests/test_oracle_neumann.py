"""Oracle pins for the Neumann BVP (reading R38): K_N ψ = ∂_n V⁺ of the
interface problem with [v] = 0, [∂_n v] = ψ, read off the gradient rows of the local quadratic fit."""
import numpy as np
import pytest

import workloads as W
from oracle.bie import Oracle2D


def _quad(seed):
    a = np.random.default_rng(seed).uniform(-1, 1, 6)
    q = lambda x, y: a[0] + a[1] * x + a[2] * y + a[3] * x * x + a[4] * x * y + a[5] * y * y
    gq = lambda x, y: (a[1] + 2 * a[3] * x + a[4] * y, a[2] + a[4] * x + 2 * a[5] * y)
    H = np.array([[2 * a[3], a[4]], [a[4], 2 * a[5]]])
    return q, gq, H


def test_normal_derivative_interpolation_exact_for_quadratics():
    """v = q·1_Ω with its exact jumps: the fitted gradient at every control point is ∇q."""
    prob = W.neumann(W.problem("ell-k1", 2, 128, [W.ellipse(1.0, 0.8)], 1.0))
    o = Oracle2D(prob)
    q, gq, H = _quad(3)
    st = o.st
    px, py = o.isect_points()
    zx, zy = o.ctrl_points()
    jump = lambda x, y: np.stack([q(x, y), *gq(x, y), np.full_like(x, H[0, 0]), np.full_like(x, H[0, 1]),
                                  np.full_like(x, H[1, 1])], -1)
    n = st.n
    base = np.where(st.side[1:n, 1:n], np.trace(H) - prob.kappa * q(o.X, o.Y)[1:n, 1:n], 0.0)
    _, coef = o.interface_solve(base, jump(px, py), jump(zx, zy), want_grad=True)
    gx, gy = gq(zx, zy)
    np.testing.assert_allclose(coef[:, 1], gx, atol=1e-9)
    np.testing.assert_allclose(coef[:, 2], gy, atol=1e-9)
    np.testing.assert_allclose(o.normal_derivative(coef), gx * o.z_nrm[0] + gy * o.z_nrm[1], atol=1e-9)


def test_normal_derivative_second_order_with_exact_jumps():
    """Interface problem of u*·1_Ω with exact jumps (Φ = u*, Ψ = ∂_n u*, [F] = f): ∂_n V⁺ → ∂_n u* at O(h²)."""
    errs = []
    for n in (64, 128, 256):
        prob = W.neumann(W.problem("ell-k1", 2, n, [W.ellipse(1.0, 0.8)], 1.0))
        o = Oracle2D(prob)
        zx, zy = o.ctrl_points()
        px, py = o.isect_points()
        ux, uy = W.grad_u_exact(zx, zy)
        gN = ux * o.z_nrm[0] + uy * o.z_nrm[1]
        f = lambda x, y: W.f_exact(1.0, x, y)
        jq, jz = o.jumps_from(phi=W.u_exact(zx, zy), psi=gN, Fq=f(px, py), Fz=f(zx, zy))
        _, coef = o.interface_solve(o.base_rhs(f(o.X, o.Y)[1:n, 1:n]), jq, jz, want_grad=True)
        errs.append(np.abs(o.normal_derivative(coef) - gN).max())
    ratios = np.array(errs[:-1]) / np.array(errs[1:])
    assert np.all(ratios > 3.0), (errs, ratios)


def test_neumann_solve_converges():
    """GMRES on K_N ψ = g_N − ∂_n(Yf)⁺, u = Yf − Sψ: u_h → u* (control points ∝ N, clear of ∂B)."""
    errs = []
    for n in (128, 256, 512):
        prob = W.neumann(W.problem("ell", 2, n, [W.ellipse(0.6, 0.45, n_ctrl=n)], 1.0))
        o = Oracle2D(prob)
        zx, zy = o.ctrl_points()
        ux, uy = W.grad_u_exact(zx, zy)
        gN = ux * o.z_nrm[0] + uy * o.z_nrm[1]
        u, psi, st = o.solve(gN, lambda x, y: W.f_exact(1.0, x, y))
        assert st.converged and st.iters < 20
        errs.append(o.errors(u, W.u_exact(o.X, o.Y))[0])
    assert errs[-1] < errs[0] / 8 and errs[-1] < 1e-4, errs


def test_neumann_needs_positive_kappa():
    with pytest.raises(ValueError):
        Oracle2D(W.neumann(W.C1(64)))


def test_neumann_3d_gradient_exact_and_convergence():
    """3D (R12, R38): the 10-point fit's gradient is exact for a piecewise quadratic with exact jumps,
    and the Neumann BVP on an ellipsoid converges under refinement."""
    from oracle.bie3d import Oracle3D
    prob = W.neumann(W.problem("ellipsoid-k1", 3, 32, [W.ellipsoid(0.7, 0.6, 0.5)], 1.0))
    o = Oracle3D(prob)
    rng = np.random.default_rng(4)
    a = rng.uniform(-1, 1, 10)
    H = np.array([[2 * a[4], a[7], a[8]], [a[7], 2 * a[5], a[9]], [a[8], a[9], 2 * a[6]]])
    q = lambda x, y, z: (a[0] + a[1] * x + a[2] * y + a[3] * z + a[4] * x * x + a[5] * y * y + a[6] * z * z
                         + a[7] * x * y + a[8] * x * z + a[9] * y * z)
    gq = lambda x, y, z: np.stack([a[1] + 2 * a[4] * x + a[7] * y + a[8] * z, a[2] + 2 * a[5] * y + a[7] * x + a[9] * z,
                                   a[3] + 2 * a[6] * z + a[8] * x + a[9] * y], -1)
    p = o.points()
    jq = np.concatenate([q(*p.T)[:, None], gq(*p.T),
                         np.tile([H[0, 0], H[1, 1], H[2, 2], H[0, 1], H[0, 2], H[1, 2]], (o.M, 1))], -1)
    n = prob.n
    X, Y, Z = np.meshgrid(o.st.x, o.st.x, o.st.x, indexing="ij")
    base = np.where(o.st.side, np.trace(H) - prob.kappa * q(X, Y, Z), 0.0)[1:n, 1:n, 1:n]
    _, coef = o.interface_solve(base, jq, want_grad=True)
    np.testing.assert_allclose(coef[:, 1:4], gq(*p.T), atol=1e-9)
    errs = []
    for n in (32, 64):
        prob = W.neumann(W.problem("ellipsoid-k1", 3, n, [W.ellipsoid(0.7, 0.6, 0.5)], 1.0))
        o = Oracle3D(prob)
        p = o.points()
        gN = np.sum(np.stack(W.grad_u_exact(*p.T), -1) * o.st.nrm, -1)
        u, psi, st = o.solve(gN, lambda x, y, z: W.f_exact(1.0, x, y, z))
        assert st.converged
        X, Y, Z = np.meshgrid(o.st.x, o.st.x, o.st.x, indexing="ij")
        errs.append(o.errors(u, W.u_exact(X, Y, Z))[0])
    assert errs[1] < errs[0] / 2.5, errs
