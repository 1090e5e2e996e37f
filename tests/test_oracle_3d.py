"""Pins for the 3D oracle (readings R12-R14) against closed forms and exactness identities (no GPU)."""
import numpy as np
import pytest
import scipy.sparse
import scipy.sparse.linalg

import workloads as W
from oracle import fastsolve, grid3d
from oracle.bie3d import Oracle3D, correct3d, interpolate3d, jumps3d


def _quad3(seed):
    a = np.random.default_rng(seed).uniform(-1, 1, 10)
    H = np.array([[2 * a[4], a[7], a[8]], [a[7], 2 * a[5], a[9]], [a[8], a[9], 2 * a[6]]])

    def q(x, y, z):
        return (a[0] + a[1] * x + a[2] * y + a[3] * z + a[4] * x * x + a[5] * y * y + a[6] * z * z
                + a[7] * x * y + a[8] * x * z + a[9] * y * z)

    def grad(x, y, z):
        return np.stack([a[1] + 2 * a[4] * x + a[7] * y + a[8] * z,
                         a[2] + 2 * a[5] * y + a[7] * x + a[9] * z,
                         a[3] + 2 * a[6] * z + a[8] * x + a[9] * y], -1)
    return q, grad, H


def _jump_row(Q, G, H):
    m = Q.size
    return np.concatenate([Q[:, None], G, np.tile([H[0, 0], H[1, 1], H[2, 2], H[0, 1], H[0, 2], H[1, 2]], (m, 1))], -1)


SURF = {"ellipsoid": W.ellipsoid(1.0, 0.8, 0.6), "torus": W.torus(0.7, 0.3)}


def _surface_points(comp, m=200, seed=0):
    rng = np.random.default_rng(seed)
    u, v = rng.uniform(0, 2 * np.pi, m), rng.uniform(0, 2 * np.pi, m)
    if comp.kind == W.ELLIPSOID:
        a, b, c = comp.p[:3]
        w = rng.uniform(-0.95, 0.95, m)
        s = np.sqrt(1 - w * w)
        return np.stack([a * s * np.cos(u), b * s * np.sin(u), c * w], -1)
    R, r = comp.p[:2]
    return np.stack([(R + r * np.cos(v)) * np.cos(u), (R + r * np.cos(v)) * np.sin(u), r * np.sin(v)], -1)


@pytest.mark.parametrize("name", ["ellipsoid", "torus"])
@pytest.mark.parametrize("kappa", [0.0, 1.0])
def test_jumps3d_exact_for_piecewise_quadratics(name, kappa):
    comp = SURF[name]
    p = _surface_points(comp)
    n, e1, e2, kab = grid3d.frames(comp, p)
    qi, gi, Hi = _quad3(1)
    qo, go, Ho = _quad3(2)
    Q = qi(*p.T) - qo(*p.T)
    G = gi(*p.T) - go(*p.T)
    H = Hi - Ho
    # Monge-patch derivatives of Φ = Q|Γ and Ψ = ∇Q·n (x(t) = x0 + t_a e_a + ½κ_ab t_a t_b n)
    E = np.stack([e1, e2], 1)
    Gn = (G * n).sum(1)
    dPhi = np.einsum("mai,mi->ma", E, G)
    d2 = np.einsum("mai,ij,mbj->mab", E, H, E) + kab * Gn[:, None, None]
    d2Phi = np.stack([d2[:, 0, 0], d2[:, 0, 1], d2[:, 1, 1]], -1)
    dPsi = np.einsum("mai,ij,mj->ma", E, H, n) - np.einsum("mab,mbi,mi->ma", kab, E, G)
    F = np.trace(H) - kappa * Q
    J = jumps3d(Q, dPhi, d2Phi, Gn, dPsi, F, kappa, n, e1, e2, kab)
    np.testing.assert_allclose(J, _jump_row(Q, G, H), atol=1e-11)


def test_frames_sphere_closed_form():
    p = _surface_points(W.ellipsoid(1, 1, 1))
    n, e1, e2, kab = grid3d.frames(W.ellipsoid(1, 1, 1), p)
    np.testing.assert_allclose(n, p, atol=1e-14)                       # outward unit normal
    np.testing.assert_allclose(kab, -np.eye(2)[None].repeat(len(p), 0), atol=1e-13)   # κ = −1/r
    np.testing.assert_allclose(np.linalg.det(np.stack([e1, e2, n], 1)), 1.0, atol=1e-13)


def test_lsq_fit_constants_and_convergence():
    errs = []
    q, gq, H = _quad3(3)
    for nn in (32, 64):
        st = grid3d.build(W.problem("sph", 3, nn, [W.ellipsoid(1, 1, 1)], 0.0))
        idx, pinv = grid3d.lsq_operator(st, grid3d.lsq_neighbours(st))
        c = grid3d.lsq_fit(idx, pinv, np.full(st.M, 3.0))
        assert np.abs(c).max() < 1e-9
        d = grid3d.lsq_fit(idx, pinv, q(*st.q_pos.T))
        G = gq(*st.q_pos.T)
        E = np.stack([st.e1, st.e2], 1)
        ex1 = np.einsum("mai,mi->ma", E, G)
        ex2 = np.einsum("mai,ij,mbj->mab", E, H, E) + st.kab * (G * st.nrm).sum(1)[:, None, None]
        errs.append([np.abs(d[:, :2] - ex1).max(), np.abs(d[:, 2] - ex2[:, 0, 0]).max()])
    e = np.array(errs)
    order = np.log2(e[0] / e[1])
    # unweighted one-sided fits: O(h²) first and O(h) second derivatives (max norm pre-asymptotic)
    assert order[0] > 1.5 and order[1] > 0.5, (e, order)


def test_correction3d_quadratic_witness():
    prob = W.C4(32)
    st = grid3d.build(prob)
    q, gq, H = _quad3(4)
    n, h = st.n, st.h
    X, Y, Z = np.meshgrid(st.x, st.x, st.x, indexing="ij")
    v = np.where(st.side, q(X, Y, Z), 0.0)
    G = gq(*st.q_pos.T)
    jq = _jump_row(q(*st.q_pos.T), G, H)
    base = np.where(st.side[1:n, 1:n, 1:n], np.trace(H) - prob.kappa * q(X, Y, Z)[1:n, 1:n, 1:n], 0.0)
    f = correct3d(st, base, jq)
    p = np.pad(v[1:n, 1:n, 1:n], 1)
    c = p[1:-1, 1:-1, 1:-1]
    lap = (p[2:, 1:-1, 1:-1] + p[:-2, 1:-1, 1:-1] + p[1:-1, 2:, 1:-1] + p[1:-1, :-2, 1:-1]
           + p[1:-1, 1:-1, 2:] + p[1:-1, 1:-1, :-2] - 6 * c) / h ** 2 - prob.kappa * c
    assert np.abs(lap - f).max() < 1e-8


def test_fast_solver3d_eigenfunction_and_dense():
    n, h, kap = 16, 2.4 / 16, 1.0
    i = np.arange(1, n)
    S = np.einsum("i,j,k->ijk", np.sin(np.pi * 2 * i / n), np.sin(np.pi * 5 * i / n), np.sin(np.pi * 11 * i / n))
    lam = -4 / h ** 2 * sum(np.sin(np.pi * p / (2 * n)) ** 2 for p in (2, 5, 11)) - kap
    np.testing.assert_allclose(fastsolve.solve3d(lam * S, h, kap), S, atol=1e-11)
    n, h = 8, 0.3
    m = n - 1
    T = scipy.sparse.diags([1.0, -2.0, 1.0], [-1, 0, 1], shape=(m, m))
    I = scipy.sparse.identity(m)
    A = (scipy.sparse.kron(scipy.sparse.kron(T, I), I) + scipy.sparse.kron(scipy.sparse.kron(I, T), I)
         + scipy.sparse.kron(scipy.sparse.kron(I, I), T)) / h ** 2 - kap * scipy.sparse.identity(m ** 3)
    f = np.random.default_rng(0).uniform(-1, 1, (m, m, m))
    ref = scipy.sparse.linalg.spsolve(A.tocsc(), f.ravel()).reshape(m, m, m)
    np.testing.assert_allclose(fastsolve.solve3d(f, h, kap), ref, atol=1e-12)


@pytest.mark.parametrize("prob", [W.C4(32), W.C5(64)], ids=["ellipsoid32", "torus64"])
def test_interface_solve3d_reproduces_piecewise_quadratic(prob):
    o = Oracle3D(prob)
    st = o.st
    n = st.n
    q, gq, H = _quad3(6)
    X, Y, Z = np.meshgrid(st.x, st.x, st.x, indexing="ij")
    jq = _jump_row(q(*st.q_pos.T), gq(*st.q_pos.T), H)
    base = np.where(st.side[1:n, 1:n, 1:n], np.trace(H) - prob.kappa * q(X, Y, Z)[1:n, 1:n, 1:n], 0.0)
    v, vp = o.interface_solve(base, jq)
    np.testing.assert_allclose(v, np.where(st.side, q(X, Y, Z), 0.0), atol=1e-10)
    np.testing.assert_allclose(vp, q(*st.q_pos.T), atol=1e-10)


def test_interp3d_exact_for_quadratics():
    st = grid3d.build(W.C4(32))
    q, gq, H = _quad3(7)
    X, Y, Z = np.meshgrid(st.x, st.x, st.x, indexing="ij")
    out = interpolate3d(st, q(X, Y, Z), np.zeros((st.M, 10)), grid3d.stencil(st))
    np.testing.assert_allclose(out, q(*st.q_pos.T), atol=1e-12)


def test_KD3d_constant_density():
    o = Oracle3D(W.C4(32))
    np.testing.assert_allclose(o.apply_KD(np.ones(o.M)), 1.0, atol=1e-12)


@pytest.mark.slow
def test_second_order_3d():
    errs = []
    for nn in (32, 64):
        prob = W.problem("sphere", 3, nn, [W.ellipsoid(1, 1, 1)], 0.0)
        o = Oracle3D(prob)
        X, Y, Z = np.meshgrid(o.st.x, o.st.x, o.st.x, indexing="ij")
        v, phi, s = o.solve(W.u_exact(*o.points().T), lambda a, b, c: W.f_exact(0.0, a, b, c))
        assert s.converged
        errs.append(o.errors(v, W.u_exact(X, Y, Z)))
    e = np.array(errs)
    order = np.log2(e[0] / e[1])
    assert np.all(order > 1.7), order
