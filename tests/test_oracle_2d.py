"""Pins for the 2D CPU oracle against things other than itself (no GPU).

Each test names what fixes the expected value: a worked example (tests/golden), a closed
form, an exactness property of the scheme, brute force, or a textbook identity.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.sparse
import scipy.sparse.linalg
import scipy.special

import workloads as W
from oracle import correction, fastsolve, geometry as geo, grid, interp, jumps, spline
from oracle.bie import Oracle2D
from oracle.gmres import gmres

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _quad(seed):
    """Random quadratic q = a0 + a1 x + a2 y + a3 x² + a4 xy + a5 y² with exact derivatives."""
    a = np.random.default_rng(seed).uniform(-1, 1, 6)

    def q(x, y):
        return a[0] + a[1] * x + a[2] * y + a[3] * x * x + a[4] * x * y + a[5] * y * y

    def grad(x, y):
        return np.stack([a[1] + 2 * a[3] * x + a[4] * y, a[2] + a[4] * x + 2 * a[5] * y])

    hess = np.array([[2 * a[3], a[4]], [a[4], 2 * a[5]]])
    return q, grad, hess


# ----------------------------------------------------------------- grid / geometry
def test_grid_worked_example():
    gold = json.load(open(os.path.join(GOLD, "grid_circle_h0p3.json")))
    n = gold["n"]
    p = W.problem("circle", 2, n, [W.circle(gold["radius"])], 0.0)
    st = grid.build(p, check_clearance=False)
    assert st.side.sum() == gold["interior_nodes"]
    assert st.irregular[1:n, 1:n].sum() == gold["irregular_unknowns"]
    assert (st.q_axis == 0).sum() == gold["x_crossings"]
    assert (st.q_axis == 1).sum() == gold["y_crossings"]
    row = (st.q_axis == 0) & (np.abs(st.x[st.q_j]) < 1e-12)
    np.testing.assert_allclose(np.sort(st.q_xi[row]), gold["row_y0_crossings"], atol=1e-10)


@pytest.mark.parametrize("prob", [W.C1(64), W.C2(128), W.C3(256)])
def test_intersection_invariants(prob):
    st = grid.build(prob)
    n = st.n
    # endpoints differ in side; crossing lies on Γ of its component; even count per line
    i1 = st.q_i + (st.q_axis == 0)
    j1 = st.q_j + (st.q_axis == 1)
    assert np.all(st.side[st.q_i, st.q_j] != st.side[i1, j1])
    px = np.where(st.q_axis == 0, st.q_xi, st.x[st.q_i])
    py = np.where(st.q_axis == 1, st.q_xi, st.x[st.q_j])
    for k, c in enumerate(prob.comps):
        sel = st.q_comp == k
        g = geo.curve(c, st.q_theta[sel])[0]
        np.testing.assert_allclose(g[0], px[sel], atol=1e-12)
        np.testing.assert_allclose(g[1], py[sel], atol=1e-12)
    for axis in (0, 1):
        line = st.q_j if axis == 0 else st.q_i
        cnt = np.bincount(line[st.q_axis == axis], minlength=n + 1)
        assert np.all(cnt % 2 == 0)
    # every irregular unknown is an endpoint of a recorded edge
    ends = set(zip(st.q_i.tolist(), st.q_j.tolist())) | set(zip(i1.tolist(), j1.tolist()))
    ii, jj = np.nonzero(st.irregular)
    assert set(zip(ii.tolist(), jj.tolist())) == ends


def test_arc_length_closed_forms():
    c = W.circle(1.0)
    assert abs(geo.perimeter(c) - 2 * math.pi) < 1e-13
    a, b = 1.0, 0.8
    exact = 4 * a * scipy.special.ellipe(1 - (b / a) ** 2)       # complete elliptic integral
    assert abs(geo.perimeter(W.ellipse(a, b)) - exact) < 1e-13
    th = np.linspace(0, 2 * math.pi, 7)
    np.testing.assert_allclose(geo.arc_length_ccw(W.circle(2.0), th), 2.0 * th, atol=1e-13)


def test_frame_closed_forms():
    r = 1.5
    c = W.circle(r)
    th = np.linspace(0, 6, 9)
    g, tau, taup, n = geo.frame(c, th)
    np.testing.assert_allclose(tau, np.stack([-np.sin(th), np.cos(th)]), atol=1e-14)
    np.testing.assert_allclose(taup, -np.stack([np.cos(th), np.sin(th)]) / r, atol=1e-14)
    np.testing.assert_allclose(n, np.stack([np.cos(th), np.sin(th)]), atol=1e-14)     # outward
    hole = W.circle(r, role=W.HOLE)
    _, tau_h, taup_h, n_h = geo.frame(hole, th)
    np.testing.assert_allclose(n_h, -n, atol=1e-14)        # points into the hole = out of Ω
    np.testing.assert_allclose(taup_h, taup, atol=1e-14)
    # star: τ' against a central difference of τ in arc length
    s = W.star(1.0, 0.2, 4)
    th = np.linspace(0.1, 6.0, 11)
    e = 1e-5
    _, t0, tp, _ = geo.frame(s, th)
    _, tpl, _, _ = geo.frame(s, th + e)
    _, tmi, _, _ = geo.frame(s, th - e)
    ds = np.linalg.norm(geo.curve(s, th)[1], axis=0) * 2 * e
    np.testing.assert_allclose((tpl - tmi) / ds, tp, atol=1e-8)


def test_control_points_uniform_arc_length():
    prob = W.C3(256)
    st = grid.build(prob)
    for k, c in enumerate(prob.comps):
        sel = st.z_comp == k
        L, M = st.comp_L[k], st.comp_M[k]
        s = geo.s_omega(c, st.z_theta[sel], L)
        s = np.where(s > L - 1e-9, s - L, s)
        np.testing.assert_allclose(s, np.arange(M) * L / M, atol=1e-12 * L)
        th = st.z_theta[sel]
        dth = np.mod(np.diff(th), 2 * math.pi)
        if c.role == W.HOLE:            # clockwise: θ decreases
            assert np.all(dth > math.pi)
        else:
            assert np.all(dth < math.pi)
    assert st.comp_M[0] == round(st.comp_L[0] / (1.18 * st.h))


# ----------------------------------------------------------------- spline
def test_spline_interpolates_and_constants():
    rng = np.random.default_rng(3)
    phi = rng.uniform(-1, 1, 40)
    Mk = spline.knots(phi, 0.1)
    g, gp, gpp = spline.evaluate(phi, Mk, 0.1, np.arange(40) * 0.1)
    np.testing.assert_allclose(g, phi, atol=1e-14)
    c = np.full(40, 2.5)
    g, gp, gpp = spline.evaluate(c, spline.knots(c, 0.1), 0.1, rng.uniform(0, 4, 50))
    np.testing.assert_allclose(g, 2.5, atol=1e-14)
    np.testing.assert_allclose(gp, 0.0, atol=1e-13)
    np.testing.assert_allclose(gpp, 0.0, atol=1e-12)


def test_spline_matches_dense_cyclic_solve():
    m, d = 16, 0.3
    phi = np.random.default_rng(4).uniform(-1, 1, m)
    A = np.zeros((m, m))
    for i in range(m):
        A[i, i] = 4
        A[i, (i + 1) % m] = 1
        A[i, (i - 1) % m] = 1
    rhs = np.array([6 * (phi[(i + 1) % m] - 2 * phi[i] + phi[i - 1]) / d ** 2 for i in range(m)])
    np.testing.assert_allclose(spline.knots(phi, d), np.linalg.solve(A, rhs), atol=1e-12)


def test_spline_convergence_orders():
    errs = []
    for m in (32, 64, 128):
        L = 2 * math.pi
        d = L / m
        s = np.arange(m) * d
        phi = np.sin(s) + 0.3 * np.cos(2 * s)
        Mk = spline.knots(phi, d)
        t = np.linspace(0, L, 997, endpoint=False)
        g, gp, gpp = spline.evaluate(phi, Mk, d, t)
        errs.append([np.abs(g - (np.sin(t) + 0.3 * np.cos(2 * t))).max(),
                     np.abs(gp - (np.cos(t) - 0.6 * np.sin(2 * t))).max(),
                     np.abs(gpp - (-np.sin(t) - 1.2 * np.cos(2 * t))).max()])
    errs = np.array(errs)
    orders = np.log2(errs[:-1] / errs[1:])
    assert np.all(orders[:, 0] > 3.7) and np.all(orders[:, 1] > 2.7) and np.all(orders[:, 2] > 1.8)


# ----------------------------------------------------------------- jumps
@pytest.mark.parametrize("comp", [W.ellipse(1.0, 0.8), W.star(1.0, 0.2, 4), W.circle(0.3, (0.2, 0.1), role=W.HOLE)])
@pytest.mark.parametrize("kappa", [0.0, 1.0])
def test_jumps_exact_for_piecewise_quadratics(comp, kappa):
    """Exact jumps of w = q_in in Ω, q_out outside: the appendix system must return them."""
    qi, gi, Hi = _quad(1)
    qo, go, Ho = _quad(2)
    th = np.linspace(0, 2 * math.pi, 23, endpoint=False)
    g, tau, taup, n = geo.frame(comp, th)
    Q = qi(*g) - qo(*g)
    G = gi(*g) - go(*g)
    H = Hi - Ho
    Phis = (G * tau).sum(0)
    Phiss = np.einsum("ip,ij,jp->p", tau, H, tau) + (G * taup).sum(0)
    Psi = (G * n).sum(0)
    npr = np.stack([taup[1], -taup[0]])
    Psis = np.einsum("ip,ij,jp->p", tau, H, n) + (G * npr).sum(0)
    F = np.trace(H) - kappa * Q
    J = jumps.jumps2d(Q, Phis, Phiss, Psi, Psis, F, kappa, tau, taup)
    np.testing.assert_allclose(J[:, 0], Q, atol=1e-13)
    np.testing.assert_allclose(J[:, 1:3].T, G, atol=1e-12)
    np.testing.assert_allclose(J[:, 3], H[0, 0], atol=1e-11)
    np.testing.assert_allclose(J[:, 4], H[0, 1], atol=1e-11)
    np.testing.assert_allclose(J[:, 5], H[1, 1], atol=1e-11)


def test_jumps_trivial_cases():
    tau = np.array([[0.0], [1.0]])
    taup = np.array([[-1.0], [0.0]])          # unit circle at (1, 0)
    J = jumps.jumps2d(2.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, tau, taup)
    np.testing.assert_allclose(J[0], [2, 0, 0, 0, 0, 0], atol=1e-15)
    J = jumps.jumps2d(0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, tau, taup)   # single layer, n = (1, 0)
    np.testing.assert_allclose(J[0, :3], [0, 1, 0], atol=1e-15)


# ----------------------------------------------------------------- correction (witness)
@pytest.mark.parametrize("prob", [W.C1(64), W.C2(128), W.C3(128)])
def test_correction_quadratic_witness(prob):
    """For v = q·1_Ω with exact jumps the corrected 5-point residual vanishes at every node."""
    st = grid.build(prob)
    q, gq, H = _quad(7)
    n, h, kap = st.n, st.h, prob.kappa
    X, Y = np.meshgrid(st.x, st.x, indexing="ij")
    v = np.where(st.side, q(X, Y), 0.0)
    px = np.where(st.q_axis == 0, st.q_xi, st.x[st.q_i])
    py = np.where(st.q_axis == 1, st.q_xi, st.x[st.q_j])
    G = gq(px, py)
    jq = np.stack([q(px, py), G[0], G[1], np.full_like(px, H[0, 0]), np.full_like(px, H[0, 1]),
                   np.full_like(px, H[1, 1])], -1)
    base = np.where(st.side[1:n, 1:n], np.trace(H) - kap * q(X, Y)[1:n, 1:n], 0.0)
    f = correction.correct2d(st, base, jq)
    lhs = fastsolve.apply_operator2d(v[1:n, 1:n], h, kap)
    assert np.abs(lhs - f).max() < 1e-9 / (h * h) * 1e-3
    # corrections only at irregular nodes
    diff = f != base
    assert np.all(st.irregular[1:n, 1:n][diff])


# ----------------------------------------------------------------- DST / Thomas / fast solver
@pytest.mark.parametrize("n", [8, 16, 64])
def test_dst_direct_sum_and_round_trip(n):
    f = np.random.default_rng(n).uniform(-1, 1, (3, n - 1))
    np.testing.assert_allclose(fastsolve.dst1(f), fastsolve.dst1_direct(f), atol=1e-12)
    np.testing.assert_allclose(fastsolve.idst1(fastsolve.dst1(f)), f, atol=1e-13)
    j = np.arange(1, n)
    fk = fastsolve.dst1(np.sin(np.pi * j * 3 / n))
    expect = np.zeros(n - 1)
    expect[2] = n / 2
    np.testing.assert_allclose(fk, expect, atol=1e-12)


def test_thomas_worked_example_and_dense():
    gold = json.load(open(os.path.join(GOLD, "thomas_tridiag.json")))
    # tridiag(−1,2,−1) u = f  ⇔  u_{i−1} − 2u_i + u_{i+1} = −f
    u = fastsolve.thomas(np.array([-2.0]), -np.array(gold["f"], float)[:, None])[:, 0]
    np.testing.assert_allclose(u, gold["u"], atol=1e-14)
    n, K = 50, 4
    dk = -np.array([2.1, 2.5, 3.0, 7.0])
    r = np.random.default_rng(0).uniform(-1, 1, (n, K))
    x = fastsolve.thomas(dk, r)
    for k in range(K):
        A = np.diag(np.full(n, dk[k])) + np.diag(np.ones(n - 1), 1) + np.diag(np.ones(n - 1), -1)
        np.testing.assert_allclose(x[:, k], np.linalg.solve(A, r[:, k]), atol=1e-13)


def test_fast_solver_eigenfunction():
    n, h, kap = 64, 2.4 / 64, 1.0
    i = np.arange(1, n)
    p, q = 5, 11
    S = np.outer(np.sin(np.pi * p * i / n), np.sin(np.pi * q * i / n))
    lam = -4 / h ** 2 * np.sin(np.pi * p / (2 * n)) ** 2 - 4 / h ** 2 * np.sin(np.pi * q / (2 * n)) ** 2 - kap
    np.testing.assert_allclose(fastsolve.solve2d(lam * S, h, kap), S, atol=1e-11)


@pytest.mark.parametrize("n,kap", [(16, 0.0), (32, 1.0)])
def test_fast_solver_dense_lu(n, kap):
    h = 2.4 / n
    m = n - 1
    T = scipy.sparse.diags([1.0, -2.0, 1.0], [-1, 0, 1], shape=(m, m))
    I = scipy.sparse.identity(m)
    A = (scipy.sparse.kron(T, I) + scipy.sparse.kron(I, T)) / h ** 2 - kap * scipy.sparse.identity(m * m)
    f = np.random.default_rng(1).uniform(-1, 1, (m, m))
    v = scipy.sparse.linalg.spsolve(A.tocsc(), f.ravel()).reshape(m, m)
    np.testing.assert_allclose(fastsolve.solve2d(f, h, kap), v, rtol=0, atol=1e-10 * np.abs(v).max())


def test_operator_symmetric_negative_definite():
    n, h = 24, 0.1
    a = np.random.default_rng(5).uniform(-1, 1, (2, n - 1, n - 1))
    Lu = fastsolve.apply_operator2d(a[0], h, 0.5)
    Lw = fastsolve.apply_operator2d(a[1], h, 0.5)
    assert abs((Lu * a[1]).sum() - (a[0] * Lw).sum()) < 1e-10 * np.abs(Lu).sum()
    assert (Lu * a[0]).sum() < 0


# ----------------------------------------------------------------- interpolation / interface solve
def test_interpolation_exact_for_quadratics():
    prob = W.C2(128)
    st = grid.build(prob)
    q, gq, H = _quad(11)
    X, Y = np.meshgrid(st.x, st.x, indexing="ij")
    out = interp.interpolate2d(st, q(X, Y), np.zeros((st.M, 6)), want_grad=True)
    np.testing.assert_allclose(out[:, 0], q(*st.z), atol=1e-12)
    np.testing.assert_allclose(out[:, 1:3].T, gq(*st.z), atol=1e-10)
    # piecewise quadratic with exact jumps at z: V⁺ = q_in(z)
    qo, go, Ho = _quad(12)
    v = np.where(st.side, q(X, Y), qo(X, Y))
    G = gq(*st.z) - go(*st.z)
    Hd = H - Ho
    jz = np.stack([q(*st.z) - qo(*st.z), G[0], G[1], np.full(st.M, Hd[0, 0]), np.full(st.M, Hd[0, 1]),
                   np.full(st.M, Hd[1, 1])], -1)
    np.testing.assert_allclose(interp.interpolate2d(st, v, jz), q(*st.z), atol=1e-11)


@pytest.mark.parametrize("prob", [W.C1(64), W.C2(128), W.C3(128)])
def test_interface_solve_reproduces_piecewise_quadratic(prob):
    """Correction → fast solve → interpolation is exact for v = q·1_Ω (any κ, any geometry)."""
    o = Oracle2D(prob)
    st = o.st
    n = st.n
    q, gq, H = _quad(21)
    px, py = o.isect_points()
    G = gq(px, py)
    jq = np.stack([q(px, py), G[0], G[1], np.full_like(px, H[0, 0]), np.full_like(px, H[0, 1]),
                   np.full_like(px, H[1, 1])], -1)
    Gz = gq(*st.z)
    jz = np.stack([q(*st.z), Gz[0], Gz[1], np.full(st.M, H[0, 0]), np.full(st.M, H[0, 1]), np.full(st.M, H[1, 1])], -1)
    base = np.where(st.side[1:n, 1:n], np.trace(H) - prob.kappa * q(o.X, o.Y)[1:n, 1:n], 0.0)
    v, vp = o.interface_solve(base, jq, jz)
    np.testing.assert_allclose(v, np.where(st.side, q(o.X, o.Y), 0.0), atol=1e-10)
    np.testing.assert_allclose(vp, q(*st.z), atol=1e-10)


def test_KD_constant_and_hole_nullspace():
    o = Oracle2D(W.C1(64))
    np.testing.assert_allclose(o.apply_KD(np.ones(o.M)), 1.0, atol=1e-12)       # K_D(1) = 1, κ = 0
    phi = W.random_density(o.M, 0)
    np.testing.assert_allclose(o.apply_KD(2 * phi + 3), 2 * o.apply_KD(phi) + 3, atol=1e-11)
    o = Oracle2D(W.C3(128))
    st = o.st
    e = np.zeros(o.M)
    e[st.comp_off[1]:st.comp_off[1] + st.comp_M[1]] = 1.0
    holes, o.holes, wg, o.w_gamma = o.holes, [], o.w_gamma, []
    assert np.abs(o.apply_KD(e)).max() < 1e-12                                      # discrete K_D(1_Γh) = 0 (R27)
    o.holes, o.w_gamma = holes, wg
    assert np.abs(o.apply_KD(e)).max() > 1e-4                                       # completion removes it


# ----------------------------------------------------------------- GMRES
def test_gmres_textbook_cases():
    b = np.random.default_rng(0).uniform(-1, 1, 20)
    x, s = gmres(lambda v: v, b)
    assert s.iters == 1 and np.allclose(x, b)
    d = np.where(np.arange(20) % 2 == 0, 1.0, 2.0)
    x, s = gmres(lambda v: d * v, b)
    assert s.iters <= 2 and np.allclose(x, b / d, atol=1e-12)
    rng = np.random.default_rng(1)
    A = np.eye(50) + 0.3 * rng.standard_normal((50, 50)) / np.sqrt(50)
    b = rng.uniform(-1, 1, 50)
    x, s = gmres(lambda v: A @ v, b, restart=10, tol=1e-12)
    assert s.converged and s.restarts > 1
    np.testing.assert_allclose(x, np.linalg.solve(A, b), atol=1e-8)


# ----------------------------------------------------------------- end-to-end
def _order(prob_fn, ns):
    errs = []
    its = []
    for n in ns:
        prob = prob_fn(n)
        o = Oracle2D(prob)
        zx, zy = o.ctrl_points()
        u, phi, s = o.solve(W.u_exact(zx, zy), lambda x, y: W.f_exact(prob.kappa, x, y))
        assert s.converged
        errs.append(o.errors(u, W.u_exact(o.X, o.Y)))
        its.append(s.iters)
    e = np.array(errs)
    return np.log2(e[:-1] / e[1:]), its


def test_second_order_ellipse():
    o, its = _order(W.C1, [64, 128, 256])
    assert np.all(o[:, 1] > 1.7) and np.all(o[:, 1] < 2.4), o     # scaled ℓ²
    assert np.all(o[:, 0] > 1.7), o                                  # max norm


def test_second_order_star_helmholtz():
    o, its = _order(W.C2, [128, 256, 512])
    assert np.all(o[:, 1] > 1.6) and np.all(o[:, 1] < 2.6), o
    assert o[:, 0].mean() > 1.7, o          # max-norm order fluctuates on the star; mean over 128→512


def test_second_order_multiply_connected():
    o, its = _order(W.C3, [128, 256])
    assert np.all(o[:, 1] > 1.6), o


def test_constant_solutions():
    prob = W.C1(64)
    o = Oracle2D(prob)
    u, phi, s = o.solve(np.ones(o.M), None)
    assert s.iters == 1
    assert np.abs(u[o.st.side] - 1).max() < 1e-12
    prob = W.problem("star-k1", 2, 128, [W.star(1.0, 0.2, 4)], 1.0)
    o = Oracle2D(prob)
    u, phi, s = o.solve(np.ones(o.M), lambda x, y: -np.ones_like(x), tol=1e-12)
    assert np.abs(u[o.st.side] - 1).max() < 1e-9
    np.testing.assert_allclose(phi, 1.0, atol=1e-9)


@pytest.mark.parametrize("m", [1, 2, 4, 8])
def test_arrowhead_partitions_equal_thomas(m):
    """ADM over m partitions reproduces the plain Thomas solution."""
    n, K = 127, 5
    dk = -np.array([2.0001, 2.05, 2.5, 3.0, 6.0])
    r = np.random.default_rng(m).uniform(-1, 1, (n, K))
    np.testing.assert_allclose(fastsolve.thomas_arrowhead(dk, r, m), fastsolve.thomas(dk, r), atol=1e-11)
    gold = json.load(open(os.path.join(GOLD, "thomas_tridiag.json")))
    u = fastsolve.thomas_arrowhead(np.array([-2.0]), -np.array(gold["f"], float)[:, None], 2)[:, 0]
    np.testing.assert_allclose(u, gold["u"], atol=1e-14)
