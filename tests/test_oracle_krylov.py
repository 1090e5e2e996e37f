"""Pins for the Richardson and BiCGSTAB drivers."""
import numpy as np

import workloads as W
from oracle.bie import Oracle2D
from oracle.krylov import bicgstab, richardson


def test_richardson_identity_one_step():
    b = np.random.default_rng(0).uniform(-1, 1, 50)
    x, st = richardson(lambda v: v, b, gamma=1.0)
    assert st.converged and st.iters == 1 and np.array_equal(x, b)


def test_richardson_diagonal_rate():
    """K = diag(λ): the error of component i shrinks by |1 − γλ_i| per step, so the iteration count
    is the smallest k with max_i |1 − γλ_i|^k |b_i/...| below tol — checked against the closed form."""
    lam = np.array([0.5, 0.8, 1.0, 1.2])
    b = np.ones(4)
    gamma = 0.9
    x, st = richardson(lambda v: lam * v, b, gamma=gamma, tol=1e-10)
    rho = np.abs(1 - gamma * lam)
    res = lambda k: np.sqrt(np.sum((rho ** k) ** 2)) / 2.0       # ‖r_k‖/‖r_0‖, r_k,i = (1−γλ_i)^k b_i
    k = next(k for k in range(1, 200) if res(k) <= 1e-10)
    assert st.converged and st.iters == k
    np.testing.assert_allclose(x, b / lam, rtol=1e-9)


def test_bicgstab_dense_systems():
    rng = np.random.default_rng(1)
    for n in (5, 40):
        A = np.eye(n) * 3 + rng.uniform(-0.5, 0.5, (n, n))        # nonsymmetric, well conditioned
        b = rng.uniform(-1, 1, n)
        x, st = bicgstab(lambda v: A @ v, b, tol=1e-12)
        assert st.converged and st.iters <= n
        np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=1e-9, atol=1e-11)
    x, st = bicgstab(lambda v: v, b, tol=1e-12)
    assert st.converged and st.iters == 1 and np.allclose(x, b)


def test_drivers_agree_on_the_bvp():
    """Richardson (γ = 1), BiCGSTAB and GMRES reach the same discrete solution (C1 ellipse)."""
    prob = W.C1(64)
    o = Oracle2D(prob)
    zx, zy = o.ctrl_points()
    f = lambda x, y: W.f_exact(prob.kappa, x, y)
    g = W.u_exact(zx, zy)
    u0, p0, s0 = o.solve(g, f, tol=1e-12)
    for method in ("richardson", "bicgstab"):
        u, p, s = o.solve(g, f, tol=1e-12, method=method)
        assert s.converged
        m = o.st.side
        assert np.abs(u[m] - u0[m]).max() < 1e-9 * np.abs(u0[m]).max()
        assert np.abs(p - p0).max() < 1e-9 * np.abs(p0).max()
