"""Pins for the Gray–Scott oracle (readings R40, R41)."""
import numpy as np

import workloads as W
from oracle.grayscott import GrayScott, bilinear, rates, reaction


def test_reaction_equilibrium_and_midpoint_order():
    u, v = np.ones(5), np.zeros(5)
    u1, v1 = reaction(u, v, 0.125)
    assert np.array_equal(u1, u) and np.array_equal(v1, v)          # (1, 0) is a fixed point
    # one node against RK4 with tiny steps: the midpoint rule's local error is O(dt³)
    def rk4(u, v, t, n=2000):
        h = t / n
        for _ in range(n):
            a = rates(u, v)
            b = rates(u + 0.5 * h * a[0], v + 0.5 * h * a[1])
            c = rates(u + 0.5 * h * b[0], v + 0.5 * h * b[1])
            d = rates(u + h * c[0], v + h * c[1])
            u, v = u + h / 6 * (a[0] + 2 * b[0] + 2 * c[0] + d[0]), v + h / 6 * (a[1] + 2 * b[1] + 2 * c[1] + d[1])
        return u, v
    errs = []
    for dt in (2e-3, 1e-3):
        um, vm = reaction(np.array([0.5]), np.array([0.25]), dt)
        ur, vr = rk4(np.array([0.5]), np.array([0.25]), dt)
        errs.append(max(abs(um - ur)[0], abs(vm - vr)[0]))
    assert errs[1] < 1e-8 and 6 < errs[0] / errs[1] < 10          # ≈ 8 = 2³


def test_bilinear_exact_for_bilinear_fields():
    lo, h, n = -2.0, 0.0625, 64
    x = lo + np.arange(n + 1) * h
    X, Y = np.meshgrid(x, x, indexing="ij")
    f = lambda x, y: 0.3 + 1.1 * x - 0.7 * y + 0.25 * x * y
    px, py = np.random.default_rng(0).uniform(-1.9, 1.9, (2, 50))
    np.testing.assert_allclose(bilinear(f(X, Y), lo, h, px, py), f(px, py), atol=1e-13)


def test_gray_scott_step_bounded_and_equilibrium_converges():
    g = GrayScott(64, 0.125)
    m = g.ou.st.side
    for _ in range(2):
        g.step()
    assert np.all(np.isfinite(g.u)) and np.all(np.isfinite(g.v))
    assert -0.05 <= g.u[m].min() and g.u[m].max() <= 1.3 and -0.05 <= g.v[m].min() and g.v[m].max() <= 1.0
    # the homogeneous state (1, 0): one step drifts by the diffusion solve's discretisation error, which
    # decreases under refinement (κ_cn h² ≫ 1 here: the Neumann boundary layer is under-resolved)
    drift = []
    for n in (64, 128):
        g = GrayScott(n, 0.125)
        g.u[:] = 1.0
        g.v[:] = 0.0
        g.step()
        drift.append(np.abs(g.u[g.ou.st.side] - 1.0).max())
        assert np.abs(g.v).max() == 0.0
    assert drift[1] < drift[0]
