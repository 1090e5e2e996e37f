"""GPU parity of the CUDA path (through the C ABI) against the CPU oracle, same seeded inputs.

Bars (BASELINE.json north_star): fast solve ≤ 1e-12 relative max-norm,
kfbi_apply ≤ 1e-10, final solution ≤ 1e-8 with GMRES iteration counts within ±1.
"""
import numpy as np
import pytest
import torch

import workloads as W
from oracle import fastsolve
from oracle.bie import Oracle2D
from paper_2404_15249_b200 import KFBI

pytestmark = pytest.mark.gpu

_OR, _GPU = {}, {}


def oracle(prob):
    if prob not in _OR:
        _OR[prob] = Oracle2D(prob)
    return _OR[prob]


def gpu(prob):
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback exists)"
    if prob not in _GPU:
        _GPU[prob] = KFBI(prob)
    return _GPU[prob]


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _quad(seed):
    a = np.random.default_rng(seed).uniform(-1, 1, 6)
    q = lambda x, y: a[0] + a[1] * x + a[2] * y + a[3] * x * x + a[4] * x * y + a[5] * y * y
    gq = lambda x, y: np.stack([a[1] + 2 * a[3] * x + a[4] * y, a[2] + a[4] * x + 2 * a[5] * y])
    H = np.array([[2 * a[3], a[4]], [a[4], 2 * a[5]]])
    return q, gq, H


# ------------------------------------------------------------------ fast solver (Alg. 4)
@pytest.mark.parametrize("n,kappa", [(64, 0.0), (1024, 1.0), (2048, 0.0)])
def test_fast_solve_matches_oracle(n, kappa):
    prob = W.problem(f"box{n}", 2, n, [W.ellipse(1.0, 0.8)], kappa)
    k = gpu(prob)
    rhs = np.random.default_rng(n).uniform(-1, 1, (n + 1, n + 1))
    v = k.test_fast_solve(rhs).cpu().numpy()
    ref = fastsolve.solve2d(rhs[1:n, 1:n], prob.h, kappa)
    # backward error: the GPU field solves the 5-point system to rounding — within a
    # small factor of the residual of the oracle's own FP64 solution (scipy DST-I + Thomas)
    res = fastsolve.apply_operator2d(v[1:n, 1:n], prob.h, kappa) - rhs[1:n, 1:n]
    res_oracle = fastsolve.apply_operator2d(ref, prob.h, kappa) - rhs[1:n, 1:n]
    print(f"N={n} κ={kappa}: forward rel gap {rel(v[1:n, 1:n], ref):.2e}, residual GPU {np.abs(res).max():.2e}"
          f" oracle {np.abs(res_oracle).max():.2e}")
    assert np.abs(res).max() < 4 * np.abs(res_oracle).max() + 1e-14 * np.abs(rhs).max()
    # forward difference vs the oracle's plain Thomas: bounded by cond(L_h)·ε, cond ≈ (2N/π)²
    # for the κ = 0 low modes
    assert rel(v[1:n, 1:n], ref) < 1e-11
    assert np.all(v[0] == 0) and np.all(v[:, -1] == 0)


@pytest.mark.parametrize("p,q", [(1234, 3001), (3, 4001)])
def test_fast_solve_eigenfunction_full_size(p, q):
    """A discrete eigenfunction sin(πpi/N) sin(πqj/N) of Δ_h is reproduced at N = 8192.  For a
    stiff pair (one index near N/2, the other tiny) the forward transform's rounding leaks
    ε·|f̂| into the low modes, which (Δ_h)⁻¹ amplifies by ~N²: there the bound is the FP64
    error of the same algorithm on the CPU oracle (scipy DST-I + Thomas), not a fixed 1e-10."""
    n = 8192
    prob = W.problem("box8192", 2, n, [W.ellipse(1.0, 0.8)], 0.0)
    k = gpu(prob)
    h = prob.h
    i = np.arange(n + 1)
    S = np.outer(np.sin(np.pi * p * i / n), np.sin(np.pi * q * i / n))
    lam = -4 / h ** 2 * (np.sin(np.pi * p / (2 * n)) ** 2 + np.sin(np.pi * q / (2 * n)) ** 2)
    v = k.test_fast_solve(lam * S).cpu().numpy()
    err = np.abs(v - S).max()
    print(f"eigenfunction ({p}, {q}) at N = 8192: max error {err:.2e}")
    if min(p, q) > 100:
        assert err < 1e-10
    else:
        ref = fastsolve.solve2d((lam * S)[1:n, 1:n], h, 0.0)
        err_oracle = np.abs(ref - S[1:n, 1:n]).max()
        assert err < 8 * err_oracle + 1e-13, (err, err_oracle)


# ------------------------------------------------------------------ interface solve witness
@pytest.mark.parametrize("prob", [W.C1(64), W.C2(1024), W.C3(2048)], ids=lambda p: p.name + str(p.n))
def test_interface_solve_piecewise_quadratic(prob):
    """v = q·1_Ω with exact jumps is reproduced at every node and at V⁺(z) = q(z)."""
    k = gpu(prob)
    n = prob.n
    q, gq, H = _quad(5)
    x = prob.lo + np.arange(n + 1) * prob.h
    X, Y = np.meshgrid(x, x, indexing="ij")
    mask = k.node_mask().astype(bool)
    pq = k.points("isect")
    pz = k.points("ctrl")
    Gq, Gz = gq(pq[:, 0], pq[:, 1]), gq(pz[:, 0], pz[:, 1])
    jq = np.stack([q(pq[:, 0], pq[:, 1]), Gq[0], Gq[1], np.full(k.nq, H[0, 0]), np.full(k.nq, H[0, 1]),
                   np.full(k.nq, H[1, 1])], -1)
    jz = np.stack([q(pz[:, 0], pz[:, 1]), Gz[0], Gz[1], np.full(k.M, H[0, 0]), np.full(k.M, H[0, 1]),
                   np.full(k.M, H[1, 1])], -1)
    base = np.where(mask, np.trace(H) - prob.kappa * q(X, Y), 0.0)
    v, vp = k.test_interface_solve(base, jq, jz)
    assert np.abs(v.cpu().numpy() - np.where(mask, q(X, Y), 0.0)).max() < 1e-10
    assert np.abs(vp.cpu().numpy() - q(pz[:, 0], pz[:, 1])).max() < 1e-10


# ------------------------------------------------------------------ K_D apply
DENS = ["seed0", "seed1", "seed2", "smooth"]


def density(prob, o, name):
    if name == "smooth":
        return W.smooth_density(o.st.comp_M)
    return W.random_density(o.M, int(name[-1]))


@pytest.mark.parametrize("prob", [W.C1(64), W.C2(1024), W.C3(1024)], ids=lambda p: p.name + str(p.n))
@pytest.mark.parametrize("dens", DENS)
def test_apply_matches_oracle(prob, dens):
    o, k = oracle(prob), gpu(prob)
    phi = density(prob, o, dens)
    out = k.apply(phi).cpu().numpy()
    ref = o.apply_KD(phi)
    assert rel(out, ref) < 1e-10


def test_apply_constant_density():
    k = gpu(W.C1(64))
    out = k.apply(np.ones(k.M)).cpu().numpy()
    assert np.abs(out - 1).max() < 1e-12          # K_D(1) = 1 at κ = 0 (R17)


def test_apply_deterministic():
    prob = W.C2(1024)
    k = gpu(prob)
    phi = torch.tensor(W.random_density(k.M, 7), device="cuda")
    a = k.apply(phi).clone()
    b = k.apply(phi).clone()
    assert torch.equal(a, b)


@pytest.mark.slow
def test_apply_full_size_C3():
    prob = W.C3(8192)
    o, k = oracle(prob), gpu(prob)
    phi = W.random_density(o.M, 0)
    assert rel(k.apply(phi).cpu().numpy(), o.apply_KD(phi)) < 1e-10


@pytest.mark.slow
def test_apply_full_size_C2_split_columns():
    """The star at N = 8192 puts > 512 stencil rows in one grid column where Γ runs along it:
    those columns are split into several k_inv_sparse work items (setup2d.cpp)."""
    prob = W.C2(8192)
    o, k = oracle(prob), gpu(prob)
    phi = W.random_density(o.M, 1)
    assert rel(k.apply(phi).cpu().numpy(), o.apply_KD(phi)) < 1e-10


# ------------------------------------------------------------------ full solve
@pytest.mark.parametrize("prob", [W.C1(64), W.C2(1024), W.C3(1024)], ids=lambda p: p.name + str(p.n))
def test_solve_matches_oracle(prob):
    o, k = oracle(prob), gpu(prob)
    n = prob.n
    f = lambda x, y: W.f_exact(prob.kappa, x, y)
    zx, zy = o.ctrl_points()
    u_ref, phi_ref, s_ref = o.solve(W.u_exact(zx, zy), f)
    pz, pq = k.points("ctrl"), k.points("isect")
    x = prob.lo + np.arange(n + 1) * prob.h
    X, Y = np.meshgrid(x, x, indexing="ij")
    u, phi, s = k.solve(W.u_exact(pz[:, 0], pz[:, 1]), f(X, Y), f(pq[:, 0], pq[:, 1]), f(pz[:, 0], pz[:, 1]))
    u = u.cpu().numpy()
    m = o.st.side
    assert s.converged and abs(s.iters - s_ref.iters) <= 1
    assert rel(u[m], u_ref[m]) < 1e-8
    assert rel(phi.cpu().numpy(), phi_ref) < 1e-8
    # and the solution is the manufactured one to discretisation accuracy
    assert np.abs(u[m] - W.u_exact(X, Y)[m]).max() < 50 * prob.h ** 2


@pytest.mark.parametrize("prob,restart", [(W.C1(64), 4), (W.C2(512), 5)], ids=["C1-r4", "C2-r5"])
def test_restarted_solve_matches_oracle(prob, restart):
    """GMRES(m) with restarts shorter than the iteration count (Alg. 5): the host's one-step-
    ahead enqueue of Arnoldi steps crosses cycle boundaries and convergence inside a cycle; the solve
    matches the oracle's GMRES(m) to 1e-8 with the iteration and restart counts within ±1."""
    o, k = oracle(prob), gpu(prob)
    n = prob.n
    f = lambda x, y: W.f_exact(prob.kappa, x, y)
    zx, zy = o.ctrl_points()
    u_ref, phi_ref, s_ref = o.solve(W.u_exact(zx, zy), f, restart=restart)
    pz, pq = k.points("ctrl"), k.points("isect")
    x = prob.lo + np.arange(n + 1) * prob.h
    X, Y = np.meshgrid(x, x, indexing="ij")
    u, phi, s = k.solve(W.u_exact(pz[:, 0], pz[:, 1]), f(X, Y), f(pq[:, 0], pq[:, 1]), f(pz[:, 0], pz[:, 1]),
                        restart=restart)
    print(f"{prob.name} GMRES({restart}): {s.iters} iterations, {s.restarts} cycles (oracle {s_ref.iters}, "
          f"{s_ref.restarts})")
    assert s.converged and s.restarts > 1 and abs(s.iters - s_ref.iters) <= 1
    assert rel(u.cpu().numpy()[o.st.side], u_ref[o.st.side]) < 1e-8
    assert rel(phi.cpu().numpy(), phi_ref) < 1e-8


@pytest.mark.slow
def test_solve_full_size_C3():
    """The bench workload itself: C3 8192² (κ = 0, two holes, hole completion R27) solved by
    kfbi_solve against the oracle's Alg. 5 GMRES on the same inputs — world-1 in-place bump axpy into
    the final spectrum and the k_dst_dense2<·, 8192> final field included."""
    prob = W.C3(8192)
    o, k = oracle(prob), gpu(prob)
    n = prob.n
    f = lambda x, y: W.f_exact(prob.kappa, x, y)
    zx, zy = o.ctrl_points()
    u_ref, phi_ref, s_ref = o.solve(W.u_exact(zx, zy), f)
    pz, pq = k.points("ctrl"), k.points("isect")
    x = prob.lo + np.arange(n + 1) * prob.h
    X, Y = np.meshgrid(x, x, indexing="ij")
    fg = f(X, Y)
    del X, Y
    u, phi, s = k.solve(W.u_exact(pz[:, 0], pz[:, 1]), fg, f(pq[:, 0], pq[:, 1]), f(pz[:, 0], pz[:, 1]))
    u = u.cpu().numpy()
    m = o.st.side
    assert s.converged and abs(s.iters - s_ref.iters) <= 1, (s.iters, s_ref.iters)
    assert rel(u[m], u_ref[m]) < 1e-8
    assert rel(phi.cpu().numpy(), phi_ref) < 1e-8
    _OR.pop(prob, None)
    _GPU.pop(prob, None)


def test_solve_second_order_on_gpu():
    errs = []
    for n in (256, 512, 1024, 2048):
        prob = W.C2(n)
        k = gpu(prob)
        pz, pq = k.points("ctrl"), k.points("isect")
        x = prob.lo + np.arange(n + 1) * prob.h
        X, Y = np.meshgrid(x, x, indexing="ij")
        f = lambda a, b: W.f_exact(prob.kappa, a, b)
        u, phi, s = k.solve(W.u_exact(pz[:, 0], pz[:, 1]), f(X, Y), f(pq[:, 0], pq[:, 1]), f(pz[:, 0], pz[:, 1]))
        m = k.node_mask().astype(bool)
        e = u.cpu().numpy()[m] - W.u_exact(X, Y)[m]
        errs.append(np.sqrt(np.mean(e * e)))
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(orders > 1.6) and np.all(orders < 2.6), orders


# ------------------------------------------------------------------ multi-GPU partition (emulated)
@pytest.mark.parametrize("n,world", [(2048, 2), (2048, 4), (4096, 8)])
def test_partitioned_apply_matches_single(n, world):
    """All `world` slabs in one context (rank = −1): the arrowhead split across slabs, the level-2
    slab-separator solve and the disjoint partial interpolation sums reproduce world = 1."""
    prob = W.C3(n)
    k1 = gpu(prob)
    kw = KFBI(prob, world=world, rank=-1)
    for seed in (0, 1):
        phi = W.random_density(k1.M, seed)
        a = k1.apply(phi).cpu().numpy()
        b = kw.apply(phi).cpu().numpy()
        assert rel(b, a) < 1e-12
    if n == 2048:
        o = oracle(prob)
        phi = W.random_density(o.M, 2)
        assert rel(kw.apply(phi).cpu().numpy(), o.apply_KD(phi)) < 1e-10


def test_partitioned_solve_matches_oracle():
    prob = W.C3(2048)
    o = oracle(prob)
    kw = KFBI(prob, world=4, rank=-1)
    n = prob.n
    f = lambda x, y: W.f_exact(prob.kappa, x, y)
    zx, zy = o.ctrl_points()
    u_ref, phi_ref, s_ref = o.solve(W.u_exact(zx, zy), f)
    pz, pq = kw.points("ctrl"), kw.points("isect")
    x = prob.lo + np.arange(n + 1) * prob.h
    X, Y = np.meshgrid(x, x, indexing="ij")
    u, phi, s = kw.solve(W.u_exact(pz[:, 0], pz[:, 1]), f(X, Y), f(pq[:, 0], pq[:, 1]), f(pz[:, 0], pz[:, 1]))
    m = o.st.side
    assert s.converged and abs(s.iters - s_ref.iters) <= 1
    assert rel(u.cpu().numpy()[m], u_ref[m]) < 1e-8


# ------------------------------------------------------------------ Neumann BVP (NEXT-1, R38)
NEU = [W.neumann(W.C2(1024)), W.neumann(W.problem("ellipse-k1", 2, 256, [W.ellipse(1.0, 0.8)], 1.0))]


@pytest.mark.parametrize("prob", NEU, ids=lambda p: p.name + str(p.n))
@pytest.mark.parametrize("dens", DENS)
def test_apply_neumann_matches_oracle(prob, dens):
    """K_N ψ = ∂_n V⁺ ([v] = 0, [∂_n v] = ψ) against the oracle."""
    o, k = oracle(prob), gpu(prob)
    psi = density(prob, o, dens)
    assert rel(k.apply(psi).cpu().numpy(), o.apply_KN(psi)) < 1e-10


def _ellipse_normal(x, y, a=1.0, b=0.8):
    gx, gy = x / a ** 2, y / b ** 2
    r = np.hypot(gx, gy)
    return gx / r, gy / r


def test_solve_neumann_matches_oracle():
    prob = NEU[1]
    o, k = oracle(prob), gpu(prob)
    n = prob.n
    f = lambda x, y: W.f_exact(prob.kappa, x, y)
    gN = lambda x, y: sum(g * m for g, m in zip(W.grad_u_exact(x, y), _ellipse_normal(x, y)))
    zx, zy = o.ctrl_points()
    u_ref, psi_ref, s_ref = o.solve(gN(zx, zy), f)
    pz, pq = k.points("ctrl"), k.points("isect")
    x = prob.lo + np.arange(n + 1) * prob.h
    X, Y = np.meshgrid(x, x, indexing="ij")
    u, psi, s = k.solve(gN(pz[:, 0], pz[:, 1]), f(X, Y), f(pq[:, 0], pq[:, 1]), f(pz[:, 0], pz[:, 1]))
    u = u.cpu().numpy()
    m = o.st.side
    assert s.converged and abs(s.iters - s_ref.iters) <= 1
    assert rel(u[m], u_ref[m]) < 1e-8
    assert rel(psi.cpu().numpy(), psi_ref) < 1e-8
    assert np.abs(u[m] - W.u_exact(X, Y)[m]).max() < 5e-3


# ------------------------------------------------------------------ Richardson / BiCGSTAB (NEXT-4)
@pytest.mark.parametrize("method", ["richardson", "bicgstab"])
@pytest.mark.parametrize("prob", [W.C1(64), W.C2(1024), NEU[1]], ids=lambda p: p.name + str(p.n))
def test_solve_drivers_match_oracle(prob, method):
    o, k = oracle(prob), gpu(prob)
    n = prob.n
    f = lambda x, y: W.f_exact(prob.kappa, x, y)
    if prob.bc == W.NEUMANN:
        g = lambda x, y: sum(a * b for a, b in zip(W.grad_u_exact(x, y), _ellipse_normal(x, y)))
    else:
        g = W.u_exact
    zx, zy = o.ctrl_points()
    u_ref, phi_ref, s_ref = o.solve(g(zx, zy), f, method=method)
    pz, pq = k.points("ctrl"), k.points("isect")
    x = prob.lo + np.arange(n + 1) * prob.h
    X, Y = np.meshgrid(x, x, indexing="ij")
    u, phi, s = k.solve(g(pz[:, 0], pz[:, 1]), f(X, Y), f(pq[:, 0], pq[:, 1]), f(pz[:, 0], pz[:, 1]), method=method)
    m = o.st.side
    assert s.converged and s_ref.converged and abs(s.iters - s_ref.iters) <= 1
    assert rel(u.cpu().numpy()[m], u_ref[m]) < 1e-8
    assert rel(phi.cpu().numpy(), phi_ref) < 1e-8
