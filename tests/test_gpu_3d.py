"""GPU parity of the 3D CUDA path (C4 ellipsoid, C5 torus) against the 3D oracle, via the C ABI."""
import numpy as np
import pytest
import torch

import workloads as W
from oracle import fastsolve
from oracle.bie3d import Oracle3D
from paper_2404_15249_b200 import KFBI

pytestmark = pytest.mark.gpu

_OR, _GPU = {}, {}


def oracle(prob):
    if prob not in _OR:
        _OR[prob] = Oracle3D(prob)
    return _OR[prob]


def gpu(prob):
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback exists)"
    if prob not in _GPU:
        _GPU[prob] = KFBI(prob)
    return _GPU[prob]


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _quad3(seed):
    a = np.random.default_rng(seed).uniform(-1, 1, 10)
    H = np.array([[2 * a[4], a[7], a[8]], [a[7], 2 * a[5], a[9]], [a[8], a[9], 2 * a[6]]])
    q = lambda x, y, z: (a[0] + a[1] * x + a[2] * y + a[3] * z + a[4] * x * x + a[5] * y * y + a[6] * z * z
                         + a[7] * x * y + a[8] * x * z + a[9] * y * z)
    g = lambda x, y, z: np.stack([a[1] + 2 * a[4] * x + a[7] * y + a[8] * z, a[2] + 2 * a[5] * y + a[7] * x + a[9] * z,
                                  a[3] + 2 * a[6] * z + a[8] * x + a[9] * y], -1)
    return q, g, H


def _grid(prob):
    x = prob.lo + np.arange(prob.n + 1) * prob.h
    return np.meshgrid(x, x, x, indexing="ij")


@pytest.mark.parametrize("prob", [W.C4(64), W.C5(64)], ids=["ellipsoid64", "torus64"])
def test_fast_solve3d_matches_oracle(prob):
    k = gpu(prob)
    n = prob.n
    mask = k.node_mask().astype(bool)
    rhs = np.where(mask, np.random.default_rng(3).uniform(-1, 1, mask.shape), 0.0)
    v = k.test_fast_solve(rhs).cpu().numpy()
    ref = fastsolve.solve3d(rhs[1:n, 1:n, 1:n], prob.h, prob.kappa)
    assert rel(v[1:n, 1:n, 1:n], ref) < 1e-11
    assert np.all(v[0] == 0) and np.all(v[:, -1] == 0) and np.all(v[:, :, 0] == 0)


@pytest.mark.parametrize("prob", [W.C4(64), W.C5(64), W.C4(128)], ids=["ellipsoid64", "torus64", "ellipsoid128"])
def test_interface_solve3d_piecewise_quadratic(prob):
    k = gpu(prob)
    q, gq, H = _quad3(8)
    X, Y, Z = _grid(prob)
    mask = k.node_mask().astype(bool)
    p = k.points("ctrl")
    G = gq(*p.T)
    jq = np.concatenate([q(*p.T)[:, None], G,
                         np.tile([H[0, 0], H[1, 1], H[2, 2], H[0, 1], H[0, 2], H[1, 2]], (k.M, 1))], -1)
    base = np.where(mask, np.trace(H) - prob.kappa * q(X, Y, Z), 0.0)
    v, vp = k.test_interface_solve(base, jq, jq)
    assert np.abs(v.cpu().numpy() - np.where(mask, q(X, Y, Z), 0.0)).max() < 1e-10
    assert np.abs(vp.cpu().numpy() - q(*p.T)).max() < 1e-10


@pytest.mark.parametrize("prob", [W.C4(64), W.C5(64), W.C4(128)], ids=["ellipsoid64", "torus64", "ellipsoid128"])
@pytest.mark.parametrize("seed", [0, 1])
def test_apply3d_matches_oracle(prob, seed):
    o, k = oracle(prob), gpu(prob)
    phi = W.random_density(o.M, seed)
    assert rel(k.apply(phi).cpu().numpy(), o.apply_KD(phi)) < 1e-10


def test_apply3d_constant_density():
    k = gpu(W.C4(64))
    np.testing.assert_allclose(k.apply(np.ones(k.M)).cpu().numpy(), 1.0, atol=1e-12)   # K_D(1) = 1, κ = 0


@pytest.mark.parametrize("prob", [W.C4(64), W.C5(64)], ids=["ellipsoid64", "torus64"])
def test_solve3d_matches_oracle(prob):
    o, k = oracle(prob), gpu(prob)
    f = lambda a, b, c: W.f_exact(prob.kappa, a, b, c)
    u_ref, phi_ref, s_ref = o.solve(W.u_exact(*o.points().T), f)
    X, Y, Z = _grid(prob)
    p = k.points("ctrl")
    u, phi, s = k.solve(W.u_exact(*p.T), f(X, Y, Z), f(*p.T), f(*p.T))
    u = u.cpu().numpy()
    m = o.st.side
    assert s.converged and abs(s.iters - s_ref.iters) <= 1
    assert rel(u[m], u_ref[m]) < 1e-8
    assert rel(phi.cpu().numpy(), phi_ref) < 1e-8


def test_restarted_solve3d_matches_oracle():
    """3D GMRES(m) with m shorter than the iteration count (one-step-ahead Arnoldi enqueue across cycle
    boundaries): C4 64³ with m = 6 against the oracle's GMRES(6)."""
    prob = W.C4(64)
    o, k = oracle(prob), gpu(prob)
    f = lambda a, b, c: W.f_exact(prob.kappa, a, b, c)
    u_ref, phi_ref, s_ref = o.solve(W.u_exact(*o.points().T), f, restart=6)
    X, Y, Z = _grid(prob)
    p = k.points("ctrl")
    u, phi, s = k.solve(W.u_exact(*p.T), f(X, Y, Z), f(*p.T), f(*p.T), restart=6)
    m = o.st.side
    print(f"C4 GMRES(6): {s.iters} iterations, {s.restarts} cycles (oracle {s_ref.iters}, {s_ref.restarts})")
    assert s.converged and s.restarts > 1 and abs(s.iters - s_ref.iters) <= 1
    assert rel(u.cpu().numpy()[m], u_ref[m]) < 1e-8
    assert rel(phi.cpu().numpy(), phi_ref) < 1e-8


@pytest.mark.slow
def test_interface_solve3d_full_size_C5():
    """Full-size C5 (512³): the piecewise-quadratic witness holds at any size."""
    test_interface_solve3d_piecewise_quadratic(W.C5(512))


@pytest.mark.slow
def test_apply3d_full_size_C5():
    """The K_D apply that bench.py --config C5 times (512³: k_fwd3s<512>, k_sweep3, k_reduced3,
    k_inv3y<512>, k_zeval3<512>) against the oracle's plain Alg. 4 path, seeds 0 and 1."""
    prob = W.C5(512)
    o, k = oracle(prob), gpu(prob)
    for seed in (0, 1):
        phi = W.random_density(o.M, seed)
        assert rel(k.apply(phi).cpu().numpy(), o.apply_KD(phi)) < 1e-10
    _OR.pop(prob, None)
    _GPU.pop(prob, None)


@pytest.mark.slow
def test_solve3d_C5_256():
    """C5 geometry (torus, κ = 1) solved at 256³ against the oracle's GMRES."""
    prob = W.C5(256)
    test_solve3d_matches_oracle(prob)
    _OR.pop(prob, None)
    _GPU.pop(prob, None)


# ------------------------------------------------------------------ multi-GPU partition (emulated)
@pytest.mark.parametrize("prob,world", [(W.C4(64), 2), (W.C4(64), 4), (W.C5(128), 8), (W.C5(128), 2), (W.C5(256), 4)],
                         ids=["C4-64x2", "C4-64x4", "C5-128x8", "C5-128x2", "C5-256x4"])
def test_partitioned_apply3d_matches_single(prob, world):
    """All slabs in one context (rank = −1): block sweeps per slab, the level-2 split of the reduced
    system (slab interior separators eliminated locally, L3 = P/world − 1 = 1, 0, 0, 3, 3 here; the
    world − 1 slab separators solved mode-partitioned, each owner reading the slabs' rows of its K/world
    modes as the all-to-all delivers them) and the disjoint partial interpolation sums reproduce
    world = 1 (to summation order) and the oracle."""
    k1 = gpu(prob)
    kw = KFBI(prob, world=world, rank=-1)
    for seed in (0, 1):
        phi = W.random_density(k1.M, seed)
        assert rel(kw.apply(phi).cpu().numpy(), k1.apply(phi).cpu().numpy()) < 1e-12
    if prob.n == 64:
        o = oracle(prob)
        phi = W.random_density(o.M, 2)
        assert rel(kw.apply(phi).cpu().numpy(), o.apply_KD(phi)) < 1e-10


@pytest.mark.parametrize("world", [2, 4])
def test_partitioned_solve3d_matches_oracle(world):
    """The whole solve with every stage sharded by slab: the LSQ fits, corrections and point work of
    each slab, the dense Y apply and final field of its planes, the level-2 reduced system."""
    prob = W.C4(64)
    o = oracle(prob)
    kw = KFBI(prob, world=world, rank=-1)
    f = lambda a, b, c: W.f_exact(prob.kappa, a, b, c)
    u_ref, phi_ref, s_ref = o.solve(W.u_exact(*o.points().T), f)
    X, Y, Z = _grid(prob)
    p = kw.points("ctrl")
    u, phi, s = kw.solve(W.u_exact(*p.T), f(X, Y, Z), f(*p.T), f(*p.T))
    m = o.st.side
    assert s.converged and abs(s.iters - s_ref.iters) <= 1
    assert rel(u.cpu().numpy()[m], u_ref[m]) < 1e-8


# ------------------------------------------------------------------ Neumann BVP (NEXT-1, R38)
NEU3 = W.neumann(W.problem("ellipsoid-k1", 3, 64, [W.ellipsoid(0.7, 0.6, 0.5)], 1.0))


@pytest.mark.parametrize("seed", [0, 1])
def test_apply3d_neumann_matches_oracle(seed):
    o, k = oracle(NEU3), gpu(NEU3)
    psi = W.random_density(o.M, seed)
    assert rel(k.apply(psi).cpu().numpy(), o.apply_KN(psi)) < 1e-10


def test_solve3d_neumann_matches_oracle():
    o, k = oracle(NEU3), gpu(NEU3)
    f = lambda a, b, c: W.f_exact(NEU3.kappa, a, b, c)
    p = o.points()
    u_ref, psi_ref, s_ref = o.solve(np.sum(np.stack(W.grad_u_exact(*p.T), -1) * o.st.nrm, -1), f)
    X, Y, Z = _grid(NEU3)
    pk, nk = k.points("ctrl"), k.points("normal")
    gN = np.sum(np.stack(W.grad_u_exact(*pk.T), -1) * nk, -1)
    u, psi, s = k.solve(gN, f(X, Y, Z), f(*pk.T), f(*pk.T))
    m = o.st.side
    assert s.converged and abs(s.iters - s_ref.iters) <= 1
    assert rel(u.cpu().numpy()[m], u_ref[m]) < 1e-8
    assert rel(psi.cpu().numpy(), psi_ref) < 1e-8
