"""Edge and degenerate cases of the public API on the GPU (2D and 3D)."""
import numpy as np
import pytest
import torch

import workloads as W
from oracle.bie import Oracle2D
from paper_2404_15249_b200 import KFBI, KfbiError

pytestmark = pytest.mark.gpu

_K = {}


def gpu(prob):
    assert torch.cuda.is_available()
    if prob not in _K:
        _K[prob] = KFBI(prob)
    return _K[prob]


@pytest.mark.parametrize("prob", [W.C1(64), W.C3(1024), W.C4(32), W.neumann(W.C2(256))], ids=lambda p: p.name)
def test_zero_density_gives_zero(prob):
    k = gpu(prob)
    out = k.apply(np.zeros(k.M)).cpu().numpy()
    assert np.array_equal(out, np.zeros(k.M))


def test_solve_without_volume_source_matches_oracle():
    """f ≡ 0 (d_f_grid = NULL): ĝ = g, no Y apply; the final field is Wφ alone."""
    prob = W.C1(64)
    k, o = gpu(prob), Oracle2D(prob)
    zx, zy = o.ctrl_points()
    g = np.exp(zx) * np.cos(zy)            # harmonic: u = eˣ cos y solves Δu = 0
    u_ref, phi_ref, s_ref = o.solve(g)
    pz = k.points("ctrl")
    u, phi, s = k.solve(np.exp(pz[:, 0]) * np.cos(pz[:, 1]))
    m = o.st.side
    assert s.converged and abs(s.iters - s_ref.iters) <= 1
    assert np.abs(u.cpu().numpy()[m] - u_ref[m]).max() < 1e-8 * np.abs(u_ref[m]).max()


def test_warm_start_reaches_the_same_solution():
    """x₀ = φ₀ ≠ 0: the explicit first residual ĝ − Kφ₀ (R18; the tolerance is relative to it, so a
    start at the converged density itself would ask for an unreachable further 1e-12 reduction)."""
    prob = W.C2(256)
    k = gpu(prob)
    pz, pq = k.points("ctrl"), k.points("isect")
    x = prob.lo + np.arange(prob.n + 1) * prob.h
    X, Y = np.meshgrid(x, x, indexing="ij")
    f = lambda a, b: W.f_exact(prob.kappa, a, b)
    args = (W.u_exact(pz[:, 0], pz[:, 1]), f(X, Y), f(pq[:, 0], pq[:, 1]), f(pz[:, 0], pz[:, 1]))
    u0, phi0, s0 = k.solve(*args, tol=1e-12)
    u1, phi1, s1 = k.solve(*args, tol=1e-12, phi0=0.9 * phi0)
    assert s1.converged and s1.iters <= s0.iters + 1
    assert torch.allclose(u1, u0, rtol=0, atol=1e-9 * float(u0.abs().max()))
    assert torch.allclose(phi1, phi0, rtol=0, atol=1e-9 * float(phi0.abs().max()))


def test_nonconvergence_is_reported_with_stats():
    prob = W.C2(256)
    k = gpu(prob)
    pz = k.points("ctrl")
    g = W.u_exact(pz[:, 0], pz[:, 1])
    with pytest.raises(KfbiError) as e:
        k.solve(g, tol=1e-15, restart=2, max_restarts=1)
    assert e.value.code == 3                                     # KFBI_ENOCONV
    u, phi, s = k.solve(g, tol=1e-15, restart=2, max_restarts=1, raise_on_noconv=False)
    assert not s.converged and s.iters == 2 and np.isfinite(s.rel_residual)


@pytest.mark.parametrize("opts", [dict(restart=0), dict(restart=1000), dict(tol=0.0), dict(method="richardson", gamma=1.5)])
def test_bad_solve_options(opts):
    k = gpu(W.C1(64))
    pz = k.points("ctrl")
    with pytest.raises(KfbiError) as e:
        k.solve(W.u_exact(pz[:, 0], pz[:, 1]), **opts)
    assert e.value.code == 1                                     # KFBI_EINVAL


def test_nonfinite_input_is_a_breakdown():
    """A NaN in g makes the first residual non-finite: KFBI_EBREAKDOWN, not EINVAL."""
    k = gpu(W.C1(64))
    g = W.u_exact(*k.points("ctrl").T)
    g[3] = np.nan
    with pytest.raises(KfbiError) as e:
        k.solve(g)
    assert e.value.code == 8                                     # KFBI_EBREAKDOWN


def test_output_buffers_are_validated():
    k = gpu(W.C1(64))
    phi = np.zeros(k.M)
    for bad in (torch.empty(k.M, dtype=torch.float32, device="cuda"), torch.empty(k.M + 1, dtype=torch.float64,
                device="cuda"), torch.empty(2 * k.M, dtype=torch.float64, device="cuda")[::2]):
        with pytest.raises(ValueError):
            k.apply(phi, out=bad)
    with pytest.raises(ValueError):
        k.solve(W.u_exact(*k.points("ctrl").T), u=torch.empty(k.n_nodes - 1, dtype=torch.float64, device="cuda"))


def test_explicit_stream_matches_current_stream():
    """Work on an explicit side stream waits for the inputs converted on the current stream."""
    prob = W.C2(256)
    k = gpu(prob)
    phi = W.random_density(k.M, 4)
    ref = k.apply(phi).cpu()
    s = torch.cuda.Stream()
    out = k.apply(phi, stream=s)
    s.synchronize()
    assert torch.equal(out.cpu(), ref)


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_context_on_second_device():
    """A context on device 1 created and used while device 0 is current (per-device launch caches)."""
    prob = W.C3(1024)
    k0 = gpu(prob)
    with torch.cuda.device(0):
        k1 = KFBI(prob, device=1)
        phi = W.random_density(k0.M, 5)
        assert torch.equal(k1.apply(phi).cpu(), k0.apply(phi).cpu())
        assert torch.cuda.current_device() == 0


@pytest.mark.parametrize("prob,world", [(W.C1(64), 1), (W.C4(32), 1), (W.C3(1024), 2)], ids=["C1", "C4", "C3x2-emul"])
def test_node_mask_device_matches_host(prob, world):
    k = KFBI(prob, world=world, rank=-1) if world > 1 else gpu(prob)
    assert np.array_equal(k.node_mask_device().cpu().numpy(), k.node_mask()[k.local_slice()])
