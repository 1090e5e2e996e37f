"""Ω-compact transfers (kfbi_omega_count / kfbi_scatter_omega / kfbi_gather_omega): the serving
path moves only the Ω-node values of f and u (zero extension of f; u_h valid on Ω).
Bit-exact index work: compared with NumPy masking of the same arrays."""
import numpy as np
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu


def _k(prob):
    from paper_2404_15249_b200 import KFBI
    return KFBI(prob)


@pytest.mark.parametrize("prob", [W.C1(64), W.C3(1024), W.C3(8192), W.C4(64), W.C5(128)],
                         ids=lambda p: f"{p.name}{p.n}")
def test_scatter_gather_bit_exact(prob):
    k = _k(prob)
    mask = k.node_mask().reshape(-1).astype(bool)
    assert k.omega_count() == int(mask.sum())
    rng = np.random.default_rng(5)
    x = rng.standard_normal(mask.size)
    g = k.gather_omega(torch.tensor(x, device="cuda")).cpu().numpy()
    assert np.array_equal(g, x[mask])
    full = k.scatter_omega(torch.tensor(g, device="cuda")).cpu().numpy()
    ref = np.where(mask, x, 0.0)
    assert np.array_equal(full, ref)


def test_compact_solve_matches_full():
    prob = W.C3(1024)
    k = _k(prob)
    pz, pq = k.points("ctrl"), k.points("isect")
    x = prob.lo + np.arange(prob.n + 1) * prob.h
    X, Y = np.meshgrid(x, x, indexing="ij")
    f = W.f_exact(prob.kappa, X, Y).ravel()
    dev = lambda a: torch.tensor(np.ascontiguousarray(a), device="cuda")
    g, fq, fz = dev(W.u_exact(*pz.T)), dev(W.f_exact(prob.kappa, *pq.T)), dev(W.f_exact(prob.kappa, *pz.T))
    u_full, _, _ = k.solve(g, dev(f), fq, fz)
    mask = k.node_mask().reshape(-1).astype(bool)
    fc = k.gather_omega(dev(f))
    u2, _, _ = k.solve(g, k.scatter_omega(fc), fq, fz)
    a = k.gather_omega(u_full).cpu().numpy()
    b = k.gather_omega(u2).cpu().numpy()
    assert np.array_equal(a, b)                           # f off Ω is never read (zero extension)
    assert np.array_equal(a, u_full.cpu().numpy().reshape(-1)[mask])


def test_async_final_matches_sync():
    """opts.async_final: kfbi_solve returns with the final field still on the stream; after the
    stream is synchronised u and φ equal the synchronous solve bit for bit."""
    prob = W.C3(1024)
    k = _k(prob)
    pz, pq = k.points("ctrl"), k.points("isect")
    x = prob.lo + np.arange(prob.n + 1) * prob.h
    X, Y = np.meshgrid(x, x, indexing="ij")
    dev = lambda a: torch.tensor(np.ascontiguousarray(a), device="cuda")
    args = (dev(W.u_exact(*pz.T)), dev(W.f_exact(prob.kappa, X, Y).ravel()), dev(W.f_exact(prob.kappa, *pq.T)),
            dev(W.f_exact(prob.kappa, *pz.T)))
    u1, p1, s1 = k.solve(*args)
    u2, p2, s2 = k.solve(*args, async_final=True)
    torch.cuda.synchronize()
    assert torch.equal(u1, u2) and torch.equal(p1, p2) and s1.iters == s2.iters


@pytest.mark.parametrize("prob", [W.C1(64), W.C2(512), W.C3(1024), W.C3(2048)], ids=lambda p: f"{p.name}{p.n}")
def test_omega_io_solve_bit_exact(prob):
    """kfbi_solve_opts.omega_io: f in and u out as Ω-node values only.  The dense forward reads f at
    the Ω nodes through the row bitmasks (staged row copies at N ≥ 1024, global gathers below) and
    the final field writes u there; both equal the full-grid solve bit for bit (f off Ω is never read,
    P:530; u_h on Ω), and a 3D context refuses the option."""
    k = _k(prob)
    pz, pq = k.points("ctrl"), k.points("isect")
    x = prob.lo + np.arange(prob.n + 1) * prob.h
    X, Y = np.meshgrid(x, x, indexing="ij")
    f = W.f_exact(prob.kappa, X, Y).ravel()
    dev = lambda a: torch.tensor(np.ascontiguousarray(a), device="cuda")
    g, fq, fz = dev(W.u_exact(*pz.T)), dev(W.f_exact(prob.kappa, *pq.T)), dev(W.f_exact(prob.kappa, *pz.T))
    u_full, phi_full, st_full = k.solve(g, dev(f), fq, fz)
    mask = k.node_mask().reshape(-1).astype(bool)
    u_c, phi_c, st_c = k.solve(g, dev(f[mask]), fq, fz, omega_io=True)
    assert u_c.numel() == k.omega_count() and st_c.iters == st_full.iters
    assert torch.equal(phi_c, phi_full)
    assert np.array_equal(u_c.cpu().numpy(), u_full.cpu().numpy().reshape(-1)[mask])


@pytest.mark.parametrize("prob", [W.C4(64), W.C5(128)], ids=lambda p: f"{p.name}{p.n}")
def test_omega_io_solve_bit_exact_3d(prob):
    """3D omega_io: the dense forward builds h²·f·1_Ω from the Ω-compact f (row bitmasks and counts) and
    the final field stores u at the Ω ranks — equal to the full-grid solve bit for bit."""
    k = _k(prob)
    pz, pq = k.points("ctrl"), k.points("isect")
    x = prob.lo + np.arange(prob.n + 1) * prob.h
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    f = W.f_exact(prob.kappa, X, Y, Z).ravel()
    dev = lambda a: torch.tensor(np.ascontiguousarray(a), device="cuda")
    g, fq, fz = dev(W.u_exact(*pz.T)), dev(W.f_exact(prob.kappa, *pq.T)), dev(W.f_exact(prob.kappa, *pz.T))
    u_full, phi_full, st_full = k.solve(g, dev(f), fq, fz)
    mask = k.node_mask().reshape(-1).astype(bool)
    u_c, phi_c, st_c = k.solve(g, dev(f[mask]), fq, fz, omega_io=True)
    assert u_c.numel() == k.omega_count() and st_c.iters == st_full.iters
    assert torch.equal(phi_c, phi_full)
    assert np.array_equal(u_c.cpu().numpy(), u_full.cpu().numpy().reshape(-1)[mask])
