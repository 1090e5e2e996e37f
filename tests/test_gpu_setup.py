"""GPU-side Procedure 1 phases (kfbi_setup_device) against the host setup.

Classification, the sign-change edges with their bisected intersections (R30/R31),
the irregular-node lists (App. A.3) and, in 2D, the six-point stencils with their LU-solved
weight rows (R14, R16, R38) and the sorted unique stencil-node list come from setup_gpu.cu;
everything else from the same host code, so the two setups must agree on every list.  Integer lists and
the Ω mask are compared bit-exactly; ξ is bit-exact for ellipses (only +, −, ×, ÷ on both sides)
and within 1e-13 for stars (device sin/atan2 vs libm inside the level function, amplified where Γ
grazes a grid line, R30).  The
host setup itself is pinned to the oracle by tests/test_abi.py::test_setup_matches_oracle*.
"""
import time

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


def _pair(prob):
    from paper_2404_15249_b200 import KFBI
    import torch
    t0 = time.perf_counter()
    host = KFBI(prob)
    t1 = time.perf_counter()
    dev = KFBI(prob, device_setup=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return host, dev, t1 - t0, t2 - t1


def _all_ellipses(prob):
    return all(c.kind == W.ELLIPSE for c in prob.comps)


@pytest.mark.parametrize("make,n", [(W.C1, 64), (W.C2, 256), (W.C2, 1024), (W.C3, 1024), (W.C3, 8192)])
def test_device_setup_lists_match_host(make, n):
    prob = make(n)
    host, dev, th, td = _pair(prob)
    print(f"{prob.name} N={n}: host setup {th:.3f} s, device-phase setup {td:.3f} s")
    assert (host.M, host.nq, host.nirr) == (dev.M, dev.nq, dev.nirr)
    assert np.array_equal(host.node_mask(), dev.node_mask())
    for which in (0, 1, 2):                      # irregular nodes, intersections, stencil nodes
        assert np.array_equal(host.setup_dump(which), dev.setup_dump(which)), which
    assert np.array_equal(host.points("ctrl"), dev.points("ctrl"))
    qh, qd = host.points("isect"), dev.points("isect")
    if _all_ellipses(prob):
        assert np.array_equal(qh, qd)
    else:
        # a level error of δ moves the root by δ/|∂ℓ/∂x_a|, large where Γ grazes the grid line
        d = np.max(np.abs(qh - qd))
        print(f"  max |Δξ| = {d:.2e}")
        assert d <= 1e-13


@pytest.mark.parametrize("make,n", [(W.C2, 1024), (W.C3, 2048)])
def test_device_setup_apply_matches_host(make, n):
    import torch
    prob = make(n)
    host, dev, _, _ = _pair(prob)
    phi = torch.tensor(W.random_density(host.M, seed=7), dtype=torch.float64, device="cuda")
    a, b = host.apply(phi), dev.apply(phi)
    torch.cuda.synchronize()
    err = (a - b).abs().max().item() / a.abs().max().item()
    print(f"{prob.name} N={n}: apply(host setup) vs apply(device setup) rel {err:.2e}")
    if _all_ellipses(prob):
        assert err == 0.0
    else:   # Δξ ≤ 1e-13 enters the corrections through d/h² (App. A.3): well inside the 1e-10 apply bar
        assert err <= 1e-11


@pytest.mark.parametrize("n", [64, 1024])
def test_device_stencils_neumann_apply_matches_host(n):
    """The device LU of the normal-derivative rows (st_wn, R38) equals the host's bit for bit: the
    K_N apply (Neumann, κ = 1) of an ellipse built on either setup is identical."""
    import torch
    prob = W.neumann(W.problem("ellipse-k1", 2, n, [W.ellipse(1.0, 0.8)], 1.0))
    host, dev, _, _ = _pair(prob)
    phi = torch.tensor(W.random_density(host.M, seed=3), dtype=torch.float64, device="cuda")
    a, b = host.apply(phi), dev.apply(phi)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_device_setup_errors():
    import torch
    from paper_2404_15249_b200 import KFBI, KfbiError
    from paper_2404_15249_b200 import kfbi as K
    # Γ through the band next to ∂B: R32 from the device irregular-node pass
    prob = W.problem("too-close", 2, 128, [W.ellipse(1.19, 0.8)], 0.0)
    with pytest.raises(KfbiError) as e:
        KFBI(prob, device_setup=True)
    assert e.value.code == K.EGEOM
    with pytest.raises(KfbiError) as e:
        KFBI(prob)
    assert e.value.code == K.EGEOM
    # scratch too small → ENOMEM; 3D sizes: powers of two in [32, 512], ≈ 5 GB of scratch at 512³
    import ctypes as C
    lib = K.load()
    g = K.Grid(2, (C.c_double * 3)(-1.2, -1.2, 0), (C.c_double * 3)(1.2, 1.2, 0), (C.c_int32 * 3)(256, 256, 0))
    comps = (K.Component * 1)(K.Component(W.ELLIPSE, W.OUTER, (C.c_double * 3)(0, 0, 0), (C.c_double * 4)(1, .8, 0, 0), 0))
    b = K.Boundary(1, comps)
    pde = K.Pde(0.0, 0)
    dist = K.Dist(1, 0, 0, None)
    need = C.c_size_t()
    assert lib.kfbi_setup_scratch_size(C.byref(g), C.byref(need)) == K.OK and need.value > 0
    small = torch.empty(need.value // 4, dtype=torch.uint8, device="cuda")
    ctx = C.c_void_p()
    st = lib.kfbi_setup_device(C.byref(g), C.byref(b), C.byref(pde), C.byref(dist), None,
                               C.c_void_p(small.data_ptr()), need.value // 4, C.byref(ctx))
    assert st == K.ENOMEM and not ctx.value
    g3 = K.Grid(3, (C.c_double * 3)(-1.2, -1.2, -1.2), (C.c_double * 3)(1.2, 1.2, 1.2), (C.c_int32 * 3)(64, 64, 64))
    assert lib.kfbi_setup_scratch_size(C.byref(g3), C.byref(need)) == K.OK and need.value > 0
    g3b = K.Grid(3, (C.c_double * 3)(-1.2, -1.2, -1.2), (C.c_double * 3)(1.2, 1.2, 1.2), (C.c_int32 * 3)(1024, 1024, 1024))
    assert lib.kfbi_setup_scratch_size(C.byref(g3b), C.byref(need)) == K.EINVAL


@pytest.mark.parametrize("make,n", [(W.C1, 64), (W.C2, 1024), (W.C3, 1024)])
def test_device_setup_matches_oracle(make, n):
    """The device phases against the oracle's own Procedure 1 (oracle/grid.py), as the host setup is
    in tests/test_abi.py: integer lists bit for bit, intersection points to 1e-13·h."""
    from oracle import grid
    from paper_2404_15249_b200 import KFBI
    prob = make(n)
    k = KFBI(prob, device_setup=True)
    st = grid.build(prob)
    assert k.M == st.M and k.nq == st.q_xi.size
    assert np.array_equal(k.setup_dump(0), np.argwhere(st.irregular))
    assert np.array_equal(k.setup_dump(1), np.stack([st.q_axis, st.q_i, st.q_j], -1))
    assert np.array_equal(k.setup_dump(2), grid.stencil(st))
    assert np.array_equal(k.node_mask().astype(bool), st.side)
    px = np.where(st.q_axis == 0, st.q_xi, st.x[st.q_i])
    py = np.where(st.q_axis == 1, st.q_xi, st.x[st.q_j])
    np.testing.assert_allclose(k.points("isect"), np.stack([px, py], -1), atol=1e-13 * st.h)


@pytest.mark.parametrize("make,n", [(W.C4, 32), (W.C4, 128), (W.C5, 64), (W.C5, 512)])
def test_device_setup3d_lists_match_host(make, n):
    """3D (NEXT-3): classification, the (axis, i, j, k) sign-change edges with their bisected ξ, the
    (i, j, k) irregular nodes with their ≤ 6 incident intersections and the ten-point stencils with
    their LU-solved weight rows on the device — bit-identical to the
    host setup (ellipsoid and torus levels use only +, −, ×, ÷, √ on both sides); the host setup is pinned
    to the oracle's lists by tests/test_abi.py::test_host_setup3d_matches_oracle."""
    prob = make(n)
    host, dev, th, td = _pair(prob)
    print(f"{prob.name} N={n}: host setup {th:.3f} s, device-phase setup {td:.3f} s")
    assert (host.M, host.nq, host.nirr) == (dev.M, dev.nq, dev.nirr)
    assert np.array_equal(host.node_mask(), dev.node_mask())
    for which in (0, 1, 2):                      # irregular nodes, intersections, stencil nodes
        assert np.array_equal(host.setup_dump(which), dev.setup_dump(which)), which
    assert np.array_equal(host.points("ctrl"), dev.points("ctrl"))
    assert np.array_equal(host.points("normal"), dev.points("normal"))
    phi = W.random_density(host.M, 3)
    assert np.array_equal(host.apply(phi).cpu().numpy(), dev.apply(phi).cpu().numpy())


def test_device_stencils3d_neumann_apply_matches_host():
    """3D ten-point stencils on the device (NEXT-3 stencil LU): the Neumann normal-derivative rows
    (R38) equal the host's bit for bit — the K_N apply of the C4 ellipsoid (κ = 1) built on either
    setup is identical."""
    import torch
    prob = W.neumann(W.problem("C4-ellipsoid-k1", 3, 64, list(W.C4(64).comps), 1.0))
    host, dev, _, _ = _pair(prob)
    phi = W.random_density(host.M, 5)
    assert np.array_equal(host.apply(phi).cpu().numpy(), dev.apply(phi).cpu().numpy())


@pytest.mark.parametrize("make,n", [(W.C4, 32), (W.C5, 64)])
def test_device_setup3d_matches_oracle(make, n):
    """The 3D device phases against the oracle's 3D Procedure 1 (oracle/grid3d.py)."""
    from oracle import grid3d
    from paper_2404_15249_b200 import KFBI
    prob = make(n)
    k = KFBI(prob, device_setup=True)
    st = grid3d.build(prob)
    assert k.M == st.M and k.nq == st.M
    assert np.array_equal(k.setup_dump(0), np.argwhere(st.irregular))
    assert np.array_equal(k.setup_dump(1), np.stack([st.q_axis, st.q_i, st.q_j, st.q_k], -1))
    assert np.array_equal(k.setup_dump(2), grid3d.stencil(st))
    assert np.array_equal(k.node_mask().astype(bool), st.side)
    np.testing.assert_allclose(k.points("ctrl"), st.q_pos, atol=1e-13 * st.h)
