"""C-ABI library checks that need no GPU: it loads, exports every symbol include/kfbi.h
declares, and its host-side Procedure 1 (kfbi_setup) agrees with the oracle bit for bit on
the integer setup lists (irregular nodes, intersection edges, stencils, Ω mask)."""
import os
import re

import numpy as np
import pytest

import workloads as W
from oracle import grid
from paper_2404_15249_b200 import KFBI, KfbiError, load
from paper_2404_15249_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build()
    return load()


def test_exports_every_header_symbol(lib):
    hdr = open(os.path.join(ROOT, "include", "kfbi.h")).read()
    names = set(re.findall(r"\b(kfbi_[a-z_0-9]+)\s*\(", hdr))
    assert len(names) >= 15
    for n in sorted(names):
        assert hasattr(lib, n), n
    assert b"sm_100a" in lib.kfbi_version()


@pytest.mark.parametrize("prob", [W.C1(64), W.C2(1024), W.C3(1024), W.problem("ell-k1", 2, 256, [W.ellipse(1.0, 0.8)], 1.0)])
def test_host_setup_matches_oracle(lib, prob):
    k = KFBI(prob, workspace=False)
    st = grid.build(prob)
    assert k.M == st.M and k.nq == st.q_xi.size
    assert np.array_equal(k.setup_dump(0), np.argwhere(st.irregular))
    assert np.array_equal(k.setup_dump(1), np.stack([st.q_axis, st.q_i, st.q_j], -1))
    assert np.array_equal(k.setup_dump(2), grid.stencil(st))
    assert np.array_equal(k.node_mask().astype(bool), st.side)
    np.testing.assert_allclose(k.points("ctrl"), st.z.T, atol=1e-12)
    px = np.where(st.q_axis == 0, st.q_xi, st.x[st.q_i])
    py = np.where(st.q_axis == 1, st.q_xi, st.x[st.q_j])
    np.testing.assert_allclose(k.points("isect"), np.stack([px, py], -1), atol=1e-13 * st.h)


def test_setup_errors(lib):
    with pytest.raises(KfbiError) as e:
        KFBI(W.problem("bad-n", 2, 100, [W.circle(1.0)], 0.0), workspace=False)
    assert e.value.code == 1
    with pytest.raises(KfbiError) as e:
        KFBI(W.problem("neg-k", 2, 64, [W.circle(1.0)], -1.0), workspace=False)
    assert e.value.code == 1
    with pytest.raises(KfbiError) as e:   # Neumann at κ = 0: constant null space
        KFBI(W.neumann(W.C1(64)), workspace=False)
    assert e.value.code == 7
    with pytest.raises(KfbiError) as e:   # 3D Neumann at κ = 0 (C4): constant null space
        KFBI(W.neumann(W.C4(32)), workspace=False)
    assert e.value.code == 7
    with pytest.raises(KfbiError) as e:   # an irregular node outside [2, N−2] (R32 as built)
        KFBI(W.problem("near-box", 2, 64, [W.circle(1.18)], 0.0), workspace=False)
    assert e.value.code == 2


@pytest.mark.parametrize("prob", [W.C4(32), W.C5(64)], ids=["ellipsoid32", "torus64"])
def test_host_setup3d_matches_oracle(lib, prob):
    from oracle import grid3d
    k = KFBI(prob, workspace=False)
    st = grid3d.build(prob)
    assert k.M == st.M and k.nq == st.M
    assert np.array_equal(k.setup_dump(0), np.argwhere(st.irregular))
    assert np.array_equal(k.setup_dump(1), np.stack([st.q_axis, st.q_i, st.q_j, st.q_k], -1))
    assert np.array_equal(k.setup_dump(2), grid3d.stencil(st))
    assert np.array_equal(k.node_mask().astype(bool), st.side)
    np.testing.assert_allclose(k.points("ctrl"), st.q_pos, atol=1e-13 * st.h)


def test_omega_count_matches_mask():
    """kfbi_omega_count = number of Ω nodes of the node mask (host setup only, no GPU)."""
    import workloads as W
    from paper_2404_15249_b200 import KFBI
    for prob in (W.C1(64), W.C3(256), W.C4(32)):
        k = KFBI(prob, workspace=False)
        assert k.omega_count() == int(k.node_mask().astype(bool).sum())
