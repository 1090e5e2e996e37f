"""GPU Gray–Scott stepper (kfbi_gray_scott_step) against the oracle: same seeded initial data, same
Strang/Crank–Nicolson/bilinear readings (R40, R41)."""
import numpy as np
import pytest
import torch

import workloads as W
from oracle.grayscott import GrayScott as OracleGS
from paper_2404_15249_b200 import GrayScott

pytestmark = pytest.mark.gpu


def test_gray_scott_matches_oracle():
    assert torch.cuda.is_available()
    n, dt, tol, steps = 64, 0.125, 1e-12, 3
    o = OracleGS(n, dt, tol=tol)
    g = GrayScott(n, dt, W.GS_PARAMS, W.gray_scott_problem, W.gray_scott_initial, tol=tol)
    for _ in range(steps):
        o.step()
        g.step()
    u, v = (t.cpu().numpy() for t in g.fields())
    m = o.ou.st.side
    scale = max(np.abs(o.u[m]).max(), 1.0)
    assert np.abs(u[m] - o.u[m]).max() < 1e-9 * scale
    assert np.abs(v[m] - o.v[m]).max() < 1e-9 * scale
    gi = [x for pair in g.iters for x in pair]
    assert all(abs(a - b) <= 1 for a, b in zip(gi, o.iters))
