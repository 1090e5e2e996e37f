"""Jumps of the interface solution at a boundary point (test infrastructure only).

Follows the paper's appendix "Calculation of jumps" (inside \\iffalse) step by
step: the first-order 2×2 system and the second-order 3×3 system,
each solved by a direct method (numpy.linalg.solve) as P:864 allows.

Reading R7: the second row of P:849 reads "= ψ_s"; since [∂_n w] = ψ the row is
n·[∇w] = ψ.  Reading R8: n = (τ2, −τ1) outward from Ω, [w] = w⁺ − w⁻ with + = Ω.
Output columns: [w], [w_x], [w_y], [w_xx], [w_xy], [w_yy].
"""
from __future__ import annotations

import numpy as np


def jumps2d(Phi, Phis, Phiss, Psi, Psis, F, kappa, tau, taup):
    Phi, Phis, Phiss, Psi, Psis, F = (np.broadcast_to(np.asarray(a, dtype=np.float64), np.shape(tau[0]))
                                      for a in (Phi, Phis, Phiss, Psi, Psis, F))
    t1, t2 = tau[0], tau[1]
    p1, p2 = taup[0], taup[1]
    n = t1.size
    # P:847-850 (with reading R7):  τ1[w_x] + τ2[w_y] = φ_s ;  τ2[w_x] − τ1[w_y] = ψ
    A1 = np.empty((n, 2, 2))
    A1[:, 0, 0], A1[:, 0, 1] = t1, t2
    A1[:, 1, 0], A1[:, 1, 1] = t2, -t1
    g = np.linalg.solve(A1, np.stack([Phis, Psi], -1)[..., None])[..., 0]
    wx, wy = g[:, 0], g[:, 1]
    # P:857-860
    A2 = np.empty((n, 3, 3))
    A2[:, 0, 0], A2[:, 0, 1], A2[:, 0, 2] = t1 * t1, 2 * t1 * t2, t2 * t2
    A2[:, 1, 0], A2[:, 1, 1], A2[:, 1, 2] = t1 * t2, t2 * t2 - t1 * t1, -t1 * t2
    A2[:, 2, 0], A2[:, 2, 1], A2[:, 2, 2] = 1.0, 0.0, 1.0
    b2 = np.stack([Phiss - (p1 * wx + p2 * wy),
                   Psis - p2 * wx + p1 * wy,
                   F + kappa * Phi], -1)
    d = np.linalg.solve(A2, b2[..., None])[..., 0]
    return np.stack([Phi, wx, wy, d[:, 0], d[:, 1], d[:, 2]], -1)
