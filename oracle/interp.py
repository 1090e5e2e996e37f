"""Interpolation of the one-sided boundary value at control points (test infrastructure only).

Algorithm 3 with the derivation of P:670-706 (\\iffalse block): with offsets
(ξ, η) = p − z_k the six stencil values satisfy
    V⁺ + V⁺_x ξ + V⁺_y η + ½V⁺_xx ξ² + V⁺_xy ξη + ½V⁺_yy η² = V_p (+ J_p if p ∈ Ω^c)
with J_p the jump Taylor polynomial at z_k (reading R15: jumps at the control point).
The 6×6 system is solved by LU with partial pivoting (numpy.linalg.solve, R16).
Stencil shape: reading R14 (oracle/grid.stencil).
"""
from __future__ import annotations

import numpy as np

from .grid import stencil


def interpolate2d(st, v_full, jz, nodes=None, want_grad=False):
    """v_full: (N+1, N+1) grid field (box nodes 0); jz: (M, 6) jumps at the control points."""
    if nodes is None:
        nodes = stencil(st)
    pi, pj = nodes[..., 0], nodes[..., 1]
    dx = st.x[pi] - st.z[0][:, None]
    dy = st.x[pj] - st.z[1][:, None]
    A = np.stack([np.ones_like(dx), dx, dy, 0.5 * dx * dx, dx * dy, 0.5 * dy * dy], -1)   # (M, 6, 6)
    J = (jz[:, 0:1] + jz[:, 1:2] * dx + jz[:, 2:3] * dy + 0.5 * jz[:, 3:4] * dx * dx
         + jz[:, 4:5] * dx * dy + 0.5 * jz[:, 5:6] * dy * dy)
    rhs = v_full[pi, pj] + np.where(st.side[pi, pj], 0.0, J)
    coef = np.linalg.solve(A, rhs[..., None])[..., 0]
    return coef if want_grad else coef[:, 0]
