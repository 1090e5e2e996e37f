"""Correction of the 5-point RHS at irregular nodes (test infrastructure only).

Algorithm 2 with the correction terms of P:610-659 (\\iffalse block):
for an intersection (ξ) on an axis-a edge between nodes p and p̄,
    C⁺ at the Ω endpoint p :  −(1/h²) { [v] + [v_a](x_a(p̄) − ξ) + ½ [v_aa](x_a(p̄) − ξ)² }
    C⁻ at the Ω^c endpoint p: +(1/h²) { [v] + [v_a](x_a(p̄) − ξ) + ½ [v_aa](x_a(p̄) − ξ)² }
Reading R6: P:612 labels the endpoints inconsistently with its own formula; the signs are
the ones of P:619/P:629 with p̄ the node across Γ (exact on the quadratic witness).
Reading R9: degree-2 Taylor polynomial only ("H.O.T." dropped).  Several crossed edges at one
node add up (P:569-573 loops over the node's intersection set).
"""
from __future__ import annotations

import numpy as np


def correct2d(st, base, jq):
    """base: (N−1, N−1) RHS at unknowns; jq: (nq, 6) jumps at the intersections.

    Returns f̃ = base + Σ corrections, indexed [i−1, j−1]."""
    h = st.h
    f = base.copy()
    ax = st.q_axis
    i0, j0 = st.q_i, st.q_j
    i1 = i0 + (ax == 0)
    j1 = j0 + (ax == 1)
    # jump along the edge axis: [v], [v_a], [v_aa]
    va = np.where(ax == 0, jq[:, 1], jq[:, 2])
    vaa = np.where(ax == 0, jq[:, 3], jq[:, 5])
    v0 = jq[:, 0]
    for (pi, pj, qi, qj) in ((i0, j0, i1, j1), (i1, j1, i0, j0)):   # p = endpoint, p̄ = the other
        xbar = np.where(ax == 0, st.x[qi], st.x[qj])
        d = xbar - st.q_xi
        P = v0 + va * d + 0.5 * vaa * d * d
        sgn = np.where(st.side[pi, pj], -1.0, 1.0)
        np.add.at(f, (pi - 1, pj - 1), sgn * P / (h * h))
    return f
