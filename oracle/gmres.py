"""Restarted GMRES (test infrastructure only): Algorithm 5.

Conventions (reading R18): Arnoldi with modified Gram–Schmidt exactly as P:765-768
(h_{ij} = (w, μ_i); w −= h_{ij} μ_i, for i = 1..j); least squares over R^j by Givens
rotations; stopping relative to β₀ = ‖ĝ − K x₀‖₂ of the first cycle (tol 1e-8);
restart m = 30; x₀ = 0; explicit residual r = ĝ − K x at the start of every cycle
(P:760); lucky breakdown when h_{j+1,j} ≤ 1e-14 β₀.
"""
from __future__ import annotations

import dataclasses

import numpy as np


@dataclasses.dataclass
class Stats:
    iters: int = 0
    restarts: int = 0
    n_applies: int = 0
    rel_residual: float = np.nan
    converged: bool = False
    history: list = dataclasses.field(default_factory=list)


def gmres(K, b, x0=None, tol=1e-8, restart=30, max_restarts=50):
    n = b.size
    st = Stats()
    x = np.zeros(n) if x0 is None else x0.astype(np.float64).copy()
    beta0 = None
    for cycle in range(max_restarts + 1):
        if x0 is None and cycle == 0:
            r = b.copy()
        else:
            r = b - K(x)
            st.n_applies += 1
        beta = float(np.sqrt(r @ r))
        if beta0 is None:
            beta0 = beta
        st.rel_residual = beta / beta0 if beta0 > 0 else 0.0
        st.history.append(st.rel_residual)
        if beta <= tol * beta0 or beta0 == 0.0:
            st.converged = True
            return x, st
        if cycle == max_restarts:
            break
        st.restarts = cycle + 1
        V = np.zeros((restart + 1, n))
        H = np.zeros((restart + 1, restart))
        cs = np.zeros(restart)
        sn = np.zeros(restart)
        g = np.zeros(restart + 1)
        V[0] = r / beta
        g[0] = beta
        jlast = restart - 1
        for j in range(restart):
            w = K(V[j])
            st.iters += 1
            st.n_applies += 1
            for i in range(j + 1):                 # MGS
                H[i, j] = w @ V[i]
                w = w - H[i, j] * V[i]
            H[j + 1, j] = float(np.sqrt(w @ w))
            for i in range(j):                      # apply previous rotations
                a, c = H[i, j], H[i + 1, j]
                H[i, j] = cs[i] * a + sn[i] * c
                H[i + 1, j] = -sn[i] * a + cs[i] * c
            hnext = H[j + 1, j]
            rr = np.hypot(H[j, j], hnext)
            cs[j], sn[j] = H[j, j] / rr, hnext / rr
            H[j, j] = rr
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            if abs(g[j + 1]) <= tol * beta0 or hnext <= 1e-14 * beta0:
                jlast = j
                break
            V[j + 1] = w / hnext
        k = jlast + 1
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):              # back substitution on the Givens-reduced H
            y[i] = (g[i] - H[i, i + 1:k] @ y[i + 1:k]) / H[i, i]
        x = x + V[:k].T @ y
    st.converged = False
    return x, st
