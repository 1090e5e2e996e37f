"""Richardson and BiCGSTAB drivers over the same operator (test infrastructure only; SURVEY §8(f)
NEXT-4, Table 2 of the paper compares Richardson, BiCGSTAB and GMRES).

Richardson: φ_{k+1} = φ_k + γ(ĝ − K φ_k), γ ∈ (0, 1]; the residual ĝ − Kφ_k is formed
explicitly every iteration and the loop stops when ‖r_k‖₂ ≤ tol·‖r_0‖₂ (reading R39: the same
relative criterion as GMRES, R18, with x₀ = 0 → r₀ = ĝ).
BiCGSTAB, the textbook algorithm (van der Vorst 1992) with shadow residual r̂ = r₀, stopping on
‖r‖₂ ≤ tol·‖r₀‖₂ (also tested on the intermediate s), two operator applies per iteration.
"""
from __future__ import annotations

import numpy as np

from .gmres import Stats


def richardson(K, b, gamma=1.0, x0=None, tol=1e-8, max_iter=1500):
    st = Stats()
    x = np.zeros(b.size) if x0 is None else x0.astype(np.float64).copy()
    r0 = None
    for it in range(max_iter + 1):
        if x0 is None and it == 0:
            r = b.copy()
        else:
            r = b - K(x)
            st.n_applies += 1
        nr = float(np.sqrt(r @ r))
        r0 = nr if r0 is None else r0
        st.rel_residual = nr / r0 if r0 > 0 else 0.0
        st.history.append(st.rel_residual)
        if nr <= tol * r0 or r0 == 0.0:
            st.converged = True
            return x, st
        if it == max_iter:
            break
        x = x + gamma * r
        st.iters += 1
    return x, st


def bicgstab(K, b, x0=None, tol=1e-8, max_iter=500):
    st = Stats()
    x = np.zeros(b.size) if x0 is None else x0.astype(np.float64).copy()
    if x0 is None:
        r = b.copy()
    else:
        r = b - K(x)
        st.n_applies += 1
    rhat = r.copy()
    n0 = float(np.sqrt(r @ r))
    st.rel_residual = 1.0 if n0 > 0 else 0.0
    if n0 == 0.0:
        st.converged = True
        return x, st
    rho_prev = alpha = omega = 1.0
    v = np.zeros_like(b)
    p = np.zeros_like(b)
    for _ in range(max_iter):
        rho = float(rhat @ r)
        beta = (rho / rho_prev) * (alpha / omega)
        p = r + beta * (p - omega * v)
        v = K(p)
        st.n_applies += 1
        alpha = rho / float(rhat @ v)
        s = r - alpha * v
        st.iters += 1
        ns = float(np.sqrt(s @ s))
        if ns <= tol * n0:
            x = x + alpha * p
            st.rel_residual = ns / n0
            st.converged = True
            return x, st
        t = K(s)
        st.n_applies += 1
        omega = float(t @ s) / float(t @ t)
        x = x + alpha * p + omega * s
        r = s - omega * t
        rho_prev = rho
        nr = float(np.sqrt(r @ r))
        st.rel_residual = nr / n0
        st.history.append(st.rel_residual)
        if nr <= tol * n0:
            st.converged = True
            return x, st
    return x, st
