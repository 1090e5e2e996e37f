"""FFT-based fast solver of the 5-point (7-point) modified-Helmholtz system (test infra only).

Algorithm 4: sine transform along y [and z] (FST for the Dirichlet box,
P:742, reading R3), tridiagonal solves along x, inverse transform.  What it
computes has a plain definition: the exact solution of
    Σ_a (v_{p+e_a} − 2 v_p + v_{p−e_a}) / h² − κ v_p = f_p ,   v = 0 on ∂B.

Readings: R4  forward f̂_k = Σ_{j=1}^{N−1} f_j sin(πjk/N), inverse (2/N) Σ_k.
          Per mode:  v̂_{i−1} + d_k v̂_i + v̂_{i+1} = h² f̂_i,
          d_k = −(2 + 4 sin²(πk/2N) [+ 4 sin²(πl/2N)] + κ h²)
The DST is scipy.fft.dst(type=1) (library primitive; pinned against the O(N²) sum).
Thomas follows the textbook forward/backward sweep.
"""
from __future__ import annotations

import numpy as np
import scipy.fft


def dst1(f, axis=-1):
    """f̂_k = Σ_j f_j sin(πjk/N) over the N−1 interior entries of `axis` (R4)."""
    return 0.5 * scipy.fft.dst(f, type=1, axis=axis)


def idst1(fh, axis=-1):
    """f_j = (2/N) Σ_k f̂_k sin(πjk/N) (R4)."""
    n = fh.shape[axis] + 1
    return scipy.fft.dst(fh, type=1, axis=axis) / n


def dst1_direct(f):
    """O(N²) direct sum along the last axis — used only by tests on small N."""
    n = f.shape[-1] + 1
    j = np.arange(1, n)
    S = np.sin(np.pi * np.outer(j, j) / n)
    return f @ S


def thomas(dk, r):
    """Solve x_{i−1} + d x_i + x_{i+1} = r_i (x_0 = x_n+1 = 0) for each column of r.

    dk: (K,) diagonal per system; r: (n, K).  Textbook Thomas with forward pivots
    c_1 = d, c_i = d − 1/c_{i−1}."""
    n = r.shape[0]
    c = np.empty_like(r)
    y = np.empty_like(r)
    c[0] = dk
    y[0] = r[0]
    for i in range(1, n):
        c[i] = dk - 1.0 / c[i - 1]
        y[i] = r[i] - y[i - 1] / c[i - 1]
    x = np.empty_like(r)
    x[n - 1] = y[n - 1] / c[n - 1]
    for i in range(n - 2, -1, -1):
        x[i] = (y[i] - x[i + 1]) / c[i]
    return x


def mode_mu(n):
    k = np.arange(1, n)
    return 4.0 * np.sin(np.pi * k / (2.0 * n)) ** 2


def solve2d(f, h, kappa):
    """f: (N−1, N−1) RHS at unknowns [i, j] → v with (Δ_h − κ) v = f (Alg. 4)."""
    n = f.shape[0] + 1
    fh = dst1(f, axis=1)                       # step 1: transform along y
    dk = -(2.0 + mode_mu(n) + kappa * h * h)   # per mode k
    vh = thomas(dk, h * h * fh)                # step 2: tridiagonal along x (rows i)
    return idst1(vh, axis=1)                   # step 3: inverse transform


def solve3d(f, h, kappa):
    """f: (N−1,)*3 RHS at [i, j, k]: 2D sine transform over (j, k), tridiagonal along i."""
    n = f.shape[0] + 1
    fh = dst1(dst1(f, axis=1), axis=2)
    mu = mode_mu(n)
    dk = -(2.0 + mu[:, None] + mu[None, :] + kappa * h * h)
    vh = thomas(dk.reshape(-1), (h * h * fh).reshape(n - 1, -1)).reshape(fh.shape)
    return idst1(idst1(vh, axis=1), axis=2)


def apply_operator2d(v, h, kappa):
    """(Δ_h − κ) v at the unknowns, v = 0 outside (used by tests)."""
    p = np.pad(v, 1)
    return (p[2:, 1:-1] + p[:-2, 1:-1] + p[1:-1, 2:] + p[1:-1, :-2] - 4.0 * v) / (h * h) - kappa * v


def thomas_arrowhead(dk, r, m):
    """Arrowhead decomposition (ADM) of the per-mode tridiagonal systems over m partitions
    (P:81-148): the separator of partition k < m is its last unknown (reading R21); blocks S^k are
    solved independently, z^k = S⁻¹F_s, Z_L = S⁻¹e_first, Z_R = S⁻¹e_last; the separators h
    solve the Schur system (H − W_L S⁻¹ W_R) h = F_h − W_L S⁻¹ F_s; back-substitution
    s^k = z^k − Z_L h^{k−1} − Z_R h^k (P:128 with the garble fixed, reading R20), h⁰ = h^m = 0.
    Mathematically identical to `thomas` (same system); used to pin the partitioned GPU solver."""
    n, K = r.shape
    if m == 1:
        return thomas(dk, r)
    cuts = [round(n * q / m) for q in range(m + 1)]
    seps = [cuts[q + 1] - 1 for q in range(m - 1)]            # separator = last unknown of partition q
    blocks = [(cuts[q], (cuts[q + 1] - 1) if q < m - 1 else cuts[q + 1]) for q in range(m)]
    z, ZL, ZR = [], [], []
    for (a, b) in blocks:
        L = b - a
        e1 = np.zeros((L, K))
        e1[0] = 1.0
        eL = np.zeros((L, K))
        eL[-1] = 1.0
        z.append(thomas(dk, r[a:b]))
        ZL.append(thomas(dk, e1))
        ZR.append(thomas(dk, eL))
    # Schur system on the separators: row q couples h_{q−1}, h_q, h_{q+1}
    ns = m - 1
    h = np.zeros((ns, K))
    for k in range(K):
        A = np.zeros((ns, ns))
        rhs = np.zeros(ns)
        for q in range(ns):
            A[q, q] = dk[k] - ZR[q][-1, k] - ZL[q + 1][0, k]
            if q > 0:
                A[q, q - 1] = -ZL[q][-1, k]
            if q < ns - 1:
                A[q, q + 1] = -ZR[q + 1][0, k]
            rhs[q] = r[seps[q], k] - z[q][-1, k] - z[q + 1][0, k]
        h[:, k] = np.linalg.solve(A, rhs)
    x = np.empty_like(r)
    for q, (a, b) in enumerate(blocks):
        hl = h[q - 1] if q > 0 else 0.0
        hr = h[q] if q < ns else 0.0
        x[a:b] = z[q] - ZL[q] * hl - ZR[q] * hr
        if q < ns:
            x[seps[q]] = h[q]
    return x
