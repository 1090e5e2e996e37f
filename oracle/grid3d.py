"""Procedure 1 in 3D for the oracle (test infrastructure only; see oracle/__init__).

The paper treats 3D as "analogous" and shows 3D only for Stokes.  Readings:
R12 control points = the Γ ∩ grid-edge intersection nodes, density derivatives from a tangent-plane
least-squares fit; R13 Monge-patch jump formulas; R14 ten-point stencil.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from workloads import ELLIPSOID, TORUS
from . import geometry as geo
from .grid import GeometryError


@dataclasses.dataclass
class Setup3D:
    prob: object
    n: int
    h: float
    lo: float
    x: np.ndarray
    side: np.ndarray          # (N+1)^3 bool
    irregular: np.ndarray
    q_axis: np.ndarray        # sorted by (axis, i, j, k)
    q_i: np.ndarray
    q_j: np.ndarray
    q_k: np.ndarray
    q_xi: np.ndarray
    q_pos: np.ndarray         # (nq, 3)
    nrm: np.ndarray           # (nq, 3) outward unit normal
    e1: np.ndarray
    e2: np.ndarray
    kab: np.ndarray           # (nq, 2, 2) κ_ab = −e_aᵀ D²ℓ e_b / |∇ℓ|

    @property
    def M(self):
        return self.q_xi.size


def grad_hess(comp, p):
    """∇ℓ and D²ℓ of the level set at points p (n, 3)."""
    c = np.asarray(comp.center)
    d = p - c
    n = p.shape[0]
    if comp.kind == ELLIPSOID:
        a = np.asarray(comp.p[:3])
        g = 2 * d / a ** 2
        H = np.zeros((n, 3, 3))
        for ax in range(3):
            H[:, ax, ax] = 2 / a[ax] ** 2
        return g, H
    if comp.kind == TORUS:
        R, r = comp.p[:2]
        rho = np.sqrt(d[:, 0] ** 2 + d[:, 1] ** 2)
        qq = rho - R
        g = np.stack([2 * qq * d[:, 0] / rho, 2 * qq * d[:, 1] / rho, 2 * d[:, 2]], -1)
        H = np.zeros((n, 3, 3))
        # ∂²/∂x_a∂x_b of (ρ − R)² = 2 (x_a x_b / ρ²) + 2 (ρ − R)(δ_ab/ρ − x_a x_b/ρ³), a,b ∈ {x, y}
        for a_ in range(2):
            for b_ in range(2):
                xa, xb = d[:, a_], d[:, b_]
                H[:, a_, b_] = 2 * xa * xb / rho ** 2 + 2 * qq * ((a_ == b_) / rho - xa * xb / rho ** 3)
        H[:, 2, 2] = 2.0
        return g, H
    raise ValueError(comp.kind)


def frames(comp, p):
    """n = ∇ℓ/|∇ℓ|; e1 = normalize(n × u*), u* the axis with the smallest |n_a| (ties → lowest);
    e2 = n × e1; κ_ab = −e_aᵀ D²ℓ e_b / |∇ℓ|."""
    g, H = grad_hess(comp, p)
    gn = np.linalg.norm(g, axis=1)
    n = g / gn[:, None]
    ax = np.argmin(np.abs(n), axis=1)
    u = np.eye(3)[ax]
    e1 = np.cross(n, u)
    e1 /= np.linalg.norm(e1, axis=1)[:, None]
    e2 = np.cross(n, e1)
    E = np.stack([e1, e2], 1)                          # (n, 2, 3)
    kab = -np.einsum("nai,nij,nbj->nab", E, H, E) / gn[:, None, None]
    return n, e1, e2, kab


def build(prob) -> Setup3D:
    assert prob.dim == 3
    n, lo = prob.n, prob.lo
    h = (prob.hi - prob.lo) / n
    x = lo + np.arange(n + 1) * h
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    comps = prob.comps
    side = geo.in_omega(comps, X, Y, Z)
    del X, Y, Z
    irr = np.zeros_like(side)
    recs = []
    for axis in range(3):
        a = [slice(None)] * 3
        b = [slice(None)] * 3
        a[axis] = slice(1, None)
        b[axis] = slice(None, -1)
        d = side[tuple(a)] != side[tuple(b)]
        irr[tuple(a)] |= d
        irr[tuple(b)] |= d
        ei = np.argwhere(d)
        if ei.size == 0:
            continue
        comp = comps[0]
        p0 = x[ei]
        e = np.zeros(3)
        e[axis] = h
        want = geo.omega_side(comp, *p0.T)
        prev = want.copy()
        changes = np.zeros(len(ei), dtype=np.int64)
        for t in (0.2, 0.4, 0.6, 0.8, 1.0):
            cur = geo.omega_side(comp, *(p0 + t * e).T)
            changes += cur != prev
            prev = cur
        if np.any(changes != 1):
            raise GeometryError("edge crossed more than once (R31)")
        lo_t = np.zeros(len(ei))
        hi_t = np.ones(len(ei))
        for _ in range(64):
            m = 0.5 * (lo_t + hi_t)
            same = geo.omega_side(comp, *(p0 + m[:, None] * e).T) == want
            lo_t = np.where(same, m, lo_t)
            hi_t = np.where(same, hi_t, m)
        t = 0.5 * (lo_t + hi_t)
        xi = p0[:, axis] + t * h
        pos = p0.copy()
        pos[:, axis] = xi
        recs.append((np.full(len(ei), axis), ei, xi, pos))
    if len(comps) != 1:
        raise GeometryError("3D oracle supports one outer surface")
    ii = np.argwhere(irr)
    if ii.size and (ii.min() < 2 or ii.max() > n - 2):
        raise GeometryError("Γ too close to the box boundary (R32)")
    q_axis = np.concatenate([r[0] for r in recs])
    q_idx = np.concatenate([r[1] for r in recs])
    q_xi = np.concatenate([r[2] for r in recs])
    q_pos = np.concatenate([r[3] for r in recs])
    order = np.lexsort((q_idx[:, 2], q_idx[:, 1], q_idx[:, 0], q_axis))
    q_axis, q_idx, q_xi, q_pos = q_axis[order], q_idx[order], q_xi[order], q_pos[order]
    nrm, e1, e2, kab = frames(comps[0], q_pos)
    return Setup3D(prob, n, h, lo, x, side, irr, q_axis, q_idx[:, 0], q_idx[:, 1], q_idx[:, 2], q_xi, q_pos,
                   nrm, e1, e2, kab)


def lsq_neighbours(st: Setup3D):
    """Neighbours of each control point: all other control points whose edge low-end node lies in
    the 5×5×5 node block centred at its own low-end node (integer rule)."""
    key = st.q_i * (st.n + 1) ** 2 + st.q_j * (st.n + 1) + st.q_k
    buckets = {}
    for q, kk in enumerate(key.tolist()):
        buckets.setdefault(kk, []).append(q)
    W = st.n + 1
    nb = []
    for q in range(st.M):
        i, j, k = st.q_i[q], st.q_j[q], st.q_k[q]
        lst = []
        for di in range(-2, 3):
            for dj in range(-2, 3):
                for dk in range(-2, 3):
                    lst.extend(buckets.get((i + di) * W * W + (j + dj) * W + (k + dk), ()))
        lst = [p for p in lst if p != q]
        nb.append(np.array(sorted(lst), dtype=np.int64))
    return nb


def lsq_operator(st: Setup3D, nb):
    """Unweighted LSQ φ_q − φ₀ ≈ a1 t1 + a2 t2 + ½a3 t1² + a4 t1t2 + ½a5 t2² in tangent coordinates
    t = (e1·(x_q − x₀), e2·(x_q − x₀)).  Returns the least-squares solution operator of
    every control point as padded (M, K) neighbour indices and (M, 5, K) pseudo-inverse rows
    (numpy.linalg.pinv, a library primitive), so that a = Σ_q pinv[:, q] (φ_q − φ₀)."""
    K = max(len(p) for p in nb)
    idx = np.zeros((st.M, K), dtype=np.int64)
    pinv = np.zeros((st.M, 5, K))
    for q in range(st.M):
        p = nb[q]
        if p.size < 8:
            raise GeometryError("fewer than 8 LSQ neighbours")
        d = st.q_pos[p] - st.q_pos[q]
        t1 = d @ st.e1[q]
        t2 = d @ st.e2[q]
        A = np.stack([t1, t2, 0.5 * t1 * t1, t1 * t2, 0.5 * t2 * t2], -1)
        if np.linalg.cond(A) > 1e8:
            raise GeometryError("ill-conditioned LSQ fit")
        idx[q, :p.size] = p
        idx[q, p.size:] = q
        pinv[q, :, :p.size] = np.linalg.pinv(A)
    return idx, pinv


def lsq_fit(idx, pinv, phi):
    """(M, 5): ∂1Φ, ∂2Φ, ∂11Φ, ∂12Φ, ∂22Φ of the density at every control point."""
    return np.einsum("mak,mk->ma", pinv, phi[idx] - phi[:, None])


def stencil(st: Setup3D):
    """Ten-point stencil at each control point (reading R14, 3D): centre c = nearest node,
    {c, c±e_x, c±e_y, c±e_z, c+σ_xe_x+σ_ye_y, c+σ_xe_x+σ_ze_z, c+σ_ye_y+σ_ze_z}.  (M, 10, 3)."""
    u = (st.q_pos - st.lo) / st.h
    c = np.floor(u + 0.5).astype(np.int64)
    xc = st.lo + c * st.h
    sg = np.where(st.q_pos >= xc, 1, -1)
    offs = [np.zeros((st.M, 3), np.int64)]
    for a in range(3):
        for s in (1, -1):
            o = np.zeros((st.M, 3), np.int64)
            o[:, a] = s
            offs.append(o)
    for a, b in ((0, 1), (0, 2), (1, 2)):
        o = np.zeros((st.M, 3), np.int64)
        o[:, a] = sg[:, a]
        o[:, b] = sg[:, b]
        offs.append(o)
    return c[:, None, :] + np.stack(offs, 1)
