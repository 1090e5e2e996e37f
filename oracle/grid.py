"""Procedure 1 of P:161-167 for the oracle (test infrastructure only; see oracle/__init__).

Cartesian grid on the box B, Ω/Ω^c side of every node, regular/irregular nodes
(Fig. P:583), grid-line ∩ Γ intersection nodes and quasi-uniform control
points.  2D only here; 3D lives in oracle/grid3d.py.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

from workloads import ELLIPSE, STAR, HOLE
from . import geometry as geo


class GeometryError(ValueError):
    """KFBI_EGEOM analogue: Γ not resolved by the grid (readings R31, R32)."""


@dataclasses.dataclass
class Setup2D:
    prob: object
    n: int
    h: float
    lo: float
    x: np.ndarray            # node coordinates lo + i h, i = 0..N
    side: np.ndarray         # (N+1, N+1) bool, True = Ω
    irregular: np.ndarray    # (N+1, N+1) bool
    # intersections (sorted by axis, i, j)
    q_axis: np.ndarray
    q_i: np.ndarray
    q_j: np.ndarray
    q_xi: np.ndarray         # coordinate of the crossing along the edge axis
    q_comp: np.ndarray
    q_theta: np.ndarray
    q_s: np.ndarray          # arc length in the Ω orientation
    # components
    comp_L: np.ndarray
    comp_M: np.ndarray
    comp_off: np.ndarray
    # control points (concatenated by component)
    z_comp: np.ndarray
    z_knot: np.ndarray
    z_theta: np.ndarray
    z: np.ndarray            # (2, M)

    @property
    def M(self):
        return int(self.comp_M.sum())


def _bisect(comp, x0, y0, axis, h, want):
    """Bisection on the Ω-side predicate along an edge: t ∈ [0,1], 64 halvings (R30)."""
    a = np.zeros_like(x0)
    b = np.ones_like(x0)
    for _ in range(64):
        m = 0.5 * (a + b)
        xm = x0 + (m * h if axis == 0 else 0.0)
        ym = y0 + (m * h if axis == 1 else 0.0)
        same = geo.omega_side(comp, xm, ym) == want
        a = np.where(same, m, a)
        b = np.where(same, b, m)
    return 0.5 * (a + b)


def build(prob, check_clearance=True) -> Setup2D:
    assert prob.dim == 2
    n, lo = prob.n, prob.lo
    h = (prob.hi - prob.lo) / n
    x = lo + np.arange(n + 1) * h                       # O1: x_i = lo + i h
    X, Y = np.meshgrid(x, x, indexing="ij")
    comps = prob.comps
    side = geo.in_omega(comps, X, Y)                    # O2/R30
    # O3: irregular iff an axis neighbour lies on the other side
    irr = np.zeros_like(side)
    d0 = side[1:, :] != side[:-1, :]
    d1 = side[:, 1:] != side[:, :-1]
    irr[1:, :] |= d0
    irr[:-1, :] |= d0
    irr[:, 1:] |= d1
    irr[:, :-1] |= d1
    ii, jj = np.nonzero(irr)
    if check_clearance and ii.size and (ii.min() < 2 or jj.min() < 2 or ii.max() > n - 2 or jj.max() > n - 2):
        raise GeometryError("Γ too close to the box boundary (R32)")

    # O4: intersections on sign-change edges
    recs = []
    for axis, dmask in ((0, d0), (1, d1)):
        ei, ej = np.nonzero(dmask)
        if ei.size == 0:
            continue
        x0, y0 = x[ei], x[ej]
        x1 = x0 + (h if axis == 0 else 0.0)
        y1 = y0 + (h if axis == 1 else 0.0)
        owner = np.full(ei.size, -1)
        count = np.zeros(ei.size, dtype=np.int64)
        for c, comp in enumerate(comps):
            ch = geo.omega_side(comp, x0, y0) != geo.omega_side(comp, x1, y1)
            owner = np.where(ch, c, owner)
            count += ch
        if np.any(count != 1):
            raise GeometryError("edge crossed by several components (R31)")
        for c, comp in enumerate(comps):
            sel = owner == c
            if not np.any(sel):
                continue
            a0, b0 = x0[sel], y0[sel]
            want = geo.omega_side(comp, a0, b0)
            # double-crossing check at interior samples (R31)
            prev = want.copy()
            changes = np.zeros(a0.size, dtype=np.int64)
            for t in (0.2, 0.4, 0.6, 0.8, 1.0):
                cur = geo.omega_side(comp, a0 + (t * h if axis == 0 else 0.0), b0 + (t * h if axis == 1 else 0.0))
                changes += cur != prev
                prev = cur
            if np.any(changes != 1):
                raise GeometryError("edge crossed more than once (R31)")
            t = _bisect(comp, a0, b0, axis, h, want)
            xi = (a0 if axis == 0 else b0) + t * h
            px = xi if axis == 0 else a0
            py = xi if axis == 1 else b0
            cx, cy = comp.center[0], comp.center[1]
            if comp.kind == ELLIPSE:
                th = np.arctan2((py - cy) / comp.p[1], (px - cx) / comp.p[0])
            else:
                th = np.arctan2(py - cy, px - cx)
            th = np.mod(th, 2 * math.pi)
            recs.append((np.full(a0.size, axis), ei[sel], ej[sel], xi, np.full(a0.size, c), th))
    q_axis = np.concatenate([r[0] for r in recs])
    q_i = np.concatenate([r[1] for r in recs])
    q_j = np.concatenate([r[2] for r in recs])
    q_xi = np.concatenate([r[3] for r in recs])
    q_comp = np.concatenate([r[4] for r in recs])
    q_th = np.concatenate([r[5] for r in recs])
    order = np.lexsort((q_j, q_i, q_axis))
    q_axis, q_i, q_j, q_xi, q_comp, q_th = (a[order] for a in (q_axis, q_i, q_j, q_xi, q_comp, q_th))

    # O5: control points at uniform arc length in the Ω orientation (R11)
    L = np.array([geo.perimeter(c) for c in comps])
    Mc = np.array([c.n_ctrl if c.n_ctrl > 0 else geo.default_ctrl_count(L[k], h) for k, c in enumerate(comps)])
    off = np.concatenate([[0], np.cumsum(Mc)[:-1]])
    z_comp, z_knot, z_th = [], [], []
    for k, c in enumerate(comps):
        s = np.arange(Mc[k]) * (L[k] / Mc[k])
        s_ccw = s if c.role != HOLE else np.mod(L[k] - s, L[k])
        th = geo.theta_of_s_ccw(c, s_ccw)
        z_comp.append(np.full(Mc[k], k))
        z_knot.append(np.arange(Mc[k]))
        z_th.append(th)
    z_comp = np.concatenate(z_comp)
    z_knot = np.concatenate(z_knot)
    z_th = np.concatenate(z_th)
    z = np.concatenate([geo.curve(comps[k], z_th[z_comp == k])[0] for k in range(len(comps))], axis=1)

    q_s = np.empty_like(q_xi)
    for k, c in enumerate(comps):
        sel = q_comp == k
        q_s[sel] = geo.s_omega(c, q_th[sel], L[k])

    return Setup2D(prob, n, h, lo, x, side, irr, q_axis, q_i, q_j, q_xi, q_comp, q_th, q_s,
                   L, Mc, off, z_comp, z_knot, z_th, z)


def stencil(st: Setup2D):
    """Six-point stencil per control point (reading R14).

    Centre c = nearest node floor(t + 1/2); σ_a = +1 if z_a ≥ x_a(c) else −1;
    nodes {c, c+e_x, c−e_x, c+e_y, c−e_y, c + σ_x e_x + σ_y e_y}.  Returns (M, 6, 2) ints.
    """
    u = (st.z - st.lo) / st.h
    c = np.floor(u + 0.5).astype(np.int64)
    xc = st.lo + c * st.h
    sg = np.where(st.z >= xc, 1, -1)
    ci, cj = c[0], c[1]
    si, sj = sg[0], sg[1]
    nodes = np.stack([
        np.stack([ci, cj], -1),
        np.stack([ci + 1, cj], -1),
        np.stack([ci - 1, cj], -1),
        np.stack([ci, cj + 1], -1),
        np.stack([ci, cj - 1], -1),
        np.stack([ci + si, cj + sj], -1),
    ], axis=1)
    return nodes
