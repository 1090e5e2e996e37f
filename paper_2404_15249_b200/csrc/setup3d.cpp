// Host-side setup of the 3D KFBI interface problem (Procedure 1; "analogous").
//
// Readings: R12 control points = Γ ∩ grid-edge intersection nodes with densities fitted by
// an unweighted tangent-plane least-squares quadratic over the control points whose edge low-end node
// lies in the 5×5×5 node block around the point's own; R13 Monge-patch jump formulas; R14 ten-point
// stencil {c, c±e_a, c+σ_x e_x+σ_y e_y, c+σ_x e_x+σ_z e_z, c+σ_y e_y+σ_z e_z}.
#include <algorithm>
#include <cmath>
#include <unordered_map>

#include "kfbi_impl.h"

namespace kfbi {
namespace {

double level3(const Comp& c, double x, double y, double z) {
  const double dx = x - c.c[0], dy = y - c.c[1], dz = z - c.c[2];
  if (c.kind == KFBI_ELLIPSOID) {
    const double u = dx / c.p[0], v = dy / c.p[1], w = dz / c.p[2];
    return u * u + v * v + w * w - 1.0;
  }
  const double q = std::sqrt(dx * dx + dy * dy) - c.p[0];
  return q * q + dz * dz - c.p[1] * c.p[1];
}

inline bool inside3(const Comp& c, double x, double y, double z) { return level3(c, x, y, z) <= 0.0; }

// ∇ℓ, D²ℓ
void grad_hess(const Comp& c, const double* p, double* g, double H[3][3]) {
  const double d[3] = {p[0] - c.c[0], p[1] - c.c[1], p[2] - c.c[2]};
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) H[a][b] = 0.0;
  if (c.kind == KFBI_ELLIPSOID) {
    for (int a = 0; a < 3; ++a) {
      g[a] = 2.0 * d[a] / (c.p[a] * c.p[a]);
      H[a][a] = 2.0 / (c.p[a] * c.p[a]);
    }
    return;
  }
  const double rho = std::sqrt(d[0] * d[0] + d[1] * d[1]), q = rho - c.p[0];
  g[0] = 2.0 * q * d[0] / rho;
  g[1] = 2.0 * q * d[1] / rho;
  g[2] = 2.0 * d[2];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b)
      H[a][b] = 2.0 * d[a] * d[b] / (rho * rho) + 2.0 * q * ((a == b ? 1.0 : 0.0) / rho - d[a] * d[b] / (rho * rho * rho));
  H[2][2] = 2.0;
}

bool lu_solve_n(int n, double* A, double* b) {
  for (int k = 0; k < n; ++k) {
    int piv = k;
    for (int i = k + 1; i < n; ++i)
      if (std::fabs(A[i * n + k]) > std::fabs(A[piv * n + k])) piv = i;
    if (std::fabs(A[piv * n + k]) < 1e-300) return false;
    if (piv != k) {
      for (int j = 0; j < n; ++j) std::swap(A[k * n + j], A[piv * n + j]);
      std::swap(b[k], b[piv]);
    }
    for (int i = k + 1; i < n; ++i) {
      const double f = A[i * n + k] / A[k * n + k];
      for (int j = k; j < n; ++j) A[i * n + j] -= f * A[k * n + j];
      b[i] -= f * b[k];
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int j = i + 1; j < n; ++j) s -= A[i * n + j] * b[j];
    b[i] = s / A[i * n + i];
  }
  return true;
}

}  // namespace

void build_setup3(Setup3& S, const kfbi_grid* g, const kfbi_boundary* b, const kfbi_pde* pde, const DeviceScratch* dev) {
  if (b->ncomp != 1) throw ArgError("3D: exactly one (outer) surface is supported");
  const kfbi_component& in = b->comp[0];
  if (in.kind != KFBI_ELLIPSOID && in.kind != KFBI_TORUS) throw ArgError("3D surfaces: ellipsoid or torus");
  if (in.role != KFBI_OUTER) throw ArgError("3D surface must be the outer boundary");
  const int N = g->n[0];
  if (g->n[1] != N || g->n[2] != N || N < 32 || N > 512 || (N & (N - 1)))
    throw ArgError("3D: n must be equal powers of two in [32, 512]");
  if (pde->bc != KFBI_DIRICHLET && pde->bc != KFBI_NEUMANN) throw ArgError("bc must be DIRICHLET or NEUMANN");
  if (pde->bc == KFBI_NEUMANN && !(pde->kappa > 0)) throw UnsupportedError("Neumann needs kappa > 0 (S:555)");
  S.neumann = pde->bc == KFBI_NEUMANN;
  const double h = (g->hi[0] - g->lo[0]) / N;
  for (int a = 1; a < 3; ++a)
    if (std::fabs((g->hi[a] - g->lo[a]) / N - h) > 1e-12 * h || std::fabs(g->lo[a] - g->lo[0]) > 1e-12 * h)
      throw ArgError("grid spacing must be equal on all axes (P:559) and the box a cube");
  S.N = N;
  S.P = N / BL;
  S.lo = g->lo[0];
  S.h = h;
  S.kappa = pde->kappa;
  Comp& C = S.comp;
  C = Comp{};
  C.kind = in.kind;
  C.role = in.role;
  for (int a = 0; a < 3; ++a) C.c[a] = in.center[a];
  for (int a = 0; a < 4; ++a) C.p[a] = in.p[a];
  const double lo = S.lo;
  const int W = N + 1;
  auto X = [&](int i) { return lo + i * h; };
  auto lin = [&](int i, int j, int k) { return ((size_t)i * W + j) * W + k; };

  if (dev) {   // classification, edges, bisection and the irregular-node lists on the GPU (NEXT-3)
    gpu_setup_phases3(S, dev->ptr, dev->bytes, dev->stream);
  } else {
    // classification
    S.side.assign((size_t)W * W * W, 0);
  #pragma omp parallel for schedule(static)
    for (int i = 0; i < W; ++i)
      for (int j = 0; j < W; ++j)
        for (int k = 0; k < W; ++k) S.side[lin(i, j, k)] = inside3(C, X(i), X(j), X(k)) ? 1 : 0;
    auto side = [&](int i, int j, int k) { return S.side[lin(i, j, k)]; };

    // intersections on sign-change edges, sorted by (axis, i, j, k)
    struct E { int axis, i, j, k; };
    std::vector<E> edges;
    for (int axis = 0; axis < 3; ++axis) {
      std::vector<std::vector<E>> part(W);
  #pragma omp parallel for schedule(dynamic, 4)
      for (int i = 0; i < W; ++i)
        for (int j = 0; j < W; ++j)
          for (int k = 0; k < W; ++k) {
            const int i1 = i + (axis == 0), j1 = j + (axis == 1), k1 = k + (axis == 2);
            if (i1 > N || j1 > N || k1 > N) continue;
            if (side(i, j, k) != side(i1, j1, k1)) part[i].push_back({axis, i, j, k});
          }
      for (auto& p : part) edges.insert(edges.end(), p.begin(), p.end());
    }
    const int nq = (int)edges.size();
    S.nq = nq;
    S.q_axis.resize(nq); S.q_i.resize(nq); S.q_j.resize(nq); S.q_k.resize(nq);
    S.q_xi.resize(nq);
    bool bad = false;
  #pragma omp parallel for schedule(dynamic, 256)
    for (int e = 0; e < nq; ++e) {
      const E ed = edges[e];
      double p0[3] = {X(ed.i), X(ed.j), X(ed.k)};
      const bool want = inside3(C, p0[0], p0[1], p0[2]);
      bool prev = want;
      int changes = 0;
      for (double t : {0.2, 0.4, 0.6, 0.8, 1.0}) {
        double p[3] = {p0[0], p0[1], p0[2]};
        p[ed.axis] += t * h;
        const bool cur = inside3(C, p[0], p[1], p[2]);
        changes += cur != prev;
        prev = cur;
      }
      if (changes != 1) bad = true;
      double a = 0, bb = 1;
      for (int it = 0; it < 64; ++it) {
        const double m = 0.5 * (a + bb);
        double p[3] = {p0[0], p0[1], p0[2]};
        p[ed.axis] += m * h;
        if (inside3(C, p[0], p[1], p[2]) == want) a = m; else bb = m;
      }
      const double t = 0.5 * (a + bb);
      double pos[3] = {p0[0], p0[1], p0[2]};
      pos[ed.axis] += t * h;
      S.q_axis[e] = ed.axis; S.q_i[e] = ed.i; S.q_j[e] = ed.j; S.q_k[e] = ed.k;
      S.q_xi[e] = pos[ed.axis];
    }
    if (bad) throw GeomError("grid edge crossed more than once (R31)");
    // irregular nodes (6 neighbours) sorted by (i, j, k), CSR to their incident intersections
    std::unordered_map<int64_t, int> qidx;
    qidx.reserve(2 * (size_t)nq);
    auto key = [&](int axis, int i, int j, int k) { return (int64_t)axis * W * W * W + (int64_t)lin(i, j, k); };
    for (int e = 0; e < nq; ++e) qidx[key(S.q_axis[e], S.q_i[e], S.q_j[e], S.q_k[e])] = e;
    S.irr_lin.clear(); S.irr_side.clear(); S.irr_ptr.assign(1, 0); S.pair_q.clear(); S.pair_d.clear();
    S.irr_ijk.clear();
    for (int i = 1; i < N; ++i)
      for (int j = 1; j < N; ++j)
        for (int k = 1; k < N; ++k) {
          const int s0 = side(i, j, k);
          const int nb[6][3] = {{i - 1, j, k}, {i + 1, j, k}, {i, j - 1, k}, {i, j + 1, k}, {i, j, k - 1}, {i, j, k + 1}};
          bool irr = false;
          for (auto& q : nb) irr |= side(q[0], q[1], q[2]) != s0;
          if (!irr) continue;
          if (i < 2 || j < 2 || k < 2 || i > N - 2 || j > N - 2 || k > N - 2)
            throw GeomError("Γ too close to the box boundary (R32)");
          S.irr_lin.push_back((int64_t)(i - 1) * N * N + (int64_t)j * N + k);
          S.irr_ijk.push_back(i); S.irr_ijk.push_back(j); S.irr_ijk.push_back(k);
          S.irr_side.push_back((int8_t)s0);
          for (int q = 0; q < 6; ++q) {
            const int oi = nb[q][0], oj = nb[q][1], ok = nb[q][2];
            if (side(oi, oj, ok) == s0) continue;
            const int axis = q / 2;
            const int li = std::min(i, oi), lj = std::min(j, oj), lk = std::min(k, ok);
            auto it = qidx.find(key(axis, li, lj, lk));
            if (it == qidx.end()) throw GeomError("internal: missing intersection");
            const int e = it->second;
            const double xbar = axis == 0 ? X(oi) : axis == 1 ? X(oj) : X(ok);
            S.pair_q.push_back(e);
            S.pair_d.push_back(xbar - S.q_xi[e]);
          }
          S.irr_ptr.push_back((int)S.pair_q.size());
        }
    S.nirr = (int)S.irr_lin.size();
  }
  // frames at the intersections (common to the host and device paths): the node coordinates with the
  // edge axis replaced by ξ
  const int nqf = S.nq;
  S.q_pos.resize(3 * (size_t)nqf); S.q_n.resize(3 * (size_t)nqf);
  S.q_e1.resize(3 * (size_t)nqf); S.q_e2.resize(3 * (size_t)nqf); S.q_kab.resize(3 * (size_t)nqf);
#pragma omp parallel for schedule(static)
  for (int e = 0; e < nqf; ++e) {
    double pos[3] = {X(S.q_i[e]), X(S.q_j[e]), X(S.q_k[e])};
    pos[S.q_axis[e]] = S.q_xi[e];
    // frame: n = ∇ℓ/|∇ℓ|, e1 = normalize(n × u*), e2 = n × e1, κ_ab = −e_aᵀ D²ℓ e_b / |∇ℓ|
    double gr[3], H[3][3];
    grad_hess(C, pos, gr, H);
    const double gn = std::sqrt(gr[0] * gr[0] + gr[1] * gr[1] + gr[2] * gr[2]);
    double n[3] = {gr[0] / gn, gr[1] / gn, gr[2] / gn};
    int ax = 0;
    for (int q = 1; q < 3; ++q)
      if (std::fabs(n[q]) < std::fabs(n[ax])) ax = q;
    double u[3] = {0, 0, 0};
    u[ax] = 1.0;
    double e1[3] = {n[1] * u[2] - n[2] * u[1], n[2] * u[0] - n[0] * u[2], n[0] * u[1] - n[1] * u[0]};
    const double l1 = std::sqrt(e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2]);
    for (double& v : e1) v /= l1;
    double e2[3] = {n[1] * e1[2] - n[2] * e1[1], n[2] * e1[0] - n[0] * e1[2], n[0] * e1[1] - n[1] * e1[0]};
    auto quad = [&](const double* x, const double* y) {
      double s = 0;
      for (int r = 0; r < 3; ++r)
        for (int c2 = 0; c2 < 3; ++c2) s += x[r] * H[r][c2] * y[c2];
      return s;
    };
    for (int r = 0; r < 3; ++r) {
      S.q_pos[3 * e + r] = pos[r];
      S.q_n[3 * e + r] = n[r];
      S.q_e1[3 * e + r] = e1[r];
      S.q_e2[3 * e + r] = e2[r];
    }
    S.q_kab[3 * e] = -quad(e1, e1) / gn;
    S.q_kab[3 * e + 1] = -quad(e1, e2) / gn;
    S.q_kab[3 * e + 2] = -quad(e2, e2) / gn;
  }
  const int nq = S.nq;
  auto side = [&](int i, int j, int k) { return S.side[lin(i, j, k)]; };
  bool bad = false;

  // LSQ neighbours: 5×5×5 block of edge low-end nodes; scaled normal matrix inverse
  std::unordered_map<int64_t, std::vector<int>> bucket;
  bucket.reserve(2 * (size_t)nq);
  for (int e = 0; e < nq; ++e) bucket[(int64_t)lin(S.q_i[e], S.q_j[e], S.q_k[e])].push_back(e);
  std::vector<std::vector<int>> nbl(nq);
#pragma omp parallel for schedule(dynamic, 256)
  for (int e = 0; e < nq; ++e) {
    auto& L = nbl[e];
    for (int di = -2; di <= 2; ++di)
      for (int dj = -2; dj <= 2; ++dj)
        for (int dk = -2; dk <= 2; ++dk) {
          const int i = S.q_i[e] + di, j = S.q_j[e] + dj, k = S.q_k[e] + dk;
          if (i < 0 || j < 0 || k < 0 || i > N || j > N || k > N) continue;
          auto it = bucket.find((int64_t)lin(i, j, k));
          if (it == bucket.end()) continue;
          for (int q : it->second)
            if (q != e) L.push_back(q);
        }
    std::sort(L.begin(), L.end());
  }
  S.lsq_ptr.assign(1, 0);
  S.lsq_nb.clear();
  for (int e = 0; e < nq; ++e) {
    S.lsq_nb.insert(S.lsq_nb.end(), nbl[e].begin(), nbl[e].end());
    S.lsq_ptr.push_back((int)S.lsq_nb.size());
  }
  S.lsq_G.assign(15 * (size_t)nq, 0.0);
  S.lsq_t.assign(2 * S.lsq_nb.size(), 0.0);
#pragma omp parallel for schedule(dynamic, 256)
  for (int e = 0; e < nq; ++e) {
    const auto& L = nbl[e];
    int slot = S.lsq_ptr[e];
    if (L.size() < 8) { bad = true; continue; }
    // Â columns (t1/h, t2/h, ½(t1/h)², (t1/h)(t2/h), ½(t2/h)²); G = ÂᵀÂ
    double G[25] = {0};
    for (int q : L) {
      double d[3];
      for (int r = 0; r < 3; ++r) d[r] = (S.q_pos[3 * q + r] - S.q_pos[3 * e + r]) / h;
      double t1 = 0, t2 = 0;
      for (int r = 0; r < 3; ++r) { t1 += S.q_e1[3 * e + r] * d[r]; t2 += S.q_e2[3 * e + r] * d[r]; }
      S.lsq_t[2 * (size_t)slot] = t1;   // the fit's tangent coordinates (/h), streamed by k_lsq3
      S.lsq_t[2 * (size_t)slot + 1] = t2;
      ++slot;
      const double a[5] = {t1, t2, 0.5 * t1 * t1, t1 * t2, 0.5 * t2 * t2};
      for (int r = 0; r < 5; ++r)
        for (int c2 = 0; c2 < 5; ++c2) G[r * 5 + c2] += a[r] * a[c2];
    }
    double Ginv[25];
    for (int col = 0; col < 5; ++col) {
      double A[25], rhs[5] = {0, 0, 0, 0, 0};
      for (int r = 0; r < 25; ++r) A[r] = G[r];
      rhs[col] = 1.0;
      if (!lu_solve_n(5, A, rhs)) { bad = true; break; }
      for (int r = 0; r < 5; ++r) Ginv[r * 5 + col] = rhs[r];
    }
    int w = 0;
    for (int r = 0; r < 5; ++r)
      for (int c2 = r; c2 < 5; ++c2) S.lsq_G[15 * (size_t)e + w++] = 0.5 * (Ginv[r * 5 + c2] + Ginv[c2 * 5 + r]);
  }
  if (bad) throw GeomError("LSQ fit needs ≥ 8 non-degenerate neighbours (R12)");

  // ten-point stencils + row 0 of the inverse local system (R14, R16); NEXT-3: on the device
  // with the same arithmetic when the setup runs there (setup_gpu.cu, bit-identical)
  if (dev) {
    gpu_stencil_phase3(S, dev->ptr, dev->bytes, dev->stream);
  } else {
  S.st_c.assign(3 * (size_t)nq, 0);
  S.st_code.assign(nq, 0);
  S.st_w.assign(10 * (size_t)nq, 0.0);
  S.st_wn.assign(10 * (size_t)nq, 0.0);
  S.st_nodes_ij.assign(30 * (size_t)nq, 0);
#pragma omp parallel for schedule(static)
  for (int e = 0; e < nq; ++e) {
    int c[3], sg[3];
    const double* z = &S.q_pos[3 * e];
    for (int a = 0; a < 3; ++a) {
      c[a] = (int)std::floor((z[a] - lo) / h + 0.5);
      sg[a] = z[a] >= X(c[a]) ? 1 : -1;
    }
    const int off[10][3] = {{0, 0, 0}, {1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1},
                            {sg[0], sg[1], 0}, {sg[0], 0, sg[2]}, {0, sg[1], sg[2]}};
    double A[100], w[10];
    int ext = 0;
    for (int p = 0; p < 10; ++p) {
      const int ni = c[0] + off[p][0], nj = c[1] + off[p][1], nk = c[2] + off[p][2];
      if (ni < 1 || nj < 1 || nk < 1 || ni > N - 1 || nj > N - 1 || nk > N - 1) { bad = true; continue; }
      S.st_nodes_ij[30 * (size_t)e + 3 * p] = ni;
      S.st_nodes_ij[30 * (size_t)e + 3 * p + 1] = nj;
      S.st_nodes_ij[30 * (size_t)e + 3 * p + 2] = nk;
      if (!side(ni, nj, nk)) ext |= 1 << p;
      const double dx = X(ni) - z[0], dy = X(nj) - z[1], dz = X(nk) - z[2];
      const double row[10] = {1, dx, dy, dz, 0.5 * dx * dx, 0.5 * dy * dy, 0.5 * dz * dz, dx * dy, dx * dz, dy * dz};
      for (int q = 0; q < 10; ++q) A[q * 10 + p] = row[q];   // transpose: Aᵀ w = e_0
      w[p] = p == 0 ? 1.0 : 0.0;
    }
    double A2[100], wn[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    std::copy(A, A + 100, A2);
    if (!lu_solve_n(10, A, w)) bad = true;
    for (int p = 0; p < 10; ++p) S.st_w[10 * (size_t)e + p] = w[p];
    // normal derivative n·∇ of the local quadratic (Neumann, R38): Aᵀ w_n = (0, n, 0, …)
    for (int a = 0; a < 3; ++a) wn[1 + a] = S.q_n[3 * (size_t)e + a];
    if (!lu_solve_n(10, A2, wn)) bad = true;
    for (int p = 0; p < 10; ++p) S.st_wn[10 * (size_t)e + p] = wn[p];
    for (int a = 0; a < 3; ++a) S.st_c[3 * e + a] = c[a];
    S.st_code[e] = ext | ((sg[0] > 0) << 10) | ((sg[1] > 0) << 11) | ((sg[2] > 0) << 12);
  }
  if (bad) throw GeomError("interpolation stencil leaves the grid or is singular");
  }

  // sparse K_D path: irregular nodes by grid row (i−1)·N + j, and the distinct stencil nodes by row
  {
    const size_t nrows = (size_t)(N - 1) * N;
    S.irr_row_ptr.assign(nrows + 1, 0);
    for (int n = 0; n < S.nirr; ++n) ++S.irr_row_ptr[S.irr_lin[n] / N + 1];
    for (size_t r = 0; r < nrows; ++r) S.irr_row_ptr[r + 1] += S.irr_row_ptr[r];
    S.max_plane_irr = 0;
    for (int i = 0; i < N - 1; ++i)
      S.max_plane_irr = std::max(S.max_plane_irr, S.irr_row_ptr[(size_t)(i + 1) * N] - S.irr_row_ptr[(size_t)i * N]);
    if (S.max_plane_irr > 12288) throw GeomError("more than 12288 irregular nodes in one grid plane");
    // per plane, rows by descending irregular count (the forward kernel deals them out in snake order
    // so that every thread gets a balanced share of the entries)
    S.irr_row_perm.resize(nrows);
    for (int i = 0; i < N - 1; ++i) {
      int16_t* pr = &S.irr_row_perm[(size_t)i * N];
      for (int a = 0; a < N; ++a) pr[a] = (int16_t)a;
      const int32_t* rp = &S.irr_row_ptr[(size_t)i * N];
      std::stable_sort(pr, pr + N, [&](int16_t x, int16_t y) { return rp[x + 1] - rp[x] > rp[y + 1] - rp[y]; });
    }
    // rows with more than kHeavyRow entries come first in each plane's order; the forward kernel
    // splits each of them over 8 lanes
    S.irr_row_nheavy.assign(N - 1, 0);
    for (int i = 0; i < N - 1; ++i) {
      const int32_t* rp = &S.irr_row_ptr[(size_t)i * N];
      int h = 0;
      for (int a = 0; a < N; ++a) h += rp[a + 1] - rp[a] > kHeavyRow;
      S.irr_row_nheavy[i] = h;
    }
    std::vector<int64_t> nodes(10 * (size_t)nq);
    for (size_t e = 0; e < 10 * (size_t)nq; ++e)
      nodes[e] = (int64_t)(S.st_nodes_ij[3 * e] - 1) * N * N + (int64_t)S.st_nodes_ij[3 * e + 1] * N +
                 S.st_nodes_ij[3 * e + 2];
    std::sort(nodes.begin(), nodes.end());
    nodes.erase(std::unique(nodes.begin(), nodes.end()), nodes.end());
    S.zrow_id.clear(); S.zrow_ptr.assign(1, 0); S.znode_b.clear();
    for (size_t e = 0; e < nodes.size(); ++e) {
      const int32_t row = (int32_t)(nodes[e] / N);
      if (S.zrow_id.empty() || S.zrow_id.back() != row) {
        if (!S.zrow_id.empty()) S.zrow_ptr.push_back((int32_t)e);
        S.zrow_id.push_back(row);
      }
      S.znode_b.push_back((int32_t)(nodes[e] % N));
    }
    S.zrow_ptr.push_back((int32_t)nodes.size());
    S.zplane_ptr.assign(N, 0);
    for (int i = 1; i <= N; ++i)
      S.zplane_ptr[i - 1] = (int32_t)(std::lower_bound(S.zrow_id.begin(), S.zrow_id.end(), (i - 1) * N) -
                                      S.zrow_id.begin());
    // per grid plane i ∈ [1, N): bit 0 the sparse forward source is non-zero (irregular nodes in the
    // plane), bit 1 the y-inverse reads the plane (stencil rows): the sparse K_D apply skips the rest
    S.plane_flags.assign(N + 1, 0);
    for (int i = 1; i < N; ++i)
      S.plane_flags[i] = (uint8_t)((S.irr_row_ptr[(size_t)i * N] > S.irr_row_ptr[(size_t)(i - 1) * N] ? 1 : 0) |
                                   (S.zplane_ptr[i] > S.zplane_ptr[i - 1] ? 2 : 0));
  }

  // fast-solver tables: modes m = ll·N + kk (DST along z → ll, along y → kk), tridiagonal along x
  const size_t K = (size_t)N * N;
  S.sin_tab.resize(N / 2 + 1);
  for (int r = 0; r <= N / 2; ++r) S.sin_tab[r] = std::sin(3.14159265358979323846 * (double)r / N);
  S.tw.resize(4 * (size_t)N);
  for (int m = 0; m < 2 * N; ++m) {   // folded onto the quarter wave so that symmetric entries agree exactly
    auto sn = [&](int r) { double sg = 1.0; if (r >= N) { r -= N; sg = -1.0; } if (r > N / 2) r = N - r; return sg * S.sin_tab[r]; };
    S.tw[2 * m] = sn((m + N / 2) % (2 * N));
    S.tw[2 * m + 1] = sn(m);
  }
  S.dk.assign(K, -4.0);
  S.zr.assign((size_t)LB * K, 0.0);
  S.red_a.assign(K, 0.0);
  S.red_b.assign(K, 1.0);
  for (int ll = 1; ll < N; ++ll)
    for (int kk = 1; kk < N; ++kk) {
      const size_t m = (size_t)ll * N + kk;
      const double s1 = std::sin(3.14159265358979323846 * kk / (2.0 * N));
      const double s2 = std::sin(3.14159265358979323846 * ll / (2.0 * N));
      const double d = -(2.0 + 4.0 * s1 * s1 + 4.0 * s2 * s2 + S.kappa * h * h);
      S.dk[m] = d;
      double cs[LB], c = d;
      for (int p = 0; p < LB; ++p) {
        if (p) c = d - 1.0 / c;
        cs[p] = c;
      }
      double x = 1.0 / cs[LB - 1];
      S.zr[(size_t)(LB - 1) * K + m] = x;
      for (int p = LB - 2; p >= 0; --p) {
        x = -x / cs[p];
        S.zr[(size_t)p * K + m] = x;
      }
      S.red_a[m] = -S.zr[m];
      S.red_b[m] = d - 2.0 * S.zr[(size_t)(LB - 1) * K + m];
    }
}

}  // namespace kfbi
