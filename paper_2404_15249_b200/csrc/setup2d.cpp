// Host-side setup of the 2D KFBI interface problem (Procedure 1).
//
// Grid and node classification, grid-line ∩ Γ intersection nodes,
// quasi-uniform control points, six-point interpolation stencils with their
// precomputed inverse rows, spline filters for the density (reading
// R10) and the per-mode tables of the partitioned tridiagonal solve.
// Runs once per geometry, off the timed path.  OpenMP over grid nodes.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <unordered_map>

#include "kfbi_impl.h"

#include <chrono>
#include <cstdio>
#include <cstdlib>
namespace {
// KFBI_SETUP_TIMING=1 prints the wall time of each setup phase (host profiling aid)
void setup_tick(const char* next) {
  static bool on = std::getenv("KFBI_SETUP_TIMING") != nullptr;
  static auto last = std::chrono::steady_clock::now();
  if (!on) return;
  const auto now = std::chrono::steady_clock::now();
  std::fprintf(stderr, "[setup] %.3f s → %s\n", std::chrono::duration<double>(now - last).count(), next);
  last = now;
}
}  // namespace

namespace kfbi {
namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 6.28318530717958647692;
constexpr int kPanels = 64;
constexpr int kGL = 16;

struct GaussLegendre {
  double x[kGL], w[kGL];
  GaussLegendre() {
    // Newton on the Legendre polynomial P_16 from Chebyshev initial guesses.
    for (int i = 0; i < kGL; ++i) {
      double z = std::cos(kPi * (i + 0.75) / (kGL + 0.5)), dp = 0;
      for (int it = 0; it < 100; ++it) {
        double p0 = 1, p1 = z;
        for (int k = 2; k <= kGL; ++k) {
          double p2 = ((2 * k - 1) * z * p1 - (k - 1) * p0) / k;
          p0 = p1;
          p1 = p2;
        }
        dp = kGL * (z * p1 - p0) / (z * z - 1);
        double dz = p1 / dp;
        z -= dz;
        if (std::fabs(dz) < 1e-17) break;
      }
      x[i] = z;
      w[i] = 2.0 / ((1 - z * z) * dp * dp);
    }
  }
};
const GaussLegendre& gl() {
  static GaussLegendre g;
  return g;
}

void curve(const Comp& c, double th, double* g, double* g1, double* g2) {
  if (c.kind == KFBI_ELLIPSE) {
    double cs = std::cos(th), sn = std::sin(th);
    g[0] = c.c[0] + c.p[0] * cs;
    g[1] = c.c[1] + c.p[1] * sn;
    g1[0] = -c.p[0] * sn;
    g1[1] = c.p[1] * cs;
    g2[0] = -c.p[0] * cs;
    g2[1] = -c.p[1] * sn;
  } else {  // star ρ = r(1 + ε sin(m(θ − α)))
    double r = c.p[0], e = c.p[1], m = c.p[2], a = c.p[3];
    double sa = std::sin(m * (th - a)), ca = std::cos(m * (th - a));
    double rho = r * (1 + e * sa), rho1 = r * e * m * ca, rho2 = -r * e * m * m * sa;
    double cs = std::cos(th), sn = std::sin(th);
    g[0] = c.c[0] + rho * cs;
    g[1] = c.c[1] + rho * sn;
    g1[0] = rho1 * cs - rho * sn;
    g1[1] = rho1 * sn + rho * cs;
    g2[0] = rho2 * cs - 2 * rho1 * sn - rho * cs;
    g2[1] = rho2 * sn + 2 * rho1 * cs - rho * sn;
  }
}

double speed(const Comp& c, double th) {
  double g[2], g1[2], g2[2];
  curve(c, th, g, g1, g2);
  return std::sqrt(g1[0] * g1[0] + g1[1] * g1[1]);
}

double level(const Comp& c, double x, double y) {
  if (c.kind == KFBI_ELLIPSE) {
    double u = (x - c.c[0]) / c.p[0], v = (y - c.c[1]) / c.p[1];
    return u * u + v * v - 1.0;
  }
  double dx = x - c.c[0], dy = y - c.c[1];
  return std::sqrt(dx * dx + dy * dy) - c.p[0] * (1 + c.p[1] * std::sin(c.p[2] * (std::atan2(dy, dx) - c.p[3])));
}

inline bool omega_side(const Comp& c, double x, double y) {
  double l = level(c, x, y);
  return c.role == KFBI_OUTER ? (l <= 0.0) : (l >= 0.0);
}

// composite Gauss–Legendre arc length s_ccw(θ) = ∫_0^θ |γ'|
struct ArcLength {
  const Comp* c;
  double prefix[kPanels + 1];
  explicit ArcLength(const Comp& comp) : c(&comp) {
    const auto& q = gl();
    double wdt = kTwoPi / kPanels;
    prefix[0] = 0;
    for (int k = 0; k < kPanels; ++k) {
      double a = k * wdt, s = 0;
      for (int i = 0; i < kGL; ++i) s += q.w[i] * speed(comp, a + 0.5 * wdt * (q.x[i] + 1));
      prefix[k + 1] = prefix[k] + 0.5 * wdt * s;
    }
  }
  double total() const { return prefix[kPanels]; }
  double operator()(double th) const {
    const auto& q = gl();
    double wdt = kTwoPi / kPanels;
    int k = std::min((int)std::floor(th / wdt), kPanels - 1);
    double a = k * wdt, part = th - a, s = 0;
    for (int i = 0; i < kGL; ++i) s += q.w[i] * speed(*c, a + 0.5 * part * (q.x[i] + 1));
    return prefix[k] + 0.5 * part * s;
  }
  double theta_of(double s) const {
    double L = total(), th = kTwoPi * s / L;
    for (int it = 0; it < 60; ++it) {
      double r = (*this)(th) - s;
      if (std::fabs(r) <= 1e-14 * L) break;
      th -= r / speed(*c, th);
    }
    return th;
  }
};

void frame(const Comp& c, double th, double* pos, double* tau, double* taup) {
  double g[2], g1[2], g2[2];
  curve(c, th, g, g1, g2);
  double sp2 = g1[0] * g1[0] + g1[1] * g1[1], sp = std::sqrt(sp2);
  double o = c.role == KFBI_OUTER ? 1.0 : -1.0;  // Ω orientation (R8)
  tau[0] = o * g1[0] / sp;
  tau[1] = o * g1[1] / sp;
  double dot = g1[0] * g2[0] + g1[1] * g2[1];
  taup[0] = (g2[0] * sp2 - g1[0] * dot) / (sp2 * sp2);
  taup[1] = (g2[1] * sp2 - g1[1] * dot) / (sp2 * sp2);
  pos[0] = g[0];
  pos[1] = g[1];
}

// Gaussian elimination with partial pivoting: solve A x = b, A n×n row-major (destroyed).
bool lu_solve(int n, double* A, double* b) {
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
      double f = A[i * n + k] / A[k * n + k];
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

void build_setup(Setup& S, const kfbi_grid* g, const kfbi_boundary* b, const kfbi_pde* pde, const DeviceScratch* dev) {
  setup_tick("start");
  if (!g || !b || !pde || !b->comp || b->ncomp < 1) throw ArgError("null descriptor");
  if (g->dim != 2) throw ArgError("only dim = 2 is built in this library version");
  if (pde->kappa < 0) throw ArgError("kappa must be >= 0 (P:458)");
  if (pde->bc != KFBI_DIRICHLET && pde->bc != KFBI_NEUMANN) throw ArgError("bc must be DIRICHLET or NEUMANN");
  if (pde->bc == KFBI_NEUMANN && !(pde->kappa > 0)) throw UnsupportedError("Neumann needs kappa > 0 (S:555)");
  S.neumann = pde->bc == KFBI_NEUMANN;
  int N = g->n[0];
  if (g->n[1] != N || N < 64 || N > 8192 || (N & (N - 1))) throw ArgError("n must be equal powers of two in [64, 8192]");
  double h0 = (g->hi[0] - g->lo[0]) / N, h1 = (g->hi[1] - g->lo[1]) / N;
  if (!(h0 > 0) || std::fabs(h0 - h1) > 1e-12 * h0 || std::fabs(g->lo[0] - g->lo[1]) > 1e-12 * h0)
    throw ArgError("grid spacing must be equal on both axes (P:559) and the box square");
  S.dim = 2;
  S.N = N;
  S.P = N / BL;
  S.lo = g->lo[0];
  S.h = h0;
  S.kappa = pde->kappa;
  const double lo = S.lo, h = S.h;
  int nouter = 0;
  S.comps.clear();
  for (int k = 0; k < b->ncomp; ++k) {
    const kfbi_component& in = b->comp[k];
    Comp c{};
    c.kind = in.kind;
    c.role = in.role;
    for (int a = 0; a < 3; ++a) c.c[a] = in.center[a];
    for (int a = 0; a < 4; ++a) c.p[a] = in.p[a];
    c.n_ctrl = in.n_ctrl;
    if (c.kind != KFBI_ELLIPSE && c.kind != KFBI_STAR) throw ArgError("2D components must be ellipse or star");
    if (c.kind == KFBI_ELLIPSE && !(c.p[0] > 0 && c.p[1] > 0)) throw ArgError("ellipse axes must be > 0");
    if (c.kind == KFBI_STAR && !(c.p[0] > 0 && std::fabs(c.p[1]) < 1 && c.p[2] >= 1)) throw ArgError("bad star parameters");
    if (c.role == KFBI_OUTER) ++nouter;
    else if (c.role != KFBI_HOLE) throw ArgError("bad component role");
    S.comps.push_back(c);
  }
  if (nouter != 1) throw ArgError("exactly one outer component is required");
  const int nc = (int)S.comps.size();
  const int W = N + 1;
  auto X = [&](int i) { return lo + i * h; };  // O1: node coordinate lo + i h

  setup_tick("classification (P:551): Ω side o");
  // ---- classification: Ω side of every node ----
  // the device path (NEXT-3) runs classification, edges, bisection and the irregular lists in
  // setup_gpu.cu with the same arithmetic; the host continues from its lists
  std::vector<int> q_owner;
  auto side = [&](int i, int j) { return S.side[(size_t)i * W + j]; };
  if (dev) {
    if (S.comps.size() > 8) throw ArgError("at most 8 components for the device setup");
    gpu_setup_phases(S, dev->ptr, dev->bytes, dev->stream, q_owner);
  } else {
  S.side.assign((size_t)W * W, 0);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < W; ++i)
    for (int j = 0; j < W; ++j) {
      bool in = true;
      for (int c = 0; c < nc && in; ++c) in = omega_side(S.comps[c], X(i), X(j));
      S.side[(size_t)i * W + j] = in ? 1 : 0;
    }

  setup_tick("intersections on sign-change edg");
  // ---- intersections on sign-change edges ----
  S.q_axis.clear(); S.q_i.clear(); S.q_j.clear();
  for (int axis = 0; axis < 2; ++axis)
    for (int i = 0; i < W - (axis == 0); ++i)
      for (int j = 0; j < W - (axis == 1); ++j)
        if (side(i, j) != side(i + (axis == 0), j + (axis == 1))) {
          S.q_axis.push_back(axis);
          S.q_i.push_back(i);
          S.q_j.push_back(j);
        }
  // already in (axis, i, j) order
  S.nq = (int)S.q_axis.size();
  S.q_xi.resize(S.nq);
  q_owner.resize(S.nq);
  std::string err;
#pragma omp parallel for schedule(dynamic, 64)
  for (int e = 0; e < S.nq; ++e) {
    const int axis = S.q_axis[e];
    double x0 = X(S.q_i[e]), y0 = X(S.q_j[e]);
    double x1 = x0 + (axis == 0 ? h : 0.0), y1 = y0 + (axis == 1 ? h : 0.0);
    int owner = -1, count = 0;
    for (int c = 0; c < nc; ++c)
      if (omega_side(S.comps[c], x0, y0) != omega_side(S.comps[c], x1, y1)) { owner = c; ++count; }
    if (count != 1) {
#pragma omp critical
      err = "edge crossed by several components (R31)";
      continue;
    }
    const Comp& C = S.comps[owner];
    bool want = omega_side(C, x0, y0);
    // double-crossing check at interior samples (R31)
    bool prev = want;
    int changes = 0;
    const double ts[5] = {0.2, 0.4, 0.6, 0.8, 1.0};
    for (double t : ts) {
      bool cur = omega_side(C, x0 + (axis == 0 ? t * h : 0.0), y0 + (axis == 1 ? t * h : 0.0));
      changes += cur != prev;
      prev = cur;
    }
    if (changes != 1) {
#pragma omp critical
      err = "grid edge crossed more than once (R31)";
      continue;
    }
    double a = 0, bb = 1;
    for (int it = 0; it < 64; ++it) {
      double m = 0.5 * (a + bb);
      bool same = omega_side(C, x0 + (axis == 0 ? m * h : 0.0), y0 + (axis == 1 ? m * h : 0.0)) == want;
      if (same) a = m; else bb = m;
    }
    double t = 0.5 * (a + bb);
    S.q_xi[e] = (axis == 0 ? x0 : y0) + t * h;
    q_owner[e] = owner;
  }
  if (!err.empty()) throw GeomError(err);
  }   // host phases
  const int nq = S.nq;
  S.q_comp.resize(nq); S.q_knot.resize(nq);
  S.q_t.resize(nq); S.q_theta.resize(nq); S.q_t1.resize(nq); S.q_t2.resize(nq);
  S.q_p1.resize(nq); S.q_p2.resize(nq); S.q_x.resize(nq); S.q_y.resize(nq);

  // components: perimeter, control counts (R11)
  std::vector<ArcLength> arcs;
  arcs.reserve(nc);
  int off = 0;
  for (auto& c : S.comps) {
    arcs.emplace_back(c);
    c.L = arcs.back().total();
    c.M = c.n_ctrl > 0 ? c.n_ctrl : (int)std::lround(c.L / (1.18 * h));
    if (c.M < 8) throw ArgError("fewer than 8 control points on a component");
    c.off = off;
    c.delta = c.L / c.M;
    off += c.M;
  }
  for (int c = 0; c < nc; ++c) arcs[c].c = &S.comps[c];
  S.M = off;

#pragma omp parallel for schedule(dynamic, 64)
  for (int e = 0; e < nq; ++e) {
    const int owner = q_owner[e], axis = S.q_axis[e];
    const Comp& C = S.comps[owner];
    const double x0 = X(S.q_i[e]), y0 = X(S.q_j[e]), xi = S.q_xi[e];
    double px = axis == 0 ? xi : x0, py = axis == 1 ? xi : y0;
    double th = C.kind == KFBI_ELLIPSE ? std::atan2((py - C.c[1]) / C.p[1], (px - C.c[0]) / C.p[0])
                                       : std::atan2(py - C.c[1], px - C.c[0]);
    if (th < 0) th += kTwoPi;
    if (th >= kTwoPi) th -= kTwoPi;
    double s = arcs[owner](th);
    if (C.role == KFBI_HOLE) s = std::fmod(C.L - s, C.L);
    double u = s / C.delta;
    int m = (int)std::floor(u);
    double tt = u - m;
    if (m >= C.M) m -= C.M;
    double pos[2], tau[2], taup[2];
    frame(C, th, pos, tau, taup);
    S.q_comp[e] = owner; S.q_knot[e] = m;
    S.q_t[e] = tt; S.q_theta[e] = th;
    S.q_t1[e] = tau[0]; S.q_t2[e] = tau[1]; S.q_p1[e] = taup[0]; S.q_p2[e] = taup[1];
    S.q_x[e] = px; S.q_y[e] = py;
  }

  setup_tick("irregular nodes (P:551) and thei");
  // ---- irregular nodes and their incident intersections ----
  if (!dev) {
  std::unordered_map<int64_t, int> qidx;
  qidx.reserve(nq * 2);
  auto key = [&](int axis, int i, int j) { return ((int64_t)axis * W + i) * W + j; };
  for (int e = 0; e < nq; ++e) qidx[key(S.q_axis[e], S.q_i[e], S.q_j[e])] = e;
  S.irr_i.clear(); S.irr_j.clear(); S.irr_side.clear(); S.irr_ptr.assign(1, 0); S.pair_q.clear(); S.pair_d.clear();
  S.col_ptr.assign(N + 1, 0);
  S.col_mid.assign(N + 1, 0);
  // order: column i, odd rows j first, then even rows (the sweep accumulates the two parity
  // classes separately: sin(πj(N−k)/N) = (−1)^{j+1} sin(πjk/N))
  for (int i = 1; i < N; ++i) {
    for (int jj = 0; jj < N - 1; ++jj) {
      const int half_rows = N / 2;                   // odd rows 1,3,..,N−1 then even rows 2,..,N−2
      const int j = jj < half_rows ? 2 * jj + 1 : 2 * (jj - half_rows) + 2;
      int s0 = side(i, j);
      bool irr = side(i - 1, j) != s0 || side(i + 1, j) != s0 || side(i, j - 1) != s0 || side(i, j + 1) != s0;
      if (!irr) continue;
      if (i < 2 || j < 2 || i > N - 2 || j > N - 2) throw GeomError("Γ too close to the box boundary (R32)");
      S.irr_i.push_back(i);
      S.irr_j.push_back(j);
      S.irr_side.push_back((int8_t)s0);
      // the four edges at p: (axis, low end, other endpoint)
      const int cand[4][5] = {{0, i - 1, j, i - 1, j}, {0, i, j, i + 1, j}, {1, i, j - 1, i, j - 1}, {1, i, j, i, j + 1}};
      for (auto& cd : cand) {
        int oi = cd[3], oj = cd[4];
        if (side(oi, oj) == s0) continue;
        auto it = qidx.find(key(cd[0], cd[1], cd[2]));
        if (it == qidx.end()) throw GeomError("internal: missing intersection");
        int e = it->second;
        double xbar = cd[0] == 0 ? X(oi) : X(oj);
        S.pair_q.push_back(e);
        S.pair_d.push_back(xbar - S.q_xi[e]);  // d = x_a(p̄) − ξ
      }
      S.irr_ptr.push_back((int)S.pair_q.size());
    }
  }
  S.nirr = (int)S.irr_i.size();
  }
  {
    std::vector<int> cnt(N + 1, 0);
    for (int r : S.irr_i) cnt[r]++;
    S.col_ptr.assign(N + 1, 0);
    S.col_mid.assign(N + 1, 0);
    for (int i = 0; i < N; ++i) S.col_ptr[i + 1] = S.col_ptr[i] + cnt[i];
    // col_mid[i]: first even-row entry of column i (== col_ptr[i+1] if none)
    for (int i = 0; i < N; ++i) {
      int m = S.col_ptr[i];
      while (m < S.col_ptr[i + 1] && (S.irr_j[m] & 1)) ++m;
      S.col_mid[i] = m;
    }
    // col_ptr[i] .. col_ptr[i+1] are the irregular nodes of column i (sorted order)
  }

  setup_tick("control points at uniform Ω-orie");
  // ---- control points at uniform Ω-oriented arc length (R11) ----
  S.z_comp.resize(S.M); S.z_knot.resize(S.M); S.z_x.resize(S.M); S.z_y.resize(S.M);
  S.z_t1.resize(S.M); S.z_t2.resize(S.M); S.z_p1.resize(S.M); S.z_p2.resize(S.M);
  for (int c = 0; c < nc; ++c) {
    const Comp& C = S.comps[c];
#pragma omp parallel for schedule(static)
    for (int m = 0; m < C.M; ++m) {
      double s = m * C.delta;
      double sc = C.role == KFBI_OUTER ? s : std::fmod(C.L - s, C.L);
      double th = arcs[c].theta_of(sc);
      double pos[2], tau[2], taup[2];
      frame(C, th, pos, tau, taup);
      int id = C.off + m;
      S.z_comp[id] = c; S.z_knot[id] = m; S.z_x[id] = pos[0]; S.z_y[id] = pos[1];
      S.z_t1[id] = tau[0]; S.z_t2[id] = tau[1]; S.z_p1[id] = taup[0]; S.z_p2[id] = taup[1];
    }
  }

  setup_tick("six-point stencils + inverse row");
  // ---- six-point stencils + inverse rows (R14, R16) ----
  const int M = S.M;
  if (dev) {   // NEXT-3: the same stencils and LU solves on the device (setup_gpu.cu, bit-identical)
    gpu_stencil_phase(S, dev->ptr, dev->bytes, dev->stream);
  } else {
  std::vector<int64_t> nodes((size_t)M * 6 * 2);
  S.st_ext.assign((size_t)M * 6, 0);
  S.st_w.assign((size_t)M * 6, 0);
  S.st_wn.assign((size_t)M * 6, 0);
  S.st_dx.assign((size_t)M * 6, 0);
  S.st_dy.assign((size_t)M * 6, 0);
  bool bad = false;
#pragma omp parallel for schedule(static)
  for (int m = 0; m < M; ++m) {
    double z[2] = {S.z_x[m], S.z_y[m]};
    int c[2], sg[2];
    for (int a = 0; a < 2; ++a) {
      c[a] = (int)std::floor((z[a] - lo) / h + 0.5);
      sg[a] = z[a] >= X(c[a]) ? 1 : -1;
    }
    const int off6[6][2] = {{0, 0}, {1, 0}, {-1, 0}, {0, 1}, {0, -1}, {sg[0], sg[1]}};
    double A[36], w[6];
    for (int p = 0; p < 6; ++p) {
      int ni = c[0] + off6[p][0], nj = c[1] + off6[p][1];
      if (ni < 1 || nj < 1 || ni > N - 1 || nj > N - 1) bad = true;
      nodes[((size_t)m * 6 + p) * 2] = ni;
      nodes[((size_t)m * 6 + p) * 2 + 1] = nj;
      double dx = X(ni) - z[0], dy = X(nj) - z[1];
      S.st_dx[m * 6 + p] = dx;
      S.st_dy[m * 6 + p] = dy;
      S.st_ext[m * 6 + p] = (ni >= 0 && ni <= N && nj >= 0 && nj <= N && side(ni, nj)) ? 0 : 1;
      // transpose of the local Vandermonde: A^T w = e_0 gives w = row 0 of A^{-1}
      const double row[6] = {1.0, dx, dy, 0.5 * dx * dx, dx * dy, 0.5 * dy * dy};
      for (int q = 0; q < 6; ++q) A[q * 6 + p] = row[q];
      w[p] = p == 0 ? 1.0 : 0.0;
    }
    double A2[36], wn[6] = {0, 0, 0, 0, 0, 0};
    std::copy(A, A + 36, A2);
    if (!lu_solve(6, A, w)) bad = true;
    for (int p = 0; p < 6; ++p) S.st_w[m * 6 + p] = w[p];
    // normal derivative n·∇ of the local quadratic (Neumann, R38): Aᵀ w_n = (0, n_x, n_y, 0, 0, 0),
    // n = (τ2, −τ1)
    wn[1] = S.z_t2[m];
    wn[2] = -S.z_t1[m];
    if (!lu_solve(6, A2, wn)) bad = true;
    for (int p = 0; p < 6; ++p) S.st_wn[m * 6 + p] = wn[p];
  }
  if (bad) throw GeomError("interpolation stencil leaves the grid or is singular");
  S.st_nodes_ij = nodes;
  {
    // unique stencil nodes ordered by (column i, odd rows first, row j): the sparse inverse
    // transform processes same-parity rows together (sin(πj(N−k)/N) = (−1)^{j+1} sin(πjk/N))
    // class: 0 odd rows, 1 rows ≡ 0 (mod 4), 2 rows ≡ 2 (mod 4) — see k_inv_sparse
    auto skey = [&](int64_t i, int64_t j) { return (i * 3 + ((j & 1) ? 0 : ((j & 3) == 0 ? 1 : 2))) * W + j; };
    std::vector<int64_t> keys((size_t)M * 6);
    for (size_t k = 0; k < keys.size(); ++k) keys[k] = skey(nodes[2 * k], nodes[2 * k + 1]);
    std::vector<int64_t> uk = keys;
    std::sort(uk.begin(), uk.end());
    uk.erase(std::unique(uk.begin(), uk.end()), uk.end());
    S.nsn = (int)uk.size();
    S.sn_i.resize(S.nsn);
    S.sn_j.resize(S.nsn);
    for (int u = 0; u < S.nsn; ++u) { S.sn_i[u] = (int)(uk[u] / W / 3); S.sn_j[u] = (int)(uk[u] % W); }
    S.st_node.resize(keys.size());
    for (size_t k = 0; k < keys.size(); ++k)
      S.st_node[k] = (int)(std::lower_bound(uk.begin(), uk.end(), keys[k]) - uk.begin());
  }
  }
  {
    // work items of k_inv_sparse: one per stencil column, a column with more than kMaxColRows rows
    // (Γ running along a grid line at large N) split into equal chunks of consecutive rows
    S.ocol.clear();
    S.ocol_ptr.assign(1, 0);
    for (int u0 = 0; u0 < S.nsn;) {
      int u1 = u0;
      while (u1 < S.nsn && S.sn_i[u1] == S.sn_i[u0]) ++u1;
      const int nch = (u1 - u0 + kMaxColRows - 1) / kMaxColRows, per = (u1 - u0 + nch - 1) / nch;
      for (int k = 0; k < nch; ++k) {
        S.ocol.push_back(S.sn_i[u0]);
        S.ocol_ptr.push_back(std::min(u1, u0 + (k + 1) * per));
      }
      u0 = u1;
    }
    S.max_col_rows = 1;
    S.ocol_ncls.assign(3 * (S.ocol_ptr.size() - 1), 0);   // rows per class (odd, j ≡ 0, j ≡ 2 mod 4)
    for (size_t c = 0; c + 1 < S.ocol_ptr.size(); ++c)
      for (int u = S.ocol_ptr[c]; u < S.ocol_ptr[c + 1]; ++u) {
        const int j = S.sn_j[u];
        ++S.ocol_ncls[3 * c + ((j & 1) ? 0 : ((j & 3) == 0 ? 1 : 2))];
      }
    for (size_t c = 0; c + 1 < S.ocol_ptr.size(); ++c) {
      S.max_col_rows = std::max(S.max_col_rows, S.ocol_ptr[c + 1] - S.ocol_ptr[c]);
    }
    S.ocol_order.resize(S.ocol.size());
    for (size_t c = 0; c < S.ocol.size(); ++c) S.ocol_order[c] = (int32_t)c;
    std::stable_sort(S.ocol_order.begin(), S.ocol_order.end(), [&](int32_t x, int32_t y) {
      return S.ocol_ptr[x + 1] - S.ocol_ptr[x] > S.ocol_ptr[y + 1] - S.ocol_ptr[y];
    });
    // per work position: (item, column, first row, end row, odd rows, j ≡ 0 rows) — one load per item
    S.ocol_meta.resize(6 * S.ocol_order.size());
    for (size_t kk = 0; kk < S.ocol_order.size(); ++kk) {
      const int32_t b = S.ocol_order[kk];
      const int32_t v[6] = {b, S.ocol[b], S.ocol_ptr[b], S.ocol_ptr[b + 1], S.ocol_ncls[3 * b], S.ocol_ncls[3 * b + 1]};
      std::copy(v, v + 6, S.ocol_meta.begin() + 6 * kk);
    }
  }

  setup_tick("spline filters (reading R10; SUR");
  // ---- spline filters (reading R10) ----
  // M_m = (6/Δ²) Σ_r b_r φ_{m+r},  b_r = a_{r−1} − 2a_r + a_{r+1},  a = periodic inverse of
  // the circulant [1, 4, 1]:  a_q = (ρ^q + ρ^{M−q}) / (2√3 (1 − ρ^M)),  ρ = −(2 − √3).
  S.sp_ntaps.clear(); S.sp_first.clear(); S.sp_coef_off.clear(); S.sp_coef.clear();
  const double rho = -(2.0 - std::sqrt(3.0));
  for (auto& C : S.comps) {
    int Mc = C.M;
    auto a = [&](int q) {
      q %= Mc;
      if (q < 0) q += Mc;
      return (std::pow(rho, q) + std::pow(rho, Mc - q)) / (2.0 * std::sqrt(3.0) * (1.0 - std::pow(rho, Mc)));
    };
    double sc = 6.0 / (C.delta * C.delta);
    S.sp_coef_off.push_back((int)S.sp_coef.size());
    if (Mc <= 64) {
      S.sp_ntaps.push_back(Mc);
      S.sp_first.push_back(0);
      for (int r = 0; r < Mc; ++r) S.sp_coef.push_back(sc * (a(r - 1) - 2 * a(r) + a(r + 1)));
    } else {
      S.sp_ntaps.push_back(61);
      S.sp_first.push_back(-30);
      for (int r = -30; r <= 30; ++r) S.sp_coef.push_back(sc * (a(r - 1) - 2 * a(r) + a(r + 1)));
    }
  }

  setup_tick("fast-solver tables (Alg. 4; SURV");
  // ---- fast-solver tables (Alg. 4) ----
  const int P = S.P;
  S.sin_tab.resize(N / 2 + 1);
  for (int r = 0; r <= N / 2; ++r) S.sin_tab[r] = std::sin(kPi * (double)r / N);
  S.tw.resize(4 * (size_t)N);   // (cos, sin)(π m/N), m < 2N, folded onto the quarter wave
  for (int m = 0; m < 2 * N; ++m) {
    auto sn = [&](int r) { double sg = 1.0; if (r >= N) { r -= N; sg = -1.0; } if (r > N / 2) r = N - r; return sg * S.sin_tab[r]; };
    S.tw[2 * m] = sn((m + N / 2) % (2 * N));
    S.tw[2 * m + 1] = sn(m);
  }
  S.dk.assign(N, 0.0);
  S.invc.assign((size_t)LB * N, 0.0);
  S.zr.assign((size_t)LB * N, 0.0);
  S.red_a.assign(N, 0.0);
  S.red_b.assign(N, 0.0);
  S.red_invc.assign((size_t)std::max(P - 1, 1) * N, 0.0);
#pragma omp parallel for schedule(static)
  for (int k = 1; k < N; ++k) {
    double sk = std::sin(kPi * k / (2.0 * N));
    double d = -(2.0 + 4.0 * sk * sk + S.kappa * h * h);
    S.dk[k] = d;
    double c = d, cs[LB];
    for (int p = 0; p < LB; ++p) {
      if (p > 0) c = d - 1.0 / c;
      cs[p] = c;
      S.invc[(size_t)p * N + k] = 1.0 / c;
    }
    // Z_R = S^{-1} e_L: forward y = e_L; backward x_L = 1/c_L, x_p = −x_{p+1}/c_p
    double x = 1.0 / cs[LB - 1];
    S.zr[(size_t)(LB - 1) * N + k] = x;
    for (int p = LB - 2; p >= 0; --p) {
      x = -x / cs[p];
      S.zr[(size_t)p * N + k] = x;
    }
    double al = -S.zr[k];                                   // −Z_R[1] = −Z_L[L]
    double be = d - 2.0 * S.zr[(size_t)(LB - 1) * N + k];  // d − Z_R[L] − Z_L[1]
    S.red_a[k] = al;
    S.red_b[k] = be;
    double rc = be;
    for (int gg = 0; gg < P - 1; ++gg) {
      if (gg > 0) rc = be - al * al / rc;
      S.red_invc[(size_t)gg * N + k] = 1.0 / rc;
    }
  }
  // level-2 arrowhead tables for the reduced system tridiag(a, b, a) of size P−1 (blocks of
  // L2 = BL2−1 separators, one level-2 separator between them)
  S.rinv2.assign((size_t)LB2 * N, 0.0);
  S.z2r.assign((size_t)LB2 * N, 0.0);
  S.red2_a.assign(N, 0.0);
  S.red2_b.assign(N, 0.0);
  S.red2_ci.assign((size_t)(kMaxSeg - 1) * N, 1.0);
#pragma omp parallel for schedule(static)
  for (int k = 1; k < N; ++k) {
    const double a = S.red_a[k], bb = S.red_b[k];
    double c = bb, cs[LB2];
    for (int p = 0; p < LB2; ++p) {
      if (p > 0) c = bb - a * a / c;
      cs[p] = c;
      S.rinv2[(size_t)p * N + k] = 1.0 / c;
    }
    double x = 1.0 / cs[LB2 - 1];   // S2^{-1} e_L: z_L = 1/c_L, z_p = −a z_{p+1}/c_p
    S.z2r[(size_t)(LB2 - 1) * N + k] = x;
    for (int p = LB2 - 2; p >= 0; --p) {
      x = -a * x / cs[p];
      S.z2r[(size_t)p * N + k] = x;
    }
    S.red2_a[k] = -a * a * S.z2r[k];
    S.red2_b[k] = bb - 2.0 * a * a * S.z2r[(size_t)(LB2 - 1) * N + k];
    // level-2 pivots 1/c_q of tridiag(A2, B2, A2) (c_0 = B2, c_q = B2 − A2² / c_{q−1}), q < kMaxSeg − 1
    const double A2 = S.red2_a[k], B2 = S.red2_b[k];
    double c2 = B2;
    for (int q = 0; q < kMaxSeg - 1; ++q) {
      if (q) c2 = B2 - A2 * A2 * S.red2_ci[(size_t)(q - 1) * N + k];
      S.red2_ci[(size_t)q * N + k] = 1.0 / c2;
    }
  }
  // spectral mode order: quad {t, N−t, N/2−t, N/2+t} at positions 4t..4t+3 (t ∈ [1, N/4)), and
  // {0, N/2, N/4, 3N/4} at 0..3, so that the inverse transform loads a quad as two 16-byte words
  // and the sweep writes whole 32-byte sectors.  All per-mode tables are stored in position order.
  {
    std::vector<int> posof(N);
    for (int k = 0; k < N; ++k) posof[k] = mode_position(k, N);
    auto perm = [&](std::vector<double>& v, int rows, double fill0) {
      std::vector<double> out(v.size());
#pragma omp parallel for schedule(static)
      for (int r = 0; r < rows; ++r)
        for (int k = 0; k < N; ++k) out[(size_t)r * N + posof[k]] = k == 0 ? fill0 : v[(size_t)r * N + k];
      v.swap(out);
    };
    perm(S.dk, 1, -4.0);
    perm(S.invc, LB, -0.25);
    perm(S.zr, LB, 0.0);
    perm(S.red_a, 1, 0.0);
    perm(S.red_b, 1, 1.0);
    perm(S.red_invc, std::max(P - 1, 1), 1.0);
    perm(S.rinv2, LB2, 1.0);
    perm(S.z2r, LB2, 0.0);
    perm(S.red2_a, 1, 0.0);
    perm(S.red2_b, 1, 1.0);
    perm(S.red2_ci, kMaxSeg - 1, 1.0);
  }
  // largest number of sparse corrections staged by one sweep work item (block + separator), and the
  // blocks by descending count (the sweep's work order)
  S.maxe = 1;
  std::vector<int> bcnt(P);
  for (int gg = 0; gg < P; ++gg) {
    const int last = std::min(BL * gg + BL, N - 1);
    bcnt[gg] = S.col_ptr[last + 1] - S.col_ptr[BL * gg + 1];
    S.maxe = std::max(S.maxe, bcnt[gg]);
  }
  S.blk_order.resize(P);
  for (int gg = 0; gg < P; ++gg) S.blk_order[gg] = gg;
  std::stable_sort(S.blk_order.begin(), S.blk_order.end(), [&](int32_t x, int32_t y) { return bcnt[x] > bcnt[y]; });
  // per position of that order: (block, first entry, end entry, stencil-column mask) — one load
  // instead of blk_order → col_ptr; mask bit p: grid column BL·g + 1 + p holds stencil nodes (the
  // sparse apply's inverse reads only those spectral rows, so the sweep stores only those)
  std::vector<uint8_t> scol(N + 1, 0);
  for (int u = 0; u < S.nsn; ++u) scol[S.sn_i[u]] = 1;
  S.blk_meta.resize(4 * (size_t)P);
  for (int kk = 0; kk < P; ++kk) {
    const int gg = S.blk_order[kk], c0 = BL * gg + 1, ncol = gg < P - 1 ? BL : LB;
    int msk = 0;
    for (int p = 0; p < LB; ++p) msk |= (int)scol[c0 + p] << p;
    S.blk_meta[4 * kk] = gg;
    S.blk_meta[4 * kk + 1] = S.col_ptr[c0];
    S.blk_meta[4 * kk + 2] = S.col_ptr[c0 + ncol];
    S.blk_meta[4 * kk + 3] = msk;
  }
  S.holes.clear();
  if (S.kappa == 0.0)
    for (int c = 0; c < nc; ++c)
      if (S.comps[c].role == KFBI_HOLE) {
        if (S.comps[c].kind != KFBI_ELLIPSE) throw ArgError("hole completion (R27) needs ellipse holes");
        S.holes.push_back(c);
      }
  setup_tick("end");
}

}  // namespace kfbi
