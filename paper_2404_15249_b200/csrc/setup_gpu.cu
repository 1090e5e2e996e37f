// GPU-side Procedure 1 for 2D and 3D geometries: the O(N^d) phases of the
// host setup — node classification, sign-change edges and their intersections by bisection
// (R30/R31), irregular nodes with their incident intersections (App. A.3) — as one
// thread per node / edge, the ordered lists by prefix sums (CUB).  The arithmetic is the host's
// (setup2d.cpp) operation for operation with round-to-nearest intrinsics, so no FMA contraction can
// move a node across Γ: the lists are bit-identical to the host setup (tests/test_gpu_setup.py).
// 2D also builds the interpolation stencils on the device (the six nodes, the local 6×6 Vandermonde
// solves by LU with partial pivoting — SURVEY §8(f) NEXT-3 "stencil LU on device" — and the sorted
// unique stencil-node list by a radix sort); frames, arc length, control points and the per-mode
// tables stay on the host.
#include <cuda_runtime.h>

#include <algorithm>
#include <cub/cub.cuh>

#include "kfbi_impl.h"

namespace kfbi {
namespace {

struct DevComp {
  int kind, role;
  double c0, c1, p0, p1, p2, p3;
};
struct Comps {
  int n;
  DevComp c[8];
};

__device__ __forceinline__ double node_x(double lo, double h, int i) { return __dadd_rn(lo, __dmul_rn((double)i, h)); }

// level(c, x, y) and omega_side exactly as setup2d.cpp (points on Γ are in Ω, R30)
__device__ __forceinline__ bool d_omega_side(const DevComp& c, double x, double y) {
  double l;
  if (c.kind == KFBI_ELLIPSE) {
    const double u = __ddiv_rn(__dsub_rn(x, c.c0), c.p0), v = __ddiv_rn(__dsub_rn(y, c.c1), c.p1);
    l = __dsub_rn(__dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v)), 1.0);
  } else {
    const double dx = __dsub_rn(x, c.c0), dy = __dsub_rn(y, c.c1);
    const double ang = __dmul_rn(c.p2, __dsub_rn(atan2(dy, dx), c.p3));
    l = __dsub_rn(__dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy))),
                  __dmul_rn(c.p0, __dadd_rn(1.0, __dmul_rn(c.p1, sin(ang)))));
  }
  return c.role == KFBI_OUTER ? (l <= 0.0) : (l >= 0.0);
}

__global__ void k_classify(int W, double lo, double h, Comps cs, int8_t* __restrict__ side) {
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < (long)W * W; idx += (long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / W), j = (int)(idx % W);
    const double x = node_x(lo, h, i), y = node_x(lo, h, j);
    bool in = true;
    for (int c = 0; c < cs.n && in; ++c) in = d_omega_side(cs.c[c], x, y);
    side[idx] = in ? 1 : 0;
  }
}

// flag[axis·W² + i·W + j] = 1 for a sign-change edge from (i, j) along axis (the host's (axis, i, j) order)
__global__ void k_edge_flags(int W, const int8_t* __restrict__ side, int* __restrict__ flag) {
  const long WW = (long)W * W;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < 2 * WW; idx += (long)gridDim.x * blockDim.x) {
    const int axis = (int)(idx / WW);
    const long r = idx - axis * WW;
    const int i = (int)(r / W), j = (int)(r % W);
    int f = 0;
    if (axis == 0 ? i < W - 1 : j < W - 1) f = side[r] != side[r + (axis == 0 ? W : 1)];
    flag[idx] = f;
  }
}

__global__ void k_edge_compact(int W, const int* __restrict__ flag, const int* __restrict__ qmap, int* __restrict__ qa,
                               int* __restrict__ qi, int* __restrict__ qj) {
  const long WW = (long)W * W;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < 2 * WW; idx += (long)gridDim.x * blockDim.x) {
    if (!flag[idx]) continue;
    const int q = qmap[idx], axis = (int)(idx / WW);
    const long r = idx - axis * WW;
    qa[q] = axis;
    qi[q] = (int)(r / W);
    qj[q] = (int)(r % W);
  }
}

// owner component, the double-crossing check at 4 interior samples (R31) and 64 halvings (R30)
__global__ void k_bisect(int nq, double lo, double h, Comps cs, const int* __restrict__ qa, const int* __restrict__ qi,
                         const int* __restrict__ qj, double* __restrict__ xi_out, int* __restrict__ owner_out,
                         int* __restrict__ err) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nq) return;
  const int axis = qa[e];
  const double x0 = node_x(lo, h, qi[e]), y0 = node_x(lo, h, qj[e]);
  const double x1 = axis == 0 ? __dadd_rn(x0, h) : x0, y1 = axis == 1 ? __dadd_rn(y0, h) : y0;
  int owner = -1, count = 0;
  for (int c = 0; c < cs.n; ++c)
    if (d_omega_side(cs.c[c], x0, y0) != d_omega_side(cs.c[c], x1, y1)) {
      owner = c;
      ++count;
    }
  if (count != 1) {
    atomicOr(err, 1);
    return;
  }
  const DevComp& C = cs.c[owner];
  const bool want = d_omega_side(C, x0, y0);
  bool prev = want;
  int changes = 0;
  const double ts[5] = {0.2, 0.4, 0.6, 0.8, 1.0};
  for (int k = 0; k < 5; ++k) {
    const double d = __dmul_rn(ts[k], h);
    const bool cur = d_omega_side(C, axis == 0 ? __dadd_rn(x0, d) : x0, axis == 1 ? __dadd_rn(y0, d) : y0);
    changes += cur != prev;
    prev = cur;
  }
  if (changes != 1) {
    atomicOr(err, 2);
    return;
  }
  double a = 0.0, bb = 1.0;
  for (int it = 0; it < 64; ++it) {
    const double m = __dmul_rn(0.5, __dadd_rn(a, bb));
    const double d = __dmul_rn(m, h);
    const bool same = d_omega_side(C, axis == 0 ? __dadd_rn(x0, d) : x0, axis == 1 ? __dadd_rn(y0, d) : y0) == want;
    if (same) a = m;
    else bb = m;
  }
  const double t = __dmul_rn(0.5, __dadd_rn(a, bb));
  xi_out[e] = __dadd_rn(axis == 0 ? x0 : y0, __dmul_rn(t, h));
  owner_out[e] = owner;
}

// irregular-node flags in the host's order: column i = 1..N−1, odd rows first, then even rows
__device__ __forceinline__ int row_of(int jj, int N) { return jj < N / 2 ? 2 * jj + 1 : 2 * (jj - N / 2) + 2; }

__global__ void k_irr_flags(int N, const int8_t* __restrict__ side, int* __restrict__ iflag, int* __restrict__ err) {
  const int W = N + 1;
  const long n = (long)(N - 1) * (N - 1);
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (long)gridDim.x * blockDim.x) {
    const int i = 1 + (int)(idx / (N - 1)), j = row_of((int)(idx % (N - 1)), N);
    const long p = (long)i * W + j;
    const int8_t s0 = side[p];
    const bool irr = side[p - W] != s0 || side[p + W] != s0 || side[p - 1] != s0 || side[p + 1] != s0;
    iflag[idx] = irr ? 1 : 0;
    if (irr && (i < 2 || j < 2 || i > N - 2 || j > N - 2)) atomicOr(err, 4);   // R32
  }
}

__global__ void k_irr_compact(int N, const int* __restrict__ iflag, const int* __restrict__ imap,
                              const int8_t* __restrict__ side, int* __restrict__ ii, int* __restrict__ ij,
                              int8_t* __restrict__ iside, int* __restrict__ ncnt) {
  const int W = N + 1;
  const long n = (long)(N - 1) * (N - 1);
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (long)gridDim.x * blockDim.x) {
    if (!iflag[idx]) continue;
    const int r = imap[idx];
    const int i = 1 + (int)(idx / (N - 1)), j = row_of((int)(idx % (N - 1)), N);
    const long p = (long)i * W + j;
    const int8_t s0 = side[p];
    ii[r] = i;
    ij[r] = j;
    iside[r] = s0;
    ncnt[r] = (side[p - W] != s0) + (side[p + W] != s0) + (side[p - 1] != s0) + (side[p + 1] != s0);
  }
}

// the ≤ 4 incident intersections in the host's candidate order, d = x_a(p̄) − ξ (App. A.3)
__global__ void k_irr_pairs(int N, double lo, double h, int nirr, const int* __restrict__ ii, const int* __restrict__ ij,
                            const int* __restrict__ iptr, const int8_t* __restrict__ side, const int* __restrict__ qmap,
                            const double* __restrict__ xi, int* __restrict__ pq, double* __restrict__ pd) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nirr) return;
  const int W = N + 1;
  const long WW = (long)W * W;
  const int i = ii[r], j = ij[r];
  const int8_t s0 = side[(long)i * W + j];
  const int cand[4][5] = {{0, i - 1, j, i - 1, j}, {0, i, j, i + 1, j}, {1, i, j - 1, i, j - 1}, {1, i, j, i, j + 1}};
  int o = iptr[r];
  for (int k = 0; k < 4; ++k) {
    const int oi = cand[k][3], oj = cand[k][4];
    if (side[(long)oi * W + oj] == s0) continue;
    const int q = qmap[cand[k][0] * WW + (long)cand[k][1] * W + cand[k][2]];
    const double xbar = cand[k][0] == 0 ? node_x(lo, h, oi) : node_x(lo, h, oj);
    pq[o] = q;
    pd[o] = __dsub_rn(xbar, xi[q]);
    ++o;
  }
}

inline int grid_for(long n) { return (int)std::min<long>((n + 255) / 256, 65535L * 4); }

template <class T>
T* carve(uint8_t*& p, size_t n) {
  p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));
  T* r = reinterpret_cast<T*>(p);
  p += n * sizeof(T);
  return r;
}

void ck_(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string("setup on device: ") + what + ": " + cudaGetErrorString(e));
}

size_t cub_scan_bytes(long n) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const int*)nullptr, (int*)nullptr, (int)n);
  return b;
}

// list capacities: nq ≤ kQPerW·(N+1) intersections (Γ of total length up to ~20 box sides) and
// n_irr ≤ 2·nq (every irregular node ends a sign-change edge, each edge has two ends)
constexpr long kQPerW = 64;
size_t lists_bytes(long W) {
  const long nq = kQPerW * W, ni = 2 * nq;
  return nq * (4 * sizeof(int) + sizeof(double)) + ni * (4 * sizeof(int) + 1 + 4 * (sizeof(int) + sizeof(double))) +
         32 * 256;
}

// ---------------------------------------------------------------------------------------- 2D stencils
// The host's lu_solve (setup2d.cpp) operation for operation: partial pivoting on |a|, elimination
// a_ij −= f·a_kj with f = a_ik / a_kk, back substitution — round-to-nearest intrinsics, no contraction.
__device__ bool d_lu_solve6(double* A, double* b) {
  constexpr int n = 6;
  for (int k = 0; k < n; ++k) {
    int piv = k;
    for (int i = k + 1; i < n; ++i)
      if (fabs(A[i * n + k]) > fabs(A[piv * n + k])) piv = i;
    if (fabs(A[piv * n + k]) < 1e-300) return false;
    if (piv != k) {
      for (int j = 0; j < n; ++j) {
        const double t = A[k * n + j];
        A[k * n + j] = A[piv * n + j];
        A[piv * n + j] = t;
      }
      const double t = b[k];
      b[k] = b[piv];
      b[piv] = t;
    }
    for (int i = k + 1; i < n; ++i) {
      const double f = __ddiv_rn(A[i * n + k], A[k * n + k]);
      for (int j = k; j < n; ++j) A[i * n + j] = __dsub_rn(A[i * n + j], __dmul_rn(f, A[k * n + j]));
      b[i] = __dsub_rn(b[i], __dmul_rn(f, b[k]));
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    double sacc = b[i];
    for (int j = i + 1; j < n; ++j) sacc = __dsub_rn(sacc, __dmul_rn(A[i * n + j], b[j]));
    b[i] = __ddiv_rn(sacc, A[i * n + i]);
  }
  return true;
}

// thread per control point: the six stencil nodes (R14), offsets, exterior flags, row 0 of
// the inverse local system (V⁺ weights) and the normal-derivative row (Neumann, R38), and each node's
// sort key (column, row class, row) — setup2d.cpp's stencil loop with the same arithmetic
__global__ void k_stencil2(int M, int N, double lo, double h, const double* __restrict__ zx, const double* __restrict__ zy,
                           const double* __restrict__ t1, const double* __restrict__ t2, const int8_t* __restrict__ side,
                           int64_t* __restrict__ nodes, int8_t* __restrict__ ext, double* __restrict__ w,
                           double* __restrict__ wn, double* __restrict__ sdx, double* __restrict__ sdy,
                           int64_t* __restrict__ keys, int* __restrict__ err) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  const int W = N + 1;
  const double z[2] = {zx[m], zy[m]};
  int c[2], sg[2];
  for (int a = 0; a < 2; ++a) {
    c[a] = (int)floor(__dadd_rn(__ddiv_rn(__dsub_rn(z[a], lo), h), 0.5));
    sg[a] = z[a] >= node_x(lo, h, c[a]) ? 1 : -1;
  }
  const int off6[6][2] = {{0, 0}, {1, 0}, {-1, 0}, {0, 1}, {0, -1}, {sg[0], sg[1]}};
  double A[36], A2[36], wv[6], wnv[6];
  for (int p = 0; p < 6; ++p) {
    const int ni = c[0] + off6[p][0], nj = c[1] + off6[p][1];
    if (ni < 1 || nj < 1 || ni > N - 1 || nj > N - 1) atomicOr(err, 1);
    nodes[((size_t)m * 6 + p) * 2] = ni;
    nodes[((size_t)m * 6 + p) * 2 + 1] = nj;
    const double dx = __dsub_rn(node_x(lo, h, ni), z[0]), dy = __dsub_rn(node_x(lo, h, nj), z[1]);
    sdx[m * 6 + p] = dx;
    sdy[m * 6 + p] = dy;
    ext[m * 6 + p] = (ni >= 0 && ni <= N && nj >= 0 && nj <= N && side[(size_t)ni * W + nj]) ? 0 : 1;
    const double row[6] = {1.0, dx, dy, __dmul_rn(__dmul_rn(0.5, dx), dx), __dmul_rn(dx, dy),
                           __dmul_rn(__dmul_rn(0.5, dy), dy)};
    for (int q = 0; q < 6; ++q) A[q * 6 + p] = A2[q * 6 + p] = row[q];
    wv[p] = p == 0 ? 1.0 : 0.0;
    wnv[p] = 0.0;
    const int64_t cls = (nj & 1) ? 0 : ((nj & 3) == 0 ? 1 : 2);
    keys[(size_t)m * 6 + p] = ((int64_t)ni * 3 + cls) * W + nj;
  }
  wnv[1] = t2[m];
  wnv[2] = -t1[m];
  if (!d_lu_solve6(A, wv) || !d_lu_solve6(A2, wnv)) atomicOr(err, 2);
  for (int p = 0; p < 6; ++p) {
    w[m * 6 + p] = wv[p];
    wn[m * 6 + p] = wnv[p];
  }
}

// the host's lu_solve_n (setup3d.cpp) for the 10×10 systems, same operation order, round-to-nearest
__device__ bool d_lu_solve10(double* A, double* b) {
  constexpr int n = 10;
  for (int k = 0; k < n; ++k) {
    int piv = k;
    for (int i = k + 1; i < n; ++i)
      if (fabs(A[i * n + k]) > fabs(A[piv * n + k])) piv = i;
    if (fabs(A[piv * n + k]) < 1e-300) return false;
    if (piv != k) {
      for (int j = 0; j < n; ++j) {
        const double t = A[k * n + j];
        A[k * n + j] = A[piv * n + j];
        A[piv * n + j] = t;
      }
      const double t = b[k];
      b[k] = b[piv];
      b[piv] = t;
    }
    for (int i = k + 1; i < n; ++i) {
      const double f = __ddiv_rn(A[i * n + k], A[k * n + k]);
      for (int j = k; j < n; ++j) A[i * n + j] = __dsub_rn(A[i * n + j], __dmul_rn(f, A[k * n + j]));
      b[i] = __dsub_rn(b[i], __dmul_rn(f, b[k]));
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    double sacc = b[i];
    for (int j = i + 1; j < n; ++j) sacc = __dsub_rn(sacc, __dmul_rn(A[i * n + j], b[j]));
    b[i] = __ddiv_rn(sacc, A[i * n + i]);
  }
  return true;
}

// thread per 3D control point (intersection node): the ten-point stencil {c, c ± e_a, c + σ_x e_x +
// σ_y e_y, c + σ_x e_x + σ_z e_z, c + σ_y e_y + σ_z e_z} (R14, R16), row 0 of the inverse local
// system and the Neumann normal-derivative row (R38), centre and sign/exterior code — setup3d.cpp's
// stencil loop with the same arithmetic
__global__ void k_stencil3(int nq, int N, double lo, double h, const double* __restrict__ qpos,
                           const double* __restrict__ qn, const int8_t* __restrict__ side,
                           int64_t* __restrict__ nodes, double* __restrict__ w, double* __restrict__ wn,
                           int32_t* __restrict__ stc, int32_t* __restrict__ code, int* __restrict__ err) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nq) return;
  const int W = N + 1;
  const double z[3] = {qpos[3 * (size_t)e], qpos[3 * (size_t)e + 1], qpos[3 * (size_t)e + 2]};
  int c[3], sg[3];
  for (int a = 0; a < 3; ++a) {
    c[a] = (int)floor(__dadd_rn(__ddiv_rn(__dsub_rn(z[a], lo), h), 0.5));
    sg[a] = z[a] >= node_x(lo, h, c[a]) ? 1 : -1;
  }
  const int off[10][3] = {{0, 0, 0}, {1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1},
                          {sg[0], sg[1], 0}, {sg[0], 0, sg[2]}, {0, sg[1], sg[2]}};
  double A[100], A2[100], wv[10], wnv[10];
  int ext = 0;
  bool bad = false;
  for (int p = 0; p < 10; ++p) {
    const int ni = c[0] + off[p][0], nj = c[1] + off[p][1], nk = c[2] + off[p][2];
    wv[p] = p == 0 ? 1.0 : 0.0;
    wnv[p] = 0.0;
    if (ni < 1 || nj < 1 || nk < 1 || ni > N - 1 || nj > N - 1 || nk > N - 1) {
      bad = true;
      continue;
    }
    nodes[30 * (size_t)e + 3 * p] = ni;
    nodes[30 * (size_t)e + 3 * p + 1] = nj;
    nodes[30 * (size_t)e + 3 * p + 2] = nk;
    if (!side[((size_t)ni * W + nj) * W + nk]) ext |= 1 << p;
    const double dx = __dsub_rn(node_x(lo, h, ni), z[0]), dy = __dsub_rn(node_x(lo, h, nj), z[1]),
                 dz = __dsub_rn(node_x(lo, h, nk), z[2]);
    const double row[10] = {1.0, dx, dy, dz, __dmul_rn(__dmul_rn(0.5, dx), dx), __dmul_rn(__dmul_rn(0.5, dy), dy),
                            __dmul_rn(__dmul_rn(0.5, dz), dz), __dmul_rn(dx, dy), __dmul_rn(dx, dz), __dmul_rn(dy, dz)};
    for (int q = 0; q < 10; ++q) A[q * 10 + p] = A2[q * 10 + p] = row[q];
  }
  if (bad) {
    atomicOr(err, 1);
    return;
  }
  for (int a = 0; a < 3; ++a) wnv[1 + a] = qn[3 * (size_t)e + a];
  if (!d_lu_solve10(A, wv) || !d_lu_solve10(A2, wnv)) atomicOr(err, 2);
  for (int p = 0; p < 10; ++p) {
    w[10 * (size_t)e + p] = wv[p];
    wn[10 * (size_t)e + p] = wnv[p];
  }
  for (int a = 0; a < 3; ++a) stc[3 * (size_t)e + a] = c[a];
  code[e] = ext | ((sg[0] > 0) << 10) | ((sg[1] > 0) << 11) | ((sg[2] > 0) << 12);
}

// st_node[k] = position of keys[k] in the sorted unique list uk[0, nu) (lower bound)
__global__ void k_stencil_rank(long n, const int64_t* __restrict__ keys, const int64_t* __restrict__ uk,
                               const int* __restrict__ nu, int32_t* __restrict__ st_node) {
  const long k = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t key = keys[k];
  int a = 0, b = *nu;
  while (a < b) {
    const int mid = (a + b) >> 1;
    if (uk[mid] < key) a = mid + 1;
    else b = mid;
  }
  st_node[k] = a;
}

// ---------------------------------------------------------------------------------------- 3D
// The same phases for the 3D surfaces (setup3d.cpp): level3 / inside3 with round-to-nearest intrinsics
// in the host's operation order, edges in (axis, i, j, k) order, irregular nodes in (i, j, k) order
// with their ≤ 6 incident intersections in the host's neighbour order.
struct DevComp3 {
  int kind;
  double c0, c1, c2, p0, p1, p2;
};
__device__ __forceinline__ bool d_inside3(const DevComp3& c, double x, double y, double z) {
  const double dx = __dsub_rn(x, c.c0), dy = __dsub_rn(y, c.c1), dz = __dsub_rn(z, c.c2);
  double l;
  if (c.kind == KFBI_ELLIPSOID) {
    const double u = __ddiv_rn(dx, c.p0), v = __ddiv_rn(dy, c.p1), w = __ddiv_rn(dz, c.p2);
    l = __dsub_rn(__dadd_rn(__dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v)), __dmul_rn(w, w)), 1.0);
  } else {
    const double q = __dsub_rn(__dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy))), c.p0);
    l = __dsub_rn(__dadd_rn(__dmul_rn(q, q), __dmul_rn(dz, dz)), __dmul_rn(c.p1, c.p1));
  }
  return l <= 0.0;
}

__global__ void k_classify3(int W, double lo, double h, DevComp3 c, int8_t* __restrict__ side) {
  const long WWW = (long)W * W * W;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < WWW; idx += (long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / ((long)W * W)), j = (int)((idx / W) % W), k = (int)(idx % W);
    side[idx] = d_inside3(c, node_x(lo, h, i), node_x(lo, h, j), node_x(lo, h, k)) ? 1 : 0;
  }
}

// flag[axis·W³ + lin(i, j, k)] = 1 for a sign-change edge from (i, j, k) along axis
__global__ void k_edge_flags3(int W, const int8_t* __restrict__ side, int* __restrict__ flag) {
  const long WWW = (long)W * W * W;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < 3 * WWW; idx += (long)gridDim.x * blockDim.x) {
    const int axis = (int)(idx / WWW);
    const long r = idx - axis * WWW;
    const int i = (int)(r / ((long)W * W)), j = (int)((r / W) % W), k = (int)(r % W);
    const bool ok = axis == 0 ? i < W - 1 : axis == 1 ? j < W - 1 : k < W - 1;
    const long st = axis == 0 ? (long)W * W : axis == 1 ? W : 1;
    flag[idx] = ok && side[r] != side[r + st] ? 1 : 0;
  }
}

__global__ void k_edge_compact3(int W, const int* __restrict__ flag, const int* __restrict__ qmap, int* __restrict__ qa,
                                int* __restrict__ qi, int* __restrict__ qj, int* __restrict__ qk) {
  const long WWW = (long)W * W * W;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < 3 * WWW; idx += (long)gridDim.x * blockDim.x) {
    if (!flag[idx]) continue;
    const int q = qmap[idx], axis = (int)(idx / WWW);
    const long r = idx - axis * WWW;
    qa[q] = axis;
    qi[q] = (int)(r / ((long)W * W));
    qj[q] = (int)((r / W) % W);
    qk[q] = (int)(r % W);
  }
}

// the double-crossing check at 5 samples (R31) and 64 halvings (R30), as setup3d.cpp
__global__ void k_bisect3(int nq, double lo, double h, DevComp3 c, const int* __restrict__ qa, const int* __restrict__ qi,
                          const int* __restrict__ qj, const int* __restrict__ qk, double* __restrict__ xi_out,
                          int* __restrict__ err) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nq) return;
  const int axis = qa[e];
  const double p0[3] = {node_x(lo, h, qi[e]), node_x(lo, h, qj[e]), node_x(lo, h, qk[e])};
  auto at = [&](double t) {
    double p[3] = {p0[0], p0[1], p0[2]};
    p[axis] = __dadd_rn(p[axis], __dmul_rn(t, h));
    return d_inside3(c, p[0], p[1], p[2]);
  };
  const bool want = d_inside3(c, p0[0], p0[1], p0[2]);
  bool prev = want;
  int changes = 0;
  const double ts[5] = {0.2, 0.4, 0.6, 0.8, 1.0};
  for (int s = 0; s < 5; ++s) {
    const bool cur = at(ts[s]);
    changes += cur != prev;
    prev = cur;
  }
  if (changes != 1) atomicOr(err, 2);
  double a = 0.0, bb = 1.0;
  for (int it = 0; it < 64; ++it) {
    const double m = __dmul_rn(0.5, __dadd_rn(a, bb));
    if (at(m) == want) a = m;
    else bb = m;
  }
  const double t = __dmul_rn(0.5, __dadd_rn(a, bb));
  xi_out[e] = __dadd_rn(p0[axis], __dmul_rn(t, h));
}

__global__ void k_irr_flags3(int N, const int8_t* __restrict__ side, int* __restrict__ iflag, int* __restrict__ err) {
  const long W = N + 1, WW = W * W, M = N - 1, n = M * M * M;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (long)gridDim.x * blockDim.x) {
    const int i = 1 + (int)(idx / (M * M)), j = 1 + (int)((idx / M) % M), k = 1 + (int)(idx % M);
    const long p = ((long)i * W + j) * W + k;
    const int8_t s0 = side[p];
    const bool irr = side[p - WW] != s0 || side[p + WW] != s0 || side[p - W] != s0 || side[p + W] != s0 ||
                     side[p - 1] != s0 || side[p + 1] != s0;
    iflag[idx] = irr ? 1 : 0;
    if (irr && (i < 2 || j < 2 || k < 2 || i > N - 2 || j > N - 2 || k > N - 2)) atomicOr(err, 4);   // R32
  }
}

__global__ void k_irr_compact3(int N, const int* __restrict__ iflag, const int* __restrict__ imap,
                               const int8_t* __restrict__ side, int64_t* __restrict__ ilin, int* __restrict__ ijk,
                               int8_t* __restrict__ iside, int* __restrict__ ncnt) {
  const long W = N + 1, WW = W * W, M = N - 1, n = M * M * M;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (long)gridDim.x * blockDim.x) {
    if (!iflag[idx]) continue;
    const int r = imap[idx];
    const int i = 1 + (int)(idx / (M * M)), j = 1 + (int)((idx / M) % M), k = 1 + (int)(idx % M);
    const long p = ((long)i * W + j) * W + k;
    const int8_t s0 = side[p];
    ilin[r] = (int64_t)(i - 1) * N * N + (int64_t)j * N + k;
    ijk[3 * r] = i;
    ijk[3 * r + 1] = j;
    ijk[3 * r + 2] = k;
    iside[r] = s0;
    ncnt[r] = (side[p - WW] != s0) + (side[p + WW] != s0) + (side[p - W] != s0) + (side[p + W] != s0) +
              (side[p - 1] != s0) + (side[p + 1] != s0);
  }
}

__global__ void k_irr_pairs3(int N, double lo, double h, int nirr, const int* __restrict__ ijk,
                             const int* __restrict__ iptr, const int8_t* __restrict__ side, const int* __restrict__ qmap,
                             const double* __restrict__ xi, int* __restrict__ pq, double* __restrict__ pd) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nirr) return;
  const long W = N + 1, WWW = W * W * W;
  const int i = ijk[3 * r], j = ijk[3 * r + 1], k = ijk[3 * r + 2];
  auto lin = [&](int a, int b, int cc) { return ((long)a * W + b) * W + cc; };
  const int8_t s0 = side[lin(i, j, k)];
  const int nb[6][3] = {{i - 1, j, k}, {i + 1, j, k}, {i, j - 1, k}, {i, j + 1, k}, {i, j, k - 1}, {i, j, k + 1}};
  int o = iptr[r];
  for (int q = 0; q < 6; ++q) {
    const int oi = nb[q][0], oj = nb[q][1], ok = nb[q][2];
    if (side[lin(oi, oj, ok)] == s0) continue;
    const int axis = q / 2;
    const int li = min(i, oi), lj = min(j, oj), lk = min(k, ok);
    const int e = qmap[axis * WWW + lin(li, lj, lk)];
    const double xbar = axis == 0 ? node_x(lo, h, oi) : axis == 1 ? node_x(lo, h, oj) : node_x(lo, h, ok);
    pq[o] = e;
    pd[o] = __dsub_rn(xbar, xi[e]);
    ++o;
  }
}

// list capacities (3D): nq ≤ kQPerW2·W² intersections, n_irr ≤ 2·nq
constexpr long kQPerW2 = 16;
size_t lists_bytes3(long W) {
  const long nq = kQPerW2 * W * W, ni = 2 * nq;
  return nq * (4 * sizeof(int) + sizeof(double)) + ni * (sizeof(int64_t) + 3 * sizeof(int) + 3 * sizeof(int) + 1 +
                                                         6 * (sizeof(int) + sizeof(double))) + 32 * 256;
}

}  // namespace

size_t gpu_setup_scratch_bytes(int N) {
  const long W = N + 1, WW = W * W, n2 = (long)(N - 1) * (N - 1);
  return WW + 2 * (2 * WW) * sizeof(int) + 2 * n2 * sizeof(int) + lists_bytes(W) + cub_scan_bytes(2 * WW) + 16 * 256;
}

size_t gpu_setup_scratch_bytes3(int N) {
  const long W = N + 1, WWW = W * W * W, n3 = (long)(N - 1) * (N - 1) * (N - 1);
  return WWW + 2 * (3 * WWW) * sizeof(int) + 2 * n3 * sizeof(int) + lists_bytes3(W) + cub_scan_bytes(3 * WWW) +
         16 * 256;
}

// fills S.side, the intersection lists (axis, i, j, k, ξ) and the irregular-node lists of the 3D setup
void gpu_setup_phases3(Setup3& S, void* scratch, size_t bytes, cudaStream_t s) {
  const int N = S.N, W = N + 1;
  const long WWW = (long)W * W * W, n3 = (long)(N - 1) * (N - 1) * (N - 1);
  if (bytes < gpu_setup_scratch_bytes3(N)) throw ScratchError("device setup scratch too small (kfbi_setup_scratch_size)");
  const Comp& C = S.comp;
  const DevComp3 c{C.kind, C.c[0], C.c[1], C.c[2], C.p[0], C.p[1], C.p[2]};
  uint8_t* p = reinterpret_cast<uint8_t*>(scratch);
  int8_t* side = carve<int8_t>(p, WWW);
  int* flag = carve<int>(p, 3 * WWW);
  int* qmap = carve<int>(p, 3 * WWW);
  int* iflag = carve<int>(p, n3);
  int* imap = carve<int>(p, n3);
  int* err = carve<int>(p, 4);
  const size_t tb = cub_scan_bytes(3 * WWW);
  void* temp = carve<uint8_t>(p, tb);
  const long qcap = kQPerW2 * W * W, icap = 2 * qcap;
  int* qa = carve<int>(p, qcap);
  int* qi = carve<int>(p, qcap);
  int* qj = carve<int>(p, qcap);
  int* qk = carve<int>(p, qcap);
  double* qx = carve<double>(p, qcap);
  int64_t* ilin = carve<int64_t>(p, icap);
  int* ijk = carve<int>(p, 3 * icap);
  int* cnt = carve<int>(p, icap + 1);
  int* iptr = carve<int>(p, icap + 1);
  int8_t* isd = carve<int8_t>(p, icap);
  int* pqv = carve<int>(p, 6 * icap);
  double* pdv = carve<double>(p, 6 * icap);
  if ((size_t)(p - reinterpret_cast<uint8_t*>(scratch)) > bytes) throw ScratchError("device setup scratch layout overflow");
  ck_(cudaMemsetAsync(err, 0, sizeof(int), s), "memset");
  k_classify3<<<grid_for(WWW), 256, 0, s>>>(W, S.lo, S.h, c, side);
  k_edge_flags3<<<grid_for(3 * WWW), 256, 0, s>>>(W, side, flag);
  size_t tbb = tb;
  ck_(cub::DeviceScan::ExclusiveSum(temp, tbb, flag, qmap, (int)(3 * WWW), s), "scan edges");
  int h_last[2];
  ck_(cudaMemcpyAsync(&h_last[0], qmap + 3 * WWW - 1, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(&h_last[1], flag + 3 * WWW - 1, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaStreamSynchronize(s), "sync");
  const int nq = h_last[0] + h_last[1];
  if (nq > qcap) throw ScratchError("more intersections than the device setup scratch holds (16 per grid plane line)");
  k_edge_compact3<<<grid_for(3 * WWW), 256, 0, s>>>(W, flag, qmap, qa, qi, qj, qk);
  if (nq > 0) k_bisect3<<<(nq + 127) / 128, 128, 0, s>>>(nq, S.lo, S.h, c, qa, qi, qj, qk, qx, err);
  ck_(cudaGetLastError(), "edge kernels");
  S.nq = nq;
  S.q_axis.resize(nq); S.q_i.resize(nq); S.q_j.resize(nq); S.q_k.resize(nq); S.q_xi.resize(nq);
  ck_(cudaMemcpyAsync(S.q_axis.data(), qa, nq * sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.q_i.data(), qi, nq * sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.q_j.data(), qj, nq * sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.q_k.data(), qk, nq * sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.q_xi.data(), qx, nq * sizeof(double), cudaMemcpyDeviceToHost, s), "d2h");
  int h_err = 0;
  ck_(cudaMemcpyAsync(&h_err, err, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  S.side.resize(WWW);
  ck_(cudaMemcpyAsync(S.side.data(), side, WWW, cudaMemcpyDeviceToHost, s), "d2h side");
  ck_(cudaStreamSynchronize(s), "sync");
  if (h_err & 2) throw GeomError("grid edge crossed more than once (R31)");
  k_irr_flags3<<<grid_for(n3), 256, 0, s>>>(N, side, iflag, err);
  size_t tb2 = tb;
  ck_(cub::DeviceScan::ExclusiveSum(temp, tb2, iflag, imap, (int)n3, s), "scan irregular");
  ck_(cudaMemcpyAsync(&h_last[0], imap + n3 - 1, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(&h_last[1], iflag + n3 - 1, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(&h_err, err, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaStreamSynchronize(s), "sync");
  if (h_err & 4) throw GeomError("Γ too close to the box boundary (R32)");
  const int nirr = h_last[0] + h_last[1];
  if (nirr > icap) throw ScratchError("internal: more irregular nodes than 2·nq");
  k_irr_compact3<<<grid_for(n3), 256, 0, s>>>(N, iflag, imap, side, ilin, ijk, isd, cnt);
  ck_(cudaMemsetAsync(cnt + nirr, 0, sizeof(int), s), "memset");
  size_t tb3 = tb;
  ck_(cub::DeviceScan::ExclusiveSum(temp, tb3, cnt, iptr, nirr + 1, s), "scan pairs");
  if (nirr > 0) k_irr_pairs3<<<(nirr + 127) / 128, 128, 0, s>>>(N, S.lo, S.h, nirr, ijk, iptr, side, qmap, qx, pqv, pdv);
  ck_(cudaGetLastError(), "irregular-node kernels");
  S.nirr = nirr;
  S.irr_lin.resize(nirr); S.irr_ijk.resize(3 * (size_t)nirr); S.irr_side.resize(nirr); S.irr_ptr.resize(nirr + 1);
  ck_(cudaMemcpyAsync(S.irr_lin.data(), ilin, nirr * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.irr_ijk.data(), ijk, 3 * (size_t)nirr * sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.irr_side.data(), isd, nirr, cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.irr_ptr.data(), iptr, (nirr + 1) * sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaStreamSynchronize(s), "sync");
  const int npair = S.irr_ptr[nirr];
  S.pair_q.resize(npair);
  S.pair_d.resize(npair);
  ck_(cudaMemcpyAsync(S.pair_q.data(), pqv, npair * sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.pair_d.data(), pdv, npair * sizeof(double), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaStreamSynchronize(s), "sync");
}

// fills S.side, the intersection base lists (axis, i, j, ξ, owner) and the irregular-node lists
void gpu_setup_phases(Setup& S, void* scratch, size_t bytes, cudaStream_t s, std::vector<int>& q_owner) {
  const int N = S.N, W = N + 1;
  const long WW = (long)W * W, n2 = (long)(N - 1) * (N - 1);
  if (bytes < gpu_setup_scratch_bytes(N)) throw ScratchError("device setup scratch too small (kfbi_setup_scratch_size)");
  if (S.comps.size() > 8) throw ArgError("at most 8 components for the device setup");
  Comps cs{};
  cs.n = (int)S.comps.size();
  for (int c = 0; c < cs.n; ++c) {
    const Comp& C = S.comps[c];
    cs.c[c] = DevComp{C.kind, C.role, C.c[0], C.c[1], C.p[0], C.p[1], C.p[2], C.p[3]};
  }
  uint8_t* p = reinterpret_cast<uint8_t*>(scratch);
  int8_t* side = carve<int8_t>(p, WW);
  int* flag = carve<int>(p, 2 * WW);
  int* qmap = carve<int>(p, 2 * WW);
  int* iflag = carve<int>(p, n2);
  int* imap = carve<int>(p, n2);
  int* err = carve<int>(p, 4);
  const size_t tb = cub_scan_bytes(2 * WW);
  void* temp = carve<uint8_t>(p, tb);
  const long qcap = kQPerW * W, icap = 2 * qcap;
  int* qa = carve<int>(p, qcap);
  int* qi = carve<int>(p, qcap);
  int* qj = carve<int>(p, qcap);
  int* qo = carve<int>(p, qcap);
  double* qx = carve<double>(p, qcap);
  int* ii = carve<int>(p, icap);
  int* ij = carve<int>(p, icap);
  int* cnt = carve<int>(p, icap + 1);
  int* iptr = carve<int>(p, icap + 1);
  int8_t* isd = carve<int8_t>(p, icap);
  int* pqv = carve<int>(p, 4 * icap);
  double* pdv = carve<double>(p, 4 * icap);
  if ((size_t)(p - reinterpret_cast<uint8_t*>(scratch)) > bytes) throw ScratchError("device setup scratch layout overflow");
  ck_(cudaMemsetAsync(err, 0, sizeof(int), s), "memset");
  k_classify<<<grid_for(WW), 256, 0, s>>>(W, S.lo, S.h, cs, side);
  k_edge_flags<<<grid_for(2 * WW), 256, 0, s>>>(W, side, flag);
  size_t tbb = tb;
  ck_(cub::DeviceScan::ExclusiveSum(temp, tbb, flag, qmap, (int)(2 * WW), s), "scan edges");
  int h_last[2];
  ck_(cudaMemcpyAsync(&h_last[0], qmap + 2 * WW - 1, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(&h_last[1], flag + 2 * WW - 1, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaStreamSynchronize(s), "sync");
  const int nq = h_last[0] + h_last[1];
  if (nq > qcap) throw ScratchError("more intersections than the device setup scratch holds (64 per grid line)");
  k_edge_compact<<<grid_for(2 * WW), 256, 0, s>>>(W, flag, qmap, qa, qi, qj);
  if (nq > 0) k_bisect<<<(nq + 127) / 128, 128, 0, s>>>(nq, S.lo, S.h, cs, qa, qi, qj, qx, qo, err);
  ck_(cudaGetLastError(), "edge kernels");
  S.nq = nq;
  S.q_axis.resize(nq); S.q_i.resize(nq); S.q_j.resize(nq); S.q_xi.resize(nq);
  q_owner.resize(nq);
  ck_(cudaMemcpyAsync(S.q_axis.data(), qa, nq * sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.q_i.data(), qi, nq * sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.q_j.data(), qj, nq * sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.q_xi.data(), qx, nq * sizeof(double), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(q_owner.data(), qo, nq * sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  int h_err = 0;
  ck_(cudaMemcpyAsync(&h_err, err, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  S.side.resize(WW);
  ck_(cudaMemcpyAsync(S.side.data(), side, WW, cudaMemcpyDeviceToHost, s), "d2h side");
  ck_(cudaStreamSynchronize(s), "sync");
  if (h_err & 1) throw GeomError("edge crossed by several components (R31)");
  if (h_err & 2) throw GeomError("grid edge crossed more than once (R31)");
  // irregular nodes
  k_irr_flags<<<grid_for(n2), 256, 0, s>>>(N, side, iflag, err);
  size_t tb2 = tb;
  ck_(cub::DeviceScan::ExclusiveSum(temp, tb2, iflag, imap, (int)n2, s), "scan irregular");
  ck_(cudaMemcpyAsync(&h_last[0], imap + n2 - 1, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(&h_last[1], iflag + n2 - 1, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(&h_err, err, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaStreamSynchronize(s), "sync");
  if (h_err & 4) throw GeomError("Γ too close to the box boundary (R32)");
  const int nirr = h_last[0] + h_last[1];
  if (nirr > icap) throw ScratchError("internal: more irregular nodes than 2·nq");
  k_irr_compact<<<grid_for(n2), 256, 0, s>>>(N, iflag, imap, side, ii, ij, isd, cnt);
  ck_(cudaMemsetAsync(cnt + nirr, 0, sizeof(int), s), "memset");
  size_t tb3 = tb;
  ck_(cub::DeviceScan::ExclusiveSum(temp, tb3, cnt, iptr, nirr + 1, s), "scan pairs");
  if (nirr > 0)
    k_irr_pairs<<<(nirr + 127) / 128, 128, 0, s>>>(N, S.lo, S.h, nirr, ii, ij, iptr, side, qmap, qx, pqv, pdv);
  ck_(cudaGetLastError(), "irregular-node kernels");
  S.nirr = nirr;
  S.irr_i.resize(nirr); S.irr_j.resize(nirr); S.irr_side.resize(nirr); S.irr_ptr.resize(nirr + 1);
  ck_(cudaMemcpyAsync(S.irr_i.data(), ii, nirr * sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.irr_j.data(), ij, nirr * sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.irr_side.data(), isd, nirr, cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.irr_ptr.data(), iptr, (nirr + 1) * sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaStreamSynchronize(s), "sync");
  const int npair = S.irr_ptr[nirr];
  S.pair_q.resize(npair);
  S.pair_d.resize(npair);
  ck_(cudaMemcpyAsync(S.pair_q.data(), pqv, npair * sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.pair_d.data(), pdv, npair * sizeof(double), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaStreamSynchronize(s), "sync");
}

// 2D stencils on the device (after the host's control points): fills S.st_nodes_ij, st_ext, st_w,
// st_wn, st_dx, st_dy, the unique stencil nodes (nsn, sn_i, sn_j) and st_node.  The Ω side array of
// gpu_setup_phases is still at the head of the scratch (same carve order).
void gpu_stencil_phase(Setup& S, void* scratch, size_t bytes, cudaStream_t s) {
  const int N = S.N, W = N + 1, M = S.M;
  const long WW = (long)W * W, n6 = 6L * M;
  uint8_t* p = reinterpret_cast<uint8_t*>(scratch);
  const int8_t* side = carve<int8_t>(p, WW);
  double* zx = carve<double>(p, M);
  double* zy = carve<double>(p, M);
  double* t1 = carve<double>(p, M);
  double* t2 = carve<double>(p, M);
  int64_t* nodes = carve<int64_t>(p, 2 * n6);
  int8_t* ext = carve<int8_t>(p, n6);
  double* w = carve<double>(p, n6);
  double* wn = carve<double>(p, n6);
  double* sdx = carve<double>(p, n6);
  double* sdy = carve<double>(p, n6);
  int64_t* keys = carve<int64_t>(p, n6);
  int64_t* sorted = carve<int64_t>(p, n6);
  int64_t* uk = carve<int64_t>(p, n6);
  int32_t* st_node = carve<int32_t>(p, n6);
  int* nu = carve<int>(p, 1);
  int* err = carve<int>(p, 1);
  size_t tb_sort = 0, tb_uniq = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tb_sort, keys, sorted, (int)n6, 0, 64, s);
  cub::DeviceSelect::Unique(nullptr, tb_uniq, sorted, uk, nu, (int)n6, s);
  const size_t tb = std::max(tb_sort, tb_uniq);
  void* temp = carve<uint8_t>(p, tb);
  if ((size_t)(p - reinterpret_cast<uint8_t*>(scratch)) > bytes) throw ScratchError("device setup scratch too small for the stencils");
  ck_(cudaMemcpyAsync(zx, S.z_x.data(), M * sizeof(double), cudaMemcpyHostToDevice, s), "h2d");
  ck_(cudaMemcpyAsync(zy, S.z_y.data(), M * sizeof(double), cudaMemcpyHostToDevice, s), "h2d");
  ck_(cudaMemcpyAsync(t1, S.z_t1.data(), M * sizeof(double), cudaMemcpyHostToDevice, s), "h2d");
  ck_(cudaMemcpyAsync(t2, S.z_t2.data(), M * sizeof(double), cudaMemcpyHostToDevice, s), "h2d");
  ck_(cudaMemsetAsync(err, 0, sizeof(int), s), "memset");
  if (M > 0)
    k_stencil2<<<(M + 127) / 128, 128, 0, s>>>(M, N, S.lo, S.h, zx, zy, t1, t2, side, nodes, ext, w, wn, sdx, sdy, keys, err);
  size_t tbs = tb;
  ck_(cub::DeviceRadixSort::SortKeys(temp, tbs, keys, sorted, (int)n6, 0, 64, s), "sort stencil keys");
  size_t tbu = tb;
  ck_(cub::DeviceSelect::Unique(temp, tbu, sorted, uk, nu, (int)n6, s), "unique stencil keys");
  if (n6 > 0) k_stencil_rank<<<grid_for(n6), 256, 0, s>>>(n6, keys, uk, nu, st_node);
  ck_(cudaGetLastError(), "stencil kernels");
  int h_nu = 0, h_err = 0;
  ck_(cudaMemcpyAsync(&h_nu, nu, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(&h_err, err, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  S.st_nodes_ij.resize(2 * n6);
  S.st_ext.resize(n6); S.st_w.resize(n6); S.st_wn.resize(n6); S.st_dx.resize(n6); S.st_dy.resize(n6);
  S.st_node.resize(n6);
  ck_(cudaMemcpyAsync(S.st_nodes_ij.data(), nodes, 2 * n6 * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.st_ext.data(), ext, n6, cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.st_w.data(), w, n6 * sizeof(double), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.st_wn.data(), wn, n6 * sizeof(double), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.st_dx.data(), sdx, n6 * sizeof(double), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.st_dy.data(), sdy, n6 * sizeof(double), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.st_node.data(), st_node, n6 * sizeof(int32_t), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaStreamSynchronize(s), "sync");
  if (h_err) throw GeomError("interpolation stencil leaves the grid or is singular");
  std::vector<int64_t> hu(h_nu);
  ck_(cudaMemcpyAsync(hu.data(), uk, h_nu * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaStreamSynchronize(s), "sync");
  S.nsn = h_nu;
  S.sn_i.resize(h_nu);
  S.sn_j.resize(h_nu);
  for (int u = 0; u < h_nu; ++u) {
    S.sn_i[u] = (int)(hu[u] / W / 3);
    S.sn_j[u] = (int)(hu[u] % W);
  }
}

// 3D ten-point stencils on the device (after the host's frames): fills S.st_nodes_ij, st_w, st_wn, st_c,
// st_code.  The Ω side array of gpu_setup_phases3 is still at the head of the scratch.
void gpu_stencil_phase3(Setup3& S, void* scratch, size_t bytes, cudaStream_t s) {
  const int N = S.N, W = N + 1, nq = S.nq;
  const long WWW = (long)W * W * W;
  uint8_t* p = reinterpret_cast<uint8_t*>(scratch);
  const int8_t* side = carve<int8_t>(p, WWW);
  double* qpos = carve<double>(p, 3L * nq);
  double* qn = carve<double>(p, 3L * nq);
  int64_t* nodes = carve<int64_t>(p, 30L * nq);
  double* w = carve<double>(p, 10L * nq);
  double* wn = carve<double>(p, 10L * nq);
  int32_t* stc = carve<int32_t>(p, 3L * nq);
  int32_t* code = carve<int32_t>(p, nq);
  int* err = carve<int>(p, 1);
  if ((size_t)(p - reinterpret_cast<uint8_t*>(scratch)) > bytes) throw ScratchError("device setup scratch too small for the stencils");
  ck_(cudaMemcpyAsync(qpos, S.q_pos.data(), 3L * nq * sizeof(double), cudaMemcpyHostToDevice, s), "h2d");
  ck_(cudaMemcpyAsync(qn, S.q_n.data(), 3L * nq * sizeof(double), cudaMemcpyHostToDevice, s), "h2d");
  ck_(cudaMemsetAsync(nodes, 0, 30L * nq * sizeof(int64_t), s), "memset");
  ck_(cudaMemsetAsync(err, 0, sizeof(int), s), "memset");
  if (nq > 0) k_stencil3<<<(nq + 127) / 128, 128, 0, s>>>(nq, N, S.lo, S.h, qpos, qn, side, nodes, w, wn, stc, code, err);
  ck_(cudaGetLastError(), "stencil kernel");
  int h_err = 0;
  ck_(cudaMemcpyAsync(&h_err, err, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  S.st_nodes_ij.resize(30L * nq);
  S.st_w.resize(10L * nq);
  S.st_wn.resize(10L * nq);
  S.st_c.resize(3L * nq);
  S.st_code.resize(nq);
  ck_(cudaMemcpyAsync(S.st_nodes_ij.data(), nodes, 30L * nq * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.st_w.data(), w, 10L * nq * sizeof(double), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.st_wn.data(), wn, 10L * nq * sizeof(double), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.st_c.data(), stc, 3L * nq * sizeof(int32_t), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaMemcpyAsync(S.st_code.data(), code, nq * sizeof(int32_t), cudaMemcpyDeviceToHost, s), "d2h");
  ck_(cudaStreamSynchronize(s), "sync");
  if (h_err) throw GeomError("interpolation stencil leaves the grid or is singular");
}

}  // namespace kfbi
