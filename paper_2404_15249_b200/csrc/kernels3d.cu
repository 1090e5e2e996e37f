// sm_100a kernels of the 3D KFBI interface-problem apply (arXiv 2404.15249; readings R12-R14):
//   k_lsq3       A1  tangent-plane LSQ fit of the density (control points = intersections, R12)
//   k_correct3   A2+A3 Monge-patch jumps + seven-point corrections (compact list)
//   k_fwd3s      A4  sparse z-DST evaluated directly from the corrections, fused with the y-DST
//   k_sweep3 / k_reduced3   A5 block tridiagonal solves along x + separator system (ADM)
//   k_inv3y      A6  fixed-up y-inverse rows (transposed store); k_zeval3 z-inverse at stencil nodes
//   k_interp3    A7  ten-point jump-corrected interpolation (R14)
//   k_dst_rows3t / k_transpose3 / k_base3   dense rows for the once-per-solve applies
#include <cuda_runtime.h>

#include <algorithm>

#include "device.cuh"
#include "kernels.h"

// =============================================================================== 3D path
// Working array layout: work[(i−1)·N² + a·N + b], i = 1..N−1 (x), a, b ∈ [0, N) padded (index 0 ≡ 0).
// Forward: rows (i, j) DST along z (b: l → ll) → plane transpose → rows (i, ll) DST along y
// (j → kk): spectral layout [i][ll][kk], mode m = ll·N + kk.  Tridiagonal along x per mode
// (same two-level arrowhead as 2D).  Inverse: rows (i, ll) with the fix-up (kk → j) → transpose →
// rows (i, j) (ll → l).
namespace kfbi {
namespace {

struct Jump10 {
  double v, g[3], H[6];   // H: xx, yy, zz, xy, xz, yz
};

// Monge-patch closed form (reading R13): [∇v] = Σ_a ∂_aΦ e_a + Ψ n,
// A_ab = ∂_abΦ − κ_ab Ψ, A_an = ∂_aΨ + Σ_b κ_ab ∂_bΦ, A_nn = [F] + κΦ − A_11 − A_22, [D²v] = F A Fᵀ.
__device__ __forceinline__ Jump10 jumps3d(double Phi, const double* dP, double Psi, const double* dPsi, double F,
                                          double kappa, const double* n, const double* e1, const double* e2,
                                          const double* kab) {
  // [∇v] = ∂_aΦ e_a + Ψ n; A_ab = ∂_abΦ − κ_ab Ψ; A_an = ∂_aΨ + κ_ab ∂_bΦ
  Jump10 J;
  J.v = Phi;
#pragma unroll
  for (int r = 0; r < 3; ++r) J.g[r] = dP[0] * e1[r] + dP[1] * e2[r] + Psi * n[r];
  const double A11 = dP[2] - kab[0] * Psi, A12 = dP[3] - kab[1] * Psi, A22 = dP[4] - kab[2] * Psi;
  const double A1n = dPsi[0] + kab[0] * dP[0] + kab[1] * dP[1];
  const double A2n = dPsi[1] + kab[1] * dP[0] + kab[2] * dP[1];
  const double Ann = F + kappa * Phi - A11 - A22;
  auto h = [&](int r, int c) {
    return A11 * e1[r] * e1[c] + A12 * (e1[r] * e2[c] + e2[r] * e1[c]) + A22 * e2[r] * e2[c] +
           A1n * (e1[r] * n[c] + n[r] * e1[c]) + A2n * (e2[r] * n[c] + n[r] * e2[c]) + Ann * n[r] * n[c];
  };
  J.H[0] = h(0, 0);
  J.H[1] = h(1, 1);
  J.H[2] = h(2, 2);
  J.H[3] = h(0, 1);
  J.H[4] = h(0, 2);
  J.H[5] = h(1, 2);
  return J;
}

__device__ __forceinline__ void load_jump3(const DevTables3& T, int q, const double* phi, const double* dphi,
                                           const double* fq, const double* jg, Jump10& J) {
  if (jg) {
    J.v = jg[10 * q];
#pragma unroll
    for (int r = 0; r < 3; ++r) J.g[r] = jg[10 * q + 1 + r];
#pragma unroll
    for (int r = 0; r < 6; ++r) J.H[r] = jg[10 * q + 4 + r];
    return;
  }
  double dP[5] = {0, 0, 0, 0, 0}, dPs[2] = {0, 0};
  double Phi = 0.0, Psi = 0.0;
  if (phi && T.neumann) {   // density ψ = [∂_n v], [v] = 0 (R38)
    Psi = phi[q];
    dPs[0] = dphi[5 * q];
    dPs[1] = dphi[5 * q + 1];
  } else if (phi) {
    Phi = phi[q];
#pragma unroll
    for (int r = 0; r < 5; ++r) dP[r] = dphi[5 * q + r];
  }
  J = jumps3d(Phi, dP, Psi, dPs, fq ? fq[q] : 0.0, T.kappa, T.q_n + 3 * q, T.q_e1 + 3 * q, T.q_e2 + 3 * q,
              T.q_kab + 3 * q);
}

// A1 (3D): tangent-plane LSQ fit (reading R12) with the precomputed scaled normal-matrix inverse and the
// neighbours' tangent coordinates from setup (streamed; only φ is gathered).  Eight lanes per control
// point stride over its ~30 neighbours; the five moments are summed by a fixed xor tree.
constexpr int kLsqLanes = 8;
__global__ void k_lsq3(DevTables3 T, const double* __restrict__ phi, double* __restrict__ dphi) {
  pdl_wait();   // φ from the previous kernel
  // point p → the p-th control point of the slab's three per-axis ranges
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  int e = gt / kLsqLanes;
  const int sub = gt % kLsqLanes;
  const int n0 = T.q_hi[0] - T.q_lo[0], n1 = T.q_hi[1] - T.q_lo[1], n2 = T.q_hi[2] - T.q_lo[2];
  const bool valid = e < n0 + n1 + n2;
  e = !valid ? 0 : (e < n0 ? T.q_lo[0] + e : (e < n0 + n1 ? T.q_lo[1] + e - n0 : T.q_lo[2] + e - n0 - n1));
  double b[5] = {0, 0, 0, 0, 0};
  if (valid) {
    const double f0 = phi[e];
    const double2* __restrict__ tt = reinterpret_cast<const double2*>(T.lsq_t);
    for (int u = T.lsq_ptr[e] + sub; u < T.lsq_ptr[e + 1]; u += kLsqLanes) {
      const double2 t = tt[u];
      const double df = phi[T.lsq_nb[u]] - f0;
      b[0] = fma(t.x, df, b[0]);
      b[1] = fma(t.y, df, b[1]);
      b[2] = fma(0.5 * t.x * t.x, df, b[2]);
      b[3] = fma(t.x * t.y, df, b[3]);
      b[4] = fma(0.5 * t.y * t.y, df, b[4]);
    }
  }
#pragma unroll
  for (int o = kLsqLanes / 2; o > 0; o >>= 1)
#pragma unroll
    for (int r = 0; r < 5; ++r) b[r] += __shfl_xor_sync(0xffffffffu, b[r], o);
  if (!valid || sub) return;
  const double ih = 1.0 / T.h;
  const double* G = T.lsq_G + 15 * (size_t)e;
  // symmetric 5×5 from its upper triangle
  const double g[5][5] = {{G[0], G[1], G[2], G[3], G[4]},
                          {G[1], G[5], G[6], G[7], G[8]},
                          {G[2], G[6], G[9], G[10], G[11]},
                          {G[3], G[7], G[10], G[12], G[13]},
                          {G[4], G[8], G[11], G[13], G[14]}};
  double a[5];
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 5; ++c) s = fma(g[r][c], b[c], s);
    a[r] = s;
  }
  dphi[5 * e] = a[0] * ih;
  dphi[5 * e + 1] = a[1] * ih;
  dphi[5 * e + 2] = a[2] * ih * ih;
  dphi[5 * e + 3] = a[3] * ih * ih;
  dphi[5 * e + 4] = a[4] * ih * ih;
}

// dense base h²·f·1_Ω (or 0) into the padded working layout
__global__ void k_base3(DevTables3 T, const double* __restrict__ f, double* __restrict__ work) {
  const int N = T.N, W = N + 1;
  const size_t total = (size_t)(N - 1) * N * N;
  const double h2 = T.h * T.h;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx / ((size_t)N * N)) + 1;
    const int a = (int)((idx / N) % N), b = (int)(idx % N);
    double v = 0.0;
    if (f && a > 0 && b > 0) {
      const size_t u = ((size_t)i * W + a) * W + b;
      if (T.side[u]) v = h2 * f[u];
    }
    work[idx] = v;
  }
}

// A2+A3 (3D): seven-point correction at irregular nodes, added in place (×h²)
__global__ void k_correct3(DevTables3 T, const double* __restrict__ phi, const double* __restrict__ dphi,
                           const double* __restrict__ fq, const double* __restrict__ jg, double* __restrict__ work,
                           double* __restrict__ corr) {
  pdl_wait();   // φ and its LSQ derivatives from k_lsq3
  const int n = T.n_lo + blockIdx.x * blockDim.x + threadIdx.x;   // the slab's irregular nodes
  if (n >= T.n_hi) return;
  double acc = 0.0;
  for (int e = T.irr_ptr[n]; e < T.irr_ptr[n + 1]; ++e) {
    const int q = T.pair_q[e];
    KFBI_CHECK(q >= 0 && q < T.nq, q, T.nq);
    const double d = T.pair_d[e];
    const int ax = T.q_axis[q];
    Jump10 J;
    load_jump3(T, q, phi, dphi, fq, jg, J);
    acc += J.v + J.g[ax] * d + 0.5 * J.H[ax] * d * d;   // H[0..2] = xx, yy, zz
  }
  if (corr) corr[n] = T.irr_side[n] ? -acc : acc;   // compact (sparse K_D path)
  else work[T.irr_lin[n]] += T.irr_side[n] ? -acc : acc;
}

// the fixed-up spectral row (i, m0/N) (R20: x = z − h_{g−1} Z_L − h_g Z_R; separators x = h) as pairs
// z[zpad(m)] = (x_2m, x_2m+1), x_0 := 0; loads in batches of 4 pairs so that all 20 are in flight
template <int N>
__device__ __forceinline__ void load_fixed_row(const DevTables3& T, const double* __restrict__ spec,
                                               const double* __restrict__ hsep, int i, size_t m0, double2* z,
                                               int tid) {
  constexpr int NTL = N / 32;
  {
    const size_t K = (size_t)N * N;
    const int q = i / BL, r = i - q * BL, p = r - 1;
    const double* xs = r == 0 ? hsep + (size_t)(q - 1) * K : spec + (size_t)(i - 1) * K;
    const bool left = r != 0 && q > 0, right = r != 0 && q < T.P - 1;
    const double* hl = hsep + (size_t)(q - 1) * K;
    const double* zl = T.zr + (size_t)(LB - 1 - p) * K;
    const double* hr = hsep + (size_t)q * K;
    const double* zrr = T.zr + (size_t)p * K;
#pragma unroll
    for (int sb = 0; sb < 16; sb += 4) {
      double2 x[4], a1[4], b1[4], a2[4], b2[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const size_t mm = m0 + 2 * (tid + (sb + u) * NTL);
        x[u] = __ldcs(reinterpret_cast<const double2*>(xs + mm));
        if (left) {
          a1[u] = __ldg(reinterpret_cast<const double2*>(hl + mm));
          b1[u] = __ldg(reinterpret_cast<const double2*>(zl + mm));
        }
        if (right) {
          a2[u] = __ldg(reinterpret_cast<const double2*>(hr + mm));
          b2[u] = __ldg(reinterpret_cast<const double2*>(zrr + mm));
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        double2 t = x[u];
        if (left) {
          t.x = fma(-a1[u].x, b1[u].x, t.x);
          t.y = fma(-a1[u].y, b1[u].y, t.y);
        }
        if (right) {
          t.x = fma(-a2[u].x, b2[u].x, t.x);
          t.y = fma(-a2[u].y, b2[u].y, t.y);
        }
        const int m = tid + (sb + u) * NTL;
        if (m == 0) t.x = 0.0;
        z[zpad(m)] = t;
      }
    }
  }
}

// batched DST-I of the rows of length N (index 0 ≡ 0): one row per N/32 lanes, 8192/N rows per CTA.
// MODE 0: in place (× scale); 1: in place from the fixed-up spectral rows; 2: into the (N+1)³ grid u.
// MODE 3: the forward source is built on load — h²·f·1_Ω from the full grid `src` plus the row's
// compact corrections (the dense base is never written).
template <int MODE, int N>
__global__ void __launch_bounds__(256, 2) k_dst_rows3t(DevTables3 T, double* work, const double* __restrict__ hsep,
                                                       double scale, double* __restrict__ out,
                                                       const double* __restrict__ src,
                                                       const double* __restrict__ corr, int compact) {
  pdl_wait();   // the rows from the previous kernel
  constexpr int NTL = N / 32, RPC = 256 / NTL, ZS = N / 2 + N / 32 + 1;
  extern __shared__ double2 smz[];
  const int rl = threadIdx.x / NTL, tid = threadIdx.x % NTL;
  double2* z = smz + rl * ZS;
  const double2* __restrict__ tw = reinterpret_cast<const double2*>(T.tw);
  const size_t row = (size_t)(T.i_lo - 1) * N + (size_t)blockIdx.x * RPC + rl;   // (i−1)·N + a, slab planes
  const bool live = row < (size_t)T.i_hi * N;
  const int i = (int)(row / N) + 1, a = (int)(row % N);
  double* rp = work + row * N;
  if (MODE == 1 && live) {
    load_fixed_row<N>(T, work, hsep, i, (size_t)a * N, z, tid);
  } else if (MODE == 3) {
    const int W = N + 1;
    const double h2 = T.h * T.h;
    const size_t gbase = ((size_t)i * W + a) * W;
    const size_t gr = (size_t)i * W + a;   // grid row (i, a)
    const uint32_t* info = compact ? T.om_info + gr * 2 * T.om_nsegp : nullptr;
    // Ω-compact f: the value at node j of the row has rank om_row + (count before j's segment) + popc
    auto cval = [&](int j) {
      const uint32_t b = info[j >> 5];
      if (!((b >> (j & 31)) & 1u)) return 0.0;
      const int r = T.om_row[gr] + (int)info[T.om_nsegp + (j >> 5)] + __popc(b & ((1u << (j & 31)) - 1u));
      KFBI_CHECK(r < T.om_row[gr + 1], r, (int)gr);
      return h2 * src[r];
    };
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const int m = tid + s * NTL;
      double v0 = 0.0, v1 = 0.0;
      if (live && a > 0 && src) {
        if (compact) {
          if (m > 0) v0 = cval(2 * m);
          v1 = cval(2 * m + 1);
        } else {
          if (m > 0 && T.side[gbase + 2 * m]) v0 = h2 * src[gbase + 2 * m];
          if (T.side[gbase + 2 * m + 1]) v1 = h2 * src[gbase + 2 * m + 1];
        }
      }
      z[zpad(m)] = make_double2(v0, v1);
    }
    __syncwarp();
    if (live && a > 0 && corr) {   // the row's irregular nodes (distinct z indices)
      double* fz = reinterpret_cast<double*>(z);
      for (int e = T.irr_row_ptr[row] + tid; e < T.irr_row_ptr[row + 1]; e += NTL) {
        const int b = (int)(T.irr_lin[e] & (N - 1));
        fz[2 * zpad(b >> 1) + (b & 1)] += corr[e];
      }
    }
  } else {
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const int m = tid + s * NTL;   // pair (f_2m, f_2m+1)
      double2 t = make_double2(0.0, 0.0);
      if (live) t = __ldcs(reinterpret_cast<const double2*>(rp + 2 * m));
      if (m == 0) t.x = 0.0;
      z[zpad(m)] = t;
    }
  }
  __syncwarp();
  dst2_core<N>(z, tw, tid);
  if (!live) return;
  const double* F = reinterpret_cast<const double*>(z);
  const double sc = a == 0 ? 0.0 : scale;
  if (MODE == 2 && compact) {   // u at the row's Ω nodes only (row-major ranks)
    const size_t gr = (size_t)i * (N + 1) + a;
    const uint32_t* info = T.om_info + gr * 2 * T.om_nsegp;
    const int r0 = T.om_row[gr];
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const int j = 2 * (tid + s * NTL);
      const double2 f = *reinterpret_cast<const double2*>(F + fpos(j));
      const uint32_t b = info[j >> 5];   // j, j + 1 share a segment (j even)
      const int r = r0 + (int)info[T.om_nsegp + (j >> 5)] + __popc(b & ((1u << (j & 31)) - 1u));
      if ((b >> (j & 31)) & 1u) {
        KFBI_CHECK(r < T.om_row[gr + 1], r, (int)gr);
        out[r] = sc * f.x;
      }
      if ((b >> ((j + 1) & 31)) & 1u) {
        const int r1 = r + (int)((b >> (j & 31)) & 1u);
        KFBI_CHECK(r1 < T.om_row[gr + 1], r1, (int)gr);
        out[r1] = sc * f.y;
      }
    }
  } else if (MODE == 2) {
    double* op = out + ((size_t)i * (N + 1) + a) * (N + 1);
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const int j = 2 * (tid + s * NTL);
      const double2 f = *reinterpret_cast<const double2*>(F + fpos(j));
      op[j] = sc * f.x;
      op[j + 1] = sc * f.y;
    }
    if (tid == 0) op[N] = 0.0;
  } else {
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const int j = 2 * (tid + s * NTL);
      const double2 f = *reinterpret_cast<const double2*>(F + fpos(j));
      __stcs(reinterpret_cast<double2*>(rp + j), make_double2(sc * f.x, sc * f.y));
    }
  }
}

// ---- sparse K_D path (3D): the source of (Δ_h − κ)v = F is nonzero only at irregular nodes, and
// only the distinct stencil nodes of the result are read, so the z-direction transforms are sparse.
// forward: plane i, columns ll ∈ [l0, l0 + RPC): G_a = Σ_{irregular (i,a,b)} c · sin(π b ll/N) (the
// z-DST of the sparse rows, evaluated directly), then the y-DST of G along a → work[(i−1)][ll][kk].
#ifndef KFBI_FWD_GROUPS
#define KFBI_FWD_GROUPS 8
#endif
constexpr int kFwdGroups = KFBI_FWD_GROUPS;
template <int N>
__global__ void __launch_bounds__(256, 2) k_fwd3s(DevTables3 T, const double* __restrict__ corr,
                                                  double* __restrict__ work) {
  constexpr int NTL = N / 32, RPC = 256 / NTL < N ? 256 / NTL : N, NTHR = RPC * NTL, ZS = N / 2 + N / 32 + 1;
  constexpr int CPT = RPC < 16 ? RPC : 16, NG = RPC / CPT;
  extern __shared__ double2 smz[];
  const double2* __restrict__ tw = reinterpret_cast<const double2*>(T.tw);
  const int i = blockIdx.y + T.i_lo;
  if (!(T.plane_flags[i] & 1)) return;   // no irregular node in the plane: k_sweep3 reads it as zero
  __shared__ int s_ptr[N + 1];
  __shared__ double s_q[N / 2 + 1];   // quarter-wave sin(π r/N): staging rotations from smem, not L1/L2
  for (int r = threadIdx.x; r <= N / 2; r += NTHR) s_q[r] = T.sin_tab[r];
  // the plane's irregular entries (value, z index) staged once, coalesced: one round trip to L2
  double* s_val = reinterpret_cast<double*>(smz + RPC * ZS);
  int16_t* s_b = reinterpret_cast<int16_t*>(s_val + T.max_plane_irr);
  const int E0 = T.irr_row_ptr[(size_t)(i - 1) * N];
  for (int a = threadIdx.x; a <= N; a += NTHR) s_ptr[a] = T.irr_row_ptr[(size_t)(i - 1) * N + a] - E0;
  pdl_wait();   // the corrections from k_correct3
  {
    const int ne = T.irr_row_ptr[(size_t)i * N] - E0;
    for (int e = threadIdx.x; e < ne; e += NTHR) {
      s_val[e] = corr[E0 + e];
      s_b[e] = (int16_t)(T.irr_lin[E0 + e] & (N - 1));
    }
  }
  __syncthreads();
  // CTA rows = RPC/4 mode quads {t, N−t, N/2−t, N/2+t} (quad t = 0: {0, N/2, N/4, 3N/4}); with
  // s, c = sin, cos(πbt/N): sin(πb(N−t)/N) = (−1)^{b+1} s, sin(πb(N/2 ± t)/N) = sin(πb/2) c ± cos(πb/2) s,
  // so one rotation per entry serves four columns (the 2D sweep's quad symmetry, along z).
  constexpr int QPI = CPT / 4;   // quads per item
  // kFwdGroups consecutive mode groups per CTA: the plane's entries are staged once for all of them
  for (int grp = blockIdx.x * kFwdGroups; grp < (blockIdx.x + 1) * kFwdGroups && grp * RPC < N; ++grp) {
  const int tq0 = grp * (RPC / 4);
  if (grp != blockIdx.x * kFwdGroups) __syncthreads();   // the previous group's rows have been written out
  // G rows: entries e of grid row a (sorted by count) → CPT mode sums.  Rows with more than
  // kHeavyRow entries (the first H of the plane's order) are split over 8 lanes and summed by a fixed
  // xor tree; the rest take one thread each.  Keeps the longest per-thread chain near the mean.
  auto accumulate = [&](int e, int t0, double (&g)[CPT]) {
    const double v = s_val[e];
    const int b = s_b[e];
    const double sg1 = (b & 1) ? v : -v;                                   // (−1)^{b+1} v
    const double sg2 = ((b & 3) == 0 || (b & 3) == 3) ? -v : v, sg3 = (b & 3) <= 1 ? v : -v;
    const int r0 = (b * t0) & (2 * N - 1);
    double2 w = make_double2(sin_lookup(s_q, (r0 + N / 2) & (2 * N - 1), N), sin_lookup(s_q, r0, N));
    const double2 d = make_double2(sin_lookup(s_q, (b + N / 2) & (2 * N - 1), N), sin_lookup(s_q, b, N));
#pragma unroll
    for (int u = 0; u < QPI; ++u) {
      const double sv = w.y, cv = w.x, A = (b & 1) ? cv : sv;
      if (t0 + u == 0) {   // special quad: modes 0 (unused), N/2, N/4, 3N/4
        g[4 * u + 1] = fma(v, sin_lookup(s_q, (b * (N / 2)) & (2 * N - 1), N), g[4 * u + 1]);
        g[4 * u + 2] = fma(v, sin_lookup(s_q, (b * (N / 4)) & (2 * N - 1), N), g[4 * u + 2]);
        g[4 * u + 3] = fma(v, sin_lookup(s_q, (b * (3 * N / 4)) & (2 * N - 1), N), g[4 * u + 3]);
      } else {
        g[4 * u + 0] = fma(v, sv, g[4 * u + 0]);
        g[4 * u + 1] = fma(sg1, sv, g[4 * u + 1]);
        g[4 * u + 2] = fma(sg2, A, g[4 * u + 2]);
        g[4 * u + 3] = fma(sg3, A, g[4 * u + 3]);
      }
      if (u + 1 < QPI) w = cmul(w, d);
    }
  };
  auto store = [&](int a, int cg, const double (&g)[CPT]) {
    const int off = 2 * zpad(a >> 1) + (a & 1);
#pragma unroll
    for (int c = 0; c < CPT; ++c) reinterpret_cast<double*>(smz + (cg * CPT + c) * ZS)[off] = a ? g[c] : 0.0;
  };
  const int16_t* perm = T.irr_row_perm + (size_t)(i - 1) * N;
  const int H = T.irr_row_nheavy[i - 1];
  {   // heavy rows: 4 per warp per round, warp-uniform trip count (all lanes take part in the shuffles)
    const int lane = threadIdx.x & 31, sub = lane & 7;
    const int nitem = H * NG;
    for (int base = (threadIdx.x >> 5) * 4; base < nitem; base += NTHR / 8) {
      const int hi = base + (lane >> 3);
      const bool act = hi < nitem;
      const int cg = act ? hi / H : 0, a = act ? perm[hi % H] : 0;
      double g[CPT];
#pragma unroll
      for (int c = 0; c < CPT; ++c) g[c] = 0.0;
      if (act) {
        const int e1 = s_ptr[a + 1], t0 = tq0 + cg * QPI;
        for (int e = s_ptr[a] + sub; e < e1; e += 8) accumulate(e, t0, g);
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1)
#pragma unroll
        for (int c = 0; c < CPT; ++c) g[c] += __shfl_xor_sync(0xffffffffu, g[c], o);
      if (act && sub == 0) store(a, cg, g);
    }
  }
  const int NL = N - H;   // light rows (≤ kHeavyRow entries, incl. the empty ones): one thread each
  // rows in descending entry count, dealt in snake order over the threads (thread t takes the t-th and
  // the (2·NTHR − 1 − t)-th heaviest, …): the barrier below waits for the slowest thread
  for (int it0 = threadIdx.x; it0 < NL * NG; it0 += NTHR) {
    const int rnd = it0 / NTHR, pos = it0 - rnd * NTHR;
    const int rem = min(NTHR, NL * NG - rnd * NTHR);   // items in this round
    const int it = (rnd & 1) ? rnd * NTHR + (rem - 1 - pos) : it0;
    const int cg = it / NL, a = perm[H + it % NL];
    double g[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) g[c] = 0.0;
    const int e1 = s_ptr[a + 1], t0 = tq0 + cg * QPI;
    for (int e = s_ptr[a]; e < e1; ++e) accumulate(e, t0, g);
    store(a, cg, g);
  }
  const int rl = threadIdx.x / NTL, tid = threadIdx.x % NTL;
  const double2 wa = __ldg(tw + 2 * tid), wb = __ldg(tw + 2 * tid + 1);   // in flight across the barrier
  __syncthreads();
  double2* z = smz + rl * ZS;
  dst2_core_w<N>(z, tw, tid, wa, wb);
  const int tq = tq0 + (rl >> 2), mem = rl & 3;   // this row's mode: member of quad tq
  const int ll = tq ? (mem == 0 ? tq : mem == 1 ? N - tq : mem == 2 ? N / 2 - tq : N / 2 + tq)
                    : (mem == 0 ? 0 : mem == 1 ? N / 2 : mem == 2 ? N / 4 : 3 * N / 4);
  const double sc = ll ? 1.0 : 0.0;
  const double* F = reinterpret_cast<const double*>(z);
  KFBI_CHECK(i >= T.i_lo && i <= T.i_hi && ll >= 0 && ll < N, i, ll);
  double* op = work + ((size_t)(i - 1) * N + ll) * N;
#pragma unroll
  for (int s = 0; s < 16; ++s) {
    const int j = 2 * (tid + s * NTL);
    const double2 f = *reinterpret_cast<const double2*>(F + fpos(j));
    __stcs(reinterpret_cast<double2*>(op + j), make_double2(sc * f.x, sc * f.y));
  }
  }
}

// inverse along y: spectral rows (i, ll) fixed up with the separators (R20), DST along kk → a, stored
// transposed to out[(i−1)][a][ll] so that the z-direction evaluation reads contiguous rows.
template <int N>
#ifndef KFBI_INV3Y_MINB
#define KFBI_INV3Y_MINB 2
#endif
__global__ void __launch_bounds__(256, KFBI_INV3Y_MINB) k_inv3y(DevTables3 T, const double* __restrict__ spec,
                                                  const double* __restrict__ hsep, double scale,
                                                  double* __restrict__ out) {
  constexpr int NTL = N / 32, RPC = 256 / NTL < N ? 256 / NTL : N, NTHR = RPC * NTL, ZS = N / 2 + N / 32 + 1;
  extern __shared__ double2 smz[];
  const double2* __restrict__ tw = reinterpret_cast<const double2*>(T.tw);
  const int i = blockIdx.y + T.i_lo, l0 = blockIdx.x * RPC;
  const int rl = threadIdx.x / NTL, tid = threadIdx.x % NTL;
  double2* z = smz + rl * ZS;
  const size_t m0 = (size_t)(l0 + rl) * N;
  __shared__ int16_t s_row[N];   // visible after the barrier below
  const int w0 = T.zplane_ptr[i - 1], nn = T.zplane_ptr[i] - w0;
  if (nn == 0) return;   // no stencil row in the plane (CTA-uniform, before any barrier)
  for (int w = threadIdx.x; w < nn; w += NTHR) s_row[w] = (int16_t)(T.zrow_id[w0 + w] - (i - 1) * N);
  pdl_wait();   // the spectrum (k_sweep3) and the separators (k_reduced3 / the level-2 fix-up)
  load_fixed_row<N>(T, spec, hsep, i, m0, z, tid);
  __syncwarp();
  dst2_core<N>(z, tw, tid);
  __syncthreads();
  // only the grid rows (i, a) that hold stencil nodes are read by the z-evaluation: the others are
  // not stored (≈ 80 % of the y-inverse's writes at C5)
  for (int idx = threadIdx.x; idx < nn * RPC; idx += NTHR) {
    const int c = idx % RPC, a = s_row[idx / RPC];
    const double v = (a == 0 || l0 + c == 0) ? 0.0 : scale * reinterpret_cast<const double*>(smz + c * ZS)[fpos(a)];
    out[((size_t)(i - 1) * N + a) * N + l0 + c] = v;
  }
}

// z-direction inverse at the distinct stencil nodes only: v(i,a,b) = scale · Σ_ll R[ll] sin(π ll b/N)
// for the row R = rows[(i−1)][a][·].  A warp per row (grid-stride, next row prefetched); lane l holds
// ll = U·l + 32U·s + u (coalesced double2 loads); per u the sum over s is a Clenshaw recurrence in
// e^{i·32Uθ} (θ = πb/N), combined as Im(e^{iUlθ}(S_0 + e^{iθ} S_1)); warp reduction.
template <int N>
__global__ void __launch_bounds__(256) k_zeval3(DevTables3 T, const double* __restrict__ rows, double scale,
                                                double* __restrict__ work) {
  constexpr int V = N / 32, U = V >= 2 ? 2 : 1, S = V / U;
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * 8;
  const double2* __restrict__ tw = reinterpret_cast<const double2*>(T.tw);
  auto load = [&](int w, double (&c)[S][U]) {
    const double* rp = rows + (size_t)T.zrow_id[w] * N + U * lane;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      if constexpr (U == 2) {
        const double2 v = __ldcs(reinterpret_cast<const double2*>(rp + 32 * U * s));
        c[s][0] = v.x;
        c[s][U - 1] = v.y;
      } else {
        c[s][0] = __ldcs(rp + 32 * s);
      }
    }
  };
  int w = T.w_lo + (int)(((size_t)blockIdx.x * 256 + threadIdx.x) >> 5);
  pdl_wait();   // the y-inverse rows from k_inv3y
  if (w >= T.w_hi) return;
  double cur[S][U];
  load(w, cur);
  while (w < T.w_hi) {
    const int wn = w + nw;
    double nxt[S][U];
    if (wn < T.w_hi) load(wn, nxt);
    const size_t rbase = (size_t)T.zrow_id[w] * N;
    KFBI_CHECK(T.zrow_id[w] / N + 1 >= T.i_lo && T.zrow_id[w] / N + 1 <= T.i_hi, T.zrow_id[w], w);
    const int e1 = T.zrow_ptr[w + 1];
    for (int e0 = T.zrow_ptr[w]; e0 < e1; e0 += 8) {   // 8 nodes per transpose-reduction
    double vv[8];
#pragma unroll
    for (int nd = 0; nd < 8; ++nd) {
      const int e = e0 + nd;
      if (e >= e1) {
        vv[nd] = 0.0;
        continue;
      }
      const int b = T.znode_b[e];
      const double2 w1 = __ldg(tw + b);                                   // e^{iθ}
      const double2 wz = __ldg(tw + ((32 * U * b) & (2 * N - 1)));        // e^{i·32Uθ}
      const double2 wl = __ldg(tw + ((U * lane * b) & (2 * N - 1)));      // e^{iUlθ}
      const double twoc = 2.0 * wz.x;
      double sr[U], si[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        double b1 = 0.0, b2 = 0.0;
#pragma unroll
        for (int s = S - 1; s >= 0; --s) {
          const double b0 = fma(twoc, b1, cur[s][u] - b2);
          b2 = b1;
          b1 = b0;
        }
        sr[u] = fma(-b2, wz.x, b1);   // Σ_s c z^s = b_0 − b_1 z̄
        si[u] = b2 * wz.y;
      }
      double tr = sr[0], ti = si[0];
      if constexpr (U == 2) {
        tr += w1.x * sr[1] - w1.y * si[1];
        ti += w1.x * si[1] + w1.y * sr[1];
      }
      vv[nd] = wl.y * tr + wl.x * ti;
    }
    const double tot = warp_transpose_reduce8(vv);   // lane l: node 4·(l>>4&1) + 2·(l>>3&1) + (l>>2&1)
    const int nd = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
    if ((lane & 3) == 0 && e0 + nd < e1) work[rbase + T.znode_b[e0 + nd]] = scale * tot;
    }
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
      for (int u = 0; u < U; ++u) cur[s][u] = nxt[s][u];
    w = wn;
  }
}

// in-place transpose of every N×N plane by 32×32 tile pairs
__global__ void k_transpose3(int N, double* work) {
  __shared__ double ta[32][33], tb[32][33];
  const int T = N / 32;
  int p = blockIdx.x;   // tile pair index within a plane: (a, b) with a ≤ b
  int ta_i = 0;
  while (p >= T - ta_i) {
    p -= T - ta_i;
    ++ta_i;
  }
  const int tb_i = ta_i + p;
  double* plane = work + (size_t)blockIdx.y * N * N;
  const int tx = threadIdx.x, ty = threadIdx.y;   // 32 × 8
  for (int r = ty; r < 32; r += 8) {
    ta[r][tx] = plane[(size_t)(ta_i * 32 + r) * N + tb_i * 32 + tx];
    tb[r][tx] = plane[(size_t)(tb_i * 32 + r) * N + ta_i * 32 + tx];
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    plane[(size_t)(tb_i * 32 + r) * N + ta_i * 32 + tx] = ta[tx][r];
    plane[(size_t)(ta_i * 32 + r) * N + tb_i * 32 + tx] = tb[tx][r];
  }
}

// A5 (3D): per mode m, all P blocks of BL−1 rows in turn; pivots in registers
#ifndef KFBI_SWEEP3_SPLIT
#define KFBI_SWEEP3_SPLIT 4
#endif
constexpr int kSweep3Threads = 128;
__global__ void __launch_bounds__(kSweep3Threads) k_sweep3(DevTables3 T, double* spec, double* __restrict__ zB,
                                                          double* __restrict__ zA, bool sparse) {
  const int N = T.N, P = T.P;
  const size_t K = (size_t)N * N;
  const size_t m = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= K) return;
  const int ll = (int)(m / N), kk = (int)(m % N);
  if (ll == 0 || kk == 0) return;
  const double d = T.dk[m];
  double ic[LB];
  {
    double c = d;
#pragma unroll
    for (int p = 0; p < LB; ++p) {
      if (p) c = d - ic[p - 1];
      ic[p] = 1.0 / c;
    }
  }
  pdl_wait();   // the spectrum from k_fwd3s (the pivots above come from the setup table dk)
  // the next block's LB source planes and its separator plane are loaded while this block is solved
  // and stored (software pipelining: twice the loads in flight per thread)
  auto load = [&](int g, double (&x)[BL]) {
#pragma unroll
    for (int p = 0; p < BL; ++p) {   // plane-uniform branches (flags of grid plane BL·g + p + 1)
      const bool live = (p < LB || g < P - 1) && !(sparse && !(T.plane_flags[BL * g + p + 1] & 1));
      x[p] = live ? __ldcs(spec + (size_t)(BL * g + p) * K + m) : 0.0;
    }
  };
  // blockIdx.y: a contiguous share of the slab's blocks (more, shorter CTAs: a smaller last wave)
  const int nb = T.b_hi - T.b_lo;
  const int g0 = T.b_lo + (int)((long)nb * blockIdx.y / gridDim.y), g1 = T.b_lo + (int)((long)nb * (blockIdx.y + 1) / gridDim.y);
  double nx[BL];
  if (g0 < g1) load(g0, nx);
  for (int g = g0; g < g1; ++g) {
    double y[BL];
#pragma unroll
    for (int p = 0; p < BL; ++p) y[p] = nx[p];
    if (g + 1 < g1) load(g + 1, nx);
#pragma unroll
    for (int p = 1; p < LB; ++p) y[p] = fma(-y[p - 1], ic[p - 1], y[p]);
    y[LB - 1] *= ic[LB - 1];
#pragma unroll
    for (int p = LB - 2; p >= 0; --p) y[p] = (y[p] - y[p + 1]) * ic[p];
#pragma unroll
    for (int p = 0; p < LB; ++p)
      if (!sparse || (T.plane_flags[BL * g + p + 1] & 2)) __stcs(spec + (size_t)(BL * g + p) * K + m, y[p]);
    zB[(size_t)g * K + m] = y[0];
    if (g < P - 1) zA[(size_t)g * K + m] = y[LB] - y[LB - 1];
  }
}

__global__ void k_reduced3(DevTables3 T, const double* __restrict__ zB, const double* __restrict__ zA,
                           double* __restrict__ hsep) {
  pdl_wait();   // zB, zA from k_sweep3
  // thread per mode: the P − 1 ≤ 31 right-hand sides loaded in one batch, the forward values kept in
  // registers (no re-read of hsep), pivots recomputed for the backward pass
  constexpr int PM = 31;
  const int N = T.N, P = T.P;
  const size_t K = (size_t)N * N;
  const size_t m = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= K || P < 2) return;
  const int ll = (int)(m / N), kk = (int)(m % N);
  if (ll == 0 || kk == 0) {
    for (int g = 0; g < P - 1; ++g) hsep[(size_t)g * K + m] = 0.0;
    return;
  }
  const double a = T.red_a[m], b = T.red_b[m];
  double y[PM];
#pragma unroll
  for (int g = 0; g < PM; ++g)
    if (g < P - 1) y[g] = zA[(size_t)g * K + m] - zB[(size_t)(g + 1) * K + m];
  double c = b, ci = 0.0;
#pragma unroll
  for (int g = 0; g < PM; ++g) {
    if (g >= P - 1) break;
    if (g) {
      c = b - a * a * ci;
      y[g] = y[g] - a * y[g - 1] * ci;
    }
    ci = 1.0 / c;
  }
  // backward: h_g = (y_g − a h_{g+1}) / c_g with the pivots regenerated from the top
  double cinv[PM];
  double cc = b;
#pragma unroll
  for (int g = 0; g < PM; ++g) {
    if (g >= P - 1) break;
    if (g) cc = b - a * a * cinv[g - 1];
    cinv[g] = 1.0 / cc;
  }
  double hn = 0.0;
#pragma unroll
  for (int g = PM - 1; g >= 0; --g) {
    if (g >= P - 1) continue;
    hn = g == P - 2 ? y[g] * cinv[g] : (y[g] - a * hn) * cinv[g];
    hsep[(size_t)g * K + m] = hn;
  }
}

// ---- multi-GPU level-2 split of the reduced system (slab r = blocks [b_lo, b_hi), see api.cu) ----
// The world − 1 slab separators' level-2 system is solved mode-partitioned: owner q of
// the modes [q·Kq, (q+1)·Kq) receives 4 rows per mode from every slab and returns each slab the 2 rows
// it needs — two all-to-alls of 4·K and 2·K doubles in total per rank instead of an all-gather.
// Buffer layouts (Kq = ⌈K / W⌉, m' = m − q·Kq): seg (from local) [q][4][Kq] per slab; the owner's input
// [r][4][Kq] (slab r's rows at stride `in_r`); the owner's output [r][2][Kq] (slab r's (h_{r−1}, h_r)
// at stride `out_r`); a slab's fix-up input [q][2][Kq].
// (1) the slab's L3 interior separators b_lo .. b_hi − 2 (right-hand sides zA[g] − zB[g + 1] from the
// slab's own blocks) by Thomas with the level-2 pivots; rows (first, last, zA[b_hi − 1], zB[b_lo])
__global__ void k_red3_local(DevTables3 T, const double* __restrict__ zB, const double* __restrict__ zA,
                             double* __restrict__ hsep, double* __restrict__ seg, int Kq) {
  const int N = T.N, L3 = T.L3, g0 = T.b_lo;
  const size_t K = (size_t)N * N;
  const size_t m = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= K) return;
  const int q = (int)(m / Kq), mp = (int)(m - (size_t)q * Kq);
  double* sb = seg + (size_t)q * 4 * Kq + mp;
  const int ll = (int)(m / N), kk = (int)(m % N);
  if (ll == 0 || kk == 0) {   // not a mode (k_sweep3 leaves these rows untouched)
    for (int p = 0; p < L3; ++p) hsep[(size_t)(g0 + p) * K + m] = 0.0;
    sb[0] = sb[Kq] = sb[2 * Kq] = sb[3 * Kq] = 0.0;
    return;
  }
  const double a = T.red_a[m];
  double z = 0.0;
  for (int p = 0; p < L3; ++p) {
    const int g = g0 + p;
    const double r = zA[(size_t)g * K + m] - zB[(size_t)(g + 1) * K + m];
    z = p ? fma(-a * z, T.rinv3[(size_t)(p - 1) * K + m], r) : r;
    hsep[(size_t)g * K + m] = z;
  }
  double first = 0.0, last = 0.0;
  if (L3 > 0) {
    z *= T.rinv3[(size_t)(L3 - 1) * K + m];
    last = z;
    hsep[(size_t)(g0 + L3 - 1) * K + m] = z;
    for (int p = L3 - 2; p >= 0; --p) {
      z = (hsep[(size_t)(g0 + p) * K + m] - a * z) * T.rinv3[(size_t)p * K + m];
      hsep[(size_t)(g0 + p) * K + m] = z;
    }
    first = z;
  }
  sb[0] = first;
  sb[Kq] = last;
  sb[2 * Kq] = T.b_hi < T.P ? zA[(size_t)(T.b_hi - 1) * K + m] : 0.0;
  sb[3 * Kq] = zB[(size_t)g0 * K + m];
}

// (2) owner q (= T.rank): tridiag(A2, B2, A2) on the world − 1 slab separators for its modes, right-hand
// side zA[s] − zB[s + 1] − a·last_s − a·first_{s+1} (slab s and s + 1 rows); separator s goes to slab s
// as its h_r and to slab s + 1 as its h_{r−1}
__global__ void k_red3_solve(DevTables3 T, const double* __restrict__ in, size_t in_r, double* __restrict__ out,
                             size_t out_r, int Kq) {
  const int N = T.N, W = T.world, L3 = T.L3, q = T.rank;
  const size_t K = (size_t)N * N;
  const int mp = blockIdx.x * blockDim.x + threadIdx.x;
  const size_t m = (size_t)q * Kq + mp;
  if (mp >= Kq || m >= K || W < 2) return;
  const int ll = (int)(m / N), kk = (int)(m % N);
  const bool mode = ll != 0 && kk != 0;
  const double a = mode ? T.red_a[m] : 0.0, A2 = mode ? T.red3_a[m] : 0.0, B2 = mode ? T.red3_b[m] : 1.0;
  double c = B2, y = 0.0, ci = 0.0;
  double cinv[64], yv[64];   // world ≤ 64
  for (int s = 0; s < W - 1; ++s) {
    const double* sl = in + s * in_r + mp;          // slab s: (first, last, zA_sep, zB_first) at stride Kq
    const double* sr = in + (s + 1) * in_r + mp;
    double r = sl[2 * Kq] - sr[3 * Kq];
    if (L3 > 0) r -= a * sl[Kq] + a * sr[0];
    if (s) c = B2 - A2 * A2 * ci;
    y = s ? r - A2 * y * ci : r;
    ci = 1.0 / c;
    cinv[s] = ci;
    yv[s] = y;
  }
  double hn = 0.0;
  for (int s = W - 2; s >= 0; --s) {
    hn = s == W - 2 ? yv[s] * cinv[s] : (yv[s] - A2 * hn) * cinv[s];
    if (!mode) hn = 0.0;
    out[s * out_r + Kq + mp] = hn;              // slab s: h_r
    out[(s + 1) * out_r + mp] = hn;             // slab s + 1: h_{r−1}
  }
  out[mp] = 0.0;                                // slab 0 has no left slab separator
  out[(W - 1) * out_r + Kq + mp] = 0.0;         // the last slab has no right one
}

// (3) slab r: interior separators x = z − a h_{r−1} Z2_L[p] − a h_r Z2_R[p], and its two slab
// separators (the values the fixed-up inverse of the slab's planes reads); hin = [q][2][Kq]
__global__ void k_red3_fixup(DevTables3 T, const double* __restrict__ hin, double* __restrict__ hsep, int Kq) {
  const int N = T.N, W = T.world, L3 = T.L3, r = T.rank, g0 = T.b_lo;
  const size_t K = (size_t)N * N;
  const size_t m = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= K) return;
  const int q = (int)(m / Kq), mp = (int)(m - (size_t)q * Kq);
  const double hlv = hin[(size_t)q * 2 * Kq + mp], hrv = hin[(size_t)q * 2 * Kq + Kq + mp];
  const int ll = (int)(m / N), kk = (int)(m % N);
  const bool mode = ll != 0 && kk != 0;
  const double a = mode ? T.red_a[m] : 0.0;
  const double hl = r > 0 ? a * hlv : 0.0;
  const double hr = r < W - 1 ? a * hrv : 0.0;
  for (int p = 0; p < L3; ++p) {
    double x = hsep[(size_t)(g0 + p) * K + m];
    if (mode) {
      x = fma(-hl, T.z3r[(size_t)(L3 - 1 - p) * K + m], x);   // Z2_L[p] = Z2_R[L3 − 1 − p]
      x = fma(-hr, T.z3r[(size_t)p * K + m], x);
    }
    hsep[(size_t)(g0 + p) * K + m] = x;
  }
  if (r < W - 1) hsep[(size_t)(T.b_hi - 1) * K + m] = mode ? hrv : 0.0;
  if (r > 0) hsep[(size_t)(g0 - 1) * K + m] = mode ? hlv : 0.0;
}

// A7 (3D): ten-point interpolation at the control points
__global__ void k_interp3(DevTables3 T, const double* __restrict__ phi, const double* __restrict__ dphi,
                          const double* __restrict__ fz, const double* __restrict__ jg, const double* __restrict__ work,
                          double* __restrict__ out, int partial) {
  pdl_wait();   // the z-evaluated stencil values from k_zeval3
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= T.nq) return;
  const int N = T.N;
  const int c0 = T.st_c[3 * e], c1 = T.st_c[3 * e + 1], c2 = T.st_c[3 * e + 2];
  if (partial && (c0 + 1 < T.i_lo || c0 - 1 > T.i_hi)) {   // no stencil node in the slab
    out[e] = 0.0;
    return;
  }
  Jump10 J;
  load_jump3(T, e, phi, dphi, fz, jg, J);
  const int code = T.st_code[e];
  const int s0 = (code >> 10) & 1 ? 1 : -1, s1 = (code >> 11) & 1 ? 1 : -1, s2 = (code >> 12) & 1 ? 1 : -1;
  const int off[10][3] = {{0, 0, 0}, {1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1},
                          {s0, s1, 0}, {s0, 0, s2}, {0, s1, s2}};
  const double zx = T.q_pos[3 * e], zy = T.q_pos[3 * e + 1], zz = T.q_pos[3 * e + 2];
  double acc = 0.0;
#pragma unroll
  for (int p = 0; p < 10; ++p) {
    const int ni = c0 + off[p][0], nj = c1 + off[p][1], nk = c2 + off[p][2];
    if (partial && (ni < T.i_lo || ni > T.i_hi)) continue;   // multi-GPU: the plane owner contributes
    KFBI_CHECK(ni >= 1 && ni < N && nj >= 1 && nj < N && nk >= 1 && nk < N, ni, (long long)nj * N + nk);
    double v = work[(size_t)(ni - 1) * N * N + (size_t)nj * N + nk];
    if ((code >> p) & 1) {
      const double dx = T.lo + ni * T.h - zx, dy = T.lo + nj * T.h - zy, dz = T.lo + nk * T.h - zz;
      v += J.v + J.g[0] * dx + J.g[1] * dy + J.g[2] * dz + 0.5 * (J.H[0] * dx * dx + J.H[1] * dy * dy + J.H[2] * dz * dz) +
           J.H[3] * dx * dy + J.H[4] * dx * dz + J.H[5] * dy * dz;
    }
    acc = fma((T.neumann ? T.st_wn : T.st_w)[10 * (size_t)e + p], v, acc);   // V⁺ or ∂_n V⁺ (R38)
  }
  out[e] = acc;
}

inline int cdiv3(long a, long b) { return (int)((a + b - 1) / b); }

}  // namespace

void launch_lsq3(const DevTables3& T, const double* phi, double* dphi, cudaStream_t s) {
  const int n = T.q_hi[0] - T.q_lo[0] + T.q_hi[1] - T.q_lo[1] + T.q_hi[2] - T.q_lo[2];
  if (n <= 0) return;
  ++g_launches;
  launch_pdl(k_lsq3, dim3(cdiv3((long)n * kLsqLanes, 256)), dim3(256), 0, s, T, phi, dphi);
}
void launch_base3(const DevTables3& T, const double* fgrid, double* work, cudaStream_t s) {
  ++g_launches;
  k_base3<<<num_sms() * 8, 256, 0, s>>>(T, fgrid, work);
}
void launch_correct3(const DevTables3& T, const double* phi, const double* dphi, const double* fq,
                     const double* jq_given, double* work, cudaStream_t s, double* corr) {
  if (T.n_hi <= T.n_lo) return;
  ++g_launches;
  launch_pdl(k_correct3, dim3(cdiv3(T.n_hi - T.n_lo, 128)), dim3(128), 0, s, T, phi, dphi, fq, jq_given, work, corr);
}
template <int N>
static void dst_rows3_n(const DevTables3& T, int mode, double* work, const double* hsep, double scale, double* out,
                        cudaStream_t s, const double* src, const double* corr, int compact) {
  constexpr int RPC = 256 / (N / 32);
  const size_t sm = (size_t)RPC * (N / 2 + N / 32 + 1) * sizeof(double2);
  const int grid = cdiv3((long)(T.i_hi - T.i_lo + 1) * N, RPC);
  smem_optin((const void*)k_dst_rows3t<0, N>, sm);
  smem_optin((const void*)k_dst_rows3t<1, N>, sm);
  smem_optin((const void*)k_dst_rows3t<2, N>, sm);
  smem_optin((const void*)k_dst_rows3t<3, N>, sm);
  if (mode == 0) launch_pdl(k_dst_rows3t<0, N>, dim3(grid), dim3(256), sm, s, T, work, hsep, scale, out, src, corr, 0);
  else if (mode == 1) launch_pdl(k_dst_rows3t<1, N>, dim3(grid), dim3(256), sm, s, T, work, hsep, scale, out, src, corr, 0);
  else if (mode == 2) launch_pdl(k_dst_rows3t<2, N>, dim3(grid), dim3(256), sm, s, T, work, hsep, scale, out, src, corr, compact);
  else launch_pdl(k_dst_rows3t<3, N>, dim3(grid), dim3(256), sm, s, T, work, hsep, scale, out, src, corr, compact);
}
void launch_dst_rows3(const DevTables3& T, int mode, double* work, const double* hsep, double scale, double* out,
                      cudaStream_t s, const double* src, const double* corr, bool compact) {
  ++g_launches;
  const int cm = compact ? 1 : 0;
  switch (T.N) {
    case 32: dst_rows3_n<32>(T, mode, work, hsep, scale, out, s, src, corr, cm); break;
    case 64: dst_rows3_n<64>(T, mode, work, hsep, scale, out, s, src, corr, cm); break;
    case 128: dst_rows3_n<128>(T, mode, work, hsep, scale, out, s, src, corr, cm); break;
    case 256: dst_rows3_n<256>(T, mode, work, hsep, scale, out, s, src, corr, cm); break;
    default: dst_rows3_n<512>(T, mode, work, hsep, scale, out, s, src, corr, cm); break;
  }
}
template <int N>
static void sparse3_n(const DevTables3& T, int which, const double* src, const double* hsep, double scale,
                      double* dst, cudaStream_t s) {
  constexpr int RPC = 256 / (N / 32) < N ? 256 / (N / 32) : N, NTHR = RPC * (N / 32);
  const size_t sm = (size_t)RPC * (N / 2 + N / 32 + 1) * sizeof(double2);
  smem_optin((const void*)k_inv3y<N>, sm);
  const dim3 grid(N / RPC, T.i_hi - T.i_lo + 1);
  if (which == 0) {
    const size_t sm0 = sm + (size_t)T.max_plane_irr * (sizeof(double) + sizeof(int16_t));
    smem_optin((const void*)k_fwd3s<N>, sm0);
    const dim3 gridf((N / RPC + kFwdGroups - 1) / kFwdGroups, T.i_hi - T.i_lo + 1);
    launch_pdl(k_fwd3s<N>, gridf, dim3(NTHR), sm0, s, T, src, dst);
  }
  else if (which == 1) launch_pdl(k_inv3y<N>, grid, dim3(NTHR), sm, s, T, src, hsep, scale, dst);
  else if (T.w_hi > T.w_lo)
    launch_pdl(k_zeval3<N>, dim3(std::min(cdiv3(T.w_hi - T.w_lo, 8), num_sms() * 2)), dim3(256), 0, s, T, src, scale, dst);
}
// which: 0 forward (corr → work), 1 inverse along y (work, hsep → work2), 2 z-evaluation (work2 → work)
void launch_sparse3(const DevTables3& T, int which, const double* src, const double* hsep, double scale, double* dst,
                    cudaStream_t s) {
  ++g_launches;
  switch (T.N) {
    case 32: sparse3_n<32>(T, which, src, hsep, scale, dst, s); break;
    case 64: sparse3_n<64>(T, which, src, hsep, scale, dst, s); break;
    case 128: sparse3_n<128>(T, which, src, hsep, scale, dst, s); break;
    case 256: sparse3_n<256>(T, which, src, hsep, scale, dst, s); break;
    default: sparse3_n<512>(T, which, src, hsep, scale, dst, s); break;
  }
}
void launch_transpose3(const DevTables3& T, double* work, cudaStream_t s) {
  const int t = T.N / 32;
  dim3 grid(t * (t + 1) / 2, T.i_hi - T.i_lo + 1);   // the slab's planes
  ++g_launches;
  k_transpose3<<<grid, dim3(32, 8), 0, s>>>(T.N, work + (size_t)(T.i_lo - 1) * T.N * T.N);
}
void launch_sweep3(const DevTables3& T, double* work, double* zB, double* zA, cudaStream_t s, bool sparse) {
  ++g_launches;
  launch_pdl(k_sweep3, dim3(cdiv3((long)T.N * T.N, kSweep3Threads), std::max(1, std::min(KFBI_SWEEP3_SPLIT, T.b_hi - T.b_lo))),
             dim3(kSweep3Threads), 0, s, T, work, zB, zA, sparse);
}
void launch_reduced3(const DevTables3& T, const double* zB, const double* zA, double* hsep, cudaStream_t s) {
  if (T.P < 2) return;
  ++g_launches;
  launch_pdl(k_reduced3, dim3(cdiv3((long)T.N * T.N, 128)), dim3(128), 0, s, T, zB, zA, hsep);
}
void launch_red3_local(const DevTables3& T, const double* zB, const double* zA, double* hsep, double* seg, int Kq,
                       cudaStream_t s) {
  ++g_launches;
  k_red3_local<<<cdiv3((long)T.N * T.N, 128), 128, 0, s>>>(T, zB, zA, hsep, seg, Kq);
}
void launch_red3_solve(const DevTables3& T, const double* in, size_t in_r, double* out, size_t out_r, int Kq,
                       cudaStream_t s) {
  ++g_launches;
  k_red3_solve<<<cdiv3(Kq, 128), 128, 0, s>>>(T, in, in_r, out, out_r, Kq);
}
void launch_red3_fixup(const DevTables3& T, const double* hin, double* hsep, int Kq, cudaStream_t s) {
  ++g_launches;
  k_red3_fixup<<<cdiv3((long)T.N * T.N, 128), 128, 0, s>>>(T, hin, hsep, Kq);
}
void launch_interp3(const DevTables3& T, const double* phi, const double* dphi, const double* fz,
                    const double* jz_given, const double* work, double* out, cudaStream_t s, bool partial) {
  ++g_launches;
  launch_pdl(k_interp3, dim3(cdiv3(T.nq, 128)), dim3(128), 0, s, T, phi, dphi, fz, jz_given, work, out, partial ? 1 : 0);
}

}  // namespace kfbi
