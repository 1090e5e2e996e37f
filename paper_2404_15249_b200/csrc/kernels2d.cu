// sm_100a kernels of the 2D KFBI interface-problem apply (arXiv 2404.15249), the GMRES vector
// kernels and the Gray–Scott pointwise kernels; the 3D path is in kernels3d.cu, shared device
// helpers (tables, reductions, FFT/DST cores) in device.cuh.
//
// One pass of the apply:
//   k_spline        A1  density interpolant (periodic cubic spline knots, reading R10)
//   k_correct       A2+A3 jumps at intersections (App. "Calculation of jumps")
//                   + correction at irregular nodes (Alg. 2)
//   k_sweep         A4+A5 sine transform of the sparse corrections computed on the fly and
//                   fused into a partitioned (arrowhead) tridiagonal solve along x
//   k_reduced       A5  reduced separator system per mode
//   k_inv_sparse    A6  inverse sine transform at interpolation-stencil rows only, with the
//                   arrowhead back-substitution s = z − Z_L h_{g−1} − Z_R h_g fused
//   k_interp        A7  jump-corrected six-point interpolation (Alg. 3)
//   k_dst_dense2    A4/A6 dense rows (FFT-based DST-I in shared memory) for the volume and
//                   final applies (once per solve)
// plus deterministic GMRES vector kernels (Alg. 5: k_mgs_cluster, one thread-block
// cluster per MGS step with DSMEM partial sums; k_mgs_step/k_norm_scale for large M) and the
// Ω-compact serving transfers (k_omega_map).  FP64 on CUDA cores: the path is HBM/latency bound,
// not a dense contraction (no tensor cores).
#include <cooperative_groups.h>
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <utility>

#include "device.cuh"
#include "kernels.h"

namespace kfbi {
namespace {

// the density and its arc-length derivatives on [s_m, s_{m+1}] (t = (s − s_m)/Δ) from the
// point's precomputed knot pair (global density indices of knots m and m + 1)
__device__ __forceinline__ void spline_eval2(const double* __restrict__ phi, const double* __restrict__ mk, int2 g01,
                                             double delta, double t, double& g, double& gp, double& gpp) {
  const double g0 = phi[g01.x], g1 = phi[g01.y], a = mk[g01.x], b = mk[g01.y];
  const double w = 1.0 - t;
  g = w * g0 + t * g1 + (delta * delta / 6.0) * ((w * w * w - w) * a + (t * t * t - t) * b);
  gp = (g1 - g0) / delta + (delta / 6.0) * (-(3.0 * w * w - 1.0) * a + (3.0 * t * t - 1.0) * b);
  gpp = w * a + t * b;
}

struct Jump6 {
  double v, vx, vy, vxx, vxy, vyy;
};


// Closed form of the appendix 2×2 + 3×3 systems (reading R7 ψ for ψ_s):
//   [v] = Φ, [∇v] = Φ_s τ + Ψ n, frame components A_ττ, A_τn, A_nn, [D²v] = F A Fᵀ.
__device__ __forceinline__ Jump6 jumps2d(double Phi, double Phis, double Phiss, double Psi, double Psis, double F,
                                         double kappa, double t1, double t2, double p1, double p2) {
  Jump6 J;
  J.v = Phi;
  J.vx = t1 * Phis + t2 * Psi;
  J.vy = t2 * Phis - t1 * Psi;
  double Att = Phiss - (p1 * J.vx + p2 * J.vy);
  double Atn = Psis - (p2 * J.vx - p1 * J.vy);
  double Ann = F + kappa * Phi - Att;
  J.vxx = Att * t1 * t1 + 2.0 * Atn * t1 * t2 + Ann * t2 * t2;
  J.vxy = (Att - Ann) * t1 * t2 + Atn * (t2 * t2 - t1 * t1);
  J.vyy = Att * t2 * t2 - 2.0 * Atn * t1 * t2 + Ann * t1 * t1;
  return J;
}

// ------------------------------------------------------------------------------ A1
// blocks [0, nsb): one thread per control point; blocks nsb + h: the hole-completion coefficient
// a_h = Δs_h Σ_{Γ_h} φ (reading R27) by a deterministic block reduction (saves a launch per apply)
constexpr int kSplineLanes = 8;
__global__ void k_spline(DevTables T, const double* __restrict__ phi, double* __restrict__ mk, int nh,
                         const int* __restrict__ hoff, const int* __restrict__ hcnt,
                         const double* __restrict__ hdelta, double* __restrict__ ahole) {
  if ((int)blockIdx.x < nh) {   // hole blocks first: they are the longest, the spline blocks fill in
    __shared__ double scratch[32];
    pdl_wait();   // φ from the previous kernel
    const int hh = blockIdx.x;
    const int cnt = hcnt[hh], o = hoff[hh];
    double v[1] = {0.0};
    for (int m = threadIdx.x; m < cnt; m += 4 * blockDim.x) {   // four loads in flight, summed in order
      double x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = m + u * (int)blockDim.x < cnt ? phi[o + m + u * blockDim.x] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) v[0] += x[u];
    }
    block_reduce<1>(v, scratch);
    if (threadIdx.x == 0) ahole[hh] = hdelta[hh] * v[0];
    return;
  }
  // kSplineLanes lanes per control point, each with ≤ 64 / kSplineLanes taps whose loads are all issued
  // before the FMAs (the one-thread loop waited on one phi load per tap); a fixed xor tree sums the lanes
  const int gt = (blockIdx.x - nh) * blockDim.x + threadIdx.x;
  const int m = gt / kSplineLanes, sub = gt % kSplineLanes;
  double acc = 0.0;
  if (m >= T.M) pdl_wait();
  if (m < T.M) {
    const int c = T.z_comp[m], ml = T.z_knot[m];
    const int off = T.c_off[c], Mc = T.c_M[c], nt = T.sp_ntaps[c], first = T.sp_first[c];
    const double* b = T.sp_coef + T.sp_coef_off[c];
    int base = (ml + first + sub) % Mc;   // periodic knots
    if (base < 0) base += Mc;
    constexpr int U = 64 / kSplineLanes;
    double bv[U], pv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) bv[u] = sub + kSplineLanes * u < nt ? b[sub + kSplineLanes * u] : 0.0;
    pdl_wait();   // φ from the previous kernel (the filter taps above are setup constants)
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = sub + kSplineLanes * u;
      pv[u] = 0.0;
      if (r < nt) pv[u] = phi[off + (base + kSplineLanes * u) % Mc];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc = fma(bv[u], pv[u], acc);
  }
#pragma unroll
  for (int o = kSplineLanes / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (m < T.M && sub == 0) mk[m] = acc;
}

// ------------------------------------------------------------------------------ A2+A3
__global__ void k_correct(DevTables T, const double* __restrict__ phi, const double* __restrict__ mk,
                          const double* __restrict__ fq, const double* __restrict__ jqg, double* __restrict__ cval) {
  int n = T.irr_lo + blockIdx.x * blockDim.x + threadIdx.x;   // the slab's irregular nodes
  pdl_wait();   // φ and the spline knots M from k_spline
  if (n >= T.irr_hi) return;
  double acc = 0.0;
  for (int e = T.irr_ptr[n]; e < T.irr_ptr[n + 1]; ++e) {
    int q = T.pair_q[e];
    KFBI_CHECK(q >= 0 && q < T.nq, q, T.nq);
    double d = T.pair_d[e];
    int ax = T.q_axis[q];
    double v, va, vaa;
    if (jqg) {
      v = jqg[q * 6];
      va = jqg[q * 6 + 1 + ax];
      vaa = jqg[q * 6 + (ax == 0 ? 3 : 5)];
    } else {
      double Phi = 0, Phis = 0, Phiss = 0;
      if (phi) {
        spline_eval2(phi, mk, reinterpret_cast<const int2*>(T.q_g01)[q], T.q_dl[q], T.q_t[q], Phi, Phis, Phiss);
      }
      double F = fq ? fq[q] : 0.0;
      // Neumann (R38): the density is ψ = [∂_n v] with [v] = 0
      Jump6 J = T.neumann ? jumps2d(0.0, 0.0, 0.0, Phi, Phis, F, T.kappa, T.q_t1[q], T.q_t2[q], T.q_p1[q], T.q_p2[q])
                          : jumps2d(Phi, Phis, Phiss, 0.0, 0.0, F, T.kappa, T.q_t1[q], T.q_t2[q], T.q_p1[q], T.q_p2[q]);
      v = J.v;
      va = ax == 0 ? J.vx : J.vy;
      vaa = ax == 0 ? J.vxx : J.vyy;
    }
    acc += v + va * d + 0.5 * vaa * d * d;   // P(d), SURVEY App. A.3
  }
  // Ω endpoint: −P/h² (C⁺); Ω^c endpoint: +P/h² (C⁻).  Stored ×h².
  cval[n] = T.irr_side[n] ? -acc : acc;
}

// ------------------------------------------------------------------------------ A4+A5
// Persistent CTAs, each owning a fixed chunk of 256 mode pairs (k, N−k) (k = t, t = 0 → mode
// N/2 alone) and iterating over blocks g of BL−1 columns.  sin(πj(N−k)/N) = (−1)^{j+1}
// sin(πjk/N): one lookup serves both modes.  The block's sparse corrections (j, c) are staged
// in shared memory; sines come from a half-period table sin(πr/N), r ∈ [0, N), stored at
// r + r/16 (one pad per 16 doubles breaks the stride-j bank conflicts of a warp's lanes).
// Local Thomas in registers with the block pivots c_1 = d, c_p = d − 1/c_{p−1} computed once
// per CTA lifetime: y_p = r_p − y_{p−1}/c_{p−1}, z_p = (y_p − z_{p+1})/c_p, r = h² f̂.
// Outputs: z at the block rows, B[g] = z_g[1], A[g] = h² f̂_sep,g − z_g[L] (reduced-system
// right-hand side pieces).
constexpr int kSweepThreads = 256;
constexpr int kEntCap = 768;                 // sparse entries staged per pass (k_sweep shared memory)
constexpr int kQuads = kSweepThreads / 2;   // 128 quads {t, N−t, N/2−t, N/2+t} per CTA chunk
constexpr int kRs = kQuads + 8;              // sum-row stride: rows 2r and 2r + 1 start 16 banks apart,
                                             // so phase 2's paired reads (w = 0, 1) do not conflict
constexpr int kRotSteps = 8;                 // quads per phase-1 item (t = base + kRotStride·s)
constexpr int kRotStride = kQuads / kRotSteps;  // 16
// Persistent CTAs, each owning a fixed chunk of 256 quads of sine modes {t, N−t, N/2−t, N/2+t}
// (spectral positions 4t..4t+3, see mode_position) and iterating over blocks g of BL−1 columns
// (+ the separator column).  Phase 1 (A4, DST of the staged sparse corrections): with
// s, c = sin, cos(πjt/N), sin(πj(N−t)/N) = (−1)^{j+1} s and sin(πj(N/2 ± t)/N) = sin(πj/2) c ±
// cos(πj/2) s, so per correction (j, c_j) one rotation step serves the whole quad:
//   odd j:  A_o += c_j s,   B_o += c_j sin(πj/2) c        even j: A_e += c_j s,  B_e += c_j cos(πj/2) s
//   r_t = A_o + A_e, r_{N−t} = A_o − A_e, r_{N/2−t} = B_o − B_e, r_{N/2+t} = B_o + B_e.
// An item covers kRotSteps quads t = t0 + qg + kRotStride·s, the sines along s generated by
// rotation with the per-entry step e^{iπ·kRotStride·j/N}.  Phase 2 (A5): thread τ owns positions (4q + 2w, 4q + 2w + 1),
// q = τ/2, w = τ mod 2; local Thomas per mode, pivots in registers for the CTA's lifetime; writes
// z (block rows), B[g] = z_g[1], A[g] = h² f̂_sep,g − z_g[L].
template <int DENSE>   // 0: sparse corrections only, 1: + dense base spectrum, 2: + base and hole bumps
__global__ void __launch_bounds__(kSweepThreads, 2) k_sweep(DevTables T, const double* __restrict__ cval, DenseSrc D,
                                                           double* spec, double* __restrict__ zB,
                                                           double* __restrict__ zA) {
  extern __shared__ double sm[];
  const int N = T.N, half = N >> 1, quarter = N >> 2, m2 = 2 * N - 1, B = kSweepThreads;
  double* R = sm;                                            // [4·BL sums][kRs]
  double4* ent = reinterpret_cast<double4*>(R + (size_t)BL * 4 * kRs);   // (c, j, cos Δ, sin Δ)
  // ent = (c, c·sin(πj/2) (odd j) or c·cos(πj/2) (even j), cos Δ, sin Δ), Δ = π·kRotStride·j/N
  const int ecap = T.maxe < kEntCap ? T.maxe : kEntCap;     // entries staged per pass
  int* ent_j = reinterpret_cast<int*>(ent + ecap);
  double2* th = reinterpret_cast<double2*>(ent_j + ((ecap + 3) & ~3));   // e^{iπ 64k/N} (padded, eipi_p)
  double2* tl = th + eipi_pad(2 * N / 64) + 1;                // e^{iπ l/N}, l < 64 (padded)
  int* s_cnt = reinterpret_cast<int*>(tl + 72);               // per-column [start, mid, end)
  build_eipi_p(T.sin_tab, N, th, tl);
  auto E = [&](int r) { return eipi_p(th, tl, r); };
  const int nch = (quarter + kQuads - 1) / kQuads;
  const int G = gridDim.x / nch;
  const int ch = blockIdx.x % nch;
  const int q0 = ch * kQuads;
  // phase 2: thread τ owns half w = τ mod 2 of quad slot τ/2 (a warp's z stores fill whole 32-byte
  // sectors; the bank-conflict-free mapping w = τ/128 measured 12% slower: half-sector stores)
  const int qq = q0 + (threadIdx.x >> 1), w = threadIdx.x & 1;
  const bool active = qq < quarter;
  const int p1 = active ? 4 * qq + 2 * w : 0;   // spectral positions p1, p1 + 1 of this thread
  // block pivots 1/c_p of this thread's two modes from the setup table (bitwise the recurrence
  // c_1 = d, c_p = d − 1/c_{p−1}); read per block from L1/L2 instead of held in 60 registers, which
  // phase 1's eight-quad items use
  auto icp = [&](int p) { return __ldg(reinterpret_cast<const double2*>(T.invc + (size_t)p * N + p1)); };
  const double h2 = T.h * T.h;
  const int slot = threadIdx.x >> 1;
  double* Rs = R + slot;           // Rs[(4c + u)·kRs], u: 0 A_o, 1 B_o, 2 A_e, 3 B_e
  // blocks in descending count of sparse entries (setup order `blk_order`), snake-dealt over the
  // G block groups so that the groups that draw the blocks where Γ runs along x are not the tail
  const int grp = blockIdx.x / nch;
  // the next block's (block, entry range) is loaded one round ahead (three registers)
  auto meta = [&](int rnd, int4& m) {
    const int kk = rnd * G + ((rnd & 1) ? G - 1 - grp : grp);
    m.x = -1;
    if (kk >= T.P) return;
    m = __ldg(reinterpret_cast<const int4*>(T.blk_meta) + kk);
  };
  int4 nm = make_int4(-1, 0, 0, 0);
  meta(0, nm);
  pdl_wait();   // the corrections (k_correct) and the dense source are ready
  for (int rnd = 0; rnd * G < T.P; ++rnd) {
  const int g = nm.x, e0 = nm.y, e1m = nm.z;
  const int keep = D.stencil_only ? nm.w : 0x7fff;   // positions whose spectral rows are stored
  meta(rnd + 1, nm);
  if (g < T.g_lo || g >= T.g_hi) continue;   // CTA-uniform (g = −1: no block)
    const int c0 = BL * g + 1;
    KFBI_CHECK(c0 - 1 >= T.col_lo - 1 && c0 - 1 + LB - 1 <= T.col_hi - 1, c0, T.col_hi);   // spectral rows of the slab
    const int ncol = g < T.P - 1 ? BL : LB;   // block columns + separator column
    const int e1 = cval ? e1m : e0;
    // the block's entries are staged kEntCap at a time (a block where Γ runs along x holds up to
    // ~1,700 on the 8192² star: staging them all would leave one CTA per SM); later passes add into R
    for (int cb = e0, pass = 0; pass == 0 || cb < e1; cb += kEntCap, ++pass) {
    const int ce = e1 - cb < kEntCap ? e1 : cb + kEntCap;
    __syncthreads();
    for (int e = cb + threadIdx.x; e < ce; e += B) {
      KFBI_CHECK(e >= 0 && e < T.nirr, e, T.nirr);
      const int j = T.irr_j[e];
      KFBI_CHECK(j >= 1 && j < N, j, N);
      const int rd = (j * kRotStride) & m2;
      const double c = cval[e];
      // odd j: sin(πj/2) = ±1; even j: cos(πj/2) = ±1
      const bool neg = (j >> 1) & 1;
      const double2 dr = E(rd);   // e^{iπ·kRotStride·j/N} from the shared tables (no global lookups)
      ent[e - cb] = make_double4(c, neg ? -c : c, dr.x, dr.y);
      ent_j[e - cb] = j;
    }
    if (threadIdx.x < ncol) {
      const int i = c0 + threadIdx.x;
      auto clampc = [&](int v) { return (v < cb ? cb : v > ce ? ce : v) - cb; };   // this pass's part
      s_cnt[3 * threadIdx.x] = cval ? clampc(T.col_ptr[i]) : 0;
      s_cnt[3 * threadIdx.x + 1] = cval ? clampc(T.col_mid[i]) : 0;
      s_cnt[3 * threadIdx.x + 2] = cval ? clampc(T.col_ptr[i + 1]) : 0;
    }
    __syncthreads();
    // ---- phase 1: sparse DST of every column, 8 quads per item by rotation ----
    for (int it = threadIdx.x; it < ncol * kRotStride; it += B) {
      const int c = it / kRotStride, qg = it - c * kRotStride;
      const int tb = q0 + qg;
      const int a0 = s_cnt[3 * c], am = s_cnt[3 * c + 1], a1 = s_cnt[3 * c + 2];
      double Ao[kRotSteps], Bo[kRotSteps], Ae[kRotSteps], Be[kRotSteps];
#pragma unroll
      for (int q = 0; q < kRotSteps; ++q) Ao[q] = Bo[q] = Ae[q] = Be[q] = 0.0;
      for (int e = a0; e < am; ++e) {   // odd rows
        const double4 en = ent[e];
        const double c2 = en.y;
        const double2 e0 = E((ent_j[e] * tb) & m2);
        double sn = e0.y, cs = e0.x;
#pragma unroll
        for (int q = 0; q < kRotSteps; ++q) {
          Ao[q] = fma(en.x, sn, Ao[q]);
          Bo[q] = fma(c2, cs, Bo[q]);
          const double cn = fma(cs, en.z, -sn * en.w);
          sn = fma(sn, en.z, cs * en.w);
          cs = cn;
        }
      }
      for (int e = am; e < a1; ++e) {   // even rows
        const double4 en = ent[e];
        const double c2 = en.y;
        const double2 e0 = E((ent_j[e] * tb) & m2);
        double sn = e0.y, cs = e0.x;
#pragma unroll
        for (int q = 0; q < kRotSteps; ++q) {
          Ae[q] = fma(en.x, sn, Ae[q]);
          Be[q] = fma(c2, sn, Be[q]);
          const double cn = fma(cs, en.z, -sn * en.w);
          sn = fma(sn, en.z, cs * en.w);
          cs = cn;
        }
      }
#pragma unroll
      for (int q = 0; q < kRotSteps; ++q) {
        const int sl = qg + kRotStride * q;
        if (ch == 0 && sl == 0) continue;     // quad slot 0 of chunk 0: the special modes below
        double* r = R + 4 * c * kRs + sl;   // only this item writes these slots: no barrier needed
        r[0] = pass ? r[0] + Ao[q] : Ao[q];
        r[kRs] = pass ? r[kRs] + Bo[q] : Bo[q];
        r[2 * kRs] = pass ? r[2 * kRs] + Ae[q] : Ae[q];
        r[3 * kRs] = pass ? r[3 * kRs] + Be[q] : Be[q];
      }
    }
    if (ch == 0) {   // CTA-uniform: all lanes take part in the shuffles
      // quad slot 0 holds modes {0, N/2, N/4, 3N/4}: r_{N/2} = Σ c sin(πj/2), r_{N/4}, r_{3N/4};
      // 16 lanes per column (strided entries, fixed shuffle tree), pass sums added in pass order
      const int c = threadIdx.x >> 4, sub = threadIdx.x & 15;
      double rh = 0.0, rq = 0.0, r3 = 0.0;
      for (int e = s_cnt[3 * c] + sub; c < ncol && e < s_cnt[3 * c + 2]; e += 16) {
        const double cv = ent[e].x;
        const int j = ent_j[e];
        rh = fma(cv, E((j * half) & m2).y, rh);
        rq = fma(cv, E((j * quarter) & m2).y, rq);
        r3 = fma(cv, E((j * 3 * quarter) & m2).y, r3);
      }
#pragma unroll
      for (int o = 8; o; o >>= 1) {
        rh += __shfl_xor_sync(0xffffffffu, rh, o);
        rq += __shfl_xor_sync(0xffffffffu, rq, o);
        r3 += __shfl_xor_sync(0xffffffffu, r3, o);
      }
      if (sub == 0 && c < ncol) {
        double* r = R + 4 * c * kRs;
        const double v0 = 0.5 * rh, v2 = -0.5 * rh;                   // (A_o + A_e, A_o − A_e) = (0, r_{N/2})
        const double v1 = 0.5 * (rq + r3), v3 = 0.5 * (r3 - rq);     // (B_o − B_e, B_o + B_e) = (r_{N/4}, r_{3N/4})
        r[0] = pass ? r[0] + v0 : v0;
        r[kRs] = pass ? r[kRs] + v1 : v1;
        r[2 * kRs] = pass ? r[2 * kRs] + v2 : v2;
        r[3 * kRs] = pass ? r[3 * kRs] + v3 : v3;
      }
    }
    }   // entry passes
    __syncthreads();
    if (!active) continue;
    // ---- phase 2: local Thomas, y_p = r_p − y_{p−1}/c_{p−1}, z_p = (y_p − z_{p+1})/c_p ----
    // this thread's two right-hand sides from the quad sums (w = 0: t, N−t; w = 1: N/2−t, N/2+t)
    auto rhs = [&](int c, double& r1, double& r2) {
      const double A = Rs[(4 * c + w) * kRs], E = Rs[(4 * c + 2 + w) * kRs];
      r1 = w ? A - E : A + E;
      r2 = w ? A + E : A - E;
      if (DENSE) {   // f̂ = base + Σ a_h bump_h, one fma per bump in order
        const size_t off = (size_t)(c0 + c - 1) * N + p1;
        double2 d = DENSE == 1 || D.base ? *reinterpret_cast<const double2*>(D.base + off) : make_double2(0.0, 0.0);
        if (DENSE == 2) {
          const int col = c0 + c;   // the bumps' spectra vanish outside their supports' columns
#pragma unroll 1
          for (int q = 0; q < D.nb; ++q) {
            if (col < D.blo[q] || col > D.bhi[q]) continue;
            const double2 b = __ldcs(reinterpret_cast<const double2*>(D.bump + (size_t)q * D.ldb + off));
            const double a = __ldg(D.coef + q);
            d.x = fma(a, b.x, d.x);
            d.y = fma(a, b.y, d.y);
          }
        }
        r1 = fma(h2, d.x, r1);
        r2 = fma(h2, d.y, r2);
      }
    };
    // y_p overwrites this thread's own two sum slots of row p (the partner thread owns the others)
    // the forward values y stay in registers (no shared-memory round trip); pivots per step
    double y1[LB], y2[LB];
    rhs(0, y1[0], y2[0]);
#pragma unroll
    for (int p = 1; p < LB; ++p) {
      double r1, r2;
      rhs(p, r1, r2);
      const double2 c = icp(p - 1);
      y1[p] = fma(-y1[p - 1], c.x, r1);
      y2[p] = fma(-y2[p - 1], c.y, r2);
    }
    double sep1 = 0.0, sep2 = 0.0;
    if (g < T.P - 1) rhs(LB, sep1, sep2);
    const double2 cl = icp(LB - 1);
    double z1 = y1[LB - 1] * cl.x, z2 = y2[LB - 1] * cl.y;
    const double zl1 = z1, zl2 = z2;
    // the block's spectral rows by one pointer walked down a row per step (one 64-bit add per store
    // instead of a row index product)
    double2* zp = reinterpret_cast<double2*>(spec + (size_t)(c0 - 1 + LB - 1) * N + p1);
    const size_t rowN = (size_t)N / 2;   // one spectral row in double2 units
    if ((keep >> (LB - 1)) & 1) *zp = make_double2(z1, z2);
#pragma unroll
    for (int p = LB - 2; p >= 0; --p) {
      const double2 c = icp(p);
      z1 = (y1[p] - z1) * c.x;
      z2 = (y2[p] - z2) * c.y;
      zp -= rowN;
      if ((keep >> p) & 1) *zp = make_double2(z1, z2);
    }
    *reinterpret_cast<double2*>(zB + (size_t)g * N + p1) = make_double2(z1, z2);
    if (g < T.P - 1) *reinterpret_cast<double2*>(zA + (size_t)g * N + p1) = make_double2(sep1 - zl1, sep2 - zl2);
  }
}

// ------------------------------------------------------------------------------ A5 reduced
// −Z_L[L] h_{g−1} + (d − Z_R[L] − Z_L[1]) h_g − Z_R[1] h_{g+1} = f_sep,g − z_g[L] − z_{g+1}[1]
// (SURVEY App. A.5): tridiag(a, b, a) per mode, a = red_a, b = red_b, rhs_g = A[g] − B[g+1].
// Small P: one thread per mode, plain Thomas.
__global__ void k_reduced_small(DevTables T, const double* __restrict__ zB, const double* __restrict__ zA,
                                double* __restrict__ hsep) {
  const int N = T.N, P = T.P;
  const int k = blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (k >= N || P < 2) return;
  const double a = T.red_a[k];
  double y = zA[k] - zB[(size_t)N + k];
  hsep[k] = y;
  for (int g = 1; g < P - 1; ++g) {
    const double r = zA[(size_t)g * N + k] - zB[(size_t)(g + 1) * N + k];
    y = fma(-a * y, T.red_invc[(size_t)(g - 1) * N + k], r);
    hsep[(size_t)g * N + k] = y;
  }
  double hn = y * T.red_invc[(size_t)(P - 2) * N + k];
  hsep[(size_t)(P - 2) * N + k] = hn;
  for (int g = P - 3; g >= 0; --g) {
    hn = (hsep[(size_t)g * N + k] - a * hn) * T.red_invc[(size_t)g * N + k];
    hsep[(size_t)g * N + k] = hn;
  }
}

// Large P: the same arrowhead split applied to the reduced system (P − 1 = BL2·S − 1):
// thread (mode lane, segment σ) solves its BL2−1 separators locally in registers, the S−1
// level-2 separators per mode are solved from shared memory, then each segment is fixed up
// with the level-2 spikes (z − a h2_{σ−1} Z2_L − a h2_σ Z2_R).
#ifndef KFBI_RED2_MODES
#define KFBI_RED2_MODES 32
#endif
constexpr int kRed2Modes = KFBI_RED2_MODES;   // modes per CTA (× one thread per level-2 segment)
__global__ void __launch_bounds__(kRed2Modes * kMaxSeg) k_reduced2(DevTables T, const double* __restrict__ zB,
                                                  const double* __restrict__ zA, double* __restrict__ hsep) {
  __shared__ double s_first[kMaxSeg][kRed2Modes], s_last[kMaxSeg][kRed2Modes], s_rs[kMaxSeg][kRed2Modes], s_h2[kMaxSeg][kRed2Modes];
  __shared__ double s_rinv[LB2][kRed2Modes], s_z2r[LB2][kRed2Modes];   // the CTA's modes of the level-2 tables
  const int N = T.N, P = T.P, S = P / BL2;
  const int lane = threadIdx.x, sg = threadIdx.y;
  const int k = blockIdx.x * kRed2Modes + lane + 1;
  const bool ok = k < N;
  const int kk = ok ? k : 1;
  const double a = T.red_a[kk];
  const int gbase = sg * BL2;
  // the per-mode pivot and spike rows (setup tables, shared by the S segments) are staged once per CTA
  // while the sweep drains (PDL), then all of this segment's right-hand sides in one batch
  for (int p = sg; p < LB2; p += blockDim.y) {
    s_rinv[p][lane] = T.rinv2[(size_t)p * N + kk];
    s_z2r[p][lane] = T.z2r[(size_t)p * N + kk];
  }
  pdl_wait();   // zA, zB from k_sweep
  double z[LB2];
#pragma unroll
  for (int p = 0; p < LB2; ++p) {
    const int g = gbase + p;
    z[p] = zA[(size_t)g * N + kk] - zB[(size_t)(g + 1) * N + kk];
  }
  double rsep = 0.0;
  if (sg < S - 1) {
    const int gs = gbase + LB2;
    rsep = zA[(size_t)gs * N + kk] - zB[(size_t)(gs + 1) * N + kk];
  }
  __syncthreads();
#pragma unroll
  for (int p = 1; p < LB2; ++p) z[p] = fma(-a * z[p - 1], s_rinv[p - 1][lane], z[p]);
  z[LB2 - 1] *= s_rinv[LB2 - 1][lane];
#pragma unroll
  for (int p = LB2 - 2; p >= 0; --p) z[p] = (z[p] - a * z[p + 1]) * s_rinv[p][lane];
  s_first[sg][lane] = z[0];
  s_last[sg][lane] = z[LB2 - 1];
  if (sg < S - 1) s_rs[sg][lane] = rsep;
  __syncthreads();
  if (sg == 0 && S > 1) {
    // level-2 reduced system: tridiag(A2, B2, A2), rhs = r_s − a z_σ[L] − a z_{σ+1}[1];
    // pivots → s_rs, forward values → s_h2 (in place, per lane)
    // pivots 1/c_q from the setup table (no divisions on the critical path), loaded up front
    const double A2 = T.red2_a[kk];
    double cis[kMaxSeg - 1];
#pragma unroll
    for (int q = 0; q < kMaxSeg - 1; ++q) cis[q] = q < S - 1 ? T.red2_ci[(size_t)q * N + kk] : 1.0;
    double yprev = 0.0;
#pragma unroll
    for (int q = 0; q < kMaxSeg - 1; ++q) {
      if (q >= S - 1) break;
      const double r = s_rs[q][lane] - a * s_last[q][lane] - a * s_first[q + 1][lane];
      const double y = q ? r - A2 * yprev * cis[q - 1] : r;
      s_rs[q][lane] = cis[q];
      s_h2[q][lane] = y;
      yprev = y;
    }
    double hn = s_h2[S - 2][lane] * s_rs[S - 2][lane];
    s_h2[S - 2][lane] = hn;
    for (int q = S - 3; q >= 0; --q) {
      hn = (s_h2[q][lane] - A2 * hn) * s_rs[q][lane];
      s_h2[q][lane] = hn;
    }
  }
  __syncthreads();
  if (!ok) return;
  const double hl = sg > 0 ? a * s_h2[sg - 1][lane] : 0.0;
  const double hr = sg < S - 1 ? a * s_h2[sg][lane] : 0.0;
#pragma unroll
  for (int p = 0; p < LB2; ++p) {
    double x = z[p];
    x = fma(-hl, s_z2r[LB2 - 1 - p][lane], x);   // Z2_L[p] = Z2_R[L2 − 1 − p]
    x = fma(-hr, s_z2r[p][lane], x);
    hsep[(size_t)(gbase + p) * N + k] = x;
  }
  if (sg < S - 1) hsep[(size_t)(gbase + LB2) * N + k] = s_h2[sg][lane];
}

// ---- multi-GPU split of k_reduced2: the level-2 segments are the slabs' separator groups ----
// (1) owned segments: local level-2 block solve, z kept in hsep; segbuf[sg][4][N] = (first z, last z,
// zA of the segment's right boundary separator, zB of its first block).  The boundary separator's
// right-hand side zA[gs] − zB[gs + 1] joins one value from each side of a slab cut, so it is formed
// after the exchange from rows both owners publish (no rank reads another slab's blocks).
__global__ void k_red2_local(DevTables T, const double* __restrict__ zB, const double* __restrict__ zA,
                             double* __restrict__ hsep, double* __restrict__ segbuf) {
  pdl_wait();
  const int N = T.N, S = T.nseg;
  const int k = blockIdx.x * blockDim.x + threadIdx.x + 1;
  const int sg = T.seg_lo + blockIdx.y;
  if (k >= N) return;
  const double a = T.red_a[k];
  const int gbase = sg * BL2;
  double z[LB2];
#pragma unroll
  for (int p = 0; p < LB2; ++p) {
    const int g = gbase + p;
    z[p] = zA[(size_t)g * N + k] - zB[(size_t)(g + 1) * N + k];
  }
#pragma unroll
  for (int p = 1; p < LB2; ++p) z[p] = fma(-a * z[p - 1], T.rinv2[(size_t)(p - 1) * N + k], z[p]);
  z[LB2 - 1] *= T.rinv2[(size_t)(LB2 - 1) * N + k];
#pragma unroll
  for (int p = LB2 - 2; p >= 0; --p) z[p] = (z[p] - a * z[p + 1]) * T.rinv2[(size_t)p * N + k];
#pragma unroll
  for (int p = 0; p < LB2; ++p) hsep[(size_t)(gbase + p) * N + k] = z[p];
  double* sb = segbuf + (size_t)sg * 4 * N;
  sb[k] = z[0];
  sb[N + k] = z[LB2 - 1];
  sb[2 * N + k] = sg < S - 1 ? zA[(size_t)(gbase + LB2) * N + k] : 0.0;
  sb[3 * N + k] = zB[(size_t)gbase * N + k];
}

// (2) every rank: the level-2 tridiagonal system of the S − 1 slab separators per mode
__global__ void k_red2_solve(DevTables T, const double* __restrict__ segbuf, double* __restrict__ h2) {
  pdl_wait();
  const int N = T.N, S = T.nseg;
  const int k = blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (k >= N || S < 2) return;
  const double a = T.red_a[k], A2 = T.red2_a[k], B2 = T.red2_b[k];
  double c = B2, yprev = 0.0, ciprev = 0.0;
  for (int q = 0; q < S - 1; ++q) {
    const double* sq = segbuf + (size_t)q * 4 * N;
    const double* sn = segbuf + (size_t)(q + 1) * 4 * N;
    const double r = (sq[2 * N + k] - sn[3 * N + k]) - a * sq[N + k] - a * sn[k];
    if (q) c = B2 - A2 * A2 * ciprev;
    const double ci = 1.0 / c;
    const double y = q ? r - A2 * yprev * ciprev : r;
    h2[(size_t)q * N + k] = y;
    yprev = y;
    ciprev = ci;
  }
  // backward needs the pivots again: recompute them (S − 1 ≤ 15 per mode)
  double ci_all[16];
  c = B2;
  for (int q = 0; q < S - 1; ++q) {
    if (q) c = B2 - A2 * A2 * ci_all[q - 1];
    ci_all[q] = 1.0 / c;
  }
  double hn = h2[(size_t)(S - 2) * N + k] * ci_all[S - 2];
  h2[(size_t)(S - 2) * N + k] = hn;
  for (int q = S - 3; q >= 0; --q) {
    hn = (h2[(size_t)q * N + k] - A2 * hn) * ci_all[q];
    h2[(size_t)q * N + k] = hn;
  }
}

// (3) owned segments: z − a h2_{σ−1} Z2_L − a h2_σ Z2_R, and the slab separators on both sides
__global__ void k_red2_fixup(DevTables T, const double* __restrict__ h2, double* __restrict__ hsep) {
  pdl_wait();
  const int N = T.N, S = T.nseg;
  const int k = blockIdx.x * blockDim.x + threadIdx.x + 1;
  const int sg = T.seg_lo + blockIdx.y;
  if (k >= N) return;
  const double a = T.red_a[k];
  const int gbase = sg * BL2;
  const double hl = sg > 0 ? a * h2[(size_t)(sg - 1) * N + k] : 0.0;
  const double hr = sg < S - 1 ? a * h2[(size_t)sg * N + k] : 0.0;
#pragma unroll
  for (int p = 0; p < LB2; ++p) {
    double x = hsep[(size_t)(gbase + p) * N + k];
    x = fma(-hl, T.z2r[(size_t)(LB2 - 1 - p) * N + k], x);
    x = fma(-hr, T.z2r[(size_t)p * N + k], x);
    hsep[(size_t)(gbase + p) * N + k] = x;
  }
  if (sg < S - 1) hsep[(size_t)(gbase + LB2) * N + k] = h2[(size_t)sg * N + k];
  if (sg > 0) hsep[(size_t)(gbase - 1) * N + k] = h2[(size_t)(sg - 1) * N + k];
}

// value of v̂ at column i, mode k: separator → h; block row → z − h_{g−1} Z_L − h_g Z_R
// fixup with the row's primary value (separator row or spectral row) already in shared memory
__device__ __forceinline__ double fixup_staged(const DevTables& T, const double* row, const double* __restrict__ hsep,
                                               int i, int k) {
  const int N = T.N, P = T.P;
  const int q = i / BL, r = i - q * BL;
  if (r == 0) return row[k];
  const int p = r - 1, g = q;
  double x = row[k];
  if (g > 0) x = fma(-hsep[(size_t)(g - 1) * N + k], __ldg(T.zr + (size_t)(LB - 1 - p) * N + k), x);
  if (g < P - 1) x = fma(-hsep[(size_t)g * N + k], __ldg(T.zr + (size_t)p * N + k), x);
  return x;
}

// ------------------------------------------------------------------------------ A6 sparse
// One CTA per column holding stencil nodes: v_j = (2/N) Σ_k v̂_k sin(πjk/N) at those rows.
// Modes are taken in quads {t, N−t, N/2−t, N/2+t}, t ∈ [1, N/4), using
//   sin(πj(N−t)/N) = (−1)^{j+1} s,  sin(πj(N/2 ± t)/N) = sin(πj/2) c ± cos(πj/2) s,
// s, c = sin, cos(πjt/N):  odd j:  Σ_t s P_t + σ_j Σ_t c R_t,   σ_j = sin(πj/2)
//                          even j: Σ_t s (Q_t + τ_j D_t),          τ_j = cos(πj/2)
// with P = x_t + x_{N−t}, Q = x_t − x_{N−t}, R = x_{N/2−t} + x_{N/2+t}, D = x_{N/2+t} − x_{N/2−t}.
// Modes N/4, N/2, 3N/4 are added by thread 0.  Thread `tid` owns t = tid + s·B; (s, c) along s
// follow by rotation with the per-row step e^{iπjB/N}.  Rows come grouped by class (odd,
// j ≡ 0, j ≡ 2 mod 4; setup order) and are processed up to four at a time.
#ifndef KFBI_INV_THREADS
#define KFBI_INV_THREADS 256
#endif
constexpr int kInvThreads = KFBI_INV_THREADS;
static_assert(kMaxColRows <= kInvThreads, "k_inv_sparse stages a column's rows one per thread");

template <int QPT>
__global__ void __launch_bounds__(kInvThreads, 2) k_inv_sparse(DevTables T, const double* __restrict__ spec,
                                                               const double* __restrict__ hsep, double* __restrict__ vsten) {
  extern __shared__ double smx[];
  __shared__ int s_rows[kMaxColRows];
  __shared__ double2 s_step[kMaxColRows];   // (cos, sin)(πjB/N) of each row: the recurrence step
  __shared__ double s_xq[3];                // modes N/4, N/2, 3N/4 of the column (thread 0's quad slot)
  const int N = T.N, half = N >> 1, quarter = N >> 2, m2 = 2 * N - 1, B = kInvThreads, P = T.P;
  double* tab = smx;   // sin(πr/N), r ∈ [0, N), at r + r/16
  double* red = smx + N + N / 16 + 1;   // [warp][2·row]: per-warp partial sums of the column's rows
  for (int r = threadIdx.x; r < N; r += B) tab[r + (r >> 4)] = sin_lookup(T.sin_tab, r, N);
  auto sinr = [&](int r) {   // sin(πr/N), r ∈ [0, 2N)
    const int idx = r & (N - 1);
    const double v = tab[idx + (idx >> 4)];
    return (r & N) ? -v : v;
  };
  // persistent over the owned stencil columns: the sine table is staged once per CTA.  Items are
  // taken in descending row count (setup order `ocol_order`), dealt in snake order over the CTAs:
  // a few columns along which Γ runs hold up to ~200 rows against a mean of 12, and a plain
  // round-robin left the CTAs that drew them as the kernel's tail.
  const int G = gridDim.x, nit = T.nocol;
  // the next item's (column, row range, class counts) are loaded one round ahead from the per-position
  // table ocol_meta (one load level), so that the column's row loads do not wait behind an index chain
  struct Item { int b, i, u0, u1, ncl0, ncl1; };
  auto item = [&](int r) {   // item of round r for this CTA (b = −1: none)
    Item it{-1, 0, 0, 0, 0, 0};
    const int kk = r * G + ((r & 1) ? G - 1 - (int)blockIdx.x : (int)blockIdx.x);
    if (kk >= nit) return it;
    const int2* m = reinterpret_cast<const int2*>(T.ocol_meta + 6 * (size_t)kk);
    const int2 m0 = m[0], m1 = m[1], m2v = m[2];
    it.b = m0.x; it.i = m0.y; it.u0 = m1.x; it.u1 = m1.y; it.ncl0 = m2v.x; it.ncl1 = m2v.y;
    if (it.b < T.o_lo || it.b >= T.o_hi) it.b = -1;
    return it;
  };
  Item nx = item(0);
  pdl_wait();   // the spectral rows (k_sweep) and separators (k_reduced2 / the level-2 fix-up) are ready
  for (int rnd = 0; rnd * G < nit; ++rnd) {
  const Item cur = nx;
  nx = item(rnd + 1);
  if (cur.b < 0) continue;   // CTA-uniform
  const int i = cur.i, u0 = cur.u0, u1 = cur.u1;
  __syncthreads();
  // row indices: loaded now, stored to shared memory after the row loads (kMaxColRows ≤ B)
  const int srow = u0 + (int)threadIdx.x < u1 ? T.sn_j[u0 + threadIdx.x] : 0;
  // column i: separator → x = h; block row → x = z − h_{g−1} Z_L[p] − h_g Z_R[p].
  // Spectral positions 4t..4t+3 hold the quad {t, N−t, N/2−t, N/2+t}: two 16-byte loads per array.
  const int q = i / BL, rr = i - q * BL;
  const bool sep = rr == 0;
  KFBI_CHECK(i >= T.col_lo && i <= T.col_hi && u1 - u0 <= T.mcr, i, u1 - u0);
  const double* xrow = sep ? hsep + (size_t)(q - 1) * N : spec + (size_t)(i - 1) * N;
  const double* hl = (!sep && q > 0) ? hsep + (size_t)(q - 1) * N : nullptr;
  const double* hr = (!sep && q < P - 1) ? hsep + (size_t)q * N : nullptr;
  const double* zl = T.zr + (size_t)(sep ? 0 : LB - rr) * N;     // Z_L[p] = Z_R[LB−1−p], p = rr − 1
  const double* zrr = T.zr + (size_t)(sep ? 0 : rr - 1) * N;
  double Pv[QPT], Qp[QPT], Qm[QPT], Rv[QPT];
  double xq1 = 0.0, xq2 = 0.0, xq3 = 0.0;   // modes N/4, N/2, 3N/4 (quad slot 0)
  // the row's own quads are loaded first, all QPT of them (their registers are the final ones), and
  // the fix-up rows after: more loads in flight per thread than quad-by-quad X4 (L2-latency bound)
#pragma unroll
  for (int s = 0; s < QPT; ++s) {
    const int t = threadIdx.x + s * B;
    if (t >= quarter) {
      Pv[s] = Qp[s] = Qm[s] = Rv[s] = 0.0;
      continue;
    }
    const double2* xp = reinterpret_cast<const double2*>(xrow + 4 * t);
    const double2 a = xp[0], b2 = xp[1];
    Pv[s] = a.x; Qp[s] = a.y; Qm[s] = b2.x; Rv[s] = b2.y;
  }
  auto fix = [&](const double* hrow, const double* zrow) {
#pragma unroll
    for (int s = 0; s < QPT; ++s) {
      const int t = threadIdx.x + s * B;
      if (t >= quarter) continue;
      const double2* hp = reinterpret_cast<const double2*>(hrow + 4 * t);
      const double2* zp = reinterpret_cast<const double2*>(zrow + 4 * t);
      const double2 h0 = hp[0], h1 = hp[1], z0 = __ldg(zp), z1 = __ldg(zp + 1);
      Pv[s] = fma(-h0.x, z0.x, Pv[s]); Qp[s] = fma(-h0.y, z0.y, Qp[s]);
      Qm[s] = fma(-h1.x, z1.x, Qm[s]); Rv[s] = fma(-h1.y, z1.y, Rv[s]);
    }
  };
  if (hl) fix(hl, zl);
  if (hr) fix(hr, zrr);
#pragma unroll
  for (int s = 0; s < QPT; ++s) {
    const int t = threadIdx.x + s * B;
    if (t >= quarter) continue;
    if (t == 0) {   // positions 0..3 = modes 0, N/2, N/4, 3N/4
      xq2 = Qp[s];
      xq1 = Qm[s];
      xq3 = Rv[s];
      Pv[s] = Qp[s] = Qm[s] = Rv[s] = 0.0;
    } else {
      const double a = Pv[s], bb = Qp[s], c = Qm[s], d = Rv[s];
      Pv[s] = a + bb;
      Rv[s] = c + d;
      Qp[s] = (a - bb) + (d - c);
      Qm[s] = (a - bb) - (d - c);
    }
  }
  {   // warm L2 with the next column's spectral row while this one is evaluated
    if (nx.b >= 0) {
      const int qn = nx.i / BL, rn = nx.i - qn * BL;
      const double* nrow = rn == 0 ? hsep + (size_t)(qn - 1) * N : spec + (size_t)(nx.i - 1) * N;
      for (int o = threadIdx.x * 16; o < N; o += B * 16)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(nrow + o));
    }
  }
  if (u0 + (int)threadIdx.x < u1) {
    s_rows[threadIdx.x] = srow;
    const int rd = (srow * B) & m2;
    s_step[threadIdx.x] = make_double2(sinr((rd + half) & m2), sinr(rd));
  }
  if (threadIdx.x == 0) {
    s_xq[0] = xq1;
    s_xq[1] = xq2;
    s_xq[2] = xq3;
  }
  __syncthreads();
  const double scale = 2.0 / N;
  const int nrows = u1 - u0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = B >> 5;
  // rows come sorted by class (odd, j ≡ 0, j ≡ 2 mod 4): groups of ≤ 4 rows of one class.  Sines along
  // the thread's quads t = tid + s·B by the three-term recurrence S_{s+1} = 2 cos(πjB/N) S_s − S_{s−1}
  // (one FMA per step; cosines likewise for odd rows).
  const int ncl0 = cur.ncl0, ncl1 = cur.ncl1;
#pragma unroll 1
  for (int c0 = 0; c0 < 3; ++c0) {
    const int cbeg = c0 == 0 ? 0 : (c0 == 1 ? ncl0 : ncl0 + ncl1);
    const int cend = c0 == 0 ? ncl0 : (c0 == 1 ? ncl0 + ncl1 : nrows);
#pragma unroll 1
    for (int u = cbeg; u < cend; u += 4) {
      const int nr = cend - u < 4 ? cend - u : 4;
      double accs[4] = {0.0, 0.0, 0.0, 0.0}, accc[4] = {0.0, 0.0, 0.0, 0.0};
      double S[4], Sm[4], C[4], Cm[4], twocd[4];
      int js[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        js[k] = k < nr ? s_rows[u + k] : 0;
        const int r0 = (js[k] * (int)threadIdx.x) & m2;
        const double2 st = s_step[k < nr ? u + k : u];
        const double s0 = sinr(r0), c0v = sinr((r0 + half) & m2);
        const double sd = st.y, cd = st.x;
        S[k] = s0;
        C[k] = c0v;
        Sm[k] = fma(s0, cd, -c0v * sd);   // angle − πjB/N
        Cm[k] = fma(c0v, cd, s0 * sd);
        twocd[k] = 2.0 * cd;
      }
      if (c0 == 0) {
#pragma unroll
        for (int s = 0; s < QPT; ++s) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            accs[k] = fma(Pv[s], S[k], accs[k]);
            accc[k] = fma(Rv[s], C[k], accc[k]);
            const double sn = fma(twocd[k], S[k], -Sm[k]), cn = fma(twocd[k], C[k], -Cm[k]);
            Sm[k] = S[k];
            S[k] = sn;
            Cm[k] = C[k];
            C[k] = cn;
          }
        }
      } else {
#pragma unroll
        for (int s = 0; s < QPT; ++s) {
          const double xv = c0 == 1 ? Qp[s] : Qm[s];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            accs[k] = fma(xv, S[k], accs[k]);
            const double sn = fma(twocd[k], S[k], -Sm[k]);
            Sm[k] = S[k];
            S[k] = sn;
          }
        }
      }
      double acc[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc[k] = accs[k];
        acc[4 + k] = accc[k];
      }
      const double ws = warp_transpose_reduce8(acc);
      if ((lane & 3) == 0) {   // value index v = 4·(lane>>4 & 1) + 2·(lane>>3 & 1) + (lane>>2 & 1): acc[v]
        const int v = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
        const int k = v & 3;
        if (k < nr) red[(size_t)wid * 2 * T.mcr + 2 * (u + k) + (v >> 2)] = ws;
      }
    }
  }
  __syncthreads();   // one barrier per column: sum the warps' partials in a fixed order
  for (int t = threadIdx.x; t < nrows; t += B) {
    double s1 = 0.0, s2 = 0.0;
    for (int w = 0; w < nw; ++w) {
      s1 += red[(size_t)w * 2 * T.mcr + 2 * t];
      s2 += red[(size_t)w * 2 * T.mcr + 2 * t + 1];
    }
    const int j = s_rows[t];
    // the special modes, per row here rather than by thread 0 inside every group (no warp-0 divergence)
    s1 += s_xq[0] * sinr((j * quarter) & m2) + s_xq[1] * sinr((j * half) & m2) +
          s_xq[2] * sinr((j * (half + quarter)) & m2);
    const double sig = ((j >> 1) & 1) ? -1.0 : 1.0;   // σ_j = sin(πj/2) for odd j
    KFBI_CHECK(u0 + t < T.nsn && j >= 1 && j < N, u0 + t, j);
    vsten[u0 + t] = scale * ((j & 1) ? s1 + sig * s2 : s1);
  }
  }
}

// ------------------------------------------------------------------------------ A7
__global__ void k_interp(DevTables T, const double* __restrict__ phi, const double* __restrict__ mk,
                         const double* __restrict__ fz, const double* __restrict__ jzg,
                         const double* __restrict__ vsten, int nh, const double* __restrict__ wg,
                         const double* __restrict__ ahole, double* __restrict__ out, int partial) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= T.M) return;
  if (partial) {   // multi-GPU: a control point whose stencil columns c − 1 … c + 1 miss the slab adds 0
    const int col = T.sn_i[T.st_node[m * 6]];
    if (col + 1 < T.col_lo || col - 1 > T.col_hi) {
      pdl_wait();
      double acc = 0.0;   // rank 0 still adds the hole-completion term (R27) of every control point
      if (T.rank == 0)
        for (int hh = 0; hh < nh; ++hh) acc = fma(ahole[hh], wg[(size_t)hh * T.M + m], acc);
      out[m] = acc;
      return;
    }
  }
  // the stencil's loads (node ids → values, weights, offsets) and the hole terms are issued before the
  // jump chain (spline knots → φ, M → jumps), so the two dependent load chains overlap
  int sn[6];
  double v[6], wt[6], dx[6], dy[6];
  bool ext[6];
#pragma unroll
  for (int p = 0; p < 6; ++p) {
    const int idx = m * 6 + p;
    sn[p] = T.st_node[idx];
    ext[p] = T.st_ext[idx];
    dx[p] = T.st_dx[idx];
    dy[p] = T.st_dy[idx];
    wt[p] = T.neumann ? T.st_wn[idx] : T.st_w[idx];   // V⁺ or ∂_n V⁺ (Neumann, R38)
  }
  pdl_wait();   // vsten (k_inv_sparse), the spline knots and hole coefficients (k_spline)
#pragma unroll
  for (int p = 0; p < 6; ++p) {
    KFBI_CHECK(sn[p] >= 0 && sn[p] < T.nsn, sn[p], T.nsn);
    v[p] = vsten[sn[p]];
    if (partial) {   // multi-GPU: only stencil nodes in the owned columns contribute (partial sum)
      const int col = T.sn_i[sn[p]];
      if (col < T.col_lo || col > T.col_hi) wt[p] = 0.0, v[p] = 0.0, ext[p] = false;
    }
  }
  double hole = 0.0;
  if (!partial || T.rank == 0)
    for (int hh = 0; hh < nh; ++hh) hole = fma(ahole[hh], wg[(size_t)hh * T.M + m], hole);
  Jump6 J;
  if (jzg) {
    J.v = jzg[m * 6];
    J.vx = jzg[m * 6 + 1];
    J.vy = jzg[m * 6 + 2];
    J.vxx = jzg[m * 6 + 3];
    J.vxy = jzg[m * 6 + 4];
    J.vyy = jzg[m * 6 + 5];
  } else {
    double Phi = 0, Phis = 0, Phiss = 0;
    if (phi) {
      spline_eval2(phi, mk, reinterpret_cast<const int2*>(T.z_g01)[m], T.z_dl[m], 0.0, Phi, Phis, Phiss);
    }
    J = T.neumann ? jumps2d(0.0, 0.0, 0.0, Phi, Phis, fz ? fz[m] : 0.0, T.kappa, T.z_t1[m], T.z_t2[m], T.z_p1[m], T.z_p2[m])
                  : jumps2d(Phi, Phis, Phiss, 0.0, 0.0, fz ? fz[m] : 0.0, T.kappa, T.z_t1[m], T.z_t2[m], T.z_p1[m], T.z_p2[m]);
  }
  double acc = 0.0;
#pragma unroll
  for (int p = 0; p < 6; ++p) {
    double vp = v[p];
    if (ext[p])   // exterior node: shift by the jump Taylor polynomial
      vp += J.v + J.vx * dx[p] + J.vy * dy[p] + 0.5 * J.vxx * dx[p] * dx[p] + J.vxy * dx[p] * dy[p] +
            0.5 * J.vyy * dy[p] * dy[p];
    acc = fma(wt[p], vp, acc);
  }
  out[m] = acc + hole;
}

__global__ void k_hole_coeffs(const int* __restrict__ off, const int* __restrict__ cnt,
                              const double* __restrict__ delta, const double* __restrict__ phi,
                              double* __restrict__ a) {
  pdl_wait();
  __shared__ double scratch[32];
  const int hh = blockIdx.x;
  double v[1] = {0.0};
  for (int m = threadIdx.x; m < cnt[hh]; m += blockDim.x) v[0] += phi[off[hh] + m];
  block_reduce<1>(v, scratch);
  if (threadIdx.x == 0) a[hh] = delta[hh] * v[0];
}

// ------------------------------------------------------------------------------ Gray–Scott (NEXT-2)
// pointwise reaction by the explicit midpoint rule (reading R40), rates (1/ε₀)[γ(1−u) − uv², uv² − (γ+κ_r)v]
__device__ __forceinline__ void gs_rates(double u, double v, const GsParams& p, double& du, double& dv) {
  const double uv2 = u * v * v;
  du = (p.gamma * (1.0 - u) - uv2) / p.eps0;
  dv = (uv2 - (p.gamma + p.kr) * v) / p.eps0;
}
__global__ void k_gs_reaction(double* __restrict__ u, double* __restrict__ v, long n, double dt, GsParams p) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const double u0 = u[i], v0 = v[i];
    double du, dv;
    gs_rates(u0, v0, p, du, dv);
    const double um = u0 + 0.5 * dt * du, vm = v0 + 0.5 * dt * dv;
    gs_rates(um, vm, p, du, dv);
    u[i] = u0 + dt * du;
    v[i] = v0 + dt * dv;
  }
}
__device__ __forceinline__ double bilinear(const double* __restrict__ w, int N, double lo, double h, double px,
                                           double py) {
  const double sx = (px - lo) / h, sy = (py - lo) / h;
  const int i = (int)floor(sx), j = (int)floor(sy);
  const double tx = sx - i, ty = sy - j;
  const size_t W = (size_t)N + 1, b = (size_t)i * W + j;
  return (1 - tx) * (1 - ty) * w[b] + tx * (1 - ty) * w[b + W] + (1 - tx) * ty * w[b + 1] + tx * ty * w[b + W + 1];
}
// diffusion source f = −κ w at the full grid, the intersections and the control points (R41: bilinear)
__global__ void k_gs_rhs(DevTables T, const double* __restrict__ w, double* __restrict__ fg,
                         double* __restrict__ fq, double* __restrict__ fz) {
  const long nn = (long)(T.N + 1) * (T.N + 1);
  const double k = T.kappa;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < nn + T.nq + T.M; i += (long)gridDim.x * blockDim.x) {
    if (i < nn) fg[i] = -k * w[i];
    else if (i < nn + T.nq) fq[i - nn] = -k * bilinear(w, T.N, T.lo, T.h, T.q_x[i - nn], T.q_y[i - nn]);
    else fz[i - nn - T.nq] = -k * bilinear(w, T.N, T.lo, T.h, T.z_x[i - nn - T.nq], T.z_y[i - nn - T.nq]);
  }
}
__global__ void k_gs_combine(double* __restrict__ w, const double* __restrict__ y, long n) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    w[i] = 2.0 * y[i] - w[i];   // Crank–Nicolson: (I − aΔ)^{-1}(I + aΔ) w = 2y − w
}
// out = base + Σ_q coef[q] · V_q (coefficients in device memory; base may be NULL)
__global__ void k_fill(double* __restrict__ x, long n, double val) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) x[i] = val;
}

// ---- dense DST-I rows (2D), half-length core: forward from the full grid (volume term + bumps)
// into spectral positions (MODE 0), inverse from the fixed-up spectrum into the full grid (MODE 1).
// N ≤ 1024: 256/(N/32) rows per CTA, a row on N/32 lanes of a warp; N ≥ 2048: one row per CTA.
__device__ __forceinline__ double dense_src(const DevTables& T, const double* __restrict__ src, int mask_omega,
                                            const BumpParams& bp, int i, int j) {
  const int N = T.N;
  double v = 0.0;
  if (j == 0) return v;
  const size_t idx = (size_t)i * (N + 1) + j;
  if (src && mask_omega == 2) {   // Ω-compact input: the node's rank among the Ω nodes (row-major)
    const uint32_t* info = T.om_info + (size_t)i * 2 * T.om_nsegp;
    const uint32_t bits = info[j >> 5];
    if ((bits >> (j & 31)) & 1u) {
      const int r = T.om_row[i] + (int)info[T.om_nsegp + (j >> 5)] + __popc(bits & ((1u << (j & 31)) - 1u));
      KFBI_CHECK(r < T.om_row[i + 1], r, i);
      v = src[r];
    }
  } else if (src && (!mask_omega || T.side[idx])) {
    v = src[idx];
  }
  if (bp.nh) {
    const double x = T.lo + i * T.h, yy = T.lo + j * T.h;
    for (int hh = 0; hh < bp.nh; ++hh) {
      const double dx = x - bp.cx[hh], dy = yy - bp.cy[hh], r = bp.rad[hh];
      if (fabs(dx) >= r || fabs(dy) >= r) continue;   // outside the support's bounding box
      const double rho2 = (dx * dx + dy * dy) / (r * r);
      if (rho2 < 1.0) v += bp.a[hh] * exp(1.0 - 1.0 / (1.0 - rho2));   // bump, SURVEY App. A.8
    }
  }
  return v;
}

#ifndef KFBI_DST_SPLIT
#define KFBI_DST_SPLIT 1
#endif
template <int N>
struct DenseCfg {
  static constexpr int NTH = N / 16, RPC = NTH > 32 ? 1 : 256 / NTH, NTHR = NTH * RPC, ZS = N + N / 16 + 1;
  // one row per CTA: the next row's input streams into shared memory by a bulk copy (TMA engine)
  // while the current row is transformed
  static constexpr bool STAGE = RPC == 1;
  static constexpr int STAGE_D = N + 2;            // doubles: one row (+1 for 8-byte misalignment)
  static constexpr int STAGE_B = N + 1 + 32;       // bytes of the Ω-mask row (+ alignment), or the
                                                   // Ω-compact row's segment bits and counts (2·nsegp words)
  static constexpr size_t smem(bool staged) {
    return (size_t)RPC * ZS * 16 + (staged ? (size_t)STAGE_D * 8 + STAGE_B + 16 : 0);
  }
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// one thread: arm the barrier with the byte count, then the bulk copies (16-byte aligned, sizes % 16 == 0)
__device__ __forceinline__ void bulk_load(uint64_t* bar, void* dst0, const void* src0, uint32_t n0, void* dst1,
                                          const void* src1, uint32_t n1) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // earlier generic reads of the buffer
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(n0 + n1) : "memory");
  if (n0)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst0)),
                 "l"(src0), "r"(n0), "r"(smem_u32(bar))
                 : "memory");
  if (n1)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst1)),
                 "l"(src1), "r"(n1), "r"(smem_u32(bar))
                 : "memory");
}

// Dense rows (A4 forward of the volume term / A6 inverse of the final field), one row per NTH
// threads, accurate N-point core.  MODE 0: row i of the (N+1)² grid (Ω-masked, + hole bumps) →
// spectral positions of row i−1.  MODE 1: spectral row (fixed up by the separator values) →
// grid row i scaled by 2/N.  With STAGE the row's primary input (grid row + mask row, or spectral /
// separator row) is bulk-copied into shared memory one row ahead.
template <int MODE, int N>
__global__ void __launch_bounds__(DenseCfg<N>::NTHR, 1) k_dst_dense2(DevTables T, const double* __restrict__ src,
                                                                    int mask_omega, BumpParams bp,
                                                                    const double* __restrict__ hsep,
                                                                    double* __restrict__ dst) {
  pdl_wait();   // the input rows / spectra from the previous kernel
  using C = DenseCfg<N>;
  constexpr int NTH = C::NTH, RPC = C::RPC;
  extern __shared__ double2 smz[];
  __shared__ uint64_t bar;
  const int rl = threadIdx.x / NTH, tid = threadIdx.x % NTH;
  double2* z = smz + rl * C::ZS;
  const double2* __restrict__ tw = reinterpret_cast<const double2*>(T.tw);
  double* stage = reinterpret_cast<double*>(smz + RPC * C::ZS);
  uint8_t* smask = reinterpret_cast<uint8_t*>(stage + C::STAGE_D);
  // staged input for the forward rows only: the inverse rows' spectral row was measured slower
  // staged (1150 vs 1048 µs at N = 8192) than with the L2 prefetch below
  const bool staged = C::STAGE && MODE == 0 && src != nullptr;
  const int step = gridDim.x * RPC;
  // bulk copies of row `in`'s primary input; returns nothing, offsets recomputed by the reader
  const bool compact = mask_omega == 2;   // MODE 0: src holds f at the Ω nodes only (row-major ranks)
  auto issue = [&](int in) {
    if (MODE == 0 && compact) {
      // the row's Ω values are contiguous: [om_row[in], om_row[in + 1]); the copy is rounded down to
      // whole 16-byte words (the last value, if cut, is read from global memory), plus the row's
      // segment bits and counts
      const char* a = reinterpret_cast<const char*>(src + T.om_row[in]);
      const char* al = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(a) & ~uintptr_t(15));
      const uint32_t n0 = (uint32_t)(((a - al) + (size_t)(T.om_row[in + 1] - T.om_row[in]) * 8) & ~size_t(15));
      const uint32_t* info = T.om_info + (size_t)in * 2 * T.om_nsegp;
      bulk_load(&bar, stage, al, n0, smask, info, (uint32_t)T.om_nsegp * 8u);
    } else if (MODE == 0) {
      const char* a = reinterpret_cast<const char*>(src + (size_t)in * (N + 1));
      const char* al = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(a) & ~uintptr_t(15));
      const uint32_t n0 = (uint32_t)((((a - al) + (N + 1) * 8) + 15) & ~15);
      const char* m = reinterpret_cast<const char*>(T.side + (size_t)in * (N + 1));
      const char* ml = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(m) & ~uintptr_t(15));
      const uint32_t n1 = mask_omega ? (uint32_t)((((m - ml) + (N + 1)) + 15) & ~15) : 0u;
      bulk_load(&bar, stage, al, n0, smask, ml, n1);
    } else {
      const int qn = in / BL, rn = in - qn * BL;
      const double* row = rn == 0 ? hsep + (size_t)(qn - 1) * N : src + (size_t)(in - 1) * N;
      bulk_load(&bar, stage, row, (uint32_t)N * 8, nullptr, nullptr, 0u);
    }
  };
  uint32_t phase = 0;
  if (staged) {
    if (threadIdx.x == 0) {
      mbar_init(&bar);
      if (T.col_lo + (int)blockIdx.x <= T.col_hi) issue(T.col_lo + blockIdx.x);
    }
    __syncthreads();
  }
  // persistent over row groups; unstaged: the next group's input rows are prefetched into L2 first
  for (int rb = blockIdx.x; T.col_lo + rb * RPC <= T.col_hi; rb += gridDim.x) {
  const int i = T.col_lo + rb * RPC + rl;
  const bool live = i <= T.col_hi;
  // MODE 1 with Ω-compact output: a grid row without Ω nodes has no output — its loads, transform and
  // stores are skipped
  const bool skip1 = MODE == 1 && compact && live && !T.row_omega[i];
  if (!staged) {
    const int in = i + step;
    if (in <= T.col_hi && src) {
      if (MODE == 0 && compact) {
        const double* row = src + T.om_row[in];
        for (int o = 16 * tid; o < T.om_row[in + 1] - T.om_row[in]; o += 16 * NTH)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(row + o));
      } else if (MODE == 0) {
        const double* row = src + (size_t)in * (N + 1);
        for (int o = 16 * tid; o <= N; o += 16 * NTH) asm volatile("prefetch.global.L2 [%0];" ::"l"(row + o));
        if (mask_omega && tid < (N + 128) / 128)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(T.side + (size_t)in * (N + 1) + 128 * tid));
      } else {
        const int qn = in / BL, rn = in - qn * BL;
        const double* row = rn == 0 ? hsep + (size_t)(qn - 1) * N : src + (size_t)(in - 1) * N;
        for (int o = 16 * tid; o < N; o += 16 * NTH) asm volatile("prefetch.global.L2 [%0];" ::"l"(row + o));
      }
    }
  }
  rsync<NTH>();   // the previous group's outputs have been read out of z
  if (staged) {
    mbar_wait(&bar, phase);
    phase ^= 1u;
  }
  double2 fp[8];
  if (MODE == 0) {
    if (staged && compact) {   // Ω values from the staged compact row (segment bits / counts staged too)
      const int r0 = T.om_row[i], nv = T.om_row[i + 1] - r0;
      const int off = (int)((reinterpret_cast<uintptr_t>(src + r0) & 15) >> 3);
      const int nst = ((off + nv) & ~1) - off;   // values held by the stage
      const uint32_t* bits = reinterpret_cast<const uint32_t*>(smask);
      const uint32_t* cnt = bits + T.om_nsegp;
      auto val = [&](int j) {
        const uint32_t b = bits[j >> 5];
        if (!((b >> (j & 31)) & 1u)) return 0.0;
        const int r = (int)cnt[j >> 5] + __popc(b & ((1u << (j & 31)) - 1u));
        KFBI_CHECK(r < nv, r, nv);
        return r < nst ? stage[off + r] : src[r0 + r];
      };
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int m = tid + NTH * s;
        double v0 = m ? val(2 * m) : 0.0, v1 = val(2 * m + 1);
        if (bp.nh) {
          v0 += dense_src(T, nullptr, 0, bp, i, 2 * m);
          v1 += dense_src(T, nullptr, 0, bp, i, 2 * m + 1);
        }
        fp[s] = make_double2(v0, v1);
      }
      __syncthreads();   // every read of the staging buffer is done: stream the next row in
      if (threadIdx.x == 0 && i + step <= T.col_hi) issue(i + step);
    } else if (staged) {   // the row and its mask from shared memory (8-byte / byte offsets of the aligned copies)
      const size_t a = reinterpret_cast<uintptr_t>(src + (size_t)i * (N + 1));
      const double* row = stage + ((a & 15) >> 3);
      const uint8_t* mrow = smask + (reinterpret_cast<uintptr_t>(T.side + (size_t)i * (N + 1)) & 15);
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int m = tid + NTH * s;
        double v0 = 0.0, v1 = row[2 * m + 1];
        if (m) v0 = row[2 * m];
        if (mask_omega) {
          if (!mrow[2 * m]) v0 = 0.0;
          if (!mrow[2 * m + 1]) v1 = 0.0;
        }
        if (bp.nh) {
          v0 += dense_src(T, nullptr, 0, bp, i, 2 * m);
          v1 += dense_src(T, nullptr, 0, bp, i, 2 * m + 1);
        }
        fp[s] = make_double2(v0, v1);
      }
      __syncthreads();   // every read of the staging buffer is done: stream the next row in
      if (threadIdx.x == 0 && i + step <= T.col_hi) issue(i + step);
    } else {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int m = tid + NTH * s;
        fp[s] = live ? make_double2(dense_src(T, src, mask_omega, bp, i, 2 * m), dense_src(T, src, mask_omega, bp, i, 2 * m + 1))
                     : make_double2(0.0, 0.0);
      }
    }
  } else {   // spectral positions → modes (coalesced reads, scattered shared-memory writes), then pairs
    double* f = reinterpret_cast<double*>(z);
    if (!staged) {
      // a quad of positions {t, N−t, N/2−t, N/2+t} per step: two 16-byte loads per row (x, h_{g−1},
      // Z_L[p], h_g, Z_R[p]), fixed up and scattered to the four modes
      const int q = i / BL, rr = i - q * BL;
      const bool sep = rr == 0;
      const double* xrow = sep ? hsep + (size_t)(q - 1) * N : src + (size_t)(i - 1) * N;
      const double* hl = (!sep && q > 0) ? hsep + (size_t)(q - 1) * N : nullptr;
      const double* hr = (!sep && q < T.P - 1) ? hsep + (size_t)q * N : nullptr;
      const double* zl = T.zr + (size_t)(sep ? 0 : LB - rr) * N;   // Z_L[p] = Z_R[LB−1−p], p = rr − 1
      const double* zrr = T.zr + (size_t)(sep ? 0 : rr - 1) * N;
      for (int t = tid; t < N / 4; t += NTH) {
        double2 a = make_double2(0.0, 0.0), b = a;
        if (live && !skip1) {
          a = reinterpret_cast<const double2*>(xrow + 4 * t)[0];
          b = reinterpret_cast<const double2*>(xrow + 4 * t)[1];
          if (hl) {
            const double2 h0 = reinterpret_cast<const double2*>(hl + 4 * t)[0], h1 = reinterpret_cast<const double2*>(hl + 4 * t)[1];
            const double2 z0 = __ldg(reinterpret_cast<const double2*>(zl + 4 * t)), z1 = __ldg(reinterpret_cast<const double2*>(zl + 4 * t) + 1);
            a.x = fma(-h0.x, z0.x, a.x); a.y = fma(-h0.y, z0.y, a.y);
            b.x = fma(-h1.x, z1.x, b.x); b.y = fma(-h1.y, z1.y, b.y);
          }
          if (hr) {
            const double2 h0 = reinterpret_cast<const double2*>(hr + 4 * t)[0], h1 = reinterpret_cast<const double2*>(hr + 4 * t)[1];
            const double2 z0 = __ldg(reinterpret_cast<const double2*>(zrr + 4 * t)), z1 = __ldg(reinterpret_cast<const double2*>(zrr + 4 * t) + 1);
            a.x = fma(-h0.x, z0.x, a.x); a.y = fma(-h0.y, z0.y, a.y);
            b.x = fma(-h1.x, z1.x, b.x); b.y = fma(-h1.y, z1.y, b.y);
          }
        }
        const int p = 4 * t;
        f[position_mode(p, N)] = position_mode(p, N) ? a.x : 0.0;   // mode 0 (t = 0, r = 0) is not a mode
        f[position_mode(p + 1, N)] = a.y;
        f[position_mode(p + 2, N)] = b.x;
        f[position_mode(p + 3, N)] = b.y;
      }
    } else {
      for (int p = tid; p < N; p += NTH) {
        const int k = position_mode(p, N);
        f[k] = (live && k) ? fixup_staged(T, stage, hsep, i, p) : 0.0;
      }
    }
    rsync<NTH>();
    if (staged && threadIdx.x == 0 && i + step <= T.col_hi) issue(i + step);
#pragma unroll
    for (int s = 0; s < 8; ++s) fp[s] = reinterpret_cast<const double2*>(f)[tid + NTH * s];
    rsync<NTH>();
  }
  // a forward row of f·1_Ω with no Ω node (a grid column outside Γ's x-extent) has a zero spectrum:
  // no transform (CTA-uniform when a CTA holds one row, N ≥ 2048)
  const bool empty = (MODE == 0 && RPC == 1 && mask_omega && bp.nh == 0 && live && !T.row_omega[i]) ||
                     (RPC == 1 && skip1);
  if (!empty) {
    if constexpr (N >= 2048 && KFBI_DST_SPLIT) dst1s_core<N>(z, tw, tid, fp);   // split radix: half the FFT points
    else dst1_core<N>(z, tw, tid, fp);
  }
  if (!live) continue;
  if (MODE == 0) {
    for (int p = tid; p < N; p += NTH) {   // modes → spectral positions
      const int k = position_mode(p, N);
      __stcs(dst + (size_t)(i - 1) * N + p, (k && !empty) ? z[zpad(k)].x : 0.0);
    }
  } else {
    const double sc = 2.0 / N;
    if (mask_omega == 2) {   // Ω-compact output: u at the row's Ω nodes only (never j = 0, N)
      const uint32_t* info = T.om_info + (size_t)i * 2 * T.om_nsegp;
      const int r0 = T.om_row[i];
      for (int j = tid; j <= N; j += NTH) {
        const uint32_t b = info[j >> 5];
        if ((b >> (j & 31)) & 1u) {
          const int r = r0 + (int)info[T.om_nsegp + (j >> 5)] + __popc(b & ((1u << (j & 31)) - 1u));
          KFBI_CHECK(r < T.om_row[i + 1], r, i);
          __stcs(dst + r, sc * z[zpad(j)].x);
        }
      }
    } else {
      for (int j = tid; j <= N; j += NTH)
        __stcs(dst + (size_t)i * (N + 1) + j, (j == 0 || j == N) ? 0.0 : sc * z[zpad(j)].x);
    }
  }
  }
}

// ------------------------------------------------------------------------------ A8 GMRES
// sum of the kRedBlocks per-CTA partials in a fixed order (deterministic), by one warp: lane l adds
// p[l], p[l+32], … (independent loads), then a fixed xor tree; every lane returns the total
__device__ __forceinline__ double warp_ordered_sum(const double* __restrict__ p) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
#pragma unroll
  for (int b = 0; b < kRedBlocks / 32; ++b) s += p[lane + 32 * b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}
// the same total broadcast to the whole CTA (warp 0 sums, one barrier)
__device__ __forceinline__ double block_ordered_sum(const double* __restrict__ p) {
  __shared__ double s_tot;
  if (threadIdx.x < 32) {
    const double t = warp_ordered_sum(p);
    if (threadIdx.x == 0) s_tot = t;
  }
  __syncthreads();
  return s_tot;
}

__global__ void k_mgs_step(int n, double* w, const double* Vprev, const double* Vcur, const double* pprev,
                           double* pcur, double* hout) {
  pdl_wait();
  __shared__ double scratch[32];
  const int per = (n + gridDim.x - 1) / gridDim.x;
  const int b0 = blockIdx.x * per, b1 = min(n, b0 + per);
  double hp = 0.0;
  if (Vprev) {
    hp = block_ordered_sum(pprev);
    if (blockIdx.x == 0 && threadIdx.x == 0) *hout = hp;
  }
  double a0 = 0.0, a1 = 0.0;   // two independent chains
  int i = b0 + threadIdx.x;
  for (; i + (int)blockDim.x < b1; i += 2 * blockDim.x) {
    double w0 = w[i], w1 = w[i + blockDim.x];
    if (Vprev) {
      w0 = fma(-hp, Vprev[i], w0);
      w1 = fma(-hp, Vprev[i + blockDim.x], w1);
      w[i] = w0;
      w[i + blockDim.x] = w1;
    }
    a0 = fma(w0, Vcur[i], a0);
    a1 = fma(w1, Vcur[i + blockDim.x], a1);
  }
  if (i < b1) {
    double w0 = w[i];
    if (Vprev) {
      w0 = fma(-hp, Vprev[i], w0);
      w[i] = w0;
    }
    a0 = fma(w0, Vcur[i], a0);
  }
  double v[1] = {a0 + a1};
  block_reduce<1>(v, scratch);
  if (threadIdx.x == 0) pcur[blockIdx.x] = v[0];
}

__global__ void k_norm_scale(int n, double* w, const double* __restrict__ partial, double* hout) {
  pdl_wait();
  const double hn = sqrt(block_ordered_sum(partial));
  if (blockIdx.x == 0 && threadIdx.x == 0) *hout = hn;
  if (hn == 0.0) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) w[i] = w[i] / hn;
}

// Whole MGS step of Arnoldi iteration j: h_i = (w, μ_i), w −= h_i μ_i for i = 0..j, then
// h_{j+1} = ‖w‖ and w /= h_{j+1}, on one thread-block cluster: CTA c of kMgsCl owns the contiguous
// slice [c·n_c, (c+1)·n_c) of w in registers (KPT per thread).  Per projection i: slice dot with v_i
// (v_{i+1} already loading), warp shuffles + per-warp partials summed in order by thread 0, the CTA
// partial stored into every CTA's shared slot over DSMEM, one cluster barrier, and every thread sums
// the kMgsCl partials in rank order — so all CTAs hold the same h_i, then w −= h_i v_i.  Slots are
// double-buffered by the parity of i: a slot is rewritten two barriers after it was read.
constexpr int kMgsCl = 8, kMgsClThreads = 512;
template <int KPT>
__global__ void __cluster_dims__(kMgsCl, 1, 1) __launch_bounds__(kMgsClThreads)
    k_mgs_cluster(int n, int j, const double* __restrict__ V, double* w, double* hcol) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  pdl_wait();   // w from the apply's k_interp
  __shared__ double warp_part[kMgsClThreads / 32];
  __shared__ double slot[2][kMgsCl];
  const int rank = (int)cl.block_rank(), lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nc = (n + kMgsCl - 1) / kMgsCl, c0 = rank * nc, c1 = min(n, c0 + nc);
  double x[KPT], v[KPT];
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    const int idx = c0 + threadIdx.x + k * kMgsClThreads;
    x[k] = idx < c1 ? w[idx] : 0.0;
    v[k] = idx < c1 ? V[idx] : 0.0;
  }
  auto cluster_sum = [&](double a, int parity) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) warp_part[wid] = a;
    __syncthreads();
    if (threadIdx.x < kMgsCl) {   // thread r stores this CTA's partial into CTA r's slot
      double t = 0.0;
      for (int q = 0; q < kMgsClThreads / 32; ++q) t += warp_part[q];
      double* remote = cl.map_shared_rank(&slot[parity][0], (int)threadIdx.x);
      remote[rank] = t;
    }
    cl.sync();
    double tot = 0.0;
#pragma unroll
    for (int r = 0; r < kMgsCl; ++r) tot += slot[parity][r];
    return tot;
  };
  for (int i = 0; i <= j; ++i) {
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < KPT; ++k) a = fma(x[k], v[k], a);
    double vn[KPT];
    if (i < j) {
      const double* vi = V + (size_t)(i + 1) * n;
#pragma unroll
      for (int k = 0; k < KPT; ++k) {
        const int idx = c0 + threadIdx.x + k * kMgsClThreads;
        vn[k] = idx < c1 ? vi[idx] : 0.0;
      }
    }
    const double h = cluster_sum(a, i & 1);
    if (rank == 0 && threadIdx.x == 0) hcol[i] = h;
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
      x[k] = fma(-h, v[k], x[k]);
      if (i < j) v[k] = vn[k];
    }
  }
  double a = 0.0;
#pragma unroll
  for (int k = 0; k < KPT; ++k) a = fma(x[k], x[k], a);
  const double hn = sqrt(cluster_sum(a, (j + 1) & 1));
  if (rank == 0 && threadIdx.x == 0) hcol[j + 1] = hn;
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    const int idx = c0 + threadIdx.x + k * kMgsClThreads;
    if (idx < c1) w[idx] = hn == 0.0 ? x[k] : x[k] / hn;
  }
  cl.sync();   // no CTA may exit while another can still write into its slots
}

__global__ void k_dot(int n, const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ partial) {
  pdl_wait();
  __shared__ double scratch[32];
  const int per = (n + gridDim.x - 1) / gridDim.x;
  const int b0 = blockIdx.x * per, b1 = min(n, b0 + per);
  double v[1] = {0.0};
  for (int i = b0 + threadIdx.x; i < b1; i += blockDim.x) v[0] = fma(a[i], b[i], v[0]);
  block_reduce<1>(v, scratch);
  if (threadIdx.x == 0) partial[blockIdx.x] = v[0];
}

__global__ void k_finish_sum(const double* __restrict__ partial, double* out, int take_sqrt) {
  pdl_wait();
  if (threadIdx.x < 32 && blockIdx.x == 0) {
    const double s = warp_ordered_sum(partial);
    if (threadIdx.x == 0) *out = take_sqrt ? sqrt(s) : s;
  }
}

__global__ void k_axpy_basis(int n, int k, const double* __restrict__ V, int ldv, const YCoef y,
                             double* __restrict__ x) {
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int q = 0; q < k; ++q) acc = fma(y.v[q], V[(size_t)q * ldv + i], acc);
    x[i] += acc;
  }
}

// plain copy on the SMs (device or host-mapped memory): keeps the solve's small transfers off the copy
// engines, which a concurrent bulk H2D/D2H (pipelined serving) would otherwise queue them behind
__global__ void k_copy(int n, const double* __restrict__ src, double* __restrict__ dst) {
  pdl_wait();   // src from the previous kernel
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

__global__ void k_sub(int n, const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ o) {
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) o[i] = a[i] - b[i];
}

__global__ void k_scale_copy(int n, const double* __restrict__ a, const double* __restrict__ scal,
                             double* __restrict__ o) {
  pdl_wait();
  const double s = *scal;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) o[i] = a[i] / s;
}

inline int cdiv(long a, long b) { return (int)((a + b - 1) / b); }

}  // namespace

// ============================================================================== launchers
long long g_launches = 0;

void launch_spline(const DevTables& T, const double* phi, double* mk, cudaStream_t s, const int* hole_off,
                   const int* hole_M, const double* hole_delta, int nh, double* ahole) {
  const int nsb = cdiv(T.M * kSplineLanes, 256);
  { ++g_launches; launch_pdl(k_spline, dim3(nsb + nh), dim3(256), 0, s, T, phi, mk, nh, hole_off, hole_M, hole_delta, ahole); }
}

void launch_correct(const DevTables& T, const double* phi, const double* mk, const double* fq,
                    const double* jq_given, double* cval, cudaStream_t s) {
  if (T.irr_hi <= T.irr_lo) return;
  { ++g_launches; launch_pdl(k_correct, dim3(cdiv(T.irr_hi - T.irr_lo, 128)), dim3(128), 0, s, T, phi, mk, fq, jq_given, cval); }
}



void launch_sweep(const DevTables& T, const double* cval, const DenseSrc& D, double* spec, double* zfirst,
                  double* zlast, double* fsep, cudaStream_t s) {
  const int dense = !D.any() ? 0 : D.nb > 0 ? 2 : 1;
  (void)zlast;
  const size_t sm = (size_t)BL * 4 * kRs * sizeof(double) + (size_t)std::min(T.maxe, kEntCap) * 5 * sizeof(double) +
                    (size_t)(2 * T.N / 64 + 2 * T.N / 512 + 2 + 72 + 1) * sizeof(double2) + 3 * BL * sizeof(int);
  smem_optin((const void*)k_sweep<0>, 227 * 1024);
  smem_optin((const void*)k_sweep<1>, 227 * 1024);
  smem_optin((const void*)k_sweep<2>, 227 * 1024);
  const int nch = (T.N / 4 + kQuads - 1) / kQuads;
  const int per = occupancy((const void*)k_sweep<0>, kSweepThreads, sm);
  int G = num_sms() * per / nch;
  if (G < 1) G = 1;
  if (G > T.g_hi - T.g_lo) G = T.g_hi - T.g_lo;
  const int grid = nch * G;
  ++g_launches;
  if (dense == 2) launch_pdl(k_sweep<2>, grid, kSweepThreads, sm, s, T, cval, D, spec, zfirst, fsep);
  else if (dense == 1) launch_pdl(k_sweep<1>, grid, kSweepThreads, sm, s, T, cval, D, spec, zfirst, fsep);
  else launch_pdl(k_sweep<0>, grid, kSweepThreads, sm, s, T, cval, D, spec, zfirst, fsep);
}

void launch_reduced(const DevTables& T, const double* zfirst, const double* zlast, const double* fsep, double* hsep,
                    cudaStream_t s) {
  (void)zlast;
  if (T.P < 2) return;
  if (T.P >= 2 * BL2 && T.P % BL2 == 0 && T.P / BL2 <= kMaxSeg) {
    dim3 blk(kRed2Modes, T.P / BL2);
    { ++g_launches; launch_pdl(k_reduced2, dim3(cdiv(T.N - 1, kRed2Modes)), blk, 0, s, T, zfirst, fsep, hsep); }
  } else {
    { ++g_launches; k_reduced_small<<<cdiv(T.N - 1, 64), 64, 0, s>>>(T, zfirst, fsep, hsep); }
  }
}

void launch_inverse_sparse(const DevTables& T, const double* spec, const double* hsep, double* vsten,
                           cudaStream_t s) {
  const int ncols = T.o_hi - T.o_lo;
  if (ncols <= 0) return;
  const int quarter = T.N / 4;
  const int qpt = (quarter + kInvThreads - 1) / kInvThreads;
  const size_t red_b = (size_t)(kInvThreads / 32) * 2 * T.mcr * sizeof(double);
  const int grid = ncols < 2 * num_sms() ? ncols : 2 * num_sms();
  const size_t sm = (size_t)(T.N + T.N / 16 + 1) * sizeof(double) + red_b;
  ++g_launches;
  switch (qpt) {
    case 1: smem_optin((const void*)k_inv_sparse<1>, sm); launch_pdl(k_inv_sparse<1>, grid, kInvThreads, sm, s, T, spec, hsep, vsten); break;
    case 2: smem_optin((const void*)k_inv_sparse<2>, sm); launch_pdl(k_inv_sparse<2>, grid, kInvThreads, sm, s, T, spec, hsep, vsten); break;
    case 4: smem_optin((const void*)k_inv_sparse<4>, sm); launch_pdl(k_inv_sparse<4>, grid, kInvThreads, sm, s, T, spec, hsep, vsten); break;
    case 8: smem_optin((const void*)k_inv_sparse<8>, sm); launch_pdl(k_inv_sparse<8>, grid, kInvThreads, sm, s, T, spec, hsep, vsten); break;
    default: break;
  }
}

void launch_red2_local(const DevTables& T, const double* zB, const double* zA, double* hsep, double* segbuf,
                       cudaStream_t s) {
  dim3 grid(cdiv(T.N - 1, 128), T.seg_hi - T.seg_lo);
  ++g_launches;
  launch_pdl(k_red2_local, grid, dim3(128), 0, s, T, zB, zA, hsep, segbuf);
}
void launch_red2_solve(const DevTables& T, const double* segbuf, double* h2, cudaStream_t s) {
  ++g_launches;
  launch_pdl(k_red2_solve, dim3(cdiv(T.N - 1, 128)), dim3(128), 0, s, T, segbuf, h2);
}
void launch_red2_fixup(const DevTables& T, const double* h2, double* hsep, cudaStream_t s) {
  dim3 grid(cdiv(T.N - 1, 128), T.seg_hi - T.seg_lo);
  ++g_launches;
  launch_pdl(k_red2_fixup, grid, dim3(128), 0, s, T, h2, hsep);
}

namespace {
__global__ void k_sum_parts(int n, int nparts, const double* __restrict__ parts, double* __restrict__ out) {
  pdl_wait();
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < n; m += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < nparts; ++r) s += parts[(size_t)r * n + m];
    out[m] = s;
  }
}
}  // namespace
void launch_sum_parts(int n, int nparts, const double* parts, double* out, cudaStream_t s) {
  ++g_launches;
  launch_pdl(k_sum_parts, dim3(cdiv(n, 256)), dim3(256), 0, s, n, nparts, parts, out);
}

void launch_hole_coeffs(const DevTables& T, const int* hole_off, const int* hole_M, const double* hole_delta, int nh,
                        const double* phi, double* a, cudaStream_t s) {
  (void)T;
  if (nh == 0) return;
  { ++g_launches; launch_pdl(k_hole_coeffs, dim3(nh), dim3(256), 0, s, hole_off, hole_M, hole_delta, phi, a); }
}

void launch_interp(const DevTables& T, const double* phi, const double* mk, const double* fz, const double* jz_given,
                   const double* vsten, int nh, const double* wg, const double* a, double* out, cudaStream_t s,
                   bool partial) {
  { ++g_launches; launch_pdl(k_interp, dim3(cdiv(T.M, 128)), dim3(128), 0, s, T, phi, mk, fz, jz_given, vsten, wg ? nh : 0, wg, a, out, partial ? 1 : 0); }
}

void launch_mgs_step(int n, double* w, const double* Vprev, const double* Vcur, const double* partial_prev,
                     double* partial_cur, double* hout, cudaStream_t s) {
  { ++g_launches; launch_pdl(k_mgs_step, dim3(kRedBlocks), dim3(256), 0, s, n, w, Vprev, Vcur, partial_prev, partial_cur, hout); }
}

bool launch_mgs_fused(int n, int j, const double* V, double* w, double* hcol, cudaStream_t s) {
  const int per = (n + kMgsCl * kMgsClThreads - 1) / (kMgsCl * kMgsClThreads);   // elements per thread
  switch (per <= 1 ? 1 : per <= 2 ? 2 : per <= 4 ? 4 : per <= 8 ? 8 : 0) {
    case 1: ++g_launches; launch_pdl(k_mgs_cluster<1>, dim3(kMgsCl), dim3(kMgsClThreads), 0, s, n, j, V, w, hcol); return true;
    case 2: ++g_launches; launch_pdl(k_mgs_cluster<2>, dim3(kMgsCl), dim3(kMgsClThreads), 0, s, n, j, V, w, hcol); return true;
    case 4: ++g_launches; launch_pdl(k_mgs_cluster<4>, dim3(kMgsCl), dim3(kMgsClThreads), 0, s, n, j, V, w, hcol); return true;
    case 8: ++g_launches; launch_pdl(k_mgs_cluster<8>, dim3(kMgsCl), dim3(kMgsClThreads), 0, s, n, j, V, w, hcol); return true;
    default: return false;
  }
}

void launch_norm_scale(int n, double* w, const double* partial, double* hout, cudaStream_t s) {
  { ++g_launches; launch_pdl(k_norm_scale, dim3(kRedBlocks), dim3(256), 0, s, n, w, partial, hout); }
}

void launch_dot(int n, const double* a, const double* b, double* partial, cudaStream_t s) {
  { ++g_launches; launch_pdl(k_dot, dim3(kRedBlocks), dim3(256), 0, s, n, a, b, partial); }
}

void launch_finish_sum(const double* partial, double* out, bool take_sqrt, cudaStream_t s) {
  { ++g_launches; launch_pdl(k_finish_sum, dim3(1), dim3(32), 0, s, partial, out, take_sqrt ? 1 : 0); }
}

void launch_axpy_basis(int n, int k, const double* V, int ldv, const double* y_host, double* x, cudaStream_t s) {
  YCoef y{};
  for (int q = 0; q < k && q < kYMax; ++q) y.v[q] = y_host[q];   // by value: no copy engine
  { ++g_launches; launch_pdl(k_axpy_basis, dim3(cdiv(n, 256)), dim3(256), 0, s, n, k, V, ldv, y, x); }
}
void launch_copy(int n, const double* src, double* dst, cudaStream_t s) {
  if (n <= 0) return;
  const int grid = cdiv(n, 256) < 4 * num_sms() ? cdiv(n, 256) : 4 * num_sms();
  { ++g_launches; launch_pdl(k_copy, dim3(grid), dim3(256), 0, s, n, src, dst); }
}

void launch_sub(int n, const double* a, const double* b, double* out, cudaStream_t s) {
  { ++g_launches; launch_pdl(k_sub, dim3(cdiv(n, 256)), dim3(256), 0, s, n, a, b, out); }
}

void launch_scale_copy(int n, const double* a, const double* scal, double* out, cudaStream_t s) {
  { ++g_launches; launch_pdl(k_scale_copy, dim3(cdiv(n, 256)), dim3(256), 0, s, n, a, scal, out); }
}

template <int MODE, int N>
static void dense_n(const DevTables& T, const double* src, int mask, const BumpParams& bp, const double* hsep,
                    double* dst, cudaStream_t s) {
  using C = DenseCfg<N>;
  const size_t sm = C::smem(C::STAGE && MODE == 0);
  smem_optin((const void*)k_dst_dense2<MODE, N>, sm);
  const int rows = T.col_hi - T.col_lo + 1;
  const int per = occupancy((const void*)k_dst_dense2<MODE, N>, C::NTHR, sm);
  const int groups = (rows + C::RPC - 1) / C::RPC;
  const int grid = groups < per * num_sms() ? groups : per * num_sms();
  launch_pdl(k_dst_dense2<MODE, N>, dim3(grid), dim3(C::NTHR), sm, s, T, src, mask, bp, hsep, dst);
}
template <int MODE>
static void dense_dispatch(const DevTables& T, const double* src, int mask, const BumpParams& bp, const double* hsep,
                           double* dst, cudaStream_t s) {
  ++g_launches;
  switch (T.N) {
    case 64: dense_n<MODE, 64>(T, src, mask, bp, hsep, dst, s); break;
    case 128: dense_n<MODE, 128>(T, src, mask, bp, hsep, dst, s); break;
    case 256: dense_n<MODE, 256>(T, src, mask, bp, hsep, dst, s); break;
    case 512: dense_n<MODE, 512>(T, src, mask, bp, hsep, dst, s); break;
    case 1024: dense_n<MODE, 1024>(T, src, mask, bp, hsep, dst, s); break;
    case 2048: dense_n<MODE, 2048>(T, src, mask, bp, hsep, dst, s); break;
    case 4096: dense_n<MODE, 4096>(T, src, mask, bp, hsep, dst, s); break;
    default: dense_n<MODE, 8192>(T, src, mask, bp, hsep, dst, s); break;
  }
}
void launch_dst_forward(const DevTables& T, const double* fgrid, bool mask, const BumpParams& bp, double* spec,
                        cudaStream_t s, bool compact) {
  dense_dispatch<0>(T, fgrid, compact ? 2 : (mask ? 1 : 0), bp, nullptr, spec, s);
}

void launch_inverse_dense(const DevTables& T, const double* spec, const double* hsep, double* vgrid,
                          cudaStream_t s, bool compact) {
  BumpParams bp{};
  dense_dispatch<1>(T, spec, compact ? 2 : 0, bp, hsep, vgrid, s);
}

void launch_gs_reaction(double* u, double* v, long n, double dt, const GsParams& p, cudaStream_t s) {
  ++g_launches;
  k_gs_reaction<<<(int)std::min<long>((n + 255) / 256, 8L * num_sms()), 256, 0, s>>>(u, v, n, dt, p);
}
void launch_gs_rhs(const DevTables& T, const double* w, double* fg, double* fq, double* fz, cudaStream_t s) {
  const long n = (long)(T.N + 1) * (T.N + 1) + T.nq + T.M;
  ++g_launches;
  k_gs_rhs<<<(int)std::min<long>((n + 255) / 256, 8L * num_sms()), 256, 0, s>>>(T, w, fg, fq, fz);
}
void launch_gs_combine(double* w, const double* y, long n, cudaStream_t s) {
  ++g_launches;
  k_gs_combine<<<(int)std::min<long>((n + 255) / 256, 8L * num_sms()), 256, 0, s>>>(w, y, n);
}
// one warp per 32-node segment of a grid row (no block synchronisation): rank of an Ω node = the
// segment's offset (setup) + the Ω lanes below it in the segment's ballot
template <bool SCATTER>
__global__ void __launch_bounds__(256) k_omega_map(long rows, long width, const int8_t* __restrict__ side,
                                                   const int32_t* __restrict__ om_seg,
                                                   const double* __restrict__ src, double* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const long nseg = (width + 31) / 32, nw = rows * nseg;
  for (long w = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nw; w += ((long)gridDim.x * blockDim.x) >> 5) {
    const long r = w / nseg, j = (w - r * nseg) * 32 + lane;
    const long p = r * width + j;
    const bool live = j < width;
    const bool in = live && side[p] != 0;
    const unsigned bal = __ballot_sync(0xffffffffu, in);
    const long q = (long)om_seg[w] + __popc(bal & lt);
    if (SCATTER) {
      if (live) dst[p] = in ? src[q] : 0.0;
    } else if (in) {
      dst[q] = src[p];
    }
  }
}

void launch_omega_map(long rows, long width, const int8_t* side, const int32_t* om_seg, const double* src,
                      double* dst, bool scatter, cudaStream_t s) {
  if (rows <= 0) return;
  const long warps = rows * ((width + 31) / 32);
  const int grid = (int)std::min<long>((warps + 7) / 8, 16L * num_sms());
  ++g_launches;
  if (scatter) k_omega_map<true><<<grid, 256, 0, s>>>(rows, width, side, om_seg, src, dst);
  else k_omega_map<false><<<grid, 256, 0, s>>>(rows, width, side, om_seg, src, dst);
}

void launch_fill(double* x, long n, double val, cudaStream_t s) {
  if (n <= 0) return;
  ++g_launches;
  k_fill<<<(int)std::min<long>((n + 255) / 256, 8L * num_sms()), 256, 0, s>>>(x, n, val);
}

__global__ void k_axpy_dcoef(long n, const double* __restrict__ coef, const double* __restrict__ x,
                             double* __restrict__ y) {
  pdl_wait();
  const double a = *coef;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    y[i] = fma(a, __ldcs(x + i), y[i]);
}
void launch_axpy_dcoef(long n, const double* coef, const double* x, double* y, cudaStream_t s) {
  if (n <= 0) return;
  ++g_launches;
  launch_pdl(k_axpy_dcoef, dim3((int)std::min<long>((n + 255) / 256, 8L * num_sms())), dim3(256), 0, s, n, coef, x, y);
}
}  // namespace kfbi

