// Device helpers shared by the 2D and 3D kernels: sine/twiddle tables, complex products, deterministic
// block/warp reductions, register DFTs and the shared-memory Stockham FFT with the two DST-I cores
// (half-length for 3D rows, N-point odd extension for 2D rows).  Included by kernels2d.cu and
// kernels3d.cu inside namespace kfbi (anonymous: one copy per translation unit).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <utility>

#include "kernels.h"

// Bounds checks of the hot kernels' computed indices (compute-sanitizer is closed on this GPU pool):
// built with -DKFBI_BOUNDS (KFBI_NVCC_EXTRA=-DKFBI_BOUNDS python -m paper_2404_15249_b200.build --force),
// a violated check prints the kernel, line and values and traps; compiled out otherwise.
#ifdef KFBI_BOUNDS
#include <cstdio>
#define KFBI_CHECK(cond, a, b)                                                                            \
  do {                                                                                                     \
    if (!(cond)) {                                                                                         \
      printf("KFBI_CHECK failed %s:%d (%s): %lld %lld block %d thread %d\n", __FILE__, __LINE__, #cond,  \
             (long long)(a), (long long)(b), (int)blockIdx.x, (int)threadIdx.x);                           \
      __trap();                                                                                            \
    }                                                                                                      \
  } while (0)
#else
#define KFBI_CHECK(cond, a, b) \
  do {                         \
  } while (0)
#endif

namespace kfbi {
namespace {

__device__ __forceinline__ double sin_lookup(const double* __restrict__ tab, int r, int N) {
  // sin(π r / N) for r ∈ [0, 2N) from the quarter table sin(π r / N), r ∈ [0, N/2]
  double sg = 1.0;
  if (r >= N) { r -= N; sg = -1.0; }
  if (r > (N >> 1)) r = N - r;
  return sg * tab[r];
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// e^{iπ r/N} = th[r >> 6] · tl[r & 63] from two small shared tables (2N/64 and 64 entries)
__device__ __forceinline__ double2 eipi(const double2* th, const double2* tl, int r) {
  return cmul(th[r >> 6], tl[r & 63]);
}
// the same two tables with one 16-byte pad slot after every 8 entries (th: 2N/64 + 2N/512 + 1 slots,
// tl: 72): lanes whose indices agree mod 8 (even multipliers j) then fall in different bank groups
__device__ __forceinline__ int eipi_pad(int y) { return y + (y >> 3); }
__device__ __forceinline__ double2 eipi_p(const double2* th, const double2* tl, int r) {
  return cmul(th[eipi_pad(r >> 6)], tl[eipi_pad(r & 63)]);
}
__device__ __forceinline__ void build_eipi_p(const double* __restrict__ sin_tab, int N, double2* th, double2* tl) {
  const int m2 = 2 * N - 1;
  for (int k = threadIdx.x; k < 2 * N / 64; k += blockDim.x) {
    const int r = 64 * k;
    th[eipi_pad(k)] = make_double2(sin_lookup(sin_tab, (r + N / 2) & m2, N), sin_lookup(sin_tab, r & m2, N));
  }
  for (int l = threadIdx.x; l < 64; l += blockDim.x)
    tl[eipi_pad(l)] = make_double2(sin_lookup(sin_tab, (l + N / 2) & m2, N), sin_lookup(sin_tab, l & m2, N));
}
__device__ __forceinline__ void build_eipi(const double* __restrict__ sin_tab, int N, double2* th, double2* tl) {
  const int m2 = 2 * N - 1;
  for (int k = threadIdx.x; k < 2 * N / 64; k += blockDim.x) {
    const int r = 64 * k;
    th[k] = make_double2(sin_lookup(sin_tab, (r + N / 2) & m2, N), sin_lookup(sin_tab, r & m2, N));
  }
  for (int l = threadIdx.x; l < 64; l += blockDim.x)
    tl[l] = make_double2(sin_lookup(sin_tab, (l + N / 2) & m2, N), sin_lookup(sin_tab, l & m2, N));
}


template <int NV>
__device__ __forceinline__ void block_reduce(double (&v)[NV], double* scratch) {
  // deterministic: warp shuffle tree, then warp 0 sums the per-warp partials in order
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) scratch[wid * NV + q] = v[q];
  __syncthreads();
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = 0;
      for (int w = 0; w < nw; ++w) s += scratch[w * NV + q];
      v[q] = s;
    }
}


// Sum v[0..7] over the 32 lanes of a warp by a transpose-reduce (16 doubles exchanged instead
// of 80): on return lane l holds the warp total of value (l & 7).
__device__ __forceinline__ double warp_transpose_reduce8(double (&v)[8]) {
  const int lane = threadIdx.x & 31;
  // level 16: keep 4 of 8
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const bool up = lane & 16;
    const double send = up ? v[q] : v[q + 4];
    const double keep = up ? v[q + 4] : v[q];
    v[q] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  // level 8: keep 2 of 4
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const bool up = lane & 8;
    const double send = up ? v[q] : v[q + 2];
    const double keep = up ? v[q + 2] : v[q];
    v[q] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  {
    const bool up = lane & 4;
    const double send = up ? v[0] : v[1];
    const double keep = up ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  // lane l now holds value index ((l>>4)&1)*4 + ((l>>3)&1)*2 + ((l>>2)&1)
  return v[0];
}


// ------------------------------------------------------------------------------ FFT building blocks
// (register DFTs, padded shared-memory slots; the DST-I cores are with the 2D/3D row kernels below)

// e^{+2πi m/16}
__device__ __forceinline__ double w16c(int m) {
  switch (m & 15) {
    case 0: return 1.0;
    case 1: return 0.92387953251128675613;
    case 2: return 0.70710678118654752440;
    case 3: return 0.38268343236508977173;
    case 4: return 0.0;
    case 5: return -0.38268343236508977173;
    case 6: return -0.70710678118654752440;
    case 7: return -0.92387953251128675613;
    case 8: return -1.0;
    case 9: return -0.92387953251128675613;
    case 10: return -0.70710678118654752440;
    case 11: return -0.38268343236508977173;
    case 12: return 0.0;
    case 13: return 0.38268343236508977173;
    case 14: return 0.70710678118654752440;
    default: return 0.92387953251128675613;
  }
}
__device__ __forceinline__ double w16s(int m) { return w16c(m - 4); }

// R-point DFT in registers, sign +:  V_q = Σ_r v_r e^{+2πi rq/R}  (radix-2 DIT, constant twiddles)
template <int R>
__device__ __forceinline__ void dft_reg(double2* v) {
  constexpr int LG = R == 2 ? 1 : R == 4 ? 2 : R == 8 ? 3 : 4;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    int r = 0;
#pragma unroll
    for (int b = 0; b < LG; ++b) r |= ((i >> b) & 1) << (LG - 1 - b);
    if (r > i) {
      const double2 t = v[i];
      v[i] = v[r];
      v[r] = t;
    }
  }
#pragma unroll
  for (int len = 1; len < R; len <<= 1)
#pragma unroll
    for (int i = 0; i < R; i += 2 * len)
#pragma unroll
      for (int jj = 0; jj < len; ++jj) {
        const int m = jj * (8 / len);   // e^{iπ jj/len} = W16^{8 jj/len}; m ∈ [0, 8)
        const double2 u = v[i + jj], t = v[i + jj + len];
        double tr, ti;
        if (m == 0) {            // trivial twiddles folded at compile time
          tr = t.x;
          ti = t.y;
        } else if (m == 4) {     // ·i
          tr = -t.y;
          ti = t.x;
        } else if (m == 2) {     // ·(1+i)/√2
          tr = 0.70710678118654752440 * (t.x - t.y);
          ti = 0.70710678118654752440 * (t.x + t.y);
        } else if (m == 6) {     // ·(−1+i)/√2
          tr = -0.70710678118654752440 * (t.x + t.y);
          ti = 0.70710678118654752440 * (t.x - t.y);
        } else {
          const double c = w16c(m), sn = w16s(m);
          tr = c * t.x - sn * t.y;
          ti = c * t.y + sn * t.x;
        }
        v[i + jj] = make_double2(u.x + tr, u.y + ti);
        v[i + jj + len] = make_double2(u.x - tr, u.y - ti);
      }
}

// complex slot i of the FFT buffer lives at i + i/16 (breaks the stride-R conflicts of the
// first Stockham pass's writes)
__device__ __forceinline__ int zpad(int i) { return i + (i >> 4); }


// cos(2πm/32), sin(2πm/32) (folded at compile time for constant m)
__device__ __forceinline__ double c32q(int m) {
  switch (m) {
    case 0: return 1.0;
    case 1: return 0.98078528040323043058;
    case 2: return 0.92387953251128673848;
    case 3: return 0.83146961230254523567;
    case 4: return 0.70710678118654757274;
    case 5: return 0.55557023301960228867;
    case 6: return 0.38268343236508983729;
    case 7: return 0.19509032201612833135;
    default: return 0.0;
  }
}
__device__ __forceinline__ double w32c(int m) {
  m &= 31;
  return m <= 8 ? c32q(m) : m <= 16 ? -c32q(16 - m) : m <= 24 ? -c32q(m - 16) : c32q(32 - m);
}
__device__ __forceinline__ double w32s(int m) { return w32c(m - 8); }

// the lanes of one row synchronise: within a warp (N ≤ 1024) or across the CTA (row = CTA)
// BAR > 0: a thread team of NTL threads (a multiple of 32) synchronises on named barrier BAR
template <int NTL, int BAR = 0>
__device__ __forceinline__ void rsync() {
  if constexpr (BAR > 0) asm volatile("bar.sync %0, %1;" ::"r"(BAR), "r"(NTL) : "memory");
  else if constexpr (NTL > 32) __syncthreads();
  else __syncwarp();
}

// Compile-time Stockham radix-R pass over one row z[0..M) held by M/16 lanes of one warp (rows never
// straddle warps, so __syncwarp orders the in-place smem exchange).  Twiddles e^{+2πi r k/(Ns R)} =
// tw[r k 2NT/(Ns R) mod 2NT] from the (cos, sin)(π m/NT) table of the grid size NT (L1-resident).
template <int R, int M, int Ns, int NT, int BAR = 0>
__device__ __forceinline__ void st_pass(double2* z, const double2* __restrict__ tw, int tid) {
  constexpr int NTH = M / 16, NI = M / R, IT = NI / NTH;
  double2 v[IT * R];
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int j = tid + it * NTH;
#pragma unroll
    for (int r = 0; r < R; ++r) v[it * R + r] = z[zpad(j + r * NI)];
    if (Ns > 1) {   // w^r, r < R, from one lookup by products of depth ≤ 4 (w, w², w⁴, w⁸)
      const int k = j & (Ns - 1);
      double2 wp[R];
      wp[1] = __ldg(tw + ((k * (2 * NT / (Ns * R))) & (2 * NT - 1)));
#pragma unroll
      for (int r = 2; r < R; ++r) {
        const int hi = (r & (r - 1)) ? (1 << (31 - __clz(r))) : r / 2;   // highest power of two < r, or r/2
        wp[r] = cmul(wp[hi], wp[r - hi]);
      }
#pragma unroll
      for (int r = 1; r < R; ++r) v[it * R + r] = cmul(v[it * R + r], wp[r]);
    }
    dft_reg<R>(v + it * R);
  }
  rsync<NTH, BAR>();
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int j = tid + it * NTH;
    const int base = (j / Ns) * Ns * R + (j & (Ns - 1));
#pragma unroll
    for (int q = 0; q < R; ++q) z[zpad(base + q * Ns)] = v[it * R + q];
  }
  rsync<NTH, BAR>();
}

template <int M, int Ns, int NT, int BAR = 0>
__device__ __forceinline__ void st_fft(double2* z, const double2* __restrict__ tw, int tid) {
  if constexpr (Ns * 16 <= M) {
    st_pass<16, M, Ns, NT, BAR>(z, tw, tid);
    st_fft<M, Ns * 16, NT, BAR>(z, tw, tid);
  } else if constexpr (M / Ns == 8) {
    st_pass<8, M, Ns, NT, BAR>(z, tw, tid);
  } else if constexpr (M / Ns == 4) {
    st_pass<4, M, Ns, NT, BAR>(z, tw, tid);
  } else if constexpr (M / Ns == 2) {
    st_pass<2, M, Ns, NT, BAR>(z, tw, tid);
  }
}

// position of F_j in the padded output buffer (2 doubles of pad per 32: conflict-free pair stores)
__device__ __forceinline__ int fpos(int j) { return j + 2 * (j >> 5); }

// DST-I of one row, F_k = Σ_{j=1}^{N−1} f_j sin(πjk/N), by an M = N/2 point complex FFT on N/32 lanes
// of a warp (tid ∈ [0, N/32)).  On entry z[zpad(m)] = (f_2m, f_2m+1), m ∈ [0, M), f_0 = 0.
//   y_j = sin(πj/N)(f_j + f_{N−j}) + (f_j − f_{N−j})/2  (y_0 = 0),   Y_k = Σ_j y_j e^{2πijk/N}
//   ⇒ F_2k = Im Y_k,  F_2k+1 − F_2k−1 = Re Y_k  (F_−1 = −F_1): the odd outputs are the prefix sums
//   of Re Y, taken per lane (16 terms) and across the row's lanes by a log-depth shuffle scan.
// On exit F_j sits at ((double*)z)[fpos(j)], j ∈ [0, N).
// wa, wb = e^{iπ(2 tid)/N}, e^{iπ(2 tid+1)/N} (callers may load them before their last barrier)
template <int N>
__device__ __forceinline__ void dst2_core_w(double2* z, const double2* __restrict__ tw, int tid, double2 wa, double2 wb,
                                            double* scratch = nullptr) {   // scratch: N/1024 + 1 doubles if N > 1024
  constexpr int M = N / 2, NTL = N / 32;
  double2 v[16];
#pragma unroll
  for (int s = 0; s < 16; ++s) {   // item tid of the first radix-16 pass holds m = tid + NTL·s
    const int m = tid + NTL * s;
    const double2 P = z[zpad(m)];
    const double fa = m ? z[zpad(M - m)].x : 0.0;   // f_{N−2m}
    const double fb = z[zpad(M - m - 1)].y;         // f_{N−2m−1}
    // sin(π j/N) at j = 2m, 2m+1: angle of the lane + s·π/16 (constants)
    const double sa = fma(wa.y, w32c(s), wa.x * w32s(s)), sb = fma(wb.y, w32c(s), wb.x * w32s(s));
    v[s] = make_double2(fma(sa, P.x + fa, 0.5 * (P.x - fa)), fma(sb, P.y + fb, 0.5 * (P.y - fb)));
  }
  dft_reg<16>(v);
  rsync<NTL>();
#pragma unroll
  for (int q = 0; q < 16; ++q) z[zpad(16 * tid + q)] = v[q];
  rsync<NTL>();
  st_fft<M, 16, N>(z, tw, tid);
  // Y_k = (Z_k + conj Z_{M−k})/2 − (i/2) e^{2πik/N} (Z_k − conj Z_{M−k}), k = 16·tid + t
  double R[16], I[16];
  const double2 wk0 = __ldg(tw + 32 * tid);   // e^{2πi(16 tid)/N}
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const int k = 16 * tid + t;
    const double2 A = z[zpad(k)], B = z[zpad((M - k) & (M - 1))];
    const double ex = 0.5 * (A.x + B.x), ey = 0.5 * (A.y - B.y);
    const double dx = A.x - B.x, dy = A.y + B.y;
    const double2 w = t ? cmul(wk0, __ldg(tw + 2 * t)) : wk0;   // second factor warp-uniform
    R[t] = fma(0.5, fma(w.x, dy, w.y * dx), ex);
    I[t] = fma(0.5, fma(w.y, dy, -w.x * dx), ey);
  }
  // inclusive prefix within the lane by a log-depth (Kogge-Stone) scan: rounding depth 4, not 16
#pragma unroll
  for (int d = 1; d < 16; d <<= 1)
#pragma unroll
    for (int t = 15; t >= d; --t) R[t] += R[t - d];
  const double run = R[15];
  double x = run, r0;
  if constexpr (NTL <= 32) {
#pragma unroll
    for (int d = 1; d < NTL; d <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, x, d, NTL);
      if (tid >= d) x += y;
    }
    r0 = __shfl_sync(0xffffffffu, R[0], 0, NTL);   // lane 0's R[0] = Re Y_0
  } else {   // row = CTA: warp scans, then the preceding warps' totals in a fixed order
    const int lane = tid & 31, wq = tid >> 5;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) scratch[wq] = x;
    if (tid == 0) scratch[NTL / 32] = R[0];
    __syncthreads();
    double off = 0.0;
    for (int w = 0; w < wq; ++w) off += scratch[w];
    x += off;
    r0 = scratch[NTL / 32];
  }
  const double base = (x - run) - 0.5 * r0;
  rsync<NTL>();
  double* F = reinterpret_cast<double*>(z);
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const int k = 16 * tid + t;
    *reinterpret_cast<double2*>(F + fpos(2 * k)) = make_double2(k ? I[t] : 0.0, base + R[t]);
  }
  rsync<NTL>();
}



template <int N>
__device__ __forceinline__ void dst2_core(double2* z, const double2* __restrict__ tw, int tid,
                                          double* scratch = nullptr) {
  dst2_core_w<N>(z, tw, tid, __ldg(tw + 2 * tid), __ldg(tw + 2 * tid + 1), scratch);
}

// accurate DST-I (2D rows, N up to 8192): the real DFT of the odd extension x (x_t = f_t, x_N = 0,
// x_{2N−t} = −f_t) by one N-point complex FFT of z_m = x_2m + i x_2m+1; F_k = Im(E_k + e^{iπk/N} O_k)/2.
// Every output carries O(ε log N) rounding (the half-length core's prefix sum grows as √N ε, which
// the 2D backward-error pin at N ≥ 2048 rejects).  N/16 lanes per row, 8 pairs fp[s] per lane
// (m = tid + s·N/16); on exit F_k sits in z[zpad(k)].x, k ∈ [1, N).
template <int N>
__device__ __forceinline__ void dst1_core(double2* z, const double2* __restrict__ tw, int tid, const double2* fp) {
  constexpr int NTH = N / 16;
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int m = tid + s * NTH;
    z[zpad(m)] = fp[s];
    if (m > 0) z[zpad(N - m)].x = -fp[s].x;
    else z[zpad(N / 2)].x = 0.0;
    z[zpad(N - m - 1)].y = -fp[s].y;
  }
  rsync<NTH>();
  st_fft<N, 1, N>(z, tw, tid);
  const double2 wb = __ldg(tw + 1 + tid);   // e^{iπ(1+tid)/N}; k = 1 + tid + s·N/16 adds s·π/16
  double Fk[8], Fk2[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int k = 1 + tid + s * NTH;
    const double2 A = z[zpad(k)], B = z[zpad(N - k)];
    const double2 w = make_double2(fma(wb.x, w32c(s), -wb.y * w32s(s)), fma(wb.y, w32c(s), wb.x * w32s(s)));
    Fk[s] = 0.5 * (0.5 * (A.y - B.y) - w.x * (0.5 * (A.x - B.x)) + w.y * (0.5 * (A.y + B.y)));
    Fk2[s] = 0.5 * (0.5 * (B.y - A.y) + w.x * (0.5 * (B.x - A.x)) + w.y * (0.5 * (B.y + A.y)));
  }
  rsync<NTH>();
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int k = 1 + tid + s * NTH;
    z[zpad(k)].x = Fk[s];
    if (k != N - k) z[zpad(N - k)].x = Fk2[s];
  }
  rsync<NTH>();
}


// Split-radix DST-I for one row of N ≥ 2048 on N/16 threads (the CTA), half the FFT points of
// dst1_core at the same O(ε log N) accuracy (no prefix sums): with f_j, j ∈ [0, N), f_0 = 0, M = N/2,
//   F_k = E'_k + G_k,  F_{N−k} = G_k − E'_k  (k ∈ [1, M)),  F_M = G_M,
//   E' = DST-I_M(e), e_m = f_2m  — dst1_core's odd-extension method on an M-point complex FFT;
//   G_k = Σ_m f_{2m+1} sin(π(2m+1)k/N) = C_{M−k},  C = DCT-II_M(u), u_m = (−1)^m f_{2m+1}  (sin(π(2m+1)k/N)
//     = (−1)^m cos(π(2m+1)(M−k)/N)); DCT-II by Makhoul: v_n = u_2n, v_{M−1−n} = u_{2n+1},
//     C_l = Re(e^{iπl/N} V_l), V = FFT⁺_M(v) from one M/2-point complex FFT of w_q = v_2q + i v_2q+1.
// Team E (threads [0, N/32)) runs the M-point FFT on named barrier 1 while team G (the next N/64) runs
// the M/2-point FFT on barrier 2; F_k ends in z[zpad(k)].x as with dst1_core.  Input as dst1_core:
// fp[s] = (f_2m, f_2m+1), m = tid + s·N/16.
template <int N>
__device__ __forceinline__ void dst1s_core(double2* z, const double2* __restrict__ tw, int tid, const double2* fp) {
  constexpr int NTH = N / 16, M = N / 2, TE = N / 32, TG = N / 64, H = M / 2;
  static_assert(TG % 32 == 0, "dst1s_core needs N >= 2048 (warp-aligned teams)");
  double2* zE = z;                                  // M complex slots (padded): the odd extension of e
  double2* zG = z + (M + M / 16 + 2);               // H complex slots (padded): w
  double* zGd = reinterpret_cast<double*>(zG);      // C_l after the G team's post-processing
  // scatter the row into the two teams' buffers
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int m = tid + s * NTH;
    // f_{2m}: e index 2m' (m even) or 2m'+1 (m odd), m' = m/2
    const int mp = m >> 1;
    if ((m & 1) == 0) {
      const double v = m ? fp[s].x : 0.0;
      zE[zpad(mp)].x = v;
      if (mp > 0) zE[zpad(M - mp)].x = -v;
      else zE[zpad(M / 2)].x = 0.0;
    } else {
      zE[zpad(mp)].y = fp[s].x;
      zE[zpad(M - mp - 1)].y = -fp[s].x;
    }
    // f_{2m+1} = o_m: u_m = (−1)^m o_m at v index m/2 (m even) or M − 1 − (m − 1)/2 (m odd, u = −o_m)
    const int nv = (m & 1) ? M - 1 - (m >> 1) : (m >> 1);
    const double u = (m & 1) ? -fp[s].y : fp[s].y;
    if (nv & 1) zG[zpad(nv >> 1)].y = u;
    else zG[zpad(nv >> 1)].x = u;
  }
  __syncthreads();
  if (tid < TE) {   // team E: E'_k, k ∈ [1, M), into zE[zpad(k)].x (dst1_core's post-processing at size M)
    const int te = tid;
    st_fft<M, 1, N, 1>(zE, tw, te);
    const double2 wb = __ldg(tw + 2 * (1 + te));   // e^{iπ(1+te)/M}; k = 1 + te + s·M/16 adds s·π/16
    double Fk[8], Fk2[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int k = 1 + te + s * TE;
      const double2 A = zE[zpad(k)], B = zE[zpad(M - k)];
      const double2 w = make_double2(fma(wb.x, w32c(s), -wb.y * w32s(s)), fma(wb.y, w32c(s), wb.x * w32s(s)));
      Fk[s] = 0.5 * (0.5 * (A.y - B.y) - w.x * (0.5 * (A.x - B.x)) + w.y * (0.5 * (A.y + B.y)));
      Fk2[s] = 0.5 * (0.5 * (B.y - A.y) + w.x * (0.5 * (B.x - A.x)) + w.y * (0.5 * (B.y + A.y)));
    }
    rsync<TE, 1>();
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int k = 1 + te + s * TE;
      zE[zpad(k)].x = Fk[s];
      if (k != M - k) zE[zpad(M - k)].x = Fk2[s];
    }
  } else if (tid < TE + TG) {   // team G: C_l, l ∈ [0, M), into zGd[l]
    const int tg = tid - TE;
    st_fft<H, 1, N, 2>(zG, tw, tg);
    // V_l = A_l + e^{2πil/M} B_l, A = (W_l + conj W_{−l})/2, B = (W_l − conj W_{−l})/(2i); l and
    // l + H share A_l, B_l (W has period H, the twiddle changes sign): C_l = Re(e^{iπl/N} V_l)
    constexpr int PER = H / TG;   // l ∈ [0, H) per thread: l = tg + r·TG
    double c0[PER], c1[PER];
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const int l = tg + r * TG;
      const double2 Wl = zG[zpad(l)], Wm = zG[zpad((H - l) & (H - 1))];
      const double Ax = 0.5 * (Wl.x + Wm.x), Ay = 0.5 * (Wl.y - Wm.y);   // A_l
      const double Bx = 0.5 * (Wl.y + Wm.y), By = -0.5 * (Wl.x - Wm.x);  // B_l = (W_l − conj W_{−l})/(2i)
      const double2 t = __ldg(tw + ((4 * l) & (2 * N - 1)));            // e^{2πil/M} = e^{iπ·4l/N}
      const double tBx = t.x * Bx - t.y * By, tBy = t.x * By + t.y * Bx;
      const double2 e1 = __ldg(tw + l), e2 = __ldg(tw + l + H);           // e^{iπl/N}, e^{iπ(l+H)/N}
      // V_l = A + tB, V_{l+H} = A − tB
      c0[r] = e1.x * (Ax + tBx) - e1.y * (Ay + tBy);
      c1[r] = e2.x * (Ax - tBx) - e2.y * (Ay - tBy);
    }
    rsync<TG, 2>();
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const int l = tg + r * TG;
      zGd[l] = c0[r];
      zGd[l + H] = c1[r];
    }
  }
  __syncthreads();
  // combine: k = 1 + tid + s·NTH covers [1, M]
  double Fa[8], Fb[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int k = 1 + tid + s * NTH;
    const double e = k < M ? zE[zpad(k)].x : 0.0, g = zGd[M - k];
    Fa[s] = e + g;
    Fb[s] = g - e;
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int k = 1 + tid + s * NTH;
    z[zpad(k)].x = Fa[s];
    if (k < M) z[zpad(N - k)].x = Fb[s];
  }
  __syncthreads();
}


// programmatic dependent launch: a kernel launched by launch_pdl() runs its prologue (shared tables from
// setup constants) while its predecessor drains, then waits here for the predecessor's results (a no-op
// when launched normally).  Nothing before the wait may write memory the predecessor touches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// launch with programmatic stream serialization (PDL): the kernel may start while its predecessor's
// last CTAs finish; it calls pdl_wait() before touching the predecessor's results
template <class... KArgs, class... Args>
void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  static const bool on = [] {   // KFBI_PDL=0: plain serialised launches (A/B runs)
    const char* e = std::getenv("KFBI_PDL");
    return !(e != nullptr && e[0] == '0');
  }();
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = on ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
  if (e != cudaSuccess) throw DeviceError(std::string("kernel launch: ") + cudaGetErrorString(e));
}

// Host-side launch caches, kept per device: the shared-memory opt-in of a kernel, its occupancy and
// the SM count belong to one device, and one process may drive contexts on several GPUs.
inline int cur_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

inline int num_sms() {
  static std::mutex mu;
  static std::map<int, int> n;
  const int dev = cur_device();
  std::lock_guard<std::mutex> g(mu);
  int& v = n[dev];
  if (v <= 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
  }
  return v;
}

// raise a kernel's dynamic shared-memory limit on the current device to at least `bytes`
inline void smem_optin(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  const int dev = cur_device();
  std::lock_guard<std::mutex> g(mu);
  size_t& v = done[{dev, fn}];
  if (v < bytes) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    v = bytes;
  }
}

// resident CTAs per SM of `fn` at (threads, dynamic smem) on the current device (≥ 1)
inline int occupancy(const void* fn, int threads, size_t sm) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, int, size_t>, int> done;
  const auto key = std::make_tuple(cur_device(), fn, threads, sm);
  std::lock_guard<std::mutex> g(mu);
  auto it = done.find(key);
  if (it != done.end()) return it->second;
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, sm);
  if (per < 1) per = 1;
  done[key] = per;
  return per;
}

}  // namespace
}  // namespace kfbi
