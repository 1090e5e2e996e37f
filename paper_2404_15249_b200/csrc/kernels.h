// Host-callable launchers of the sm_100a kernels (kernels2d.cu).
#pragma once
#include <cuda_runtime.h>

#include "kfbi_impl.h"

namespace kfbi {

// A1: periodic cubic-spline second-derivative knots of φ (M threads).
// spline knots of φ; with nh > 0 also the hole-completion coefficients a_h (R27) in extra blocks
void launch_spline(const DevTables& T, const double* phi, double* mk, cudaStream_t s, const int* hole_off = nullptr,
                   const int* hole_M = nullptr, const double* hole_delta = nullptr, int nh = 0,
                   double* ahole = nullptr);
// A2+A3: jumps at intersections + correction at irregular nodes (one thread per node).
//   phi/mk may be NULL (Φ ≡ 0); fq = [F] at intersections or NULL; jq_given (nq×6) replaces
//   the jump computation (test path).  Output cval[n] = h² × (correction of f̃ at node n).
void launch_correct(const DevTables& T, const double* phi, const double* mk, const double* fq,
                    const double* jq_given, double* cval, cudaStream_t s);
// A4 (dense input only): forward DST-I of rows i = 1..N−1 of a full-grid base
//   f̃ = mask·f (+ Σ_h a_h b_h), written to spec[(i−1)·N + k].
struct GsParams {   // Gray–Scott: feed γ, removal κ_r, ε₀
  double gamma, kr, eps0;
};
void launch_gs_reaction(double* u, double* v, long n, double dt, const GsParams& p, cudaStream_t s);
void launch_gs_rhs(const DevTables& T, const double* w, double* fg, double* fq, double* fz, cudaStream_t s);
void launch_gs_combine(double* w, const double* y, long n, cudaStream_t s);
void launch_fill(double* x, long n, double val, cudaStream_t s);
// y += (*coef) · x over n elements (coef on the device)
void launch_axpy_dcoef(long n, const double* coef, const double* x, double* y, cudaStream_t s);
// Ω-compact ↔ full grid (rows × width nodes, row-major; om_seg = Ω nodes before each 32-node
// segment of each row): scatter: grid[p] = compact[rank of p] on Ω nodes, 0 elsewhere;
// gather: compact[rank of p] = grid[p]
void launch_omega_map(long rows, long width, const int8_t* side, const int32_t* om_seg, const double* src,
                      double* dst, bool scatter, cudaStream_t s);


struct BumpParams {
  int nh;
  double cx[4], cy[4], rad[4];
  const double* a;   // device, nh coefficients
};
// compact: fgrid holds f at the Ω nodes only (row-major ranks, kfbi_omega_count values; mask implied)
void launch_dst_forward(const DevTables& T, const double* fgrid, bool mask, const BumpParams& bp,
                        double* spec, cudaStream_t s, bool compact = false);
// dense spectral source of a sweep: f̂ = base + Σ_{h<nb} coef[h] · bump[h·ldb] (any of them may be
// absent; base may alias the sweep's output). The final field's linear combination (R27) is formed
// as it is read instead of in a separate pass over the grid.
struct DenseSrc {
  const double* base = nullptr;
  int nb = 0;
  const double* bump = nullptr;
  long ldb = 0;
  const double* coef = nullptr;   // device, nb entries
  bool stencil_only = false;      // the sweep stores only the spectral rows of stencil columns (sparse inverse follows)
  int blo[4] = {0, 0, 0, 0}, bhi[4] = {-1, -1, -1, -1};   // grid columns i where bump h can be non-zero
  bool any() const { return base || nb > 0; }
};
// A4+A5 fused: per (mode pair, block) local solve with the sparse-correction DST computed
// on the fly, plus the dense f̂ of `D` when present.
void launch_sweep(const DevTables& T, const double* cval, const DenseSrc& D, double* spec, double* zfirst,
                  double* zlast, double* fsep, cudaStream_t s);
// A5 reduced (arrowhead) system per mode: separator values h_g.
void launch_reduced(const DevTables& T, const double* zfirst, const double* zlast, const double* fsep,
                    double* hsep, cudaStream_t s);
// A6 sparse: inverse DST-I at the stencil rows only (spike fix-up fused into the load).
void launch_inverse_sparse(const DevTables& T, const double* spec, const double* hsep, double* vsten,
                           cudaStream_t s);
// A6 dense: inverse DST-I of every row into a full (N+1)^2 grid (fix-up fused).
// compact: vgrid receives the field at the Ω nodes only (row-major ranks)
void launch_inverse_dense(const DevTables& T, const double* spec, const double* hsep, double* vgrid,
                          cudaStream_t s, bool compact = false);
// hole coefficients a_h = Δ_h Σ_{m∈Γ_h} φ_m (reading R27), one block per hole
void launch_hole_coeffs(const DevTables& T, const int* hole_off, const int* hole_M, const double* hole_delta,
                        int nh, const double* phi, double* a, cudaStream_t s);
// A7: interpolation at control points.  phi/mk NULL → Φ ≡ 0; fz = [F] at control points or
//   NULL; jz_given (M×6) test path; wg (nh×M) + a (nh) hole completion or NULL.
void launch_interp(const DevTables& T, const double* phi, const double* mk, const double* fz,
                   const double* jz_given, const double* vsten, int nh, const double* wg, const double* a,
                   double* out, cudaStream_t s, bool partial = false);
// multi-GPU split of the level-2 reduced solve (segments = slabs): local segment solves for the
// owned segments [seg_lo, seg_hi) → seg buffer [seg][4][N] (first, last, zA of the segment's boundary
// separator, zB of its first block); level-2 solve
// for all segments (after the all-gather) → h2 [seg][N]; fix-up of the owned segments' separators
void launch_red2_local(const DevTables& T, const double* zB, const double* zA, double* hsep, double* segbuf,
                       cudaStream_t s);
void launch_red2_solve(const DevTables& T, const double* segbuf, double* h2, cudaStream_t s);
void launch_red2_fixup(const DevTables& T, const double* h2, double* hsep, cudaStream_t s);
// out[m] = Σ_{r < nparts} parts[r·n + m] in rank order (single-process emulation of the all-reduce)
void launch_sum_parts(int n, int nparts, const double* parts, double* out, cudaStream_t s);

// A8: GMRES vector kernels (deterministic fixed-grid reductions)
constexpr int kRedBlocks = 512;   // per-CTA partials of the multi-CTA reductions (multiple of 32)
extern long long g_launches;   // kernels launched by this library (all launchers bump it)
void launch_mgs_step(int n, double* w, const double* Vprev, const double* Vcur, const double* partial_prev,
                     double* partial_cur, double* hout, cudaStream_t s);
void launch_norm_scale(int n, double* w, const double* partial, double* hout, cudaStream_t s);
// fused MGS step on one 8-CTA cluster for n ≤ 32768 (returns false → use the multi-kernel path)
bool launch_mgs_fused(int n, int j, const double* V, double* w, double* hcol, cudaStream_t s);
void launch_dot(int n, const double* a, const double* b, double* partial, cudaStream_t s);
void launch_finish_sum(const double* partial, double* out, bool take_sqrt, cudaStream_t s);
// GMRES update x += V y, y (k ≤ kYMax coefficients, host array) passed by value in the launch
constexpr int kYMax = 64;
struct YCoef { double v[kYMax]; };
void launch_axpy_basis(int n, int k, const double* V, int ldv, const double* y_host, double* x, cudaStream_t s);
void launch_copy(int n, const double* src, double* dst, cudaStream_t s);
void launch_sub(int n, const double* a, const double* b, double* out, cudaStream_t s);
void launch_scale_copy(int n, const double* a, const double* scal, double* out, cudaStream_t s);

// ---- 3D (kernels3d in kernels2d.cu) ----
void launch_lsq3(const DevTables3& T, const double* phi, double* dphi, cudaStream_t s);
void launch_base3(const DevTables3& T, const double* fgrid, double* work, cudaStream_t s);
void launch_correct3(const DevTables3& T, const double* phi, const double* dphi, const double* fq,
                     const double* jq_given, double* work, cudaStream_t s, double* corr = nullptr);
// sparse K_D path: which 0 = forward from the compact corrections (src = corr → dst = work, spectral
// layout); 1 = fixed-up inverse along y (src = work, hsep → dst = work2, transposed rows (i−1, a, ll));
// 2 = z-direction inverse at the distinct stencil nodes only (src = work2 → dst = work, × scale)
void launch_sparse3(const DevTables3& T, int which, const double* src, const double* hsep, double scale, double* dst,
                    cudaStream_t s);
// batched in-place DST-I of the (N−1)·N rows of the working array: mode 0 plain (× scale);
// mode 1 inverse with the arrowhead fix-up on load (rows = (i, ll), modes m = ll·N + kk);
// mode 2 final store into a full (N+1)^3 grid (× scale)
// mode 3: forward from h²·f·1_Ω (src = full (N+1)³ grid, or NULL) + the compact corrections `corr`
// compact (modes 2, 3): u / f hold the Ω-node values only (row-major node ranks, omega_io)
void launch_dst_rows3(const DevTables3& T, int mode, double* work, const double* hsep, double scale, double* out,
                      cudaStream_t s, const double* src = nullptr, const double* corr = nullptr, bool compact = false);
void launch_transpose3(const DevTables3& T, double* work, cudaStream_t s);
// sparse: the source came from k_fwd3s (planes without irregular nodes are zero and not written; the
// planes the y-inverse does not read are not stored)
void launch_sweep3(const DevTables3& T, double* work, double* zB, double* zA, cudaStream_t s, bool sparse = false);
void launch_reduced3(const DevTables3& T, const double* zB, const double* zA, double* hsep, cudaStream_t s);
// multi-GPU level-2 split of the 3D reduced system (slab = P/world blocks), mode-partitioned: the slab's
// interior separators → hsep and its 4 rows per mode in chunk-major layout seg[q][4][Kq]; owner T.rank
// of modes [rank·Kq, (rank+1)·Kq) solves the world − 1 slab separators from in[r·in_r] ([4][Kq] per slab)
// into out[r·out_r] ([2][Kq] per slab: h_{r−1}, h_r); each slab fixes up from its [q][2][Kq] rows
void launch_red3_local(const DevTables3& T, const double* zB, const double* zA, double* hsep, double* seg, int Kq,
                       cudaStream_t s);
void launch_red3_solve(const DevTables3& T, const double* in, size_t in_r, double* out, size_t out_r, int Kq,
                       cudaStream_t s);
void launch_red3_fixup(const DevTables3& T, const double* hin, double* hsep, int Kq, cudaStream_t s);
// partial: only stencil nodes in the slab's planes [i_lo, i_hi] contribute (multi-GPU partial sums)
void launch_interp3(const DevTables3& T, const double* phi, const double* dphi, const double* fz,
                    const double* jz_given, const double* work, double* out, cudaStream_t s, bool partial = false);

}  // namespace kfbi
