// Internal definitions of the KFBI library (host setup tables, device table views, context).
// Nothing here is shared with oracle/ (the CPU oracle is an independent NumPy program).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/kfbi.h"

struct CUstream_st;   // cudaStream_t without the CUDA headers (setup2d.cpp is plain C++)

namespace kfbi {

// Block structure of the in-GPU partitioned tridiagonal solve along x (arrowhead/ADM,
// P:79-148, used here across thread blocks of one GPU): blocks of BL−1 columns separated
// by one separator column (reading R21), so block g covers i ∈ [BL·g+1, BL·g+BL−1] and
// separator g sits at i = BL·(g+1).  With N = 2^p, N−1 = BL·P − 1 exactly.
constexpr int BL = 16;
constexpr int LB = BL - 1;
// The reduced separator system (P−1 unknowns per mode) is itself split the same way:
// level-2 blocks of BL2−1 separators around level-2 separators (nested arrowhead).
constexpr int BL2 = 32;
constexpr int LB2 = BL2 - 1;
constexpr int kMaxSeg = 16;   // level-2 segments per mode handled by k_reduced2 (P ≤ kMaxSeg · BL2)
// most stencil rows in one k_inv_sparse work item: longer columns are split by setup (load balance:
// rows per column reach ~200 at C3 and the cap of a few hundred on the 8192² star, mean 12)
constexpr int kMaxColRows = 64;
// 3D forward: grid rows with more irregular entries than this are split over 8 lanes
constexpr int kHeavyRow = 9;

// Position of sine mode k (0 ≤ k < N) in the 2D spectral arrays (see setup2d.cpp).
#ifdef __CUDACC__
__host__ __device__
#endif
inline int mode_position(int k, int N) {
  const int q = N >> 2, hN = N >> 1;
  if (k == 0) return 0;
  if (k == hN) return 1;
  if (k == q) return 2;
  if (k == 3 * q) return 3;
  if (k < q) return 4 * k;
  if (k > 3 * q) return 4 * (N - k) + 1;
  if (k < hN) return 4 * (hN - k) + 2;
  return 4 * (k - hN) + 3;
}
#ifdef __CUDACC__
__host__ __device__
#endif
inline int position_mode(int p, int N) {
  const int t = p >> 2, r = p & 3, hN = N >> 1;
  if (t == 0) return r == 0 ? 0 : r == 1 ? hN : r == 2 ? (N >> 2) : 3 * (N >> 2);
  return r == 0 ? t : r == 1 ? N - t : r == 2 ? hN - t : hN + t;
}

struct GeomError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ArgError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct UnsupportedError : std::runtime_error {   // → KFBI_EUNSUPPORTED
  using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {        // → KFBI_ECUDA (device setup phases)
  using std::runtime_error::runtime_error;
};
struct ScratchError : std::runtime_error {       // → KFBI_ENOMEM (device setup scratch too small)
  using std::runtime_error::runtime_error;
};

struct Comp {
  int kind, role;
  double c[3];
  double p[4];
  int n_ctrl;
  double L;      // perimeter
  int M;         // control points
  int off;       // offset of its knots in φ
  double delta;  // knot spacing L/M
};

// Host-side setup products (Procedure 1).  2D.
struct Setup {
  int dim = 2;
  int N = 0, P = 0;
  double lo = 0, h = 0, kappa = 0;
  std::vector<Comp> comps;
  std::vector<int8_t> side;          // (N+1)^2, 1 = Ω
  // intersections, sorted by (axis, i, j)
  int nq = 0;
  std::vector<int32_t> q_axis, q_i, q_j, q_comp, q_knot;
  std::vector<double> q_xi, q_t, q_theta, q_t1, q_t2, q_p1, q_p2, q_x, q_y;
  // irregular nodes sorted by (i, j) + CSR to their incident intersections
  int nirr = 0;
  std::vector<int32_t> irr_i, irr_j, irr_ptr, pair_q;
  std::vector<int8_t> irr_side;
  std::vector<double> pair_d;        // x_a(p̄) − ξ for the (node, intersection) pair
  std::vector<int32_t> col_ptr;      // N+1 entries: irregular nodes of column i in [col_ptr[i], col_ptr[i+1])
  std::vector<int32_t> col_mid;      // first even-row irregular node of column i (odd rows come first)
  // control points
  int M = 0;
  std::vector<int32_t> z_comp, z_knot;
  std::vector<double> z_x, z_y, z_t1, z_t2, z_p1, z_p2;
  // six-point stencils (reading R14): unique stencil nodes sorted by (i, j)
  int nsn = 0;
  std::vector<int32_t> sn_i, sn_j;
  std::vector<int32_t> ocol, ocol_ptr;   // columns holding stencil nodes, CSR into sn_*
  std::vector<int32_t> ocol_ncls;        // 3 per stencil column: rows of class odd, j≡0, j≡2 (mod 4)
  std::vector<int32_t> ocol_order;       // stencil-column items by descending row count (k_inv_sparse)
  std::vector<int32_t> blk_order;        // ADM blocks by descending sparse-entry count (k_sweep)
  std::vector<int32_t> blk_meta;         // 4 per position of blk_order: block, first entry, end entry, stencil-column mask
  std::vector<int32_t> ocol_meta;        // 6 per position of ocol_order: item, column, row range, class counts
  std::vector<int32_t> st_node;          // M*6 → unique stencil node index
  std::vector<int8_t> st_ext;            // M*6: 1 if the node is in Ω^c
  std::vector<double> st_w, st_dx, st_dy;   // M*6: row 0 of the inverse local system, offsets
  std::vector<double> st_wn;              // M*6: normal-derivative row n·(row 1, row 2) (Neumann)
  bool neumann = false;
  std::vector<int64_t> st_nodes_ij;      // M*6*2 (dump)
  // spline filters: per component taps, coefficients (already scaled by 6/Δ²)
  std::vector<int32_t> sp_ntaps, sp_first, sp_coef_off;
  std::vector<double> sp_coef;
  // fast solver tables, mode k = 0..N−1 (k = 0 unused)
  std::vector<double> sin_tab;       // sin(π r / N), r = 0..N/2
  std::vector<double> tw;            // 2N × (cos, sin)(π m / N)
  std::vector<double> dk;            // N
  std::vector<double> invc;          // LB × N: 1/c_p of a fresh block
  std::vector<double> zr;            // LB × N: (S⁻¹ e_L)[p]
  std::vector<double> red_a, red_b;  // N: reduced-system off-diagonal / diagonal
  std::vector<double> red_invc;      // (P−1) × N
  std::vector<double> rinv2, z2r;    // LB2 × N: level-2 block pivots / spike
  std::vector<double> red2_a, red2_b;  // N: level-2 reduced system coefficients
  std::vector<double> red2_ci;         // (kMaxSeg − 1) × N: level-2 pivots 1/c_q
  int maxe = 1;                      // max sparse entries per sweep work item
  int max_col_rows = 1;              // max stencil rows in one grid column
  // holes (κ = 0 completion, reading R27)
  std::vector<int> holes;            // component ids
};

// caller-provided device scratch for the GPU setup phases (NEXT-3, setup_gpu.cu)
struct DeviceScratch {
  void* ptr;
  size_t bytes;
  ::CUstream_st* stream;
};
// dev != nullptr: classification, sign-change edges, bisection and the irregular-node lists run on
// the device (bit-identical lists, tests/test_gpu_setup.py); the rest of Procedure 1 on the host
void build_setup(Setup& S, const kfbi_grid* g, const kfbi_boundary* b, const kfbi_pde* pde,
                 const DeviceScratch* dev = nullptr);
size_t gpu_setup_scratch_bytes(int N);
void gpu_setup_phases(Setup& S, void* scratch, size_t bytes, ::CUstream_st* s, std::vector<int>& q_owner);
// 2D stencils (nodes, LU weights, unique sorted stencil nodes) on the device, after the control points
void gpu_stencil_phase(Setup& S, void* scratch, size_t bytes, ::CUstream_st* s);

// Host-side setup products in 3D (control points = intersection nodes, reading R12).
struct Setup3 {
  int N = 0, P = 0;
  double lo = 0, h = 0, kappa = 0;
  Comp comp{};
  std::vector<int8_t> side;          // (N+1)^3
  int nq = 0;                        // intersections = control points, sorted (axis, i, j, k)
  std::vector<int32_t> q_axis, q_i, q_j, q_k;
  std::vector<double> q_xi, q_pos, q_n, q_e1, q_e2, q_kab;   // 3 per point (kab: κ11, κ12, κ22)
  int nirr = 0;                      // irregular nodes sorted (i, j, k)
  std::vector<int64_t> irr_lin;      // (i−1)·N² + j·N + k in the working array
  std::vector<int32_t> irr_ijk, irr_ptr, pair_q;
  std::vector<int8_t> irr_side;
  std::vector<double> pair_d;
  std::vector<int32_t> lsq_ptr, lsq_nb;   // LSQ neighbours (CSR)
  std::vector<double> lsq_G;              // 15 per point: (ÂᵀÂ)⁻¹ upper triangle, Â scaled by 1/h
  std::vector<double> lsq_t;              // 2 per neighbour: tangent coordinates (t1, t2)/h of the fit
  std::vector<int32_t> st_c, st_code;     // stencil centre (3) and sign/exterior code
  std::vector<double> st_w;               // 10 per point: row 0 of the inverse local system
  std::vector<double> st_wn;              // 10 per point: normal-derivative row (Neumann, R38)
  bool neumann = false;
  std::vector<int64_t> st_nodes_ij;       // dump
  std::vector<double> sin_tab, dk, zr, red_a, red_b;   // modes m = ll·N + kk
  std::vector<double> tw;            // 2N complex: (cos, sin)(π m / N), m = 0..2N−1
  std::vector<int32_t> irr_row_ptr;  // (N−1)·N + 1: irregular nodes of grid row (i−1)·N + j
  std::vector<int16_t> irr_row_perm; // (N−1)·N: per plane, rows j by descending irregular count
  std::vector<int32_t> irr_row_nheavy;   // N−1: rows of the plane with more than kHeavyRow entries
  int max_plane_irr = 0;
  std::vector<int32_t> zrow_id, zrow_ptr, znode_b;   // distinct stencil nodes grouped by grid row
  std::vector<int32_t> zplane_ptr;                   // N: zrow_id[zplane_ptr[i−1] .. zplane_ptr[i]) lie in plane i
  std::vector<uint8_t> plane_flags;                  // N+1: bit 0 irregular nodes in plane i, bit 1 stencil rows
  // multi-GPU level-2 split of the reduced system (world > 1): slabs of P/world blocks hold
  // L3 = P/world − 1 interior separators each (pivots rinv3, spike z3r: L3 × K), the world − 1 slab
  // separators solve tridiag(red3_a, red3_b, red3_a) per mode after the exchange
  int L3 = -1;
  std::vector<double> rinv3, z3r, red3_a, red3_b;
};
void build_setup3(Setup3& S, const kfbi_grid* g, const kfbi_boundary* b, const kfbi_pde* pde,
                  const DeviceScratch* dev = nullptr);
size_t gpu_setup_scratch_bytes3(int N);
void gpu_setup_phases3(Setup3& S, void* scratch, size_t bytes, ::CUstream_st* s);
// 3D ten-point stencils (nodes, LU weight rows, centre and sign/exterior code) on the device
void gpu_stencil_phase3(Setup3& S, void* scratch, size_t bytes, ::CUstream_st* s);

struct DevTables3 {
  int N, P, nq, nirr;
  double lo, h, kappa;
  const int32_t* q_axis;
  const double *q_pos, *q_n, *q_e1, *q_e2, *q_kab;
  // Ω-compact rows (grid rows (i, a), N + 1 nodes each): as DevTables::om_row / om_info
  const int32_t* om_row;
  const uint32_t* om_info;
  int om_nsegp;
  const int64_t* irr_lin;
  const int8_t* irr_side;
  const int32_t *irr_ptr, *pair_q;
  const double* pair_d;
  const int32_t *lsq_ptr, *lsq_nb;
  const double* lsq_t;
  const double* lsq_G;
  const int32_t *st_c, *st_code;
  const double *st_w, *st_wn;
  int neumann;
  const double *sin_tab, *dk, *zr, *red_a, *red_b;
  const double* tw;   // 2N × (cos, sin)
  const int32_t *irr_row_ptr, *zrow_id, *zrow_ptr, *znode_b;
  const int32_t* zplane_ptr;   // per plane, the rows the z-evaluation reads (the y-inverse writes only those)
  const uint8_t* plane_flags;  // per grid plane: bit 0 non-zero sparse source, bit 1 read by the y-inverse
  const int16_t* irr_row_perm;
  const int32_t* irr_row_nheavy;
  int max_plane_irr;
  // slab of this rank (multi-GPU): ADM blocks [b_lo, b_hi), x-planes [i_lo, i_hi],
  // stencil-node rows [w_lo, w_hi) of the zrow list; the whole problem when world = 1
  int rank, b_lo, b_hi, i_lo, i_hi, w_lo, w_hi;
  int nzrow;
  const int8_t* side;
  int world, L3;   // level-2 split of the reduced system (world > 1)
  // the slab's point work: control points (= intersections, sorted by axis, i) with low-end plane in
  // [i_lo − 2, i_hi + 2], per axis [q_lo[a], q_hi[a]); irregular nodes of its planes [n_lo, n_hi)
  int q_lo[3], q_hi[3], n_lo, n_hi;
  const double *rinv3, *z3r, *red3_a, *red3_b;
};

// ---- device views -------------------------------------------------------------------
struct DevTables {
  int N, P, M, nq, nirr, nsn, nocol, ncomp, mcr;
  double lo, h, kappa;
  // intersections
  const int32_t *q_axis, *q_comp, *q_knot;
  const double *q_t, *q_t1, *q_t2, *q_p1, *q_p2;
  const double *q_x, *q_y, *z_x, *z_y;   // point coordinates (bilinear sampling, NEXT-2)
  // irregular nodes
  const int32_t *irr_j, *irr_ptr, *pair_q, *col_ptr, *col_mid;
  const int8_t* irr_side;
  const double* pair_d;
  // control points
  const int32_t *z_comp, *z_knot;
  const int32_t *q_g01, *z_g01;   // global density indices of the knots m, m + 1 of each point
  const uint8_t* row_omega;       // grid column i holds Ω nodes
  // Ω-compact rows: om_row[i] = Ω nodes before grid row i (N + 2 entries); om_info row i = the
  // om_nsegp 32-node segment bitmasks of the row, then the Ω counts before each segment in the row
  const int32_t* om_row;
  const uint32_t* om_info;
  int om_nsegp;
  const double *q_dl, *z_dl;      // Δs of the point's component
  const double *z_t1, *z_t2, *z_p1, *z_p2;
  // stencils
  const int32_t *sn_j, *ocol, *ocol_ptr, *st_node, *ocol_ncls, *ocol_order, *blk_order, *blk_meta, *ocol_meta;
  const int8_t* st_ext;
  const double *st_w, *st_dx, *st_dy, *st_wn;
  int neumann;   // K_N: density = ψ (Φ = 0, Ψ = ψ) and the normal-derivative interpolation
  // spline
  const int32_t *c_off, *c_M, *sp_ntaps, *sp_first, *sp_coef_off;
  const double *c_delta, *sp_coef;
  // fast solver
  const double *sin_tab, *dk, *invc, *zr, *red_a, *red_b, *red_invc;
  const double* tw;   // 2N × (cos, sin)(π m/N)
  const double *rinv2, *z2r, *red2_a, *red2_b, *red2_ci;
  int maxe;
  const int8_t* side;
  const int32_t* sn_i;
  // slab of the executing rank (multi-GPU): blocks [g_lo, g_hi), level-2 segments
  // [seg_lo, seg_hi) of nseg, owned columns [col_lo, col_hi], owned stencil columns [o_lo, o_hi)
  int g_lo, g_hi, seg_lo, seg_hi, nseg, col_lo, col_hi, o_lo, o_hi, rank;
  int irr_lo, irr_hi;   // the slab's irregular nodes (sorted by column): the corrections its sweep reads
};

}  // namespace kfbi
