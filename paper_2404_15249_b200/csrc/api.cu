// C ABI of the KFBI library: context, workspace, kfbi_apply / kfbi_solve orchestration.
// See include/kfbi.h for the contract.  All device work is stream-ordered on the caller's
// stream; the only host syncs are the ones Algorithm 5 needs (one per Arnoldi step).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nccl.h>

#include "kernels.h"
#include "kfbi_impl.h"

using namespace kfbi;

namespace {
thread_local std::string g_setup_err;
constexpr int kMaxRestart = 64;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// a non-finite residual in an iterative solve (NaN/Inf in the inputs, or a breakdown): KFBI_EBREAKDOWN
struct BreakdownError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// the entry point runs on the context's device and restores the caller's current device on return
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    int cur = 0;
    if (dev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
inline void ckn(ncclResult_t e, const char* what) {
  if (e != ncclSuccess) throw NcclError(std::string(what) + ": " + ncclGetErrorString(e));
}
}  // namespace

struct kfbi_ctx {
  int dim = 2;
  // multi-GPU: slabs along x = groups of level-2 arrowhead segments.  rank == −1:
  // all `world` ranks executed by this context on one GPU (emulation, collectives in-device).
  int world = 1, rank = 0;
  bool use_nccl = false;
  ncclUniqueId nccl_id{};
  ncclComm_t comm = nullptr;
  double *segbuf = nullptr, *h2 = nullptr, *parts = nullptr;
  double *seg3 = nullptr, *seg3_in = nullptr, *h3_out = nullptr, *h3_in = nullptr;   // 3D level-2 exchange
  std::vector<DevTables> slabs;   // per-rank slab tables (2D), rebuilt with the workspace layout
  std::vector<int32_t> q_g01, z_g01;   // spline knot pairs of the intersections / control points
  std::vector<double> q_dl, z_dl;
  std::vector<uint8_t> row_omega;
  Setup S;
  DevTables T{};
  Setup3 S3;
  DevTables3 T3{};
  double *work = nullptr, *dphi = nullptr;   // 3D working array and LSQ derivatives
  double *work2 = nullptr, *corr = nullptr;  // 3D transposed inverse rows; compact corrections
  cudaStream_t stream = nullptr;
  int device = 0;
  std::string err;
  uint8_t* ws = nullptr;
  size_t ws_bytes = 0, ws_need = 0;
  // scratch
  double *spec = nullptr, *zfirst = nullptr, *zlast = nullptr, *fsep = nullptr, *hsep = nullptr;
  double *cval = nullptr, *mk = nullptr, *vsten = nullptr;
  // holes
  int nh = 0;
  int *hole_off = nullptr, *hole_M = nullptr;
  double *hole_delta = nullptr, *ahole = nullptr, *wg = nullptr, *onehot = nullptr;
  BumpParams bump{};
  // GMRES
  double *V = nullptr, *gx = nullptr, *gr = nullptr, *ghat = nullptr, *tmp = nullptr;
  double *partial = nullptr, *hcol = nullptr, *ycoef = nullptr, *scal = nullptr;
  double *spec_f = nullptr, *spec_bump = nullptr;   // cached spectra (final field by linearity)
  size_t spec_ld = 0;                                 // stride between the hole bumps' spectra
  // local-slab I/O (world > 1 with one rank per process): f and u are the rank's node slab
  // [loc_off, loc_off + loc_shape) of the full grid; the spectral and working arrays hold the slab only
  bool local_io = false;
  int64_t loc_shape[3] = {0, 0, 0}, loc_off[3] = {0, 0, 0};
  bool spec_f_valid = false;
  // Ω-compact transfers: Ω nodes per grid row (prefix), the full-grid mask on the device
  std::vector<int64_t> om_ptr;
  std::vector<int32_t> om_seg;   // Ω nodes before each 32-node segment of each row
  const int64_t* d_om_ptr = nullptr;
  const int32_t* d_om_seg = nullptr;
  std::vector<int32_t> om_row32;   // 2D: Ω nodes before each grid row (N + 2)
  std::vector<uint32_t> om_info;   // 2D: per row, the padded segment bitmasks then the in-row counts
  bool io_compact = false;         // inside kfbi_solve with opts.omega_io: f and u are Ω-compact
  const int8_t* d_side = nullptr;
  int64_t om_rows = 0, om_width = 0;
  double* hcol_host = nullptr;   // host-mapped (written by k_copy, read after a stream sync); the
  double* hcol_map = nullptr;    // first kMaxRestart + 2 doubles for scalars, then one Hessenberg
                                 // column slot per Arnoldi step (its device alias: hcol_map)
  cudaEvent_t ev_step[2] = {nullptr, nullptr};   // end of Arnoldi steps j (j even / odd)
  // Arnoldi step j (K v_j → v_{j+1}, MGS, Hessenberg column → mapped slot j) as one CUDA graph per j,
  // captured on first use (the step's pointers are fixed per j for a workspace); single-process contexts
  // only (no NCCL inside a capture).  launches = the library kernels one replay runs (kfbi_launch_count).
  struct StepGraph {
    cudaGraphExec_t exec = nullptr;
    long long launches = 0;
  };
  std::vector<StepGraph> step_graphs;
  bool graphs_off = [] {   // KFBI_GRAPHS=0: eager launches (A/B runs)
    const char* e = std::getenv("KFBI_GRAPHS");
    return e != nullptr && e[0] == '0';
  }();
  // host staging of small tables (kept alive for the async uploads)
  std::vector<int32_t> coff, cM, hoff, hM;
  std::vector<double> cdel, hdel, oneh;
};

namespace {

// two-pass bump allocator over the workspace (pass 1 sizes, pass 2 assigns + uploads)
struct Arena {
  uint8_t* base;
  size_t off = 0;
  bool assign;
  std::vector<std::pair<void*, std::pair<const void*, size_t>>> uploads;
  template <class T>
  T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T* p = assign ? reinterpret_cast<T*>(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
  // n elements addressed by global index [i0, i0 + n): the returned pointer is the buffer shifted by
  // −i0 (slab-local buffers indexed with global row numbers by the kernels)
  template <class T>
  T* take_rows(size_t n, size_t i0) {
    T* p = take<T>(n);
    return assign ? p - i0 : nullptr;
  }
  template <class T>
  const T* table(const std::vector<T>& v) {
    T* p = take<T>(v.empty() ? 1 : v.size());
    if (assign && !v.empty()) uploads.push_back({p, {v.data(), v.size() * sizeof(T)}});
    return p;
  }
};

DevTables slab(const kfbi_ctx* c, int r);
DevTables slab_build(const kfbi_ctx* c, int r);

// Ω nodes before each grid row of `width` nodes (rows × width = the full node grid, row-major)
void omega_rows(kfbi_ctx* c, const std::vector<int8_t>& side, int64_t rows, int64_t width) {
  if (c->om_rows == rows && (int64_t)c->om_ptr.size() == rows + 1) return;
  c->om_rows = rows;
  c->om_width = width;
  c->om_ptr.assign(rows + 1, 0);
  const int64_t nseg = (width + 31) / 32;
  c->om_seg.assign(rows * nseg, 0);
  for (int64_t r = 0; r < rows; ++r) {
    int64_t n = 0;
    const int8_t* row = side.data() + r * width;
    for (int64_t j = 0; j < width; ++j) {
      if ((j & 31) == 0) c->om_seg[r * nseg + (j >> 5)] = (int32_t)(c->om_ptr[r] + n);
      n += row[j] != 0;
    }
    c->om_ptr[r + 1] = c->om_ptr[r] + n;
  }
  if (c->om_ptr.back() > INT32_MAX) throw ArgError("too many Ω nodes for the compact transfers");
}

// Ω-compact row tables of the grid rows omega_rows() set up (width = N + 1 nodes per row): om_row32 =
// Ω nodes before each row, om_info = per row the nsegp 32-node segment bitmasks then the Ω counts
// before each segment within the row; returns nsegp
int omega_info(kfbi_ctx* c, const std::vector<int8_t>& side) {
  const int64_t rows = c->om_rows, W = c->om_width, nseg = (W + 31) / 32, nsegp = (nseg + 3) / 4 * 4;
  if (c->om_info.size() == (size_t)rows * 2 * nsegp && c->om_row32.size() == (size_t)rows + 1) return (int)nsegp;
  c->om_row32.assign(c->om_ptr.begin(), c->om_ptr.end());
  c->om_info.assign((size_t)rows * 2 * nsegp, 0u);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    uint32_t* info = c->om_info.data() + (size_t)r * 2 * nsegp;
    for (int64_t j = 0; j < W; ++j)
      if (side[(size_t)(r * W + j)]) info[j >> 5] |= 1u << (j & 31);
    for (int64_t g = 0; g < nseg; ++g) info[nsegp + g] = (uint32_t)(c->om_seg[r * nseg + g] - c->om_ptr[r]);
  }
  return (int)nsegp;
}

void layout(kfbi_ctx* c, Arena& A) {
  Setup& S = c->S;
  DevTables& T = c->T;
  const size_t N = S.N, P = S.P;
  T.N = S.N; T.P = S.P; T.M = S.M; T.nq = S.nq; T.nirr = S.nirr; T.nsn = S.nsn;
  T.nocol = (int)S.ocol.size(); T.ncomp = (int)S.comps.size();
  T.lo = S.lo; T.h = S.h; T.kappa = S.kappa;
  T.q_axis = A.table(S.q_axis); T.q_comp = A.table(S.q_comp); T.q_knot = A.table(S.q_knot);
  T.q_t = A.table(S.q_t); T.q_t1 = A.table(S.q_t1); T.q_t2 = A.table(S.q_t2);
  T.q_p1 = A.table(S.q_p1); T.q_p2 = A.table(S.q_p2);
  T.q_x = A.table(S.q_x); T.q_y = A.table(S.q_y); T.z_x = A.table(S.z_x); T.z_y = A.table(S.z_y);
  T.irr_j = A.table(S.irr_j); T.irr_ptr = A.table(S.irr_ptr); T.pair_q = A.table(S.pair_q);
  T.col_ptr = A.table(S.col_ptr); T.col_mid = A.table(S.col_mid); T.irr_side = A.table(S.irr_side); T.pair_d = A.table(S.pair_d);
  T.z_comp = A.table(S.z_comp); T.z_knot = A.table(S.z_knot);
  T.z_t1 = A.table(S.z_t1); T.z_t2 = A.table(S.z_t2); T.z_p1 = A.table(S.z_p1); T.z_p2 = A.table(S.z_p2);
  T.sn_j = A.table(S.sn_j); T.ocol = A.table(S.ocol); T.ocol_ptr = A.table(S.ocol_ptr);
  T.ocol_ncls = A.table(S.ocol_ncls); T.ocol_order = A.table(S.ocol_order); T.blk_order = A.table(S.blk_order);
  T.blk_meta = A.table(S.blk_meta); T.ocol_meta = A.table(S.ocol_meta);
  T.st_node = A.table(S.st_node); T.st_ext = A.table(S.st_ext);
  T.st_w = A.table(S.st_w); T.st_dx = A.table(S.st_dx); T.st_dy = A.table(S.st_dy);
  T.st_wn = A.table(S.st_wn); T.neumann = S.neumann ? 1 : 0;
  // component tables live in the setup object as small vectors
  auto& coff = c->coff; auto& cM = c->cM; auto& cdel = c->cdel;
  coff.clear(); cM.clear(); cdel.clear();
  for (auto& cc : S.comps) { coff.push_back(cc.off); cM.push_back(cc.M); cdel.push_back(cc.delta); }
  T.c_off = A.table(coff); T.c_M = A.table(cM); T.c_delta = A.table(cdel);
  // the two spline knots (global density indices) and Δs of every intersection and control point: one
  // load level for the jump kernels instead of point → component → offset, size
  auto knots = [&](const std::vector<int32_t>& comp, const std::vector<int32_t>& knot, std::vector<int32_t>& g01,
                   std::vector<double>& dl) {
    const size_t n = comp.size();
    g01.resize(2 * n);
    dl.resize(n);
    for (size_t k = 0; k < n; ++k) {
      const Comp& cc = S.comps[comp[k]];
      const int m = knot[k], m1 = m + 1 == cc.M ? 0 : m + 1;
      g01[2 * k] = cc.off + m;
      g01[2 * k + 1] = cc.off + m1;
      dl[k] = cc.delta;
    }
  };
  knots(S.q_comp, S.q_knot, c->q_g01, c->q_dl);
  knots(S.z_comp, S.z_knot, c->z_g01, c->z_dl);
  T.q_g01 = A.table(c->q_g01); T.q_dl = A.table(c->q_dl);
  T.z_g01 = A.table(c->z_g01); T.z_dl = A.table(c->z_dl);
  T.sp_ntaps = A.table(S.sp_ntaps); T.sp_first = A.table(S.sp_first); T.sp_coef_off = A.table(S.sp_coef_off);
  T.sp_coef = A.table(S.sp_coef);
  T.sin_tab = A.table(S.sin_tab); T.dk = A.table(S.dk); T.invc = A.table(S.invc); T.zr = A.table(S.zr);
  T.tw = A.table(S.tw);
  T.red_a = A.table(S.red_a); T.red_b = A.table(S.red_b); T.red_invc = A.table(S.red_invc);
  T.rinv2 = A.table(S.rinv2); T.z2r = A.table(S.z2r); T.red2_a = A.table(S.red2_a); T.red2_b = A.table(S.red2_b);
  T.red2_ci = A.table(S.red2_ci);
  T.maxe = S.maxe;
  T.mcr = S.max_col_rows;
  T.side = A.table(S.side);
  omega_rows(c, S.side, (int64_t)S.N + 1, (int64_t)S.N + 1);
  c->d_om_ptr = A.table(c->om_ptr);
  c->d_om_seg = A.table(c->om_seg);
  c->d_side = T.side;
  T.om_nsegp = omega_info(c, S.side);   // Ω-compact rows for the dense forward / final field (omega_io)
  T.om_row = A.table(c->om_row32);
  T.om_info = A.table(c->om_info);
  c->row_omega.assign(S.N + 1, 0);
  for (int i = 0; i <= S.N; ++i) c->row_omega[i] = c->om_ptr[i + 1] > c->om_ptr[i] ? 1 : 0;
  T.row_omega = A.table(c->row_omega);
  // holes
  auto& hoff = c->hoff; auto& hM = c->hM; auto& hdel = c->hdel; auto& oneh = c->oneh;
  hoff.clear(); hM.clear(); hdel.clear(); oneh.clear();
  c->nh = (int)S.holes.size();
  for (int k : S.holes) {
    hoff.push_back(S.comps[k].off); hM.push_back(S.comps[k].M); hdel.push_back(S.comps[k].delta);
  }
  for (int a = 0; a < c->nh; ++a)
    for (int b = 0; b < c->nh; ++b) oneh.push_back(a == b ? 1.0 : 0.0);
  c->hole_off = const_cast<int*>(A.table(hoff));
  c->hole_M = const_cast<int*>(A.table(hM));
  c->hole_delta = const_cast<double*>(A.table(hdel));
  c->onehot = const_cast<double*>(A.table(oneh));
  c->ahole = A.take<double>(std::max(c->nh, 1));
  c->wg = A.take<double>((size_t)std::max(c->nh, 1) * S.M);
  // scratch
  // spectral rows (row i − 1 = grid column i): the whole grid, or the rank's slab columns
  // [col_lo, col_hi] when it runs alone in its process (local-slab I/O, memory ∝ 1/world)
  size_t row0 = 0, nloc = N - 1;
  c->local_io = c->world > 1 && c->rank >= 0;
  if (c->local_io) {
    const int nseg = S.P >= 2 * BL2 ? S.P / BL2 : 1;
    const int g_lo = c->rank * nseg / c->world * BL2, g_hi = (c->rank + 1) * nseg / c->world * BL2;
    const int col_lo = BL * g_lo + 1, col_hi = std::min(BL * g_hi, S.N - 1);
    row0 = col_lo - 1;
    nloc = col_hi - col_lo + 1;
    c->loc_off[0] = col_lo; c->loc_shape[0] = nloc;
  } else {
    c->loc_off[0] = 0; c->loc_shape[0] = N + 1;
  }
  c->loc_off[1] = 0; c->loc_shape[1] = N + 1; c->loc_off[2] = 0; c->loc_shape[2] = 1;
  c->spec = A.take_rows<double>(nloc * N, row0 * N);
  // spectra reused by the final field (linearity): DST(f·1_Ω) from the solve's Y apply, DST(b_h) of the
  // hole bumps from setup — the final field's dense forward becomes spec_f + Σ a_h spec_bump_h
  c->spec_f = A.take_rows<double>(nloc * N, row0 * N);
  c->spec_ld = nloc * N;
  c->spec_bump = A.take_rows<double>((size_t)std::max(c->nh, 1) * nloc * N, row0 * N);
  c->zfirst = A.take<double>(P * N);
  c->zlast = A.take<double>(P * N);
  c->fsep = A.take<double>(std::max<size_t>(P - 1, 1) * N);
  c->hsep = A.take<double>(std::max<size_t>(P - 1, 1) * N);
  c->cval = A.take<double>(std::max(S.nirr, 1));
  c->mk = A.take<double>(S.M);
  c->vsten = A.take<double>(std::max(S.nsn, 1));
  const size_t M = S.M;
  c->V = A.take<double>((kMaxRestart + 1) * M);
  c->gx = A.take<double>(M);
  c->gr = A.take<double>(M);
  c->ghat = A.take<double>(M);
  c->tmp = A.take<double>(M);
  c->partial = A.take<double>((kMaxRestart + 2) * kRedBlocks);
  c->hcol = A.take<double>(kMaxRestart + 2);
  c->ycoef = A.take<double>(kMaxRestart + 1);
  c->scal = A.take<double>(8);
  const size_t nseg = S.P >= 2 * BL2 ? S.P / BL2 : 1;
  c->segbuf = A.take<double>(nseg * 4 * N);
  c->h2 = A.take<double>(nseg * N);
  c->parts = A.take<double>((size_t)std::max(c->world, 1) * M);
  T.sn_i = A.table(S.sn_i);
  c->slabs.clear();
  c->T = slab_build(c, c->rank >= 0 ? c->rank : 0);
  for (int r = 0; r < std::max(c->world, 1); ++r) c->slabs.push_back(slab_build(c, r));
}

void layout3(kfbi_ctx* c, Arena& A) {
  Setup3& S = c->S3;
  DevTables3& T = c->T3;
  const size_t N = S.N, P = S.P, K = N * N, M = S.nq;
  T.N = S.N; T.P = S.P; T.nq = S.nq; T.nirr = S.nirr; T.lo = S.lo; T.h = S.h; T.kappa = S.kappa;
  T.rank = 0; T.b_lo = 0; T.b_hi = S.P; T.i_lo = 1; T.i_hi = S.N - 1; T.w_lo = 0; T.w_hi = (int)S.zrow_id.size();
  T.q_axis = A.table(S.q_axis); T.q_pos = A.table(S.q_pos); T.q_n = A.table(S.q_n); T.q_e1 = A.table(S.q_e1);
  T.q_e2 = A.table(S.q_e2); T.q_kab = A.table(S.q_kab);
  T.irr_lin = A.table(S.irr_lin); T.irr_side = A.table(S.irr_side); T.irr_ptr = A.table(S.irr_ptr);
  T.pair_q = A.table(S.pair_q); T.pair_d = A.table(S.pair_d);
  T.lsq_ptr = A.table(S.lsq_ptr); T.lsq_nb = A.table(S.lsq_nb); T.lsq_G = A.table(S.lsq_G);
  T.lsq_t = A.table(S.lsq_t);
  T.st_c = A.table(S.st_c); T.st_code = A.table(S.st_code); T.st_w = A.table(S.st_w);
  T.st_wn = A.table(S.st_wn); T.neumann = S.neumann ? 1 : 0;
  T.sin_tab = A.table(S.sin_tab); T.dk = A.table(S.dk); T.zr = A.table(S.zr); T.red_a = A.table(S.red_a);
  T.red_b = A.table(S.red_b); T.side = A.table(S.side);
  omega_rows(c, S.side, ((int64_t)S.N + 1) * ((int64_t)S.N + 1), (int64_t)S.N + 1);
  c->d_om_ptr = A.table(c->om_ptr);
  c->d_om_seg = A.table(c->om_seg);
  T.om_nsegp = omega_info(c, S.side);   // Ω-compact rows for the dense forward / final field (omega_io)
  T.om_row = A.table(c->om_row32);
  T.om_info = A.table(c->om_info);
  c->d_side = T.side;
  T.tw = A.table(S.tw);
  T.irr_row_perm = A.table(S.irr_row_perm); T.irr_row_nheavy = A.table(S.irr_row_nheavy);
  T.max_plane_irr = S.max_plane_irr;
  T.irr_row_ptr = A.table(S.irr_row_ptr); T.zrow_id = A.table(S.zrow_id); T.zrow_ptr = A.table(S.zrow_ptr);
  T.znode_b = A.table(S.znode_b); T.nzrow = (int)S.zrow_id.size(); T.zplane_ptr = A.table(S.zplane_ptr);
  T.plane_flags = A.table(S.plane_flags);
  T.world = c->world; T.L3 = S.L3;
  T.q_lo[0] = 0; T.q_hi[0] = S.nq; T.q_lo[1] = T.q_hi[1] = T.q_lo[2] = T.q_hi[2] = S.nq;
  T.n_lo = 0; T.n_hi = S.nirr;
  T.rinv3 = S.L3 >= 0 ? A.table(S.rinv3) : nullptr; T.z3r = S.L3 >= 0 ? A.table(S.z3r) : nullptr;
  T.red3_a = S.L3 >= 0 ? A.table(S.red3_a) : nullptr; T.red3_b = S.L3 >= 0 ? A.table(S.red3_b) : nullptr;
  if (c->world > 1) {   // level-2 exchange buffers (reduced3_dist); the emulation holds every slab's
    const size_t W = c->world, Kq = (K + W - 1) / W, sl = c->rank >= 0 ? 1 : W;
    c->seg3 = A.take<double>(sl * W * 4 * Kq);    // from local: [slab][q][4][Kq]
    c->seg3_in = A.take<double>(W * 4 * Kq);      // owner's input [r][4][Kq] (NCCL)
    c->h3_out = A.take<double>(sl * W * 2 * Kq);  // owner's output [owner][r][2][Kq] (emulation) / [r][2][Kq]
    c->h3_in = A.take<double>(sl * W * 2 * Kq);   // slab's fix-up input [slab][q][2][Kq]
  }
  c->nh = 0;
  // working arrays: all N − 1 planes, or the rank's slab planes [i_lo, i_hi] (local-slab I/O)
  size_t pl0 = 0, npl = N - 1;
  c->local_io = c->world > 1 && c->rank >= 0;
  if (c->local_io) {
    const int b_lo = c->rank * S.P / c->world, b_hi = (c->rank + 1) * S.P / c->world;
    const int i_lo = BL * b_lo + 1, i_hi = std::min(BL * b_hi, S.N - 1);
    pl0 = i_lo - 1;
    npl = i_hi - i_lo + 1;
    c->loc_off[0] = i_lo; c->loc_shape[0] = npl;
  } else {
    c->loc_off[0] = 0; c->loc_shape[0] = N + 1;
  }
  c->loc_off[1] = c->loc_off[2] = 0; c->loc_shape[1] = c->loc_shape[2] = N + 1;
  c->work = A.take_rows<double>(npl * K, pl0 * K);
  c->work2 = A.take_rows<double>(npl * K, pl0 * K);
  c->zfirst = A.take<double>(P * K);
  c->corr = A.take<double>(std::max(S.nirr, 1));
  c->fsep = A.take<double>(P * K);   // zA: one row per block (the last block's is unused)
  c->hsep = A.take<double>(std::max<size_t>(P - 1, 1) * K);
  c->dphi = A.take<double>(5 * M);
  c->parts = A.take<double>((size_t)std::max(c->world, 1) * M);
  c->V = A.take<double>((kMaxRestart + 1) * M);
  c->gx = A.take<double>(M);
  c->gr = A.take<double>(M);
  c->ghat = A.take<double>(M);
  c->tmp = A.take<double>(M);
  c->partial = A.take<double>((kMaxRestart + 2) * kRedBlocks);
  c->hcol = A.take<double>(kMaxRestart + 2);
  c->ycoef = A.take<double>(kMaxRestart + 1);
  c->scal = A.take<double>(8);
  c->ahole = A.take<double>(1);
}

int nctrl(const kfbi_ctx* c) { return c->dim == 3 ? c->S3.nq : c->S.M; }

// DevTables restricted to the slab of rank r of `world` (full domain when world == 1)
DevTables slab_build(const kfbi_ctx* c, int r) {
  DevTables T = c->T;
  const Setup& S = c->S;
  const int world = c->world;
  T.nseg = S.P >= 2 * BL2 ? S.P / BL2 : 1;
  T.rank = r;
  if (world == 1) {
    T.g_lo = 0; T.g_hi = S.P; T.seg_lo = 0; T.seg_hi = T.nseg;
    T.col_lo = 1; T.col_hi = S.N - 1; T.o_lo = 0; T.o_hi = (int)S.ocol.size();
    T.irr_lo = 0; T.irr_hi = S.nirr;
    return T;
  }
  T.seg_lo = r * T.nseg / world;
  T.seg_hi = (r + 1) * T.nseg / world;
  T.g_lo = T.seg_lo * BL2;
  T.g_hi = T.seg_hi * BL2;
  T.col_lo = BL * T.g_lo + 1;
  T.col_hi = std::min(BL * T.g_hi, S.N - 1);
  T.o_lo = (int)(std::lower_bound(S.ocol.begin(), S.ocol.end(), T.col_lo) - S.ocol.begin());
  T.o_hi = (int)(std::upper_bound(S.ocol.begin(), S.ocol.end(), T.col_hi) - S.ocol.begin());
  T.irr_lo = S.col_ptr[T.col_lo];
  T.irr_hi = S.col_ptr[T.col_hi + 1];
  return T;
}

// the slab tables of rank r, built once per workspace (slab_build walks the stencil-column items)
DevTables slab(const kfbi_ctx* c, int r) {
  if (r >= 0 && r < (int)c->slabs.size()) return c->slabs[r];
  return slab_build(c, r);
}

// 3D slab of rank r: whole ADM blocks (15 planes + separator), P / world per rank
DevTables3 slab3(const kfbi_ctx* c, int r) {
  DevTables3 T = c->T3;
  const Setup3& S = c->S3;
  const int world = c->world;
  T.rank = r;
  if (world == 1) return T;   // c->T3 holds the full ranges (layout3)
  T.b_lo = r * S.P / world;
  T.b_hi = (r + 1) * S.P / world;
  T.i_lo = BL * T.b_lo + 1;
  T.i_hi = std::min(BL * T.b_hi, S.N - 1);
  auto row0 = [&](int i) { return (int32_t)((int64_t)(i - 1) * S.N); };
  T.w_lo = (int)(std::lower_bound(S.zrow_id.begin(), S.zrow_id.end(), row0(T.i_lo)) - S.zrow_id.begin());
  T.w_hi = (int)(std::lower_bound(S.zrow_id.begin(), S.zrow_id.end(), row0(T.i_hi + 1)) - S.zrow_id.begin());
  // point work of the slab: the control points whose LSQ derivatives the slab's corrections and
  // partial interpolation sums use (intersections of its irregular nodes' edges: low-end plane
  // i − 1 … i; stencil nodes c ± 1 of a control point in the slab: low-end plane ≥ i_lo − 2)
  for (int a = 0; a < 3; ++a) {
    auto key_lt = [&](int q, int i) { return S.q_axis[q] < a || (S.q_axis[q] == a && S.q_i[q] < i); };
    int lo = 0, hi = S.nq;
    while (lo < hi) { const int mid = (lo + hi) / 2; if (key_lt(mid, T.i_lo - 2)) lo = mid + 1; else hi = mid; }
    T.q_lo[a] = lo;
    hi = S.nq;
    while (lo < hi) { const int mid = (lo + hi) / 2; if (key_lt(mid, T.i_hi + 3)) lo = mid + 1; else hi = mid; }
    T.q_hi[a] = lo;
  }
  {
    int lo = 0, hi = S.nirr;
    while (lo < hi) { const int mid = (lo + hi) / 2; if (S.irr_ijk[3 * mid] < T.i_lo) lo = mid + 1; else hi = mid; }
    T.n_lo = lo;
    hi = S.nirr;
    while (lo < hi) { const int mid = (lo + hi) / 2; if (S.irr_ijk[3 * mid] <= T.i_hi) lo = mid + 1; else hi = mid; }
    T.n_hi = lo;
  }
  return T;
}

// level-2 arrowhead tables of the 3D reduced system tridiag(a, b, a) (P − 1 separators per mode) for
// slabs of L3 + 1 blocks: the L3 interior separators of a slab are eliminated locally (pivots and the
// right spike S₂⁻¹e_L), leaving tridiag(A2, B2, A2) on the world − 1 slab separators (App. A.5 applied
// to the reduced system).  L3 = 0: the slab separators are the whole reduced system.
void level2_tables3(Setup3& S, int L3) {
  const size_t K = (size_t)S.N * S.N;
  S.L3 = L3;
  S.rinv3.assign((size_t)std::max(L3, 1) * K, 0.0);
  S.z3r.assign((size_t)std::max(L3, 1) * K, 0.0);
  S.red3_a.assign(K, 0.0);
  S.red3_b.assign(K, 1.0);
#pragma omp parallel for schedule(static)
  for (long m = 0; m < (long)K; ++m) {
    const double a = S.red_a[m], bb = S.red_b[m];
    if (L3 == 0) {
      S.red3_a[m] = a;
      S.red3_b[m] = bb;
      continue;
    }
    std::vector<double> cs(L3);
    double cc = bb;
    for (int p = 0; p < L3; ++p) {
      if (p > 0) cc = bb - a * a / cc;
      cs[p] = cc;
      S.rinv3[(size_t)p * K + m] = 1.0 / cc;
    }
    double x = 1.0 / cs[L3 - 1];   // S₂⁻¹e_L: x_L = 1/c_L, x_p = −a x_{p+1}/c_p
    S.z3r[(size_t)(L3 - 1) * K + m] = x;
    for (int p = L3 - 2; p >= 0; --p) {
      x = -a * x / cs[p];
      S.z3r[(size_t)p * K + m] = x;
    }
    S.red3_a[m] = -a * a * S.z3r[m];
    S.red3_b[m] = bb - 2.0 * a * a * S.z3r[(size_t)(L3 - 1) * K + m];
  }
}

std::vector<int> my_ranks(const kfbi_ctx* c) {
  std::vector<int> v;
  if (c->rank >= 0) v.push_back(c->rank);
  else
    for (int r = 0; r < c->world; ++r) v.push_back(r);
  return v;
}

kfbi_status fail(kfbi_ctx* c, kfbi_status st, const std::string& msg) {
  if (c) c->err = msg;
  return st;
}

#define KFBI_TRY(ctx)                                                  \
  DeviceGuard kfbi_device_guard_((ctx)->device);                       \
  try {
#define KFBI_CATCH(ctx)                                                \
  }                                                                    \
  catch (const CudaError& e) { return fail(ctx, KFBI_ECUDA, e.what()); } \
  catch (const NcclError& e) { return fail(ctx, KFBI_ENCCL, e.what()); } \
  catch (const GeomError& e) { return fail(ctx, KFBI_EGEOM, e.what()); } \
  catch (const ArgError& e) { return fail(ctx, KFBI_EINVAL, e.what()); } \
  catch (const BreakdownError& e) { return fail(ctx, KFBI_EBREAKDOWN, e.what()); } \
  catch (const DeviceError& e) { return fail(ctx, KFBI_ECUDA, e.what()); } \
  catch (const std::exception& e) { return fail(ctx, KFBI_EINVAL, e.what()); }

cudaStream_t pick(kfbi_ctx* c, void* s) { return s ? (cudaStream_t)s : c->stream; }

void need_ws(kfbi_ctx* c) {
  if (!c->ws) throw std::runtime_error("workspace not set (kfbi_set_workspace)");
}

// --- one interface solve, sparse output at stencil nodes → V⁺ at control points ----------
// --- 2D interface solve, possibly distributed over slabs ----------------------------------
// spectral part: sweep of the owned blocks → reduced (arrowhead) system → h at every separator the
// owned columns need.  world > 1: level-2 segments = slabs; the segment end values are all-gathered
// (the only exchange of the tridiagonal solve) and every rank solves the S − 1 slab
// separators redundantly.
void spectral2(kfbi_ctx* c, const double* cval, const DenseSrc& D, cudaStream_t s) {
  for (int r : my_ranks(c)) launch_sweep(slab(c, r), cval, D, c->spec, c->zfirst, c->zlast, c->fsep, s);
  if (c->world == 1) {
    launch_reduced(c->T, c->zfirst, c->zlast, c->fsep, c->hsep, s);
    return;
  }
  for (int r : my_ranks(c)) launch_red2_local(slab(c, r), c->zfirst, c->fsep, c->hsep, c->segbuf, s);
  if (c->use_nccl) {
    const DevTables T = slab(c, c->rank);
    const size_t cnt = (size_t)(T.seg_hi - T.seg_lo) * 4 * T.N;
    ckn(ncclAllGather(c->segbuf + (size_t)T.seg_lo * 4 * T.N, c->segbuf, cnt, ncclDouble, c->comm, s), "allgather");
  }
  launch_red2_solve(c->T, c->segbuf, c->h2, s);
  for (int r : my_ranks(c)) launch_red2_fixup(slab(c, r), c->h2, c->hsep, s);
}

// stencil values of the owned columns → V⁺ (partial sums + all-reduce when distributed)
void interp2(kfbi_ctx* c, const double* phi, const double* fz, const double* jz, bool holes, double* out,
             cudaStream_t s) {
  const int nh = holes ? c->nh : 0;
  const double* wg = nh ? c->wg : nullptr;
  for (int r : my_ranks(c)) launch_inverse_sparse(slab(c, r), c->spec, c->hsep, c->vsten, s);
  if (c->world == 1) {
    launch_interp(c->T, phi, c->mk, fz, jz, c->vsten, nh, wg, c->ahole, out, s);
    return;
  }
  const int M = c->S.M;
  if (c->use_nccl) {
    launch_interp(slab(c, c->rank), phi, c->mk, fz, jz, c->vsten, nh, wg, c->ahole, c->parts, s, true);
    ckn(ncclAllReduce(c->parts, out, M, ncclDouble, ncclSum, c->comm, s), "allreduce");
    return;
  }
  for (int r : my_ranks(c))
    launch_interp(slab(c, r), phi, c->mk, fz, jz, c->vsten, nh, wg, c->ahole, c->parts + (size_t)r * M, s, true);
  launch_sum_parts(M, c->world, c->parts, out, s);
}

void dst_forward2(kfbi_ctx* c, const double* fgrid, bool mask, const BumpParams& bp, double* dst, cudaStream_t s) {
  const bool compact = c->io_compact && fgrid != nullptr;   // world = 1 only (kfbi_solve checks)
  for (int r : my_ranks(c)) launch_dst_forward(slab(c, r), fgrid, mask, bp, dst, s, compact);
}

void apply_KD2(kfbi_ctx* c, const double* phi, double* out, cudaStream_t s) {
  const DevTables& T = c->T;
  launch_spline(T, phi, c->mk, s, c->hole_off, c->hole_M, c->hole_delta, c->nh, c->ahole);   // + a_h (R27)
  for (int r : my_ranks(c)) launch_correct(slab(c, r), phi, c->mk, nullptr, nullptr, c->cval, s);   // slab's nodes
  DenseSrc D;
  D.stencil_only = true;
  spectral2(c, c->cval, D, s);
  interp2(c, phi, nullptr, nullptr, true, out, s);
}

void apply_Y2(kfbi_ctx* c, const double* fgrid, const double* fq, const double* fz, double* out, cudaStream_t s) {
  BumpParams none{};
  dst_forward2(c, fgrid, true, none, c->spec_f, s);   // kept for the final field
  c->spec_f_valid = true;
  for (int r : my_ranks(c)) launch_correct(slab(c, r), nullptr, nullptr, fq, nullptr, c->cval, s);
  DenseSrc D;
  D.base = c->spec_f;
  D.stencil_only = true;
  spectral2(c, c->cval, D, s);
  interp2(c, nullptr, fz, nullptr, false, out, s);
}

void final_field2(kfbi_ctx* c, const double* phi, const double* fgrid, const double* fq, double* u, cudaStream_t s) {
  const DevTables& T = c->T;
  BumpParams bp = c->bump;
  bp.a = c->ahole;
  launch_hole_coeffs(T, c->hole_off, c->hole_M, c->hole_delta, c->nh, phi, c->ahole, s);
  // dense source by linearity from the cached spectra: f̂ + Σ a_h ŵ_h, formed inside the sweep
  DenseSrc D;
  if (!fgrid || c->spec_f_valid) {
    D.base = fgrid ? c->spec_f : nullptr;
    D.nb = c->nh;
    D.bump = c->spec_bump;
    D.ldb = (long)c->spec_ld;
    D.coef = c->ahole;
    for (int h = 0; h < c->nh && h < 4; ++h) {   // bump h lives in |x − cx| < rad
      D.blo[h] = std::max(1, (int)std::floor((c->bump.cx[h] - c->bump.rad[h] - T.lo) / T.h) - 1);
      D.bhi[h] = std::min(T.N - 1, (int)std::ceil((c->bump.cx[h] + c->bump.rad[h] - T.lo) / T.h) + 1);
    }
    if (fgrid && c->world == 1) {
      // spec_f is not needed after the final field: add a_h ŵ_h into it on the bumps' support columns
      // only (in place, one fma per bump in order), then a base-only dense sweep
      for (int h = 0; h < c->nh && h < 4; ++h) {
        const size_t off = (size_t)(D.blo[h] - 1) * T.N;
        const long n = (long)(D.bhi[h] - D.blo[h] + 1) * T.N;
        launch_axpy_dcoef(n, c->ahole + h, c->spec_bump + (size_t)h * D.ldb + off, c->spec_f + off, s);
      }
      D.nb = 0;
    }
  } else {
    dst_forward2(c, fgrid, true, bp, c->spec_f, s);
    D.base = c->spec_f;
  }
  c->spec_f_valid = false;
  launch_spline(T, phi, c->mk, s);
  for (int r : my_ranks(c)) launch_correct(slab(c, r), phi, c->mk, fq, nullptr, c->cval, s);
  spectral2(c, c->cval, D, s);
  for (int r : my_ranks(c)) launch_inverse_dense(slab(c, r), c->spec, c->hsep, u, s, c->io_compact);   // owned columns
  if (c->local_io || c->io_compact) return;   // the box rows 0 and N belong to no slab / hold no Ω node
  const size_t W = (size_t)T.N + 1;
  ck(cudaMemsetAsync(u, 0, W * sizeof(double), s), "memset");
  ck(cudaMemsetAsync(u + (size_t)T.N * W, 0, W * sizeof(double), s), "memset");
}

// --- 3D interface solves (control points = intersection nodes, R12) -------------------
// rows: DST along z (source h²·f·1_Ω + compact corrections built on load), transpose, DST along y
// (from_work: the source is already in the working array, e.g. the test entry points)
void reduced3_dist(kfbi_ctx* c, cudaStream_t s);
// dense forward of the slab planes (all of them for world = 1 or the emulation): z-DST of the rows with
// the source built on load, transpose, y-DST, block sweeps, then the (distributed) reduced system
void forward3(kfbi_ctx* c, const double* fgrid, cudaStream_t s, bool from_work = false) {
  for (int r : my_ranks(c)) {
    const DevTables3 Ts = slab3(c, r);
    if (from_work) launch_dst_rows3(Ts, 0, c->work, nullptr, 1.0, nullptr, s);
    else launch_dst_rows3(Ts, 3, c->work, nullptr, 1.0, nullptr, s, fgrid, c->corr, c->io_compact && fgrid);
    launch_transpose3(Ts, c->work, s);
    launch_dst_rows3(Ts, 0, c->work, nullptr, 1.0, nullptr, s);
    launch_sweep3(Ts, c->work, c->zfirst, c->fsep, s);
  }
  reduced3_dist(c, s);
}
void inverse3(kfbi_ctx* c, double* u, cudaStream_t s) {   // u == NULL: result stays in work
  const double sc = 2.0 / c->T3.N;
  for (int r : my_ranks(c)) {
    const DevTables3 Ts = slab3(c, r);
    launch_dst_rows3(Ts, 1, c->work, c->hsep, sc, nullptr, s);
    launch_transpose3(Ts, c->work, s);
    if (!u) launch_dst_rows3(Ts, 0, c->work, nullptr, sc, nullptr, s);
    else launch_dst_rows3(Ts, 2, c->work, nullptr, sc, u, s, nullptr, nullptr, c->io_compact);   // the slab's planes of u
  }
  if (!u || c->io_compact) return;   // Ω-compact u: the box faces hold no Ω node
  const size_t W = (size_t)c->T3.N + 1;
  if (c->local_io) {   // the slab's planes: only their a = N faces (the box planes 0, N belong to no slab)
    const DevTables3 Ts = slab3(c, c->rank);
    ck(cudaMemset2DAsync(u + ((size_t)Ts.i_lo * W + c->T3.N) * W, W * W * sizeof(double), 0, W * sizeof(double),
                         Ts.i_hi - Ts.i_lo + 1, s), "memset");
    return;
  }
  ck(cudaMemsetAsync(u, 0, W * W * sizeof(double), s), "memset");
  ck(cudaMemsetAsync(u + (size_t)c->T3.N * W * W, 0, W * W * sizeof(double), s), "memset");
  ck(cudaMemset2DAsync(u + (W + c->T3.N) * W, W * W * sizeof(double), 0, W * sizeof(double), c->T3.N - 1, s), "memset");
}
// the slab's sparse inverse (y-rows, z at the stencil nodes) and the interpolation (partial sums of the
// slabs, all-reduced) — shared by the K_D and Y applies
void interp3_dist(kfbi_ctx* c, const double* phi, const double* fz, double* out, cudaStream_t s) {
  const DevTables3& T = c->T3;
  const double sc = 2.0 / T.N;
  for (int r : my_ranks(c)) {
    const DevTables3 Ts = slab3(c, r);
    launch_sparse3(Ts, 1, c->work, c->hsep, sc, c->work2, s);
    launch_sparse3(Ts, 2, c->work2, nullptr, sc, c->work, s);
  }
  if (c->world == 1) {
    launch_interp3(T, phi, c->dphi, fz, nullptr, c->work, out, s);
    return;
  }
  const int M = T.nq;
  if (c->use_nccl) {
    launch_interp3(slab3(c, c->rank), phi, c->dphi, fz, nullptr, c->work, c->parts, s, true);
    ckn(ncclAllReduce(c->parts, out, M, ncclDouble, ncclSum, c->comm, s), "allreduce");
    return;
  }
  for (int r : my_ranks(c))
    launch_interp3(slab3(c, r), phi, c->dphi, fz, nullptr, c->work, c->parts + (size_t)r * M, s, true);
  launch_sum_parts(M, c->world, c->parts, out, s);
}
// K_D (the GMRES operator): sparse source, sparse read-out — no dense z-direction transforms
// Multi-GPU: each rank runs the sparse forward, the block sweeps, the y-inverse
// and the z-evaluation of its own slab; the reduced system goes through reduced3_dist (below: slab-
// local elimination, mode-partitioned level-2 solve over two grouped all-to-alls), and the
// interpolation partial sums (plane owner contributes) are all-reduced.  rank = −1 emulates all slabs
// in one ctx.
// reduced (separator) system of the sweeps just run.  world > 1: every slab eliminates its interior
// separators and publishes 4 values per mode (first, last, its boundary separator's zA, its first
// block's zB); the level-2 system of the world − 1 slab separators is solved mode-partitioned (owner q
// of K/W modes; all-to-all of the 4 rows, all-to-all of the 2 rows each slab needs back: ≈ 6·K doubles
// sent per rank); every slab then fixes up its own interior separators.
void reduced3_dist(kfbi_ctx* c, cudaStream_t s) {
  const DevTables3& T = c->T3;
  if (c->world == 1) {
    launch_reduced3(T, c->zfirst, c->fsep, c->hsep, s);
    return;
  }
  const size_t W = c->world, K = (size_t)T.N * T.N, Kq = (K + W - 1) / W;
  if (c->use_nccl) {
    const int me = c->rank;
    const DevTables3 Ts = slab3(c, me);
    launch_red3_local(Ts, c->zfirst, c->fsep, c->hsep, c->seg3, (int)Kq, s);
    // all-to-all: owner q gets every slab's 4 rows of its modes
    ckn(ncclGroupStart(), "group");
    for (int q = 0; q < (int)W; ++q) {
      if (q == me) continue;
      ckn(ncclSend(c->seg3 + (size_t)q * 4 * Kq, 4 * Kq, ncclDouble, q, c->comm, s), "send seg");
      ckn(ncclRecv(c->seg3_in + (size_t)q * 4 * Kq, 4 * Kq, ncclDouble, q, c->comm, s), "recv seg");
    }
    ckn(ncclGroupEnd(), "group");
    ck(cudaMemcpyAsync(c->seg3_in + (size_t)me * 4 * Kq, c->seg3 + (size_t)me * 4 * Kq, 4 * Kq * sizeof(double),
                       cudaMemcpyDeviceToDevice, s), "self rows");
    launch_red3_solve(Ts, c->seg3_in, 4 * Kq, c->h3_out, 2 * Kq, (int)Kq, s);
    // all-to-all back: slab r gets (h_{r−1}, h_r) of every owner's modes
    ckn(ncclGroupStart(), "group");
    for (int r = 0; r < (int)W; ++r) {
      if (r == me) continue;
      ckn(ncclSend(c->h3_out + (size_t)r * 2 * Kq, 2 * Kq, ncclDouble, r, c->comm, s), "send h");
      ckn(ncclRecv(c->h3_in + (size_t)r * 2 * Kq, 2 * Kq, ncclDouble, r, c->comm, s), "recv h");
    }
    ckn(ncclGroupEnd(), "group");
    ck(cudaMemcpyAsync(c->h3_in + (size_t)me * 2 * Kq, c->h3_out + (size_t)me * 2 * Kq, 2 * Kq * sizeof(double),
                       cudaMemcpyDeviceToDevice, s), "self h");
    launch_red3_fixup(Ts, c->h3_in, c->hsep, (int)Kq, s);
    return;
  }
  // emulation (every slab in this context): the exchanges are strided reads of the other slabs' buffers —
  // owner q reads slab r's rows at seg3[r][q] (stride W·4·Kq) and writes slab r's rows to h3_in[r][q]
  for (int r = 0; r < (int)W; ++r)
    launch_red3_local(slab3(c, r), c->zfirst, c->fsep, c->hsep, c->seg3 + (size_t)r * W * 4 * Kq, (int)Kq, s);
  for (int q = 0; q < (int)W; ++q)
    launch_red3_solve(slab3(c, q), c->seg3 + (size_t)q * 4 * Kq, W * 4 * Kq, c->h3_in + (size_t)q * 2 * Kq,
                      W * 2 * Kq, (int)Kq, s);
  for (int r = 0; r < (int)W; ++r) launch_red3_fixup(slab3(c, r), c->h3_in + (size_t)r * W * 2 * Kq, c->hsep, (int)Kq, s);
}

void apply_KD3(kfbi_ctx* c, const double* phi, double* out, cudaStream_t s) {
  for (int r : my_ranks(c)) {   // the slab's control points and irregular nodes only
    const DevTables3 Ts = slab3(c, r);
    launch_lsq3(Ts, phi, c->dphi, s);
    launch_correct3(Ts, phi, c->dphi, nullptr, nullptr, nullptr, s, c->corr);
  }
  for (int r : my_ranks(c)) {
    const DevTables3 Ts = slab3(c, r);
    launch_sparse3(Ts, 0, c->corr, nullptr, 1.0, c->work, s);
    launch_sweep3(Ts, c->work, c->zfirst, c->fsep, s, true);
  }
  reduced3_dist(c, s);
  interp3_dist(c, phi, nullptr, out, s);
}
void apply_Y3(kfbi_ctx* c, const double* fgrid, const double* fq, const double* fz, double* out, cudaStream_t s) {
  for (int r : my_ranks(c)) launch_correct3(slab3(c, r), nullptr, nullptr, fq, nullptr, nullptr, s, c->corr);
  forward3(c, fgrid, s);
  interp3_dist(c, nullptr, fz, out, s);   // only the stencil nodes are read
}
void final_field3(kfbi_ctx* c, const double* phi, const double* fgrid, const double* fq, double* u, cudaStream_t s) {
  for (int r : my_ranks(c)) {
    const DevTables3 Ts = slab3(c, r);
    launch_lsq3(Ts, phi, c->dphi, s);
    launch_correct3(Ts, phi, c->dphi, fq, nullptr, nullptr, s, c->corr);
  }
  forward3(c, fgrid, s);
  inverse3(c, u, s);
}

void apply_KD(kfbi_ctx* c, const double* phi, double* out, cudaStream_t s) {
  if (c->dim == 3) apply_KD3(c, phi, out, s);
  else apply_KD2(c, phi, out, s);
}
void apply_Y(kfbi_ctx* c, const double* fgrid, const double* fq, const double* fz, double* out, cudaStream_t s) {
  if (c->dim == 3) apply_Y3(c, fgrid, fq, fz, out, s);
  else apply_Y2(c, fgrid, fq, fz, out, s);
}
void final_field(kfbi_ctx* c, const double* phi, const double* fgrid, const double* fq, double* u, cudaStream_t s) {
  if (c->dim == 3) final_field3(c, phi, fgrid, fq, u, s);
  else final_field2(c, phi, fgrid, fq, u, s);
}

}  // namespace

extern "C" {

const char* kfbi_version(void) { return "kfbi-b200 0.1 (sm_100a, 2D)"; }
const char* kfbi_last_error(const kfbi_ctx* ctx) { return ctx ? ctx->err.c_str() : g_setup_err.c_str(); }
const char* kfbi_last_setup_error(void) { return g_setup_err.c_str(); }

kfbi_status kfbi_get_unique_id(void* out128) {
  if (!out128) return KFBI_EINVAL;
  ncclUniqueId id;
  const ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) {
    g_setup_err = std::string("ncclGetUniqueId: ") + ncclGetErrorString(r);
    return KFBI_ENCCL;
  }
  std::memcpy(out128, &id, sizeof(id));
  return KFBI_OK;
}

namespace {
kfbi_status setup_impl(const kfbi_grid* grid, const kfbi_boundary* bnd, const kfbi_pde* pde,
                       const kfbi_dist* dist, void* stream, const DeviceScratch* dev, kfbi_ctx** out) {
  if (!out) return KFBI_EINVAL;
  *out = nullptr;
  auto* c = new kfbi_ctx();
  try {
    if (dist && dist->world > 1) {
      c->world = dist->world;
      c->rank = dist->rank;
      if (c->rank < -1 || c->rank >= c->world) throw ArgError("bad rank");
      if (c->rank >= 0 && dist->nccl_id) {
        c->use_nccl = true;
        std::memcpy(&c->nccl_id, dist->nccl_id, sizeof(ncclUniqueId));
      }
    }
    if (!grid || !bnd || !pde || !bnd->comp) throw ArgError("null descriptor");
    c->dim = grid->dim;
    if (c->dim == 3) build_setup3(c->S3, grid, bnd, pde, dev);
    else build_setup(c->S, grid, bnd, pde, dev);
    if (c->world > 1) {
      if (c->dim == 3) {
        if (c->S3.P < c->world || c->S3.P % c->world) throw ArgError("3D: world must divide N/16 (slabs = ADM blocks)");
        level2_tables3(c->S3, c->S3.P / c->world - 1);
      } else {
        const int nseg = c->S.P >= 2 * BL2 ? c->S.P / BL2 : 1;
        if (nseg < c->world || nseg % c->world) throw ArgError("world must divide N/512 (slabs = level-2 segments)");
      }
    }
    c->stream = (cudaStream_t)stream;
    c->device = (dist && dist->device >= 0) ? dist->device : 0;
    if (!dist || dist->device < 0) cudaGetDevice(&c->device);
    Arena A{nullptr, 0, false};
    if (c->dim == 3) layout3(c, A);
    else layout(c, A);
    c->ws_need = A.off + 256;
    c->bump.nh = c->nh;
    for (int h = 0; h < c->nh && h < 4; ++h) {
      const Comp& C = c->S.comps[c->S.holes[h]];
      c->bump.cx[h] = C.c[0];
      c->bump.cy[h] = C.c[1];
      c->bump.rad[h] = 0.5 * std::min(C.p[0], C.p[1]);
    }
    if (c->nh > 4) throw ArgError("at most 4 holes");
  } catch (const GeomError& e) {
    g_setup_err = e.what();
    delete c;
    return KFBI_EGEOM;
  } catch (const UnsupportedError& e) {
    g_setup_err = e.what();
    delete c;
    return KFBI_EUNSUPPORTED;
  } catch (const DeviceError& e) {
    g_setup_err = e.what();
    delete c;
    return KFBI_ECUDA;
  } catch (const ScratchError& e) {
    g_setup_err = e.what();
    delete c;
    return KFBI_ENOMEM;
  } catch (const std::exception& e) {
    g_setup_err = e.what();
    delete c;
    return KFBI_EINVAL;
  }
  *out = c;
  return KFBI_OK;
}

}  // namespace

kfbi_status kfbi_setup(const kfbi_grid* grid, const kfbi_boundary* bnd, const kfbi_pde* pde,
                       const kfbi_dist* dist, void* stream, kfbi_ctx** out) {
  return setup_impl(grid, bnd, pde, dist, stream, nullptr, out);
}

kfbi_status kfbi_setup_scratch_size(const kfbi_grid* grid, size_t* bytes) {
  if (!grid || !bytes) return KFBI_EINVAL;
  *bytes = 0;
  const int N = grid->n[0];
  if (grid->dim == 3) {
    if (N < 32 || N > 512 || (N & (N - 1))) {
      g_setup_err = "3D: n must be a power of two in [32, 512]";
      return KFBI_EINVAL;
    }
    *bytes = gpu_setup_scratch_bytes3(N);
    return KFBI_OK;
  }
  if (grid->dim != 2) {
    g_setup_err = "dim must be 2 or 3";
    return KFBI_EINVAL;
  }
  if (N < 64 || N > 8192 || (N & (N - 1))) {
    g_setup_err = "n must be a power of two in [64, 8192]";
    return KFBI_EINVAL;
  }
  *bytes = gpu_setup_scratch_bytes(N);
  return KFBI_OK;
}

kfbi_status kfbi_setup_device(const kfbi_grid* grid, const kfbi_boundary* bnd, const kfbi_pde* pde,
                              const kfbi_dist* dist, void* stream, void* d_scratch, size_t bytes,
                              kfbi_ctx** out) {
  if (!out) return KFBI_EINVAL;
  *out = nullptr;
  if (!grid || (grid->dim != 2 && grid->dim != 3)) {
    g_setup_err = "dim must be 2 or 3";
    return KFBI_EINVAL;
  }
  if (!d_scratch) {
    g_setup_err = "null device scratch";
    return KFBI_EINVAL;
  }
  if (dist && dist->device >= 0) cudaSetDevice(dist->device);
  const DeviceScratch dev{d_scratch, bytes, (cudaStream_t)stream};
  return setup_impl(grid, bnd, pde, dist, stream, &dev, out);
}

kfbi_status kfbi_slab(const kfbi_ctx* c, int32_t rank, int64_t* out) {
  if (!c || !out || rank < 0 || rank >= c->world) return KFBI_EINVAL;
  if (c->dim == 3) {
    const DevTables3 T = slab3(c, rank);
    const int64_t v[6] = {T.b_lo, T.b_hi, T.i_lo, T.i_hi, T.w_lo, T.w_hi};
    for (int q = 0; q < 6; ++q) out[q] = v[q];
    return KFBI_OK;
  }
  const DevTables T = slab(c, rank);
  const int64_t v[6] = {T.g_lo, T.g_hi, T.col_lo, T.col_hi, T.o_lo, T.o_hi};
  for (int q = 0; q < 6; ++q) out[q] = v[q];
  return KFBI_OK;
}

kfbi_status kfbi_workspace_size(const kfbi_ctx* ctx, size_t* bytes) {
  if (!ctx || !bytes) return KFBI_EINVAL;
  *bytes = ctx->ws_need;
  return KFBI_OK;
}

void drop_step_graphs(kfbi_ctx* c) {
  for (auto& g : c->step_graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  c->step_graphs.clear();
}

kfbi_status kfbi_set_workspace(kfbi_ctx* c, void* d_ws, size_t bytes) {
  if (!c || !d_ws) return KFBI_EINVAL;
  if (bytes < c->ws_need) return fail(c, KFBI_ENOMEM, "workspace too small");
  if (((uintptr_t)d_ws) & 255) return fail(c, KFBI_EINVAL, "workspace must be 256-byte aligned");
  KFBI_TRY(c)
  drop_step_graphs(c);   // captured pointers refer to the previous workspace
  c->ws = (uint8_t*)d_ws;
  c->ws_bytes = bytes;
  Arena A{c->ws, 0, true};
  if (c->dim == 3) layout3(c, A);
  else layout(c, A);
  cudaStream_t s = c->stream;
  for (auto& u : A.uploads) ck(cudaMemcpyAsync(u.first, u.second.first, u.second.second, cudaMemcpyHostToDevice, s), "upload");
  if (!c->hcol_host) {
    ck(cudaHostAlloc(&c->hcol_host, (size_t)(kMaxRestart + 1) * (kMaxRestart + 2) * sizeof(double),
                     cudaHostAllocMapped), "cudaHostAlloc");
    ck(cudaHostGetDevicePointer((void**)&c->hcol_map, c->hcol_host, 0), "cudaHostGetDevicePointer");
    for (auto& e : c->ev_step) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  }
  if (c->use_nccl && !c->comm) {   // a second kfbi_set_workspace keeps the communicator
    ckn(ncclCommInitRank(&c->comm, c->world, c->nccl_id, c->rank), "ncclCommInitRank");
  }
  // hole completion fields w_h|Γ (reading R27): plain fast solve of the bump, no jumps
  for (int h = 0; h < c->nh; ++h) {
    BumpParams bp = c->bump;
    bp.a = c->onehot + (size_t)h * c->nh;
    const long nspec = (long)c->spec_ld;
    dst_forward2(c, nullptr, false, bp, c->spec_bump + (size_t)h * nspec, s);
    DenseSrc D;
    D.base = c->spec_bump + (size_t)h * nspec;
    D.stencil_only = true;
    spectral2(c, nullptr, D, s);
    interp2(c, nullptr, nullptr, nullptr, false, c->wg + (size_t)h * c->S.M, s);
  }
  ck(cudaGetLastError(), "setup kernels");
  ck(cudaStreamSynchronize(s), "setup sync");
  KFBI_CATCH(c)
  return KFBI_OK;
}

kfbi_status kfbi_sizes(const kfbi_ctx* c, int64_t* M, int64_t* nq, int64_t* nirr, int64_t* nn) {
  if (!c) return KFBI_EINVAL;
  if (c->dim == 3) {
    const int64_t W = c->S3.N + 1;
    if (M) *M = c->S3.nq;
    if (nq) *nq = c->S3.nq;
    if (nirr) *nirr = c->S3.nirr;
    if (nn) *nn = W * W * W;
    return KFBI_OK;
  }
  if (M) *M = c->S.M;
  if (nq) *nq = c->S.nq;
  if (nirr) *nirr = c->S.nirr;
  if (nn) *nn = (int64_t)(c->S.N + 1) * (c->S.N + 1);
  return KFBI_OK;
}

kfbi_status kfbi_local_slab(const kfbi_ctx* c, int64_t local_shape[3], int64_t local_offset[3]) {
  if (!c || !local_shape || !local_offset) return KFBI_EINVAL;
  for (int a = 0; a < 3; ++a) {
    local_shape[a] = c->loc_shape[a];
    local_offset[a] = c->loc_off[a];
  }
  return KFBI_OK;
}

kfbi_status kfbi_points(const kfbi_ctx* c, int32_t which, double* xyz) {
  if (!c || !xyz) return KFBI_EINVAL;
  if (c->dim == 3) {
    if (which == 2) {   // outward unit normals at the control points
      std::memcpy(xyz, c->S3.q_n.data(), c->S3.q_n.size() * sizeof(double));
      return KFBI_OK;
    }
    if (which != 0 && which != 1) return KFBI_EINVAL;
    std::memcpy(xyz, c->S3.q_pos.data(), c->S3.q_pos.size() * sizeof(double));
    return KFBI_OK;
  }
  const Setup& S = c->S;
  if (which == 0) {
    for (int m = 0; m < S.M; ++m) { xyz[2 * m] = S.z_x[m]; xyz[2 * m + 1] = S.z_y[m]; }
  } else if (which == 2) {   // outward unit normals n = (τ2, −τ1) at the control points (R8)
    for (int m = 0; m < S.M; ++m) { xyz[2 * m] = S.z_t2[m]; xyz[2 * m + 1] = -S.z_t1[m]; }
  } else if (which == 1) {
    for (int q = 0; q < S.nq; ++q) { xyz[2 * q] = S.q_x[q]; xyz[2 * q + 1] = S.q_y[q]; }
  } else {
    return KFBI_EINVAL;
  }
  return KFBI_OK;
}

kfbi_status kfbi_node_mask(const kfbi_ctx* c, int8_t* mask) {
  if (!c || !mask) return KFBI_EINVAL;
  const auto& sd = c->dim == 3 ? c->S3.side : c->S.side;
  std::memcpy(mask, sd.data(), sd.size());
  return KFBI_OK;
}

kfbi_status kfbi_node_mask_device(kfbi_ctx* c, int8_t* d_mask, void* stream) {
  if (!c || !d_mask) return fail(c, KFBI_EINVAL, "null pointer");
  KFBI_TRY(c)
  need_ws(c);
  const size_t row = c->dim == 3 ? (size_t)(c->S3.N + 1) * (c->S3.N + 1) : (size_t)c->S.N + 1;
  const size_t off = (size_t)c->loc_off[0] * row;
  const size_t n = (size_t)c->loc_shape[0] * row;
  ck(cudaMemcpyAsync(d_mask, c->d_side + off, n, cudaMemcpyDeviceToDevice, pick(c, stream)), "mask copy");
  KFBI_CATCH(c)
  return KFBI_OK;
}

kfbi_status kfbi_omega_count(const kfbi_ctx* c, int64_t* n_omega) {
  if (!c || !n_omega || c->om_ptr.empty()) return KFBI_EINVAL;
  *n_omega = c->om_ptr.back();
  return KFBI_OK;
}

kfbi_status kfbi_scatter_omega(kfbi_ctx* c, const double* d_compact, double* d_grid, void* stream) {
  if (!c || !d_compact || !d_grid) return fail(c, KFBI_EINVAL, "null pointer");
  if (c->local_io) return fail(c, KFBI_EUNSUPPORTED, "Omega transfers are full-grid (world = 1 or the emulation)");
  KFBI_TRY(c)
  need_ws(c);
  launch_omega_map(c->om_rows, c->om_width, c->d_side, c->d_om_seg, d_compact, d_grid, true, pick(c, stream));
  ck(cudaGetLastError(), "kfbi_scatter_omega launch");
  KFBI_CATCH(c)
  return KFBI_OK;
}

kfbi_status kfbi_gather_omega(kfbi_ctx* c, const double* d_grid, double* d_compact, void* stream) {
  if (!c || !d_compact || !d_grid) return fail(c, KFBI_EINVAL, "null pointer");
  if (c->local_io) return fail(c, KFBI_EUNSUPPORTED, "Omega transfers are full-grid (world = 1 or the emulation)");
  KFBI_TRY(c)
  need_ws(c);
  launch_omega_map(c->om_rows, c->om_width, c->d_side, c->d_om_seg, d_grid, d_compact, false, pick(c, stream));
  ck(cudaGetLastError(), "kfbi_gather_omega launch");
  KFBI_CATCH(c)
  return KFBI_OK;
}

kfbi_status kfbi_apply(kfbi_ctx* c, const double* d_phi, double* d_out, void* stream) {
  if (!c || !d_phi || !d_out) return fail(c, KFBI_EINVAL, "null pointer");
  KFBI_TRY(c)
  need_ws(c);
  apply_KD(c, d_phi, d_out, pick(c, stream));
  ck(cudaGetLastError(), "kfbi_apply launch");
  KFBI_CATCH(c)
  return KFBI_OK;
}

// ---- Richardson and BiCGSTAB drivers (reading R39) over the same apply ----
// scalars leave the device through the host-mapped buffer (no copy engine), one sync per batch
namespace {
void dots(kfbi_ctx* c, int n, const double* const* a, const double* const* b, const bool* take_sqrt, double* out,
          cudaStream_t s) {
  const int M = nctrl(c);
  for (int q = 0; q < n; ++q) {
    launch_dot(M, a[q], b[q], c->partial + (size_t)q * kRedBlocks, s);
    launch_finish_sum(c->partial + (size_t)q * kRedBlocks, c->scal + q, take_sqrt[q], s);
  }
  launch_copy(n, c->scal, c->hcol_map, s);
  ck(cudaStreamSynchronize(s), "sync scalars");
  for (int q = 0; q < n; ++q) out[q] = c->hcol_host[q];
}
double norm2(kfbi_ctx* c, const double* a, cudaStream_t s) {
  const double* av[1] = {a};
  const bool sq[1] = {true};
  double v;
  dots(c, 1, av, av, sq, &v, s);
  return v;
}
void axpy(kfbi_ctx* c, double alpha, const double* xv, double* y, cudaStream_t s) {   // y += α x
  launch_axpy_basis(nctrl(c), 1, xv, nctrl(c), &alpha, y, s);
}

// φ_{k+1} = φ_k + γ(ĝ − Kφ_k), explicit residual every iteration, ‖r‖ ≤ tol‖r₀‖
bool solve_richardson(kfbi_ctx* c, const kfbi_solve_opts& o, bool have_x0, kfbi_solve_stats& st, cudaStream_t s) {
  const int M = nctrl(c), max_iter = o.restart * o.max_restarts;
  double r0 = -1.0;
  for (int it = 0; it <= max_iter; ++it) {
    if (!have_x0 && it == 0) {
      launch_copy(M, c->ghat, c->gr, s);
    } else {
      apply_KD(c, c->gx, c->tmp, s);
      st.n_applies++;
      launch_sub(M, c->ghat, c->tmp, c->gr, s);
    }
    const double nr = norm2(c, c->gr, s);
    if (!std::isfinite(nr)) throw BreakdownError("non-finite residual");
    if (r0 < 0) r0 = nr;
    st.rel_residual = r0 > 0 ? nr / r0 : 0.0;
    if (nr <= o.tol * r0 || r0 == 0.0) return true;
    if (it == max_iter) break;
    axpy(c, o.gamma, c->gr, c->gx, s);
    st.iters++;
  }
  return false;
}

// BiCGSTAB (van der Vorst 1992), shadow residual r̂ = r₀; vectors in the GMRES basis storage
bool solve_bicgstab(kfbi_ctx* c, const kfbi_solve_opts& o, bool have_x0, kfbi_solve_stats& st, cudaStream_t s) {
  const int M = nctrl(c), max_iter = o.restart * o.max_restarts;
  double *rhat = c->V, *r = c->V + M, *p = c->V + 2 * (size_t)M, *v = c->V + 3 * (size_t)M,
         *sv = c->V + 4 * (size_t)M, *t = c->V + 5 * (size_t)M;
  if (!have_x0) {
    launch_copy(M, c->ghat, r, s);
  } else {
    apply_KD(c, c->gx, c->tmp, s);
    st.n_applies++;
    launch_sub(M, c->ghat, c->tmp, r, s);
  }
  launch_copy(M, r, rhat, s);
  const double n0 = norm2(c, r, s);
  if (!std::isfinite(n0)) throw BreakdownError("non-finite residual");
  st.rel_residual = n0 > 0 ? 1.0 : 0.0;
  if (n0 == 0.0) return true;
  double rho_prev = 1.0, alpha = 1.0, omega = 1.0;
  const bool no_sqrt[2] = {false, false};
  for (int it = 0; it < max_iter; ++it) {
    double rho;
    {
      const double* a[1] = {rhat};
      const double* b[1] = {r};
      dots(c, 1, a, b, no_sqrt, &rho, s);
    }
    const double beta = (rho / rho_prev) * (alpha / omega);
    if (it == 0) {
      launch_copy(M, r, p, s);                       // p = r (p = v = 0 before)
    } else {                                         // p = r + β(p − ω v)
      launch_copy(M, r, c->tmp, s);
      axpy(c, beta, p, c->tmp, s);
      axpy(c, -beta * omega, v, c->tmp, s);
      launch_copy(M, c->tmp, p, s);
    }
    apply_KD(c, p, v, s);
    st.n_applies++;
    double rv;
    {
      const double* a[1] = {rhat};
      const double* b[1] = {v};
      dots(c, 1, a, b, no_sqrt, &rv, s);
    }
    alpha = rho / rv;
    launch_copy(M, r, sv, s);                        // s = r − α v
    axpy(c, -alpha, v, sv, s);
    st.iters++;
    const double ns = norm2(c, sv, s);
    if (!std::isfinite(ns)) throw BreakdownError("non-finite BiCGSTAB residual");
    if (ns <= o.tol * n0) {
      axpy(c, alpha, p, c->gx, s);
      st.rel_residual = ns / n0;
      return true;
    }
    apply_KD(c, sv, t, s);
    st.n_applies++;
    double ts_tt[2];
    {
      const double* a[2] = {t, t};
      const double* b[2] = {sv, t};
      dots(c, 2, a, b, no_sqrt, ts_tt, s);
    }
    omega = ts_tt[0] / ts_tt[1];
    axpy(c, alpha, p, c->gx, s);                     // x += α p + ω s
    axpy(c, omega, sv, c->gx, s);
    launch_copy(M, sv, r, s);                        // r = s − ω t
    axpy(c, -omega, t, r, s);
    rho_prev = rho;
    const double nr = norm2(c, r, s);
    st.rel_residual = nr / n0;
    if (nr <= o.tol * n0) return true;
  }
  return false;
}
}  // namespace

kfbi_status kfbi_solve(kfbi_ctx* c, const double* d_g, const double* d_f_grid, const double* d_f_isect,
                       const double* d_f_ctrl, const double* d_phi0, double* d_u, double* d_phi_out,
                       const kfbi_solve_opts* opts, kfbi_solve_stats* stats, void* stream) {
  if (!c || !d_g || !d_u) return fail(c, KFBI_EINVAL, "null pointer");
  if ((d_f_grid == nullptr) != (d_f_isect == nullptr) || (d_f_grid == nullptr) != (d_f_ctrl == nullptr))
    return fail(c, KFBI_EINVAL, "f_grid, f_isect, f_ctrl must all be given or all NULL");
  kfbi_solve_opts o{1e-8, 30, 50, KFBI_GMRES, 1.0, 0, 0};
  if (opts) o = *opts;
  if (o.omega_io && (c->local_io || c->world != 1))
    return fail(c, KFBI_EUNSUPPORTED, "omega_io: single-context grids only");
  if (o.restart < 1 || o.restart > kMaxRestart || o.max_restarts < 1 || !(o.tol > 0) || o.method < 0 ||
      o.method > KFBI_BICGSTAB || (o.method == KFBI_RICHARDSON && !(o.gamma > 0 && o.gamma <= 1)))
    return fail(c, KFBI_EINVAL, "bad solve options");
  kfbi_solve_stats st{};
  auto t0 = std::chrono::steady_clock::now();
  bool converged = false;
  KFBI_TRY(c)
  need_ws(c);
  struct CompactIO {   // f and u Ω-compact for this solve only (reset on every exit path)
    kfbi_ctx* c;
    CompactIO(kfbi_ctx* c_, bool on) : c(c_) { c->io_compact = on; }
    ~CompactIO() { c->io_compact = false; }
  } compact_io(c, o.omega_io != 0);
  if (c->local_io) {   // the rank's node slab: the kernels index with global node numbers
    const size_t row = c->dim == 3 ? (size_t)(c->S3.N + 1) * (c->S3.N + 1) : (size_t)c->S.N + 1;
    if (d_f_grid) d_f_grid -= (size_t)c->loc_off[0] * row;
    d_u -= (size_t)c->loc_off[0] * row;
  }
  cudaStream_t s = pick(c, stream);
  const int M = nctrl(c);
  const size_t bM = (size_t)M * sizeof(double);
  // ĝ = g − (Yf)⁺
  if (d_f_grid) {
    apply_Y(c, d_f_grid, d_f_isect, d_f_ctrl, c->tmp, s);
    st.n_applies++;
    launch_sub(M, d_g, c->tmp, c->ghat, s);
  } else {
    launch_copy(M, d_g, c->ghat, s);
  }
  // GMRES(m), Algorithm 5, reading R18
  if (d_phi0) launch_copy(M, d_phi0, c->gx, s);
  else ck(cudaMemsetAsync(c->gx, 0, bM, s), "zero x");
  if (o.method != KFBI_GMRES) {
    converged = o.method == KFBI_RICHARDSON ? solve_richardson(c, o, d_phi0 != nullptr, st, s)
                                            : solve_bicgstab(c, o, d_phi0 != nullptr, st, s);
  } else {
  double beta0 = -1.0;
  std::vector<double> H((size_t)(o.restart + 1) * o.restart), cs(o.restart), sn(o.restart), gv(o.restart + 1), y(o.restart);
  auto Hc = [&](int i, int j) -> double& { return H[(size_t)i * o.restart + j]; };
  for (int cycle = 0; cycle <= o.max_restarts; ++cycle) {
    // r = ĝ − K x  (explicit residual; skipped for x₀ = 0 on the first cycle)
    if (!d_phi0 && cycle == 0) {
      launch_copy(M, c->ghat, c->gr, s);
    } else {
      apply_KD(c, c->gx, c->tmp, s);
      st.n_applies++;
      launch_sub(M, c->ghat, c->tmp, c->gr, s);
    }
    launch_dot(M, c->gr, c->gr, c->partial, s);
    launch_finish_sum(c->partial, c->scal, true, s);
    launch_copy(1, c->scal, c->hcol_map, s);   // β into host-mapped memory (no copy engine)
    ck(cudaStreamSynchronize(s), "sync beta");
    const double beta = c->hcol_host[0];
    if (!std::isfinite(beta)) throw BreakdownError("non-finite residual");
    if (beta0 < 0) beta0 = beta;
    st.rel_residual = beta0 > 0 ? beta / beta0 : 0.0;
    if (beta <= o.tol * beta0 || beta0 == 0.0) { converged = true; break; }
    if (cycle == o.max_restarts) break;
    st.restarts = cycle + 1;
    launch_scale_copy(M, c->gr, c->scal, c->V, s);   // V_0 = r / β
    std::fill(gv.begin(), gv.end(), 0.0);
    gv[0] = beta;
    int jlast = o.restart - 1;
    // Arnoldi step j on the device: K v_j → w, MGS (deterministic reductions; one fused
    // cluster for small M) → the Hessenberg column into mapped slot j.  The host runs one step behind:
    // step j + 1 (whose input v_{j+1} is step j's MGS output, already on the stream) is enqueued before
    // the host waits for step j and does its Givens update, unless the residual history predicts that
    // step j converges — so the GPU does not idle through the per-step host round trip, nor
    // through its mapped write when PCIe is busy with the serving loop's copies.  A step enqueued past
    // convergence (mispredicted) changes nothing the solution reads and is not counted.
    auto slot = [&](int j) { return (size_t)(kMaxRestart + 2) * (size_t)(j + 1); };
    auto step_body = [&](int j) {
      double* w = c->V + (size_t)(j + 1) * M;
      apply_KD(c, c->V + (size_t)j * M, w, s);
      if (!launch_mgs_fused(M, j, c->V, w, c->hcol, s)) {
      for (int i = 0; i <= j; ++i)
        launch_mgs_step(M, w, i ? c->V + (size_t)(i - 1) * M : nullptr, c->V + (size_t)i * M,
                        i ? c->partial + (size_t)(i - 1) * kRedBlocks : nullptr, c->partial + (size_t)i * kRedBlocks,
                        i ? c->hcol + (i - 1) : nullptr, s);
      launch_mgs_step(M, w, c->V + (size_t)j * M, w, c->partial + (size_t)j * kRedBlocks,
                      c->partial + (size_t)(j + 1) * kRedBlocks, c->hcol + j, s);
      launch_norm_scale(M, w, c->partial + (size_t)(j + 1) * kRedBlocks, c->hcol + j + 1, s);
      }
      launch_copy(j + 2, c->hcol, c->hcol_map + slot(j), s);
    };
    auto enqueue_step = [&](int j) {
      if (!c->use_nccl && !c->graphs_off) {
        if ((int)c->step_graphs.size() <= j) c->step_graphs.resize(kMaxRestart);
        auto& g = c->step_graphs[j];
        if (!g.exec) {   // capture once; on any capture failure fall back to eager launches for good
          const long long l0 = g_launches;
          cudaGraph_t graph = nullptr;
          bool ok = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
          if (ok) {
            try {
              step_body(j);
            } catch (...) {
              ok = false;
            }
            ok = cudaStreamEndCapture(s, &graph) == cudaSuccess && ok;
            ok = ok && graph && cudaGraphInstantiate(&g.exec, graph, 0) == cudaSuccess;
            if (graph) cudaGraphDestroy(graph);
          }
          g.launches = g_launches - l0;
          g_launches = l0;
          if (!ok) {
            cudaGetLastError();
            if (g.exec) cudaGraphExecDestroy(g.exec);
            g.exec = nullptr;
            c->graphs_off = true;
          }
        }
        if (g.exec) {
          ck(cudaGraphLaunch(g.exec, s), "graph launch");
          g_launches += g.launches;
          ck(cudaEventRecord(c->ev_step[j & 1], s), "record step");
          return;
        }
      }
      step_body(j);
      ck(cudaEventRecord(c->ev_step[j & 1], s), "record step");
    };
    int enq = 1;           // steps enqueued in this cycle
    double rho = 0.25;     // fastest residual reduction per step seen in this cycle (prediction)
    enqueue_step(0);
    for (int j = 0; j < o.restart; ++j) {
      // speculate step j + 1 when the predicted residual after step j stays well above the target
      const bool spec = enq == j + 1 && j + 1 < o.restart && std::fabs(gv[j]) * rho > 16.0 * o.tol * beta0;
      if (spec) {
        enqueue_step(j + 1);
        enq = j + 2;
      }
      ck(cudaEventSynchronize(c->ev_step[j & 1]), "sync hcol");
      st.iters++;
      st.n_applies++;
      const double* hc = c->hcol_host + slot(j);
      for (int i = 0; i <= j + 1; ++i) Hc(i, j) = hc[i];
      for (int i = 0; i < j; ++i) {   // previous Givens rotations
        const double a = Hc(i, j), b = Hc(i + 1, j);
        Hc(i, j) = cs[i] * a + sn[i] * b;
        Hc(i + 1, j) = -sn[i] * a + cs[i] * b;
      }
      const double hnext = Hc(j + 1, j);
      const double rr = std::hypot(Hc(j, j), hnext);
      cs[j] = Hc(j, j) / rr;
      sn[j] = hnext / rr;
      Hc(j, j) = rr;
      Hc(j + 1, j) = 0.0;
      const double gj = gv[j];
      gv[j + 1] = -sn[j] * gv[j];
      gv[j] = cs[j] * gv[j];
      if (!std::isfinite(gv[j + 1])) throw BreakdownError("non-finite GMRES residual");
      if (std::fabs(gv[j + 1]) <= o.tol * beta0 || hnext <= 1e-14 * beta0) { jlast = j; break; }
      if (gj != 0.0) rho = std::min(rho, std::fabs(gv[j + 1] / gj));
      if (enq == j + 1 && j + 1 < o.restart) {   // not speculated: enqueue step j + 1 now
        enqueue_step(j + 1);
        enq = j + 2;
      }
    }
    const int k = jlast + 1;
    for (int i = k - 1; i >= 0; --i) {
      double sacc = gv[i];
      for (int q = i + 1; q < k; ++q) sacc -= Hc(i, q) * y[q];
      y[i] = sacc / Hc(i, i);
    }
    launch_axpy_basis(M, k, c->V, M, y.data(), c->gx, s);   // φ_m = φ_0 + M_m y_m
  }
  }
  if (d_phi_out) launch_copy(M, c->gx, d_phi_out, s);
  // final field u = Wφ + Yf (+ Σ a_h w_h) (R27)
  final_field(c, c->gx, d_f_grid, d_f_isect, d_u, s);
  st.n_applies++;
  ck(cudaGetLastError(), "solve kernels");
  if (!o.async_final) ck(cudaStreamSynchronize(s), "solve sync");
  KFBI_CATCH(c)
  st.converged = converged ? 1 : 0;
  st.t_solve_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (stats) *stats = st;
  return converged ? KFBI_OK : fail(c, KFBI_ENOCONV, "GMRES did not converge");
}

kfbi_status kfbi_apply_model(const kfbi_ctx* c, double* bytes_sweep, double* bytes_inverse, double* unknowns) {
  if (!c) return KFBI_EINVAL;
  if (c->dim == 3) {
    const double N = c->S3.N, U = (N - 1) * (N - 1) * (N - 1);
    double nf = 0, ni = 0;   // planes with irregular nodes (non-zero source) / with stencil rows
    for (size_t i = 1; i < c->S3.plane_flags.size(); ++i) {
      nf += c->S3.plane_flags[i] & 1;
      ni += (c->S3.plane_flags[i] >> 1) & 1;
    }
    // k_fwd3s: writes the spectrum of the planes with a non-zero sparse source (computed on chip)
    if (bytes_sweep) *bytes_sweep = 8.0 * nf * N * N;
    // k_inv3y: reads the spectrum of the planes with stencil rows, writes the y-inverse rows that hold
    // stencil nodes
    if (bytes_inverse) *bytes_inverse = 8.0 * ni * N * N + 8.0 * N * (double)c->S3.zrow_id.size();
    if (unknowns) *unknowns = U;
    return KFBI_OK;
  }
  const double N = c->S.N;
  // distinct grid columns holding stencil nodes; those inside ADM blocks (not separators) are the
  // spectral rows the sparse apply's sweep stores (8 B per mode) and its inverse reads
  std::vector<int32_t> cols(c->S.sn_i.begin(), c->S.sn_i.end());
  std::sort(cols.begin(), cols.end());
  cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
  double ncol = 0, nblk = 0;
  for (int32_t i : cols) {
    ncol += 1;
    nblk += (i % BL) != 0;
  }
  if (bytes_sweep) *bytes_sweep = 8.0 * nblk * (N - 1);
  if (bytes_inverse) *bytes_inverse = 8.0 * ncol * (N - 1);
  if (unknowns) *unknowns = (N - 1) * (N - 1);
  return KFBI_OK;
}

kfbi_status kfbi_profile_apply(kfbi_ctx* c, const double* d_phi, double* d_out, int32_t reps, double* ms,
                               void* stream) {
  if (!c || !d_phi || !d_out || !ms || reps < 1) return fail(c, KFBI_EINVAL, "bad arguments");
  KFBI_TRY(c)
  need_ws(c);
  cudaStream_t s = pick(c, stream);
  const DevTables& T = c->T;
  cudaEvent_t ev[8];
  for (auto& e : ev) ck(cudaEventCreate(&e), "event");
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (c->dim == 3) {
    // one rank per process: this rank's slab (its working arrays hold the slab's planes only)
    const DevTables3 T3 = c->local_io ? slab3(c, c->rank) : c->T3;
    const double sc = 2.0 / T3.N;
    for (int r = 0; r < reps; ++r) {
      ck(cudaEventRecord(ev[0], s), "rec");
      launch_lsq3(T3, d_phi, c->dphi, s);
      ck(cudaEventRecord(ev[1], s), "rec");
      launch_correct3(T3, d_phi, c->dphi, nullptr, nullptr, nullptr, s, c->corr);
      ck(cudaEventRecord(ev[2], s), "rec");
      launch_sparse3(T3, 0, c->corr, nullptr, 1.0, c->work, s);
      ck(cudaEventRecord(ev[3], s), "rec");
      launch_sweep3(T3, c->work, c->zfirst, c->fsep, s, true);
      launch_reduced3(T3, c->zfirst, c->fsep, c->hsep, s);
      ck(cudaEventRecord(ev[4], s), "rec");
      launch_sparse3(T3, 1, c->work, c->hsep, sc, c->work2, s);
      ck(cudaEventRecord(ev[5], s), "rec");
      launch_sparse3(T3, 2, c->work2, nullptr, sc, c->work, s);
      ck(cudaEventRecord(ev[6], s), "rec");
      launch_interp3(T3, d_phi, c->dphi, nullptr, nullptr, c->work, d_out, s, c->local_io);
      ck(cudaEventRecord(ev[7], s), "rec");
      ck(cudaEventSynchronize(ev[7]), "sync");
      for (int q = 0; q < 7; ++q) {
        float t = 0;
        ck(cudaEventElapsedTime(&t, ev[q], ev[q + 1]), "elapsed");
        acc[q] += t;
      }
      float t = 0;
      ck(cudaEventElapsedTime(&t, ev[0], ev[7]), "elapsed");
      acc[7] += t;
    }
    for (int q = 0; q < 8; ++q) ms[q] = acc[q] / reps;
    for (auto& e : ev) cudaEventDestroy(e);
    return KFBI_OK;
  }
  for (int r = 0; r < reps; ++r) {
    ck(cudaEventRecord(ev[0], s), "rec");
    launch_spline(T, d_phi, c->mk, s, c->hole_off, c->hole_M, c->hole_delta, c->nh, c->ahole);
    ck(cudaEventRecord(ev[1], s), "rec");
    for (int r : my_ranks(c)) launch_correct(slab(c, r), d_phi, c->mk, nullptr, nullptr, c->cval, s);
    ck(cudaEventRecord(ev[2], s), "rec");
    DenseSrc D;
    D.stencil_only = true;
    launch_sweep(T, c->cval, D, c->spec, c->zfirst, c->zlast, c->fsep, s);
    ck(cudaEventRecord(ev[3], s), "rec");
    launch_reduced(T, c->zfirst, c->zlast, c->fsep, c->hsep, s);
    ck(cudaEventRecord(ev[4], s), "rec");
    launch_inverse_sparse(T, c->spec, c->hsep, c->vsten, s);
    ck(cudaEventRecord(ev[5], s), "rec");
    ck(cudaEventRecord(ev[6], s), "rec");   // hole coefficients are fused into the spline launch
    launch_interp(T, d_phi, c->mk, nullptr, nullptr, c->vsten, c->nh, c->nh ? c->wg : nullptr, c->ahole, d_out, s);
    ck(cudaEventRecord(ev[7], s), "rec");
    ck(cudaEventSynchronize(ev[7]), "sync");
    for (int q = 0; q < 7; ++q) {
      float t = 0;
      ck(cudaEventElapsedTime(&t, ev[q], ev[q + 1]), "elapsed");
      acc[q] += t;
    }
    float t = 0;
    ck(cudaEventElapsedTime(&t, ev[0], ev[7]), "elapsed");
    acc[7] += t;
  }
  for (int q = 0; q < 8; ++q) ms[q] = acc[q] / reps;
  for (auto& e : ev) cudaEventDestroy(e);
  KFBI_CATCH(c)
  return KFBI_OK;
}

kfbi_status kfbi_gray_scott_step(kfbi_ctx* cu, kfbi_ctx* cv, double* d_u, double* d_v, double* d_psi_u,
                                 double* d_psi_v, int32_t warm, double* d_scratch, double dt, const double* params5,
                                 double tol, int32_t* iters2, void* stream) {
  if (!cu || !cv || !d_u || !d_v || !d_psi_u || !d_psi_v || !d_scratch || !params5 || !(dt > 0) || !(tol > 0))
    return KFBI_EINVAL;
  if (cu->dim != 2 || cv->dim != 2 || !cu->S.neumann || !cv->S.neumann || cu->S.N != cv->S.N ||
      cu->S.M != cv->S.M || cu->S.nq != cv->S.nq)
    return fail(cu, KFBI_EINVAL, "Gray-Scott needs two 2D Neumann contexts on the same geometry");
  const double eps[2] = {params5[3], params5[4]};
  kfbi_ctx* cs[2] = {cu, cv};
  for (int q = 0; q < 2; ++q)
    if (std::fabs(cs[q]->S.kappa - 2.0 / (eps[q] * dt)) > 1e-12 * cs[q]->S.kappa)
      return fail(cu, KFBI_EINVAL, "context kappa must be 2/(eps dt) (Crank-Nicolson, reading R40)");
  if (cu && cu->local_io) return fail(cu, KFBI_EUNSUPPORTED, "full-grid entry point (world = 1 or the emulation)");
  KFBI_TRY(cu)
  need_ws(cu);
  need_ws(cv);
  cudaStream_t s = pick(cu, stream);
  const long nn = (long)(cu->S.N + 1) * (cu->S.N + 1);
  const int M = cu->S.M, nq = cu->S.nq;
  double* fg = d_scratch;
  double* fq = fg + nn;
  double* fz = fq + nq;
  double* y = fz + M;
  double* g0 = y + nn;
  const GsParams p{params5[0], params5[1], params5[2]};
  launch_fill(g0, M, 0.0, s);   // homogeneous Neumann data
  launch_gs_reaction(d_u, d_v, nn, 0.5 * dt, p, s);
  double* w[2] = {d_u, d_v};
  double* psi[2] = {d_psi_u, d_psi_v};
  for (int q = 0; q < 2; ++q) {
    launch_gs_rhs(cs[q]->T, w[q], fg, fq, fz, s);
    kfbi_solve_opts o{tol, 30, 50, KFBI_GMRES, 1.0, 0};
    kfbi_solve_stats st{};
    const kfbi_status r = kfbi_solve(cs[q], g0, fg, fq, fz, warm ? psi[q] : nullptr, y, psi[q], &o, &st, s);
    if (r != KFBI_OK) return r;
    if (iters2) iters2[q] = st.iters;
    launch_gs_combine(w[q], y, nn, s);
  }
  launch_gs_reaction(d_u, d_v, nn, 0.5 * dt, p, s);
  ck(cudaGetLastError(), "gray-scott step");
  KFBI_CATCH(cu)
  return KFBI_OK;
}

kfbi_status kfbi_launch_count(int64_t* count) {
  if (!count) return KFBI_EINVAL;
  *count = (int64_t)kfbi::g_launches;
  return KFBI_OK;
}

kfbi_status kfbi_destroy(kfbi_ctx* c) {
  if (!c) return KFBI_OK;
  DeviceGuard g(c->device);
  if (c->comm) ncclCommDestroy(c->comm);
  drop_step_graphs(c);
  if (c->hcol_host) cudaFreeHost(c->hcol_host);
  for (auto& e : c->ev_step)
    if (e) cudaEventDestroy(e);
  delete c;
  return KFBI_OK;
}

kfbi_status kfbi_test_fast_solve(kfbi_ctx* c, const double* d_rhs, double* d_v, void* stream) {
  if (!c || !d_rhs || !d_v) return KFBI_EINVAL;
  if (c && c->local_io) return fail(c, KFBI_EUNSUPPORTED, "full-grid entry point (world = 1 or the emulation)");
  KFBI_TRY(c)
  need_ws(c);
  cudaStream_t s = pick(c, stream);
  if (c->dim == 3) {
    launch_base3(c->T3, d_rhs, c->work, s);   // note: masked by Ω (test inputs are Ω-supported or use 2D)
    forward3(c, nullptr, s, true);
    inverse3(c, d_v, s);
    ck(cudaGetLastError(), "fast solve 3D");
    return KFBI_OK;
  }
  BumpParams none{};
  launch_dst_forward(c->T, d_rhs, false, none, c->spec, s);
  DenseSrc D;
  D.base = c->spec;
  launch_sweep(c->T, nullptr, D, c->spec, c->zfirst, c->zlast, c->fsep, s);
  launch_reduced(c->T, c->zfirst, c->zlast, c->fsep, c->hsep, s);
  launch_inverse_dense(c->T, c->spec, c->hsep, d_v, s);
  const size_t W = (size_t)c->T.N + 1;
  ck(cudaMemsetAsync(d_v, 0, W * sizeof(double), s), "memset");
  ck(cudaMemsetAsync(d_v + (size_t)c->T.N * W, 0, W * sizeof(double), s), "memset");
  ck(cudaGetLastError(), "fast solve");
  KFBI_CATCH(c)
  return KFBI_OK;
}

kfbi_status kfbi_test_interface_solve(kfbi_ctx* c, const double* d_base, const double* d_jq, const double* d_jz,
                                      double* d_v, double* d_vplus, void* stream) {
  if (!c || !d_jq || !d_jz) return KFBI_EINVAL;
  if (c && c->local_io) return fail(c, KFBI_EUNSUPPORTED, "full-grid entry point (world = 1 or the emulation)");
  KFBI_TRY(c)
  need_ws(c);
  cudaStream_t s = pick(c, stream);
  if (c->dim == 3) {
    launch_base3(c->T3, d_base, c->work, s);
    launch_correct3(c->T3, nullptr, nullptr, nullptr, d_jq, c->work, s);
    forward3(c, nullptr, s, true);
    if (d_v) {
      inverse3(c, d_v, s);
    } else {
      inverse3(c, nullptr, s);
    }
    if (d_vplus) {
      if (d_v) {   // the field went to d_v: recompute the working copy for the interpolation
        launch_base3(c->T3, d_base, c->work, s);
        launch_correct3(c->T3, nullptr, nullptr, nullptr, d_jq, c->work, s);
        forward3(c, nullptr, s, true);
        inverse3(c, nullptr, s);
      }
      launch_interp3(c->T3, nullptr, nullptr, nullptr, d_jz, c->work, d_vplus, s);
    }
    ck(cudaGetLastError(), "interface solve 3D");
    return KFBI_OK;
  }
  BumpParams none{};
  if (d_base) launch_dst_forward(c->T, d_base, false, none, c->spec, s);
  for (int r : my_ranks(c)) launch_correct(slab(c, r), nullptr, nullptr, nullptr, d_jq, c->cval, s);
  DenseSrc D;
  D.base = d_base ? c->spec : nullptr;
  launch_sweep(c->T, c->cval, D, c->spec, c->zfirst, c->zlast, c->fsep, s);
  launch_reduced(c->T, c->zfirst, c->zlast, c->fsep, c->hsep, s);
  if (d_vplus) {
    launch_inverse_sparse(c->T, c->spec, c->hsep, c->vsten, s);
    launch_interp(c->T, nullptr, nullptr, nullptr, d_jz, c->vsten, 0, nullptr, nullptr, d_vplus, s);
  }
  if (d_v) {
    launch_inverse_dense(c->T, c->spec, c->hsep, d_v, s);
    const size_t W = (size_t)c->T.N + 1;
    ck(cudaMemsetAsync(d_v, 0, W * sizeof(double), s), "memset");
    ck(cudaMemsetAsync(d_v + (size_t)c->T.N * W, 0, W * sizeof(double), s), "memset");
  }
  ck(cudaGetLastError(), "interface solve");
  KFBI_CATCH(c)
  return KFBI_OK;
}

kfbi_status kfbi_test_setup_dump(const kfbi_ctx* c, int32_t which, int64_t* out) {
  if (!c || !out) return KFBI_EINVAL;
  if (c->dim == 3) {
    const Setup3& S = c->S3;
    if (which == 0) {
      for (size_t u = 0; u < S.irr_ijk.size(); ++u) out[u] = S.irr_ijk[u];
    } else if (which == 1) {
      for (int q = 0; q < S.nq; ++q) {
        out[4 * q] = S.q_axis[q]; out[4 * q + 1] = S.q_i[q]; out[4 * q + 2] = S.q_j[q]; out[4 * q + 3] = S.q_k[q];
      }
    } else if (which == 2) {
      std::memcpy(out, S.st_nodes_ij.data(), S.st_nodes_ij.size() * sizeof(int64_t));
    } else {
      return KFBI_EINVAL;
    }
    return KFBI_OK;
  }
  const Setup& S = c->S;
  if (which == 0) {
    std::vector<std::pair<int, int>> v(S.nirr);
    for (int n = 0; n < S.nirr; ++n) v[n] = {S.irr_i[n], S.irr_j[n]};
    std::sort(v.begin(), v.end());
    for (int n = 0; n < S.nirr; ++n) { out[2 * n] = v[n].first; out[2 * n + 1] = v[n].second; }
  } else if (which == 1) {
    for (int q = 0; q < S.nq; ++q) { out[3 * q] = S.q_axis[q]; out[3 * q + 1] = S.q_i[q]; out[3 * q + 2] = S.q_j[q]; }
  } else if (which == 2) {
    std::memcpy(out, S.st_nodes_ij.data(), S.st_nodes_ij.size() * sizeof(int64_t));
  } else {
    return KFBI_EINVAL;
  }
  return KFBI_OK;
}

}  // extern "C"
