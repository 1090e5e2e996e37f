/*
 * kfbi.h — C ABI of the B200-native kernel-free boundary integral (KFBI) library.
 *
 * Hot path of arXiv 2404.15249 ("A GPU-accelerated Cartesian grid method for PDEs on
 * irregular domain"): the interface-problem apply run once per iteration of the boundary
 * integral solve, and the GMRES solve around it.  Citations are PAPER.md line numbers (P:n).
 *
 *   PDE      Δu − κu = f in Ω, u = g_D on Γ = ∂Ω, κ ≥ 0
 *   BIE      ½φ + Wφ + Yf = g_D on Γ;  u = Wφ + Yf in Ω
 *   apply    K_D φ = ½φ + Wφ at the control points, evaluated as the interior one-sided
 *            value of the interface problem Δv − κv = 0, [v] = φ, [∂_n v] = 0,
 *            v = 0 on ∂B: jumps → correction at irregular nodes
 *            (Alg. 2) → FFT/DST + tridiagonal fast solve (Alg. 4)
 *            → jump-corrected interpolation (Alg. 3)
 *   solve    restarted GMRES on K_D φ = g_D − (Yf)⁺ (Alg. 5), then the final
 *            field u_h = Wφ + Yf
 *
 * Conventions: FP64 everywhere; N intervals per axis, N a power of
 * two ≥ 64; box B = [lo, hi]^d with equal spacing h; node coordinate lo + i·h;
 * homogeneous Dirichlet box condition.  Grid fields crossing the ABI are full node
 * grids of (N+1)^d doubles, row-major, last index contiguous ([i][j] in 2D), box nodes 0.
 *
 * Memory and ownership: every d_* pointer is caller-owned device memory on the context's
 * device; host pointers are caller-owned host memory.  The library allocates NO device
 * memory: the caller queries kfbi_workspace_size() and hands a device buffer (e.g. a
 * torch.uint8 tensor) to kfbi_set_workspace(); the context borrows it until destroyed.
 * Streams are cudaStream_t passed as void* (NULL = legacy default stream).
 * Devices: a context lives on kfbi_dist.device (the current device if dist is NULL or
 * device < 0); every entry point runs on that device and restores the caller's current device.
 *
 * Errors: every call returns a kfbi_status; no exceptions or exit() cross the ABI.
 * kfbi_last_error(ctx) / kfbi_last_setup_error() return a message for the last failure.
 * After KFBI_ECUDA or KFBI_ENCCL only kfbi_destroy() is valid on that context.
 * Threading: calls on one context are not thread-safe; distinct contexts are independent.
 * Determinism: no floating-point atomics; results are bitwise repeatable for fixed inputs.
 */
#ifndef KFBI_H_
#define KFBI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t kfbi_status;
enum {
  KFBI_OK = 0,
  KFBI_EINVAL = 1,       /* bad sizes, κ < 0, unequal h, null pointer, N not a power of two */
  KFBI_EGEOM = 2,        /* Γ leaves the box, an edge crossed twice or by two components
                            (R31), or an irregular node outside [2, N−2] on some axis — the
                            clearance reading R32 as built: every interpolation
                            stencil node is then an unknown node                               */
  KFBI_ENOCONV = 3,      /* GMRES hit max_restarts; outputs hold the last iterate + stats   */
  KFBI_ECUDA = 4,
  KFBI_ENCCL = 5,
  KFBI_ENOMEM = 6,       /* workspace missing or too small                                  */
  KFBI_EUNSUPPORTED = 7, /* feature not built (e.g. device setup in 3D, Neumann with κ = 0)   */
  KFBI_EBREAKDOWN = 8    /* kfbi_solve: a residual became NaN/Inf (non-finite inputs or a
                            breakdown of the iteration); outputs are undefined                  */
};

/* geometry kinds (2D curves parametrised CCW by θ ∈ [0, 2π)) */
enum {
  KFBI_ELLIPSE = 1,      /* p = {ra, rb}: γ = c + (ra cos θ, rb sin θ); circle: ra = rb        */
  KFBI_STAR = 2,         /* p = {r, ε, m, α}: ρ = r(1 + ε sin(m(θ − α))) (R25)    */
  KFBI_ELLIPSOID = 3,    /* p = {a, b, c}   (3D)                                     */
  KFBI_TORUS = 4         /* p = {R, r}      (3D; reading R28)                                   */
};
enum { KFBI_OUTER = 0, KFBI_HOLE = 1 };
enum { KFBI_DIRICHLET = 0, KFBI_NEUMANN = 1 };

typedef struct {
  int32_t dim;           /* 2 or 3                                           */
  double lo[3], hi[3];   /* box B; (hi − lo)/n must be equal on all axes      */
  int32_t n[3];          /* intervals per axis, all equal, power of two in [64, 8192] (2D)
                            or [32, 512] (3D)                                  */
} kfbi_grid;

typedef struct {
  int32_t kind;          /* KFBI_ELLIPSE, KFBI_STAR, …                                      */
  int32_t role;          /* KFBI_OUTER (one) or KFBI_HOLE (Ω = outer region minus holes)   */
  double center[3];
  double p[4];
  int32_t n_ctrl;        /* control points on this curve; 0 = round(L / (1.18 h)) (R11)   */
} kfbi_component;

typedef struct {
  int32_t ncomp;
  const kfbi_component* comp;
} kfbi_boundary;

typedef struct {
  double kappa;          /* κ ≥ 0                                    */
  int32_t bc;            /* KFBI_DIRICHLET, or KFBI_NEUMANN (κ > 0; κ = 0 →
                            KFBI_EUNSUPPORTED)                       */
} kfbi_pde;

typedef struct {
  int32_t world, rank, device;   /* world = 1 for a single GPU                 */
  const void* nccl_id;           /* 128-byte ncclUniqueId (world > 1), else NULL */
} kfbi_dist;

typedef struct {
  double tol;            /* relative residual, default 1e-8          */
  int32_t restart;       /* GMRES(m), default 30 (R18)                       */
  int32_t max_restarts;  /* default 50                                       */
  int32_t method;        /* KFBI_GMRES (default), KFBI_RICHARDSON (φ += γ(ĝ − Kφ)),
                            KFBI_BICGSTAB (textbook, 2 applies per iteration); the last two run
                            at most restart × max_restarts iterations (reading R39)            */
  double gamma;          /* Richardson relaxation γ ∈ (0, 1], default 1               */
  int32_t async_final;   /* 0 (default): return after the final field is computed; 1: return once
                            the iteration has converged and the final field (u) is enqueued on
                            `stream` — d_u / d_phi_out are complete when the stream reaches that
                            point (serving loops overlap their next host work with it)          */
  int32_t omega_io;      /* 0 (default): d_f_grid and d_u are full (N+1)^d node grids; 1 (one
                            context per grid): both hold only the Ω-node values in row-major node order
                            (kfbi_omega_count entries, the layout of kfbi_scatter_omega /
                            kfbi_gather_omega): the dense forward transform reads f and the final
                            field writes u in that layout directly (no full-grid f or u is formed;
                            16-byte aligned device buffers).  KFBI_EUNSUPPORTED with one rank
                            per process.                                                       */
} kfbi_solve_opts;
enum { KFBI_GMRES = 0, KFBI_RICHARDSON = 1, KFBI_BICGSTAB = 2 };

typedef struct {
  int32_t iters;         /* Arnoldi steps (applies of K inside cycles)        */
  int32_t restarts;      /* cycles started                                    */
  int32_t n_applies;     /* all interface solves incl. Y, residual and final  */
  int32_t converged;
  double rel_residual;   /* ‖ĝ − Kφ‖₂ / ‖ĝ − Kφ₀‖₂ at exit                    */
  double t_solve_s;      /* host wall clock of kfbi_solve                     */
} kfbi_solve_stats;

typedef struct kfbi_ctx kfbi_ctx;

/* Library / error introspection. */
const char* kfbi_version(void);
const char* kfbi_last_error(const kfbi_ctx* ctx);
const char* kfbi_last_setup_error(void);

/* rank 0 of a multi-GPU run writes a 128-byte NCCL unique id to out128 (host); the caller
 * broadcasts it (e.g. as a torch.uint8[128] tensor over torch.distributed) and passes it in
 * kfbi_dist.nccl_id on every rank.  Multi-GPU layout: 2D grids
 * are split along x into `world` slabs of whole level-2 arrowhead segments (512 columns each), so
 * `world` must divide N/512; 3D grids into slabs of whole ADM blocks (15 planes + separator), so
 * `world` must divide N/16.  Each slab solves its blocks, eliminates its interior separators and
 * publishes 4 values per mode (first, last, its boundary separator's zA, its first block's zB).
 * Per apply the ranks exchange those rows — 2D: one ncclAllGather, every rank solves the slab
 * separators; 3D: mode-partitioned, one grouped ncclSend/ncclRecv all-to-all to the owner of
 * K/world modes and one back with the two rows each slab needs — and sum disjoint partial
 * interpolations (one ncclAllReduce).  Corrections, LSQ fits, transforms, the once-per-solve dense
 * applies and the final field run on each rank's slab only (kfbi_local_slab); φ, the outputs and
 * GMRES are replicated.  kfbi_dist.rank = −1 with world > 1 runs all ranks' slabs in this one
 * context (single-GPU emulation of the partition; the exchanges become reads of the other slabs'
 * buffers). */
kfbi_status kfbi_get_unique_id(void* out128);

/* Slab of `rank` (host): out6 = {first block, end block, first column, last column, first
 * stencil column index, end stencil column index}; the columns are grid indices i (x).
 * 3D: {first block, end block, first x-plane, last x-plane, first stencil row, end stencil row}. */
kfbi_status kfbi_slab(const kfbi_ctx* ctx, int32_t rank, int64_t* out6);

/* Procedure 1: grid, control points, node classification, intersections,
 * stencils and per-mode fast-solver tables, on the host.  No device memory is touched
 * until kfbi_set_workspace().  `stream` is kept as the context's default stream. */
kfbi_status kfbi_setup(const kfbi_grid* grid, const kfbi_boundary* bnd, const kfbi_pde* pde,
                       const kfbi_dist* dist, void* stream, kfbi_ctx** out);

/* Procedure 1 with its O(N^d) phases on the device (2D and 3D): node
 * classification, the sign-change edges and their intersections by 64-step bisection
 * (readings R30/R31) and the irregular nodes with their incident intersections (P:551,
 * App. A.3) run as kernels on `stream` in the caller's scratch d_scratch (device, ≥ the bytes
 * kfbi_setup_scratch_size returns — ≈ 5 GB at 512³ — borrowed for the call only, contents undefined
 * after), and so do the interpolation stencils (the stencil nodes, the local Vandermonde
 * systems solved by LU with partial pivoting for the V⁺ and ∂_n V⁺ weight rows, and in 2D the sorted
 * unique stencil-node list); the lists come back to the host, and the rest of Procedure 1 (frames, arc
 * length, control points, LSQ neighbourhoods, spline filters, per-mode tables) runs there as in
 * kfbi_setup (host↔device traffic: the lists, and the control points up for the stencils).
 * The lists are identical to kfbi_setup's (same arithmetic, IEEE round-to-nearest, no contraction; the
 * star level uses the device sin/atan2, so a node within an ulp of Γ could in principle classify
 * differently).  Synchronous.  Errors as kfbi_setup plus KFBI_ENOMEM (scratch too small), KFBI_ECUDA. */
kfbi_status kfbi_setup_scratch_size(const kfbi_grid* grid, size_t* bytes);
kfbi_status kfbi_setup_device(const kfbi_grid* grid, const kfbi_boundary* bnd, const kfbi_pde* pde,
                              const kfbi_dist* dist, void* stream, void* d_scratch, size_t bytes,
                              kfbi_ctx** out);

/* Bytes of device workspace the context needs (setup tables + scratch). */
kfbi_status kfbi_workspace_size(const kfbi_ctx* ctx, size_t* bytes);

/* Borrow `bytes` of device memory at d_ws (256-byte aligned), upload the setup tables and
 * run the setup-time device work (hole-completion fields, R27).  Synchronous. */
kfbi_status kfbi_set_workspace(kfbi_ctx* ctx, void* d_ws, size_t bytes);

/* M = number of control points, nq = number of intersection nodes, n_irr = irregular
 * nodes, n_nodes = (N+1)^d grid nodes of a full field. */
kfbi_status kfbi_sizes(const kfbi_ctx* ctx, int64_t* M, int64_t* nq, int64_t* n_irr, int64_t* n_nodes);

/* The node box this context reads f from and writes u to (memory is the paper's
 * reason for going multi-GPU).  world = 1, or rank = −1 (all slabs in one context):
 * the full grid, local_shape = (N+1, N+1, 1) in 2D / (N+1)³ in 3D, offset 0.  One rank per process
 * (world > 1, rank ≥ 0): the rank's slab of grid columns / x-planes i ∈ [local_offset[0],
 * local_offset[0] + local_shape[0]) with all j (and k): 2D shape (n_i, N+1, 1), 3D (n_i, N+1, N+1).
 * kfbi_solve's d_f_grid and d_u are then arrays of that shape (row-major, last index contiguous), u is
 * valid on the slab's Ω nodes, and the context's spectral / working arrays hold the slab only (the
 * workspace shrinks ∝ 1/world).  kfbi_scatter_omega, kfbi_gather_omega, kfbi_gray_scott_step and the
 * kfbi_test_* entry points are full-grid only (KFBI_EUNSUPPORTED on a one-rank-per-process context). */
kfbi_status kfbi_local_slab(const kfbi_ctx* ctx, int64_t local_shape[3], int64_t local_offset[3]);

/* Host copies of point coordinates so the caller can evaluate g and f there:
 * which = 0: control points (M × dim, interleaved), 1: intersection nodes (nq × dim),
 * 2: outward unit normals at the control points (M × dim; Neumann data g_N = n·∇u). */
kfbi_status kfbi_points(const kfbi_ctx* ctx, int32_t which, double* host_xyz);

/* Ω mask of the full node grid ((N+1)^d int8, 1 = Ω) into host memory. */
kfbi_status kfbi_node_mask(const kfbi_ctx* ctx, int8_t* host_mask);

/* Ω mask of this context's node slab (kfbi_local_slab: the full grid unless one rank per process) into
 * device memory d_mask (int8, local_shape elements, row-major), enqueued on `stream` (a device-to-device
 * copy of the context's classification; needs the workspace). */
kfbi_status kfbi_node_mask_device(kfbi_ctx* ctx, int8_t* d_mask, void* stream);

/* Ω-compact grid transfers (serving path).  The solve uses f only on Ω nodes (zero extension,
 * P:530) and u_h is valid only there, so a caller may move just the Ω values across PCIe:
 * n_omega = number of Ω nodes of the full (N+1)^d node grid, in row-major node order (i, j[, k]) —
 * the order of kfbi_node_mask's 1 entries.  kfbi_scatter_omega: d_grid[p] = d_compact[rank of p]
 * on Ω nodes, 0 elsewhere (a full-grid f for kfbi_solve).  kfbi_gather_omega: d_compact[rank of p] =
 * d_grid[p] for the Ω nodes of a full grid (e.g. kfbi_solve's u).  Device pointers, n_omega and
 * (N+1)^d doubles; asynchronous on `stream`; single-context grids (world = 1 layouts). */
kfbi_status kfbi_omega_count(const kfbi_ctx* ctx, int64_t* n_omega);
kfbi_status kfbi_scatter_omega(kfbi_ctx* ctx, const double* d_compact, double* d_grid, void* stream);
kfbi_status kfbi_gather_omega(kfbi_ctx* ctx, const double* d_grid, double* d_compact, void* stream);

/* out = K̃φ = K_D φ (+ hole completion, R27), φ and out are M doubles on the device.
 * Neumann contexts: out = K_N ψ = ½ψ − ∂_n(Sψ) = ∂_n V⁺ of the interface problem with
 * [v] = 0, [∂_n v] = ψ (reading R38).  Asynchronous, stream-ordered, no state change. */
kfbi_status kfbi_apply(kfbi_ctx* ctx, const double* d_phi, double* d_out, void* stream);

/* Full BVP solve (Procedures 2-3; Neumann: P:795-808 with GMRES on K_N, ĝ_N =
 * g_N − ∂_n(Yf)⁺, u = Yf − Sψ; d_g then holds g_N = ∂_n u at the control points and d_phi_out ψ).  With world > 1 every rank passes the
 * same replicated g, f_isect, f_ctrl and its (full-size) f_grid; d_u receives the rank's slab
 * columns (others untouched); d_phi_out is replicated.
 *   d_g        g_D at the control points (M)
 *   d_f_grid   f at the full node grid ((N+1)^d), or NULL for f ≡ 0; values outside Ω
 *              are ignored (zero extension)
 *   d_f_isect  f at the intersection nodes (nq) and d_f_ctrl at the control points (M),
 *              both NULL iff d_f_grid is NULL
 *   d_phi0     initial density (M) or NULL for φ₀ = 0
 *   d_u        out: full node grid; u_h on Ω nodes, the interface solution elsewhere
 *   d_phi_out  out: converged density (M) or NULL
 * Synchronous (one host sync per Arnoldi step, as P:782), except that with opts->async_final the
 * final-field work is left running on `stream`. */
kfbi_status kfbi_solve(kfbi_ctx* ctx, const double* d_g, const double* d_f_grid,
                       const double* d_f_isect, const double* d_f_ctrl, const double* d_phi0,
                       double* d_u, double* d_phi_out, const kfbi_solve_opts* opts,
                       kfbi_solve_stats* stats, void* stream);

/* Algorithmic HBM bytes per launch of the two dominant kernels (model of DESIGN.md §6):
 * 2D: bytes_sweep = k_sweep (the spectral rows of the block columns that hold stencil nodes
 * written, 8 B per mode), bytes_inverse = k_inv_sparse (the spectral rows of the distinct stencil
 * columns read); 3D: bytes_sweep = k_fwd3s (spectrum of the planes with irregular nodes written),
 * bytes_inverse = k_inv3y (spectrum of the planes with stencil rows read + the y-inverse rows that
 * hold stencil nodes written).
 * unknowns = interior grid points.  Host-only, no GPU work. */
kfbi_status kfbi_apply_model(const kfbi_ctx* ctx, double* bytes_sweep, double* bytes_inverse,
                             double* unknowns);

kfbi_status kfbi_destroy(kfbi_ctx* ctx);

/* Gray–Scott reaction–diffusion (readings R40, R41): one
 * Strang step R(Δt/2) ∘ D(Δt) ∘ R(Δt/2) of u_t = ε₁Δu + (1/ε₀)[γ(1−u) − uv²],
 * v_t = ε₂Δv + (1/ε₀)[uv² − (γ+κ_r)v] with ∂_n u = ∂_n v = 0, in place on the full node grids
 * d_u, d_v ((N+1)² doubles, device).  R: explicit midpoint rule at every node.  D: Crank–Nicolson
 * per species as one Neumann solve (Δ − κ)y = −κw, ∂_n y = 0, w ← 2y − w, the boundary data of
 * the source by bilinear interpolation of w at the intersection and control points.
 *   ctx_u, ctx_v  2D Neumann contexts on the same geometry with κ = 2/(ε₁Δt) and 2/(ε₂Δt)
 *   d_psi_u/v     densities (M doubles each): GMRES warm start when warm ≠ 0, updated in place
 *   d_scratch     2(N+1)² + nq + 2M doubles of device scratch
 *   params5       host {γ, κ_r, ε₀, ε₁, ε₂};  tol  GMRES tolerance;  iters2  host out, 2 ints
 * Synchronous (two kfbi_solve calls). */
kfbi_status kfbi_gray_scott_step(kfbi_ctx* ctx_u, kfbi_ctx* ctx_v, double* d_u, double* d_v, double* d_psi_u,
                                 double* d_psi_v, int32_t warm, double* d_scratch, double dt,
                                 const double* params5, double tol, int32_t* iters2, void* stream);

/* Device time of each kernel of one kfbi_apply, averaged over `reps` applies, from CUDA
 * events recorded on `stream` between the launches (bench/roofline use; synchronous).
 * ms_out[8] = {spline (+ hole coefficients), correct, sweep, reduced, inverse, 0, interp, whole
 * apply}; in 3D:
 * {LSQ fit, correction, sparse forward DST (k_fwd3s), tridiagonal sweep + reduced system, inverse
 * y-DST (k_inv3y), z-evaluation at the stencil nodes, interp, apply}. */
kfbi_status kfbi_profile_apply(kfbi_ctx* ctx, const double* d_phi, double* d_out, int32_t reps,
                               double* ms_out, void* stream);

/* Process-wide count of kernels this library has launched (for bench gpu_launches). */
kfbi_status kfbi_launch_count(int64_t* count);

/* ---------------------------------------------------------------- test-only entry points
 * kfbi_test_fast_solve: d_v = solution of (Δ_h − κ)v = d_rhs on the unknowns (full-grid
 *   layouts, box entries of d_rhs ignored, of d_v written 0) — Alg. 4 alone.
 * kfbi_test_interface_solve: Alg. 1 steps 4-6 with GIVEN jumps: d_jq (nq × 6) at the
 *   intersections and d_jz (M × 6) at the control points, columns [v],[v_x],[v_y],[v_xx],
 *   [v_xy],[v_yy]; d_base full grid or NULL (0); d_v full grid out (or NULL) and d_vplus
 *   (M) out = V⁺ at the control points.
 * kfbi_test_setup_dump: host copies of the integer setup lists for parity with the oracle:
 *   which = 0: irregular nodes (n_irr × dim int64, sorted), 1: intersections (nq × (dim+1)
 *   int64: axis, low-end node), 2: stencil nodes (M × 6 × dim int64). */
kfbi_status kfbi_test_fast_solve(kfbi_ctx* ctx, const double* d_rhs, double* d_v, void* stream);
kfbi_status kfbi_test_interface_solve(kfbi_ctx* ctx, const double* d_base, const double* d_jq,
                                      const double* d_jz, double* d_v, double* d_vplus, void* stream);
kfbi_status kfbi_test_setup_dump(const kfbi_ctx* ctx, int32_t which, int64_t* host_out);

#ifdef __cplusplus
}
#endif
#endif /* KFBI_H_ */
