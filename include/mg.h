/*
 * mg.h — C-ABI of the B200-native adaptive multigrid Poisson solver (libmg.so).
 *
 * Solves the Poisson equation ∇²u = f (PAPER.md E1) in 3D on a
 * block-structured, collocated (node-centred) multiresolution grid (§2.1,
 * P:58-65) with per-axis periodic, unbounded or semi-unbounded directions (§2.2,
 * P:67-100), by
 * the adaptive FAS V(η1,η2)-cycle of Alg. 1, the compact
 * Mehrstellen stencils Δ_h^M u = R_h^M f (E10-E12; M = 2 uses the
 * cross stencil E8), full-weighting restriction (E6),
 * injection (E7), trilinear prolongation, ghost
 * interpolation of order M+2 at resolution jumps, and an FFT /
 * lattice-Green's-function direct solve of the coarsest level (P:67-100,
 * P:245; the 2-unbounded kernel is E14).
 *
 * Conventions (all entry points):
 *  - Return value: MG_OK (0) on success, a negative MG_ERR_* on error, a
 *    positive MG_WARN_* warning (the call did its work).  No C++ exception
 *    crosses the ABI.  mg_last_error() gives a message for the last failure.
 *  - Device pointers (suffix _dev) are CUDA device addresses of fp64 arrays the
 *    CALLER owns (e.g. torch tensors); the library never keeps them after the
 *    call returns.  Host pointers (suffix _host or plain const int32_t*) are
 *    ordinary host memory, also caller-owned and not retained.
 *  - Field layout on leaves: [n_leaf][B][B][B], x fastest, i.e. element
 *    (leaf n, node (ix,iy,iz)) is at n*B^3 + (iz*B + iy)*B + ix; leaves in the
 *    order given to mg_create.  Leaf (level, bi, bj, bk) owns the level-global
 *    nodes J = B*(bi,bj,bk) + [0,B)^3, at x = origin + J * h0 / 2^level.
 *  - A handle is bound to one CUDA stream (the one given to mg_create); every
 *    call enqueues work on that stream.  Calls that return host scalars
 *    (mg_residual_norm, mg_solve) synchronise that stream.  Handles are not
 *    thread-safe.
 *  - Only fp64.  There is no CPU fallback: without a CUDA device every call
 *    that needs one returns MG_ERR_CUDA.
 */
#ifndef MG_H
#define MG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mg_handle mg_handle;

/* boundary conditions, per face (-x,+x,-y,+y,-z,+z).  Per axis (low, high):
 * (PERIODIC, PERIODIC), (UNBOUNDED, UNBOUNDED), semi-unbounded (EVEN or ODD, UNBOUNDED)
 * (reading S1), or symmetric on both faces (ODD, ODD) / (EVEN, ODD) / (EVEN, EVEN)
 * (homogeneous Dirichlet / Neumann-Dirichlet / Neumann; readings S2, S3).  The low
 * face mirrors about the node plane x = 0 (EVEN: u(-k) = u(k); ODD: u(-k) = -u(k), so
 * u(0) = 0 and f on that plane is ignored); an ODD high face mirrors about the unstored
 * node N (u(N) = 0); an EVEN high face about the last stored node N-1 (the wall node is
 * an unknown; u(N-1+k) = u(N-1-k)).  An (EVEN, EVEN) axis needs the other axes periodic
 * or symmetric (else MG_ERR_BC); with no ODD face the problem is singular and the coarse
 * solve takes the zero-average solution (f must be compatible).  Blocks
 * touching EVEN/ODD faces stay on AMR level 0, which must be the coarse-solve level
 * (coarse_n = 0, no U1). */
enum { MG_BC_PERIODIC = 0, MG_BC_UNBOUNDED = 1, MG_BC_EVEN = 2, MG_BC_ODD = 3 };
/* smoother ("an iteration of the Gauss-Seidel method"; readings Z10) */
enum { MG_SMOOTHER_JACOBI = 0, MG_SMOOTHER_RBGS = 1 };
/* stopping criterion of mg_solve: relative ∞-norm residual or Cauchy (E20) */
enum { MG_CRIT_RESIDUAL = 0, MG_CRIT_CAUCHY = 1 };

enum {
  MG_OK = 0,
  MG_WARN_NOT_CONVERGED = 1,     /* mg_solve hit max_cycles; the partial solution is kept */
  MG_ERR_ARG = -1,               /* null pointer, bad size or enum */
  MG_ERR_LAYOUT_NESTING = -2,    /* leaves overlap, partial refinement, level 0 not covered */
  MG_ERR_LAYOUT_2TO1 = -3,       /* 26-neighbour 2:1 constraint violated */
  MG_ERR_UNBOUNDED_REFINED = -4, /* refined block touches an unbounded face */
  MG_ERR_BC = -5,                /* unsupported face pair (see MG_BC_*) */
  MG_ERR_ORDER = -6,             /* order not in {2,4,6} */
  MG_ERR_STATE = -7,             /* e.g. mg_vcycle before mg_set_rhs */
  MG_ERR_CUDA = -8,              /* CUDA / cuFFT failure or no device */
  MG_ERR_OOM = -9,               /* device allocation failed */
  MG_ERR_NONFINITE = -10,        /* NaN/Inf met in a norm */
  MG_ERR_LAYOUT_GHOST = -11      /* a ghost interpolation stencil leaves the coarse level */
};

typedef struct mg_desc {
  double origin[3];          /* physical position of level-global node 0 */
  double h0;                 /* grid spacing of AMR level 0 (isotropic) */
  int32_t base_blocks[3];    /* level-0 blocks per axis */
  int32_t block_size;        /* B: nodes per block edge; 16 (also 8) */
  int32_t bc[6];             /* per face, MG_BC_* */
  int32_t order;             /* M = 2 (cross stencil E8), 4 (Mehrstellen E12) or 6 (27-point Mehrstellen
                                E13 with its radius-2 right-hand side, reading Z24; with
                                allow_unbounded_refined the coarse solve's exterior band is 7 nodes
                                wide instead of 5, for the I = 8 c2f chain) */
  int32_t coarse_n;          /* nodes along x of the coarsest MG level (uniform sub-base
                                coarsening N0/2^j, reading Z5); 0 = AMR level 0 is coarsest */
  int32_t smoother;          /* MG_SMOOTHER_* */
  double omega;              /* relaxation factor (Jacobi ω; RB uses it too, 1 = Gauss-Seidel) */
  int32_t eta1, eta2;        /* pre-/post-smoothing sweeps */
  int32_t allow_unbounded_refined; /* accept refined levels touching unbounded faces (reading U1) */
  int64_t n_leaf;            /* number of leaf blocks */
  const int32_t* leaves;     /* host array [n_leaf][4] = (level, bi, bj, bk) */
  /* Kernel-variant controls.  0 everywhere = automatic (the production choice, what a
   * user wants).  The tests force each variant on small layouts so that the parity
   * suite runs every code path the automatic choice takes at full size.  Results are
   * identical up to rounding order for every setting. */
  int32_t pencil_blocks;     /* blocks per pencil of the z-marching kernels on B = 16 levels:
                                0 auto (by level size), 1, 2, 3 or 4 (with the wave-tail split
                                off); else MG_ERR_ARG */
  int32_t zsplit;            /* RB sweep of 1-block pencils split into two 8-plane z-parts:
                                0 auto (levels with fewer blocks than SMs), 1 never, 2 always */
  int32_t fuse;              /* 0 auto: fused pencil kernels where eligible (last pre-sweep +
                                residual + restriction; residual + restriction); 1 never fuse */
  int32_t ncomp;             /* right-hand sides solved together (0 or 1 = scalar; up to 8, e.g. 3 for
                                the Biot-Savart velocity): every call then takes and
                                returns leaf arrays [ncomp][n_leaf][B][B][B], one V-cycle and every
                                kernel launch cover all components (gridDim.y = ncomp), the norms
                                are the max over components, the coarse solve is one batched FFT */
  int32_t coarse_pruning;    /* x-periodic, y/z-unbounded coarse solve: 0 auto (1-D cuFFT passes that
                                skip the zero half of the padded source and unread outputs),
                                1 the plain 3-D transform of the padded lattice (cuFFT),
                                2 the pruned solve with the y and z transforms, the multiplier and
                                the window as three fused kernels of mixed-radix FFTs in shared
                                memory (mg_fft.cu; measured slower than 0); else MG_ERR_ARG */
  int32_t staging;           /* plane tiles of the RB sweep: 0 cp.async ring (default, the
                                fastest measured), 1 TMA tensor copies (cp.async.bulk.tensor, 9
                                boxes per field and plane) into an mbarrier ring; measured 2.5x
                                slower on B200; same values bit for bit */
  int32_t ghost_kernel;      /* c2f ghost boxes: 0 auto (on levels with >= 1024 boxes <= 2 nodes
                                thick along some axis, i.e. the layers of the distance-1 halo,
                                and no exterior chain: those boxes one warp each with the thin
                                axis interpolated first; every other box one CTA each, x, y, z
                                passes), 1 every box on the CTA kernel, 2 every thin box on the
                                warp kernel; else MG_ERR_ARG */
  int32_t pencil_order;      /* how z-runs of blocks are cut into pencils and launched: 0 auto (2 on
                                levels of >= 24 waves of 1-block pencils, else 1), 1 balanced chunks,
                                longest first, 2 chunks cut where the block's z index is a multiple
                                of the pencil length, launched in z-major order whatever their
                                length; else MG_ERR_ARG */
} mg_desc;

/* Validate the layout (nesting, 2:1, unbounded-face rule), build the level
 * hierarchy, ghost/transfer tables and coarse-solve kernels, allocate device
 * memory.  `cuda_stream` is a cudaStream_t (NULL = legacy default stream).
 * On success *out owns everything; release with mg_destroy. */
int mg_create(const mg_desc* d, void* cuda_stream, mg_handle** out);
void mg_destroy(mg_handle* h);
/* Thread-local message of the last failing call (never NULL). */
const char* mg_last_error(const mg_handle* h);

/* f on the leaves (device, leaf layout).  Injects f up the tree, fills its ghosts
 * (f := 0 beyond unbounded faces, mirror images beyond EVEN/ODD faces), stores
 * f* = R_h^M f on leaf nodes and
 * ‖f*‖∞.  Resets u to 0 (Alg. 1 initial solution, reading Z28). */
int mg_set_rhs(mg_handle* h, const double* f_dev);
/* Initial guess / read-back of u on the leaves (device, leaf layout). */
int mg_set_solution(mg_handle* h, const double* u_dev);
int mg_get_solution(mg_handle* h, double* u_dev);
/* n V(η1,η2)-cycles in place (Alg. 1), asynchronous on the handle's stream. */
int mg_vcycle(mg_handle* h, int n);
/* Composite residual max|f* - Δ_h^M u| over leaf nodes of all levels, and that
 * divided by ‖f*‖∞.  Synchronises.  Does not change the solution. */
int mg_residual_norm(mg_handle* h, double* abs_inf, double* rel_inf);
/* Cycle until the criterion value <= tol or max_cycles (MG_WARN_NOT_CONVERGED). */
int mg_solve(mg_handle* h, double tol, int max_cycles, int criterion,
             int* cycles_out, double* value_out);
/* End-to-end call on HOST buffers: copies f_host (leaf layout) to the device,
 * mg_set_rhs, runs `ncycles` V-cycles, copies u back into u_host, returns the
 * relative residual.  Buffers are caller-owned host memory (pinned is faster). */
int mg_run_host(mg_handle* h, const double* f_host, double* u_host, int ncycles, double* rel_out);
/* Capture each V-cycle as one CUDA graph (1) or launch kernels directly (0). */
int mg_use_graph(mg_handle* h, int enable);

/* ---- introspection / debug (tests and benchmarks) ---- */
enum { MG_INFO_NLEVELS = 0 };
/* info[0..9] = B, n_real, n_ghost, N[3], amr_level, n_c2f, n_inject, n_leaf_blocks */
int mg_level_info(mg_handle* h, int level, int64_t* info);
/* host int32[n][3]: block coordinates of the level's real blocks (storage order);
 * with `level | MG_ALL_BLOCKS`, real then ghost blocks (n = n_real + n_ghost) */
enum { MG_ALL_BLOCKS = 0x10000 };
int mg_level_blocks(mg_handle* h, int level, int32_t* coords_host);
int mg_num_levels(mg_handle* h);

enum { MG_FIELD_U = 0, MG_FIELD_F = 1, MG_FIELD_R = 2, MG_FIELD_UHAT = 3 };
/* dir 0: export the level's real blocks [n_real][B^3] into dev; 1: import from dev;
 * 2 / 3: export / import real then ghost blocks [n_real + n_ghost][B^3] (ghost checks).
 * field | (c << 8) selects component c (ncomp > 1). */
int mg_debug_field(mg_handle* h, int field, int level, int dir, double* dev);
enum {
  MG_OP_REFRESH = 0,        /* ghost fill of `level` (f2c injection + c2f / band) */
  MG_OP_SMOOTH = 1,         /* refresh + one smoothing sweep */
  MG_OP_RESIDUAL = 2,       /* refresh + r = f - Δu on all level nodes */
  MG_OP_RESTRICT = 3,       /* level -> level-1: residual, inject u, FW r, FAS rhs, û */
  MG_OP_PROLONG = 4,        /* u_level += P(u - û)_{level-1} */
  MG_OP_INJECT_UP = 5,      /* canonicalise: u_{k-1}[covered] <- u_k, all levels */
  MG_OP_COARSE_SOLVE = 6,   /* direct solve of the coarsest level */
  MG_OP_SMOOTH_RESIDUAL = 7 /* fused last pre-sweep + residual (ghost-free levels) */
};
int mg_debug_apply(mg_handle* h, int op, int level);
/* Debug (initcheck substitute): set every ghost-block node that no stencil, transfer
 * or interpolation is designed to read (outside the needed halo) to NaN
 * in all level fields.  Call after mg_set_rhs; a later result that reads one turns
 * non-finite.  Synchronises. */
int mg_debug_poison(mg_handle* h);
/* Time one operator: runs it `reps` times between CUDA events, returns ms per rep.
 * op: an MG_OP_*, 100 = one V-cycle, -1 = the bare fused RB sweep + residual tile kernel
 * of the level, -2 = the bare production pair (RB pencil sweep, then residual pencil
 * kernel); no ghost refresh for -1 / -2. */
int mg_time_op(mg_handle* h, int op, int level, int reps, double* ms_out);

/* Per-stage CUDA-event profiling of non-graph launches.  mg_profile(h, 1) clears
 * and starts; mg_profile_read fills ms[stage*nlev + level] and counts[...] for the
 * stages MG_ST_* below (nlev = mg_num_levels).  Synchronises the stream. */
enum { MG_ST_SMOOTH = 0, MG_ST_SMOOTH_RES = 1, MG_ST_RESIDUAL = 2, MG_ST_GHOST = 3, MG_ST_RESTRICT = 4,
       MG_ST_PROLONG = 5, MG_ST_COARSE = 6, MG_ST_INJECT_UP = 7, MG_ST_NORM = 8, MG_ST_FAS = 9, MG_ST_COUNT = 10 };
int mg_profile(mg_handle* h, int enable);
int mg_profile_read(mg_handle* h, double* ms, int64_t* counts);
/* Number of kernels this library has launched so far in the process (all handles). */
int64_t mg_kernel_launches(void);
/* Host wall time (ms) of the phases of mg_create: [0] layout validation and level
 * hierarchy, [1] ghost blocks / need masks / transfer lists, [2] ghost boxes, [3] pencils,
 * [4] device allocation and table upload, [5] coarse-solve setup (LGF tables, cuFFT
 * plans).  ms: 6 doubles, caller-owned. */
int mg_setup_times(const mg_handle* h, double* ms);

/* ---- Grid adaptation (§2.1; readings A1, A2).
 * No handle: adaptation produces a new leaf list, from which the caller creates a new
 * solver handle (mg_create).
 *
 * mg_detail: detail coefficient γ of every leaf block ("detail coefficient γ"):
 *   γ = max over the block's nodes of |u - P_W u|, P_W the order-W tensor-product
 *   Lagrange interpolation of the block's all-even nodes (x, then y, then z; an odd
 *   local index j uses the even positions j-(W-1) … j+(W-1), shifted by 2 to stay in
 *   the block).  field_dev: leaf-ordered [n_leaf][B][B][B] fp64 DEVICE array (x
 *   fastest, the mg_set_rhs layout); gamma_dev: [n_leaf] fp64 DEVICE output.  B in
 *   {8, 16}; W in {2, 4, 6} with 2(W-1) <= B-2.  Enqueued on `stream` (a cudaStream_t;
 *   NULL = legacy default stream), asynchronous.  NaN nodes are skipped by the max.
 *   Returns MG_OK, MG_ERR_ARG (bad size / pointer) or MG_ERR_CUDA (launch failure).
 */
int mg_detail(const double* field_dev, int32_t n_leaf, int32_t B, int32_t W, double* gamma_dev, void* stream);

/* mg_adapt: refine / coarsen / 2:1-balance a leaf list from per-leaf γ: leaves
 * with γ > eps_r below max_level are refined into 8; complete octets of leaves, none
 * refined, all γ < eps_c, are coarsened into their parent when the parent keeps the
 * 2:1 constraint; then refinements restore the 26-neighbour 2:1 balance.  Leaves
 * touching an unbounded face stay at level 0 unless allow_unbounded_refined;
 * suppressed refinements are counted in *n_suppressed (may be NULL).
 *   base_blocks[3], bc[6]: as in mg_desc; leaves: HOST int32 [n_leaf][4] rows
 *   (level, bi, bj, bk); gamma: HOST fp64 [n_leaf]; out_leaves: HOST int32
 *   [out_capacity][4], filled sorted by (level, bi, bj, bk); *n_out = number of output
 *   leaves (also when out_capacity is too small, then MG_ERR_ARG is returned).
 *   Caller owns every buffer.  Pure host code, no CUDA.
 */
int mg_adapt(const int32_t base_blocks[3], const int32_t bc[6], int32_t allow_unbounded_refined,
             const int32_t* leaves, int32_t n_leaf, const double* gamma, double eps_r, double eps_c,
             int32_t max_level, int32_t* out_leaves, int32_t out_capacity, int32_t* n_out,
             int32_t* n_suppressed);

/* mg_transfer: u of `dst` (an adapted grid of the same domain: same origin, h0,
 * base_blocks, B, bc, coarse_n, ncomp) from the composite solution of `src` (
 * reading A3): a dst leaf that is a block of src at the same level copies it (a leaf kept,
 * or coarsened into a parent, which holds the injected fine values, E7); a dst leaf one
 * level finer than src (refined) takes the trilinear interpolation of its src
 * parent, ghost nodes included; then inject-up.  Call after mg_set_rhs(dst) (which
 * resets u).  Device-to-device on dst's stream; synchronises both streams.  Returns
 * MG_OK, MG_ERR_ARG (different domains), MG_ERR_STATE, MG_ERR_LAYOUT_NESTING (a leaf
 * more than one level finer than src). */
int mg_transfer(mg_handle* dst, mg_handle* src);

#ifdef __cplusplus
}
#endif
#endif /* MG_H */
