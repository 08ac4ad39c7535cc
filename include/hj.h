/* include/hj.h — C-ABI of the B200-native hierarchical Jacobi solver (libhj.so).
 *
 * What it solves: the finite-difference Poisson problem of the paper
 *   1D  -u'' = f on (0,1), 3-point stencil, A = tridiag(-1,2,-1)/h^2   PAPER.md:180-207 (§3.4, Eq. 5)
 *   2D  -(u_xx+u_yy) = f, 5-point stencil, dx = dy = h                PAPER.md:393-421 (§4.2)
 * with Dirichlet data g on the ring, by
 *   HJ_CLASSIC       one global-memory Jacobi sweep per cycle          PAPER.md:114-133 (§3.2)
 *   HJ_HIERARCHICAL  the paper's cycle: copy each tile + 1-cell halo on chip, k Jacobi
 *                    sub-iterations with the halo frozen, write the interior back
 *                                                                      PAPER.md:161-166 (§3.3),
 *                                                                      :382-387 (§4.1), App. A :532-575
 * until ||f - A x_c||_2 <= tol * ||f - A x_0||_2 (relative) or
 * ||f - A x_c||_2 <= tol (absolute).  Readings of the paper: DESIGN.md §3.
 * With hj_problem.stencil set, the same methods solve the paper's general systems instead:
 *   1D  tridiagonal A with per-point a_i, d_i, c_i, x_i <- (b_i - a_i x_{i-1} - c_i x_{i+1})/d_i
 *                                                                      PAPER.md:69-83 (§3, Eq. 4)
 *   2D  pentadiagonal A with constants a, c, e, f, d,
 *       x_ij <- (b_ij - a x_{i-1,j} - c x_{i+1,j} - e x_{i,j-1} - f x_{i,j+1})/d
 *                                                                      PAPER.md:329-347 (§4, Eq. 10)
 *   (e.g. anisotropic Poisson, dx != dy: a = c = -1/dx^2, e = f = -1/dy^2, d = 2/dx^2 + 2/dy^2,
 *   PAPER.md:413-419), evaluated as the FMA chain of DESIGN.md reading c23.
 *
 * Conventions shared by every entry point
 *  - Arrays are row-major with x fastest: f[j*nx + i], 0 <= i < nx, 0 <= j < ny.
 *  - dim 1 with ny > 1: ny INDEPENDENT 1D problems of nx points each (the paper's batch of 1024
 *    copies), row-major f[b*nx + i]; the stopping test uses the norm of the stacked
 *    residual.
 *  - bc (Dirichlet ring): dim 1: [g_left, g_right] per problem (problem b at bc[2b], bc[2b+1]);
 *    dim 2: [south(nx) | north(nx) | west(ny) | east(ny)], south = the row below j = 0.  NULL
 *    means g = 0 (the paper's u = 0).
 *  - x0 NULL means a zero initial guess (the paper's protocol passes ones).
 *  - Iterates are kept in hj_params.dtype (f64 or f32); the residual is always accumulated in
 *    f64 from s = h2f - (stencil applied to x) (h^2-scaled form, reported unscaled), where
 *    h2f = h^2 f for f64 and h2f = (double)(float)(h*h*f), the right-hand side the fp32 iteration
 *    actually solves, for f32 (reading c16; pinned in tests/test_oracle_pins.py).
 *  - Ownership: every input pointer is borrowed for the duration of the call only; every
 *    output buffer is caller-allocated; the library allocates and frees its own device
 *    scratch (two padded iterate buffers, the h^2 f array, residual partials, history).
 *  - Errors: a non-OK status leaves a message in hj_last_error() (thread-local).  Invalid
 *    arguments/configurations are detected before any device work.  Not converging within
 *    max_cycles is NOT an error (HJ_NOT_CONVERGED, outputs valid).  A non-finite residual
 *    stops the solve with HJ_ERR_NUMERIC; outputs then hold the iterate whose residual was
 *    non-finite and the history up to it.
 *  - Thread-compatibility: one call per plan at a time; distinct plans may run concurrently.
 *  - There is no CPU fallback: without a usable sm_100 device every call returns HJ_ERR_CUDA.
 */
#ifndef HJ_H_
#define HJ_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HJ_OK = 0,
  HJ_NOT_CONVERGED = 1,      /* outputs valid, cycles == max_cycles                           */
  HJ_ERR_INVALID_ARG = 2,    /* NULL pointer, dim not 1/2, n < 1, h <= 0 or non-finite, ...    */
  HJ_ERR_INVALID_CONFIG = 3, /* tile < 1 or > n, k < 1 (classic: k != 1), overlap odd / < 0 /
                                >= tile, overlap with row slabs,
                                tol < 0 / >= 1 (relative) / NaN, max_cycles < 0, tile does not
                                fit on chip, slab rows not a multiple of tile_y              */
  HJ_ERR_NUMERIC = 4,        /* NaN/Inf residual                                               */
  HJ_ERR_CUDA = 5,
  HJ_ERR_NCCL = 6,
  HJ_ERR_OOM = 7,
  HJ_ERR_PEER = 8            /* peer transport: a rank did not signal within HJ_PEER_TIMEOUT_S
                                (default 30 s), or plan used before hj_plan_peer_attach        */
} hj_status;

typedef enum { HJ_F64 = 0, HJ_F32 = 1 } hj_dtype;
typedef enum {
  HJ_HIERARCHICAL = 0,  /* the paper's hierarchical cycle (§3.3, §4.1)                  */
  HJ_CLASSIC = 1,       /* one global-memory Jacobi sweep per cycle (§3.2)              */
  HJ_MULTIGRID = 2      /* V-cycles with the hierarchical cycle as DAMPED-Jacobi smoother
                           (SURVEY.md §8(f) NEXT #4; PAPER.md:17, :530 name multigrid smoothing
                           as the use of the method; reading c24 fixes the textbook
                           V-cycle: vertex-centred coarsening n -> (n-1)/2 while n is odd >= 3
                           (2D: both axes), full-weighting restriction of the residual, (bi)linear
                           interpolation, mg_coarse_cycles plain hierarchical cycles on the
                           coarsest grid).  One "cycle" = one V-cycle; the stopping test and
                           history are those of the other modes.  Poisson only (stencil NULL),
                           overlap 0, no row slabs; nx (and ny in 2D) odd >= 3; every level,
                           the finest included, uses tile = min(tile, n_level) and k
                           sub-iterations.                                                    */
} hj_mode;
typedef enum { HJ_TOL_RELATIVE = 0, HJ_TOL_ABSOLUTE = 1 } hj_tol_mode;
typedef enum {
  HJ_KERNEL_AUTO = 0,   /* register-resident warp-per-tile kernel where the tile shape allows
                           (2D 32x32; 1D tile = 32*2^m <= 1024), else the shared-memory kernel */
  HJ_KERNEL_SMEM = 1    /* the paper's design: one CTA per tile, one thread per DOF, shared-
                           memory ping-pong with __syncthreads between sub-iterations          */
} hj_kernel;

typedef struct {
  int32_t dim;           /* 1 or 2                                                           */
  int64_t nx, ny;        /* interior points per direction; dim 1: ny = number of problems     */
  double h;              /* grid spacing (hx == hy == h); unused when stencil != NULL         */
  const double *f;       /* nx*ny right-hand side of -Δu = f; with stencil: b of Ax = b       */
  const double *bc;      /* ring values (layout above) or NULL                               */
  const double *x0;      /* nx*ny initial guess or NULL                                       */
  const double *stencil; /* NULL: the Poisson problem above.  Otherwise the general
                            coefficients (reading c23), same memory space as f:
                              dim 2: 5 doubles {a, c, e, f, d} = the coefficients of the west,
                                     east, south, north neighbour and the point itself (Eq. 10);
                              dim 1: 3*nx*ny doubles, planes [a | d | c] indexed like f (Eq. 4;
                                     a of a problem's first point and c of its last multiply
                                     the ring values).
                            Every d must be non-zero and every value finite
                            (HJ_ERR_INVALID_ARG).  The residual is then r = D^-1 (b - Ax) in the
                            iterate's arithmetic; history/tolerances use ||r||*|d| in 2D
                            (= ||b - Ax||) and ||r|| in 1D.  Jacobi converges for diagonally
                            dominant A; divergence ends in HJ_ERR_NUMERIC or HJ_NOT_CONVERGED. */
} hj_problem;

typedef struct {
  hj_mode mode;
  hj_dtype dtype;
  int32_t tile_x, tile_y;  /* subdomain interior (the paper's blockDim.x/.y); dim 1: tile_y=1 */
  int32_t k;               /* sub-iterations per cycle (>= 1; classic: 1)                    */
  int32_t overlap;         /* overlapping subdomains o (x; and y unless overlap_y >= 0): even,
                              0 <= o < tile.  Block b starts at 1 + b*(tile - o), the last block
                              is shifted to end at n, overlaps are owned half/half with the left
                              block taking the odd extra point (PAPER.md:243-305 §3.5, :454-510
                              §4.3; reading c21).  0 = the paper's basic method.     */
  double tol;
  hj_tol_mode tol_mode;
  double ref_residual;     /* 0: r_0 = ||f - A x0||; > 0: use this r_0 (resume a solve)      */
  int64_t max_cycles;      /* >= 0                                                            */
  hj_kernel kernel;        /* kernel family selection (HJ_KERNEL_AUTO recommended)           */
  int32_t overlap_y;       /* 2D: overlap along y; negative = same as overlap                 */
  /* HJ_MULTIGRID only (ignored otherwise); zeros select the defaults */
  int32_t mg_nu1, mg_nu2;  /* pre-/post-smoothing hierarchical cycles per level, >= 0; both 0
                              = (1, 1)                                                         */
  double mg_omega;         /* damping of the smoothing sub-iterations, x + omega (u - x) as one
                              fma in the iterate type, 0 < omega <= 1; 0 = 4/5 (2D), 2/3 (1D)  */
  int32_t mg_coarse_cycles;/* plain (undamped) cycles on the coarsest grid, >= 0; 0 = 1        */
  int32_t mg_levels;       /* maximum number of grids incl. the finest (>= 2); 0 = no limit    */
} hj_params;

typedef struct {
  double *x;               /* caller-allocated nx*ny doubles (f64 even for f32 solves)       */
  double *history;         /* caller-allocated hj_history_capacity(params) doubles (=
                              max_cycles+1 up to 2^24) or NULL; history[c] = ||f - A x_c||_2
                              for c = 0..min(cycles, capacity-1).  jacobi_solve*, with history,
                              reject max_cycles+1 > capacity (HJ_ERR_INVALID_CONFIG);
                              hj_plan_solve truncates (never writes past capacity)            */
  int64_t cycles;          /* first c at which the test held (0 if x0 already satisfies it)  */
  int32_t converged;
  double initial_residual; /* ||f - A x0||_2                                                  */
  double final_residual;   /* ||f - A x_cycles||_2                                            */
  double seconds_solve;    /* cycle loop only (device-resident data)                          */
  double seconds_total;    /* whole call, incl. allocation and H2D/D2H copies (paper style)  */
} hj_result;

/* Host pointers in problem and result.  Blocking. */
hj_status jacobi_solve(const hj_problem *problem, const hj_params *params, hj_result *result);

/* Device pointers in problem (f, bc, x0) and result (x, history); cuda_stream is a
 * cudaStream_t (NULL = the legacy default stream).  Returns when the solve is complete. */
hj_status jacobi_solve_device(const hj_problem *problem, const hj_params *params,
                              hj_result *result, void *cuda_stream);

/* ---- plans: set up once (device pointers), run cycles many times (benchmarks, resume) ---- */
typedef struct hj_plan hj_plan;

/* Allocates the padded iterate buffers, h^2 f and scratch on the current device and
 * initialises them from problem (device pointers; copied, not retained). */
hj_status hj_plan_create(const hj_problem *problem, const hj_params *params, void *cuda_stream,
                         hj_plan **plan);
/* Re-initialise the iterate to the problem's x0 (kept in a device copy) and the cycle count to 0. */
hj_status hj_plan_reset(hj_plan *plan);
/* Launch exactly ncycles cycles from the current state without host synchronisation; each
 * cycle = the cycle kernel + residual reduction (one "step").  If kernel_ms is not NULL, CUDA
 * events on the plan's stream bracket every cycle-kernel launch and *kernel_ms receives the
 * sum of their durations (the call then synchronises once, at the end). */
hj_status hj_plan_run(hj_plan *plan, int64_t ncycles, float *kernel_ms);
/* Run to convergence (or max_cycles) from the current state and fill result
 * (x and history are DEVICE pointers or NULL).  Cycles run as CUDA graphs of G cycles with the
 * stopping test on the device (host polls once per graph).  Single-GPU hierarchical plans small
 * enough for one co-resident wave (2D: 32x32 tiles, nx and ny multiples of 32, at most 8 tiles per
 * SM, no overlap; 1D: register tiles, no ragged tile, at most 1024 problems) instead run the whole
 * solve in ONE cooperative launch with the tile iterates resident in registers — the same
 * iterates, histories and cycle counts bit for bit; the environment variable HJ_RESIDENT=0 disables
 * it (the same cycle). */
hj_status hj_plan_solve(hj_plan *plan, hj_result *result);
/* Entries of the residual history kept for these parameters: min(max_cycles + 1, 2^24) (the
 * environment variable HJ_HIST_CAP lowers the 2^24 limit, for tests).  The history buffer of
 * hj_plan_solve must hold this many doubles; 0 for params == NULL. */
int64_t hj_history_capacity(const hj_params *params);
/* The cycle kernel family the plan runs (for tests and benchmark records): 0 = REG2D (32x32 tiles in
 * registers, TMA-staged), 1 = SMEM2D (the paper's shared-memory design, any tile), 2 = CLASSIC2D,
 * 3 = REG1D, 4 = SMEM1D, 5 = CLASSIC1D, 6 = REGT (register tiles of shapes 16x16, 32x16, 16x32,
 * 64x32, 32x64, 64x64, 128x32); -1 for plan == NULL. */
int32_t hj_plan_kernel_kind(const hj_plan *plan);
/* Number of launches of library kernels per cycle (for launch accounting). */
int32_t hj_plan_launches_per_cycle(const hj_plan *plan);
hj_status hj_plan_destroy(hj_plan *plan);

/* ---- multi-GPU: row slabs, one process per GPU (PAPER.md has no multi-GPU; north star) ---- */
typedef struct {
  int32_t rank, nranks;
  const char *nccl_id;     /* 128 bytes from hj_nccl_unique_id() on rank 0, broadcast by caller */
  int64_t row_begin, row_end; /* this rank's interior rows [begin, end) of the global grid;
                                 multiples of tile_y (hierarchical) / of 8 (classic)        */
} hj_dist;

hj_status hj_nccl_unique_id(char out[128]);
/* Plan for one rank of a row-slab solve: problem->f and ->x0 are DEVICE pointers to the local
 * rows [row_begin, row_end), problem->bc a DEVICE pointer to the full ring (or NULL).  Creating
 * the plan initialises NCCL (collective over all ranks) and exchanges the initial halos. */
hj_status hj_plan_create_dist(const hj_problem *problem, const hj_params *params,
                              const hj_dist *dist, void *cuda_stream, hj_plan **plan);
/* problem: GLOBAL nx, ny, h and bc (host pointers, full ring); f and x0 hold ONLY the local
 * rows [row_begin, row_end) (host pointers).  result->x receives the local rows; history is
 * global (identical on every rank).  Cycle counts and iterates are bitwise identical to the
 * single-GPU solve for any nranks (tile rows never straddle slabs). */
hj_status jacobi_solve_dist(const hj_problem *problem, const hj_params *params,
                            hj_result *result, const hj_dist *dist);

/* ---- multi-GPU without NCCL: the peer-memory transport ----
 * Same row slabs and bitwise guarantees as above, but the per-cycle exchange is done by the
 * library's own kernels through CUDA IPC mappings of the neighbours' buffers (NVLink/NVSwitch
 * stores between GPUs; processes sharing one GPU also work): rows 1 and R of the new iterate are
 * stored into the neighbours' ghost rows, each rank's residual row sums are stored into every
 * rank's residual vector, and the finalize kernel signals every rank (fence.sys + atomic) and
 * waits for all signals of the cycle (bounded spin; HJ_ERR_PEER after HJ_PEER_TIMEOUT_S).
 * Usage (every rank, one process per GPU):
 *   hj_plan_create_peer(...)              dist->nccl_id is ignored (may be NULL)
 *   hj_plan_peer_export(plan, blob)       HJ_PEER_HANDLE_BYTES bytes
 *   -- the caller all-gathers the blobs in rank order (e.g. torch.distributed) --
 *   hj_plan_peer_attach(plan, blobs)      opens the mappings and runs the collective reset
 * after which hj_plan_run / hj_plan_solve work as for any plan.  hj_plan_reset and
 * hj_plan_destroy are collective: call them on every rank (destroy only after every rank has
 * finished its last run).  Problem pointers as for hj_plan_create_dist. */
#define HJ_PEER_HANDLE_BYTES 512
hj_status hj_plan_create_peer(const hj_problem *problem, const hj_params *params,
                              const hj_dist *dist, void *cuda_stream, hj_plan **plan);
hj_status hj_plan_peer_export(const hj_plan *plan, void *handle_out);
hj_status hj_plan_peer_attach(hj_plan *plan, const void *all_handles);

/* Resource figures of the paper: tiles = the paper's operational block count (
 * with overlap Eq. 8/13, ceiling when inexact), threads = tiles*tile_x*tile_y
 * (Eq. 9/14), smem_bytes_paper_formula = sizeof(T)*(2(Tx+2)+Tx) in 1D
 * and sizeof(T)*(2(Tx+2)(Ty+2)+TxTy) in 2D. Host-only. */
hj_status hj_resource_figures(const hj_problem *problem, const hj_params *params,
                              int64_t *tiles, int64_t *threads, int64_t *smem_bytes_paper_formula);

/* Message of the last failing call on this thread ("" if none). */
const char *hj_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* HJ_H_ */
