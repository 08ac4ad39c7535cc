// Internal declarations shared by the CUDA translation units of libhj.so.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/hj.h"

namespace hj {

// ------------------------------------------------------------------ errors ---
void set_error(const std::string& msg);

#define HJ_CUDA(call)                                                                     \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      ::hj::set_error(std::string(#call) + ": " + cudaGetErrorString(e_));              \
      return e_ == cudaErrorMemoryAllocation ? HJ_ERR_OOM : HJ_ERR_CUDA;                  \
    }                                                                                     \
  } while (0)

#define HJ_TRY(expr)                  \
  do {                                \
    hj_status s_ = (expr);            \
    if (s_ != HJ_OK) return s_;       \
  } while (0)

// --------------------------------------------------------- device control ----
// One per plan, in device memory.  Written only by the finalize kernel (and reset by
// the host); read by every cycle kernel so that cycles after convergence are no-ops.
struct Ctrl {
  long long c;          // index of the snapshot the next cycle kernel reads (x_c)
  long long c_done;     // cycle at which the solve stopped
  int done;             // 1 once converged / max_cycles reached / numeric error
  int converged;
  int status;           // hj_status of the solve
  int pad;
  double sqrtS0;        // sqrt(S_0) used by the relative test (or ref_residual * h^2)
  double S0, S_last;    // h^2-scaled squared residuals
  unsigned long long sig0;  // peer transport: own signal counter at the last reset
};

// Subdomains along one axis (0-based interior indices; §3.5, §4.3; DESIGN.md c10, c21).
//  o == 0: tiles [b*T, min((b+1)*T, n)), ragged last tile, each owns its whole interior.
//  o  > 0: block b starts at b*(T-o), the last block at n-T (shifted to end at n); all blocks
//          are T wide; an overlap of L points between blocks b, b+1 is owned ceil(L/2) / floor(L/2).
struct Axis {
  int n, T, o, nb;
};
__host__ __device__ __forceinline__ int axis_nb(int n, int T, int o) {
  return o == 0 ? (n + T - 1) / T : (n - T + (T - o) - 1) / (T - o) + 1;
}
__host__ __device__ __forceinline__ Axis make_axis(int n, int T, int o) { return Axis{n, T, o, axis_nb(n, T, o)}; }
__host__ __device__ __forceinline__ int axis_start(const Axis& a, int b) {
  return a.o == 0 ? b * a.T : (b == a.nb - 1 ? a.n - a.T : b * (a.T - a.o));
}
__host__ __device__ __forceinline__ int axis_width(const Axis& a, int b) {
  return a.o == 0 ? (a.n - b * a.T < a.T ? a.n - b * a.T : a.T) : a.T;
}
__host__ __device__ __forceinline__ int axis_own_hi(const Axis& a, int b) {  // inclusive
  if (b == a.nb - 1) return a.n - 1;
  if (a.o == 0) return (b + 1) * a.T - 1;
  const int s1 = axis_start(a, b + 1), L = axis_start(a, b) + a.T - s1;
  return s1 + (L + 1) / 2 - 1;
}
__host__ __device__ __forceinline__ int axis_own_lo(const Axis& a, int b) {
  return b == 0 ? 0 : axis_own_hi(a, b - 1) + 1;
}

// Geometry of the padded iterate buffers (both dims; 1D uses one row).
//   X[(j) * pitch + col0 - 1 + i],  i = 0..nx+1 along x (i=0: west/left ring),
//   j = 0..ny+1 along y (j=0: south ring).  col0 = 2 puts interior column 0 on a
//   16-byte boundary so that pairs of doubles are one 128-bit access.
struct Geom {
  int dim, dtype, mode, kernel_kind;
  int gen;                     // general coefficients (hj_problem.stencil, DESIGN.md c23)
  double wt[4];                // 2D general: T(-a/d), T(-c/d), T(-e/d), T(-f/d), exact in double
  double rdiv;                 // reported residual = sqrt(S) / rdiv: h^2, 1/|d| (2D general), 1
  int64_t nx, ny;            // local interior extent (dist: the slab's rows)
  int64_t pitch, col0, rows; // X layout (elements)
  int64_t fpitch, frows;     // H2F layout: H2F[j*fpitch + i]
  int tx, ty, k;
  int ox, oy;                  // overlap along x / y (0: the paper's basic method)
  Axis ax, ay;                 // block plans (hierarchical modes)
  int64_t ntx, nty, ntiles;  // tiles of this plan (classic: row-blocks x col-blocks)
  int64_t parts_per_row;     // partials per row group (ntx; classic2d: 4 per CTA)
  int64_t nparts;            // number of residual partials
  int64_t nrg_local, rg_offset, nrg_global;  // row groups (tile rows) and their global offset
  double h, h2;
  double omega = 1.0;          // damped sub-iterations (multigrid smoother, reading c24); 1 = the paper's
};

enum KernelKind { K_REG2D = 0, K_SMEM2D = 1, K_CLASSIC2D = 2, K_REG1D = 3, K_SMEM1D = 4, K_CLASSIC1D = 5,
                  K_REGT = 6 /* register tiles of other shapes, kernels_2dt.cu */ };

// Kernel launch descriptor passed to the per-dimension launchers.
struct CycleArgs {
  const void* xin;
  void* xout;
  const void* h2f;             // Q = T(h^2 f) / diag (0.25 in 2D, 0.5 in 1D), see init_q_kernel;
                               // general coefficients: Q = T(b / d)
  const void* wl;              // 1D general: T(-a_i/d_i), same layout as Q (else NULL)
  const void* wr;              // 1D general: T(-c_i/d_i)
  const CUtensorMap* tm_in;   // TMA descriptor of xin, 34 x (col0+34) box (REG2D loads)
  const CUtensorMap* tm_f;    // TMA descriptor of h2f, 32 x 32 box (REG2D loads)
  const CUtensorMap* tm_out;  // TMA descriptor of xout, 32 x 32 box (REG2D stores)
  double* part;               // per-tile residual partials of the snapshot
  const Ctrl* ctrl;
  long long max_cycles;
  // multigrid (reading c24): if cor_e != NULL, the snapshot is first corrected by the (bi)linear
  // interpolation of the next coarser iterate cor_e (a padded buffer of pitch cor_pitch) — the
  // coarse-grid correction fused into the first post-smoothing cycle (2D only)
  const void* cor_e = nullptr;
  long long cor_pitch = 0;
  const CUtensorMap* tm_cor = nullptr;  // REG2D: TMA map of cor_e, box R2::EW x 18 (tile's patch)
  // peer transport, fused halo (REG2D plans): interior column 0 of the NEIGHBOURS' ghost rows in
  // their copy of xout (rank-1's row R+1, rank+1's row 0; NULL at the slab ends).  The kernels
  // store the new first / last interior row straight into them (NVLink stores), tile by tile.
  void* peer_lo = nullptr;
  void* peer_hi = nullptr;
  // multigrid (c24): the snapshot is identically zero (a coarse level's first cycle) — x is not read
  bool zero_x = false;
  // REG2D only, plans without ragged edge tiles: run only the tile rows ty0 + j * tys, j < nty_run
  // (nty_run < 0: every tile row).  The overlapped NCCL transport launches the slab's two boundary
  // tile rows first, sends their rows while the interior tile rows run.
  int ty0 = 0, tys = 1, nty_run = -1;
};

// Launchers (kernels_2d.cu / kernels_1d.cu).  Return cudaGetLastError().
cudaError_t launch_cycle_2d(const Geom& g, const CycleArgs& a, int grid_hint, cudaStream_t st);
cudaError_t launch_cycle_1d(const Geom& g, const CycleArgs& a, int grid_hint, cudaStream_t st);
// REGT (kernels_2dt.cu): tile shapes 16x16, 32x16, 16x32, 64x32, 32x64, 64x64, 128x32 (Poisson, o = 0,
// no ragged tiles); warps per tile = (tx/32)(ty/32) for tiles of 32 and more, else 1.
bool regt_shape(int tx, int ty);
int regt_warps_per_tile(int tx, int ty);
cudaError_t launch_regt(const Geom& g, const CycleArgs& a, int grid_hint, cudaStream_t st);
cudaError_t configure_2dt();
// Resident solves (whole solve in one cooperative launch; kernels_2d.cu / kernels_1d.cu): the tiles'
// iterates stay in registers across cycles, only halos and residual partials cross the grid.
// part: 2 x ntiles doubles; bar: 2 zeroed unsigned ints.
cudaError_t launch_resident_2d(const Geom& g, void* X0, void* X1, const void* Q, double* part, Ctrl* ctrl,
                               double* hist, long long hist_cap, double tol, int tol_mode, double ref_residual,
                               long long max_cycles, int k, unsigned int* bar, cudaStream_t st);
cudaError_t launch_resident_1d(const Geom& g, void* X0, void* X1, const void* Q, double* part, Ctrl* ctrl,
                               double* hist, long long hist_cap, double tol, int tol_mode, double ref_residual,
                               long long max_cycles, int k, unsigned int* bar, cudaStream_t st);
cudaError_t launch_resident_1dm(const Geom& g, int M, void* X0, void* X1, const void* Q, double* part, double* R,
                                Ctrl* ctrl, double* hist, long long hist_cap, double tol, int tol_mode,
                                double ref_residual, long long max_cycles, int k, unsigned int* bar, cudaStream_t st);
bool res1w_ok(const Geom& g);
// res1c: one small 1D problem in one CTA (C points per lane, ghost depth D); default layout
constexpr int RES1C_C = 8, RES1C_D = 4;
bool res1c_ok(const Geom& g, int* C, int* D);
cudaError_t launch_resident_1c(const Geom& g, int C, int D, void* X0, void* X1, const void* Q, Ctrl* ctrl,
                               double* hist, long long hist_cap, double tol, int tol_mode, double ref_residual,
                               long long max_cycles, int k, cudaStream_t st);
cudaError_t launch_resident_1w(const Geom& g, void* X0, void* X1, const void* Q, Ctrl* ctrl, double* hist,
                               long long hist_cap, double tol, int tol_mode, double ref_residual,
                               long long max_cycles, int k, cudaStream_t st);
size_t reg1d_smem_bytes(int dtype, int tile);
int reg1d_warps_per_cta(int dtype, int tile);
cudaError_t reg_kernels_configure();  // opt in to large dynamic shared memory
// Multigrid transfers (mg.cu, reading c24): gf = fine level, gc = the next coarser level.
// write_zero: also zero the coarse iterate's interior (2D skips it when the coarse level's first
// cycle runs in zero-start mode, CycleArgs::zero_x; 1D always writes it)
cudaError_t launch_mg_restrict(const Geom& gf, const void* xf, const void* qf, const Geom& gc, void* qc,
                               void* xc, bool write_zero, const Ctrl* ctrl, cudaStream_t st);
cudaError_t launch_mg_correct(const Geom& gf, const void* xin, void* xout, const Geom& gc, const void* e,
                              const Ctrl* ctrl, cudaStream_t st);

// Classic kernels block geometry (CTA = 8 rows x 256 cols, one residual partial per warp).
constexpr int CLASSIC2D_ROWS = 8;
constexpr int CLASSIC2D_COLS = 256;   // 128 threads x 2 columns
constexpr int CLASSIC1D_CELLS = 2048; // 256 threads x 8 cells

// ------------------------------------------------------------- PTX helpers ---
#if defined(__CUDACC__)
__host__ __device__ __forceinline__ long long lmin(long long a, long long b) { return a < b ? a : b; }
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Plain arrive (release at CTA scope: the arriving thread's prior shared-memory writes, and those
// of its warp ordered before it by __syncwarp, are visible to threads that observe the phase).
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// 2D tensor tile global -> shared, completion on an mbarrier (TMA, SASS UTMALDG).
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// Contiguous bulk copy global -> shared (TMA bulk engine, SASS UBLKCP); 16-B aligned, size % 16 == 0.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// 2D tensor tile shared -> global (TMA store, SASS UTMASTG), tracked by bulk groups.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* tm, int c0, int c1, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(tm)),
               "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the shared-memory sources of all committed bulk stores have been read
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// all committed bulk stores are complete (globally visible)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// order this thread's generic-proxy shared-memory accesses before later async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void prefetch_tensormap(const CUtensorMap* tm) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tm)) : "memory");
}

// Canonical elemental updates, see DESIGN.md §6:
//   1D: 0.5 * ((L + R) + h2f)  ==  fma(0.5, L + R, q),   q = 0.5 * h2f  (exact)
//   2D: 0.25 * (((W + E) + (S + N)) + h2f) == fma(0.25, (W+E)+(S+N), q), q = 0.25 * h2f
// Scaling by a power of two commutes with round-to-nearest (no under/overflow), so the
// single-rounding fma equals the two-rounding form bit for bit.
__device__ __forceinline__ double upd2(double w, double e, double s, double n, double q) {
  return __fma_rn(0.25, __dadd_rn(__dadd_rn(w, e), __dadd_rn(s, n)), q);
}
__device__ __forceinline__ float upd2(float w, float e, float s, float n, float q) {
  return __fmaf_rn(0.25f, __fadd_rn(__fadd_rn(w, e), __fadd_rn(s, n)), q);
}
__device__ __forceinline__ double upd1(double l, double r, double q) {
  return __fma_rn(0.5, __dadd_rn(l, r), q);
}
__device__ __forceinline__ float upd1(float l, float r, float q) {
  return __fmaf_rn(0.5f, __fadd_rn(l, r), q);
}
// h^2-scaled residual contributions in double (h2f64 = h2f of the iterate type, widened).
__device__ __forceinline__ double res2(double x, double w, double e, double s, double n, double h2f) {
  return h2f - (4.0 * x - ((w + e) + (s + n)));
}
__device__ __forceinline__ double res1(double x, double l, double r, double h2f) {
  return h2f - (2.0 * x - (l + r));
}

// General coefficients (PAPER.md:80-83 Eq. 4, :344-347 Eq. 10; reading c23): the
// division distributed over the terms, weights w = T(-coef/d), q = T(b/d):
//   2D: fma(wN, N, fma(wS, S, fma(wE, E, fma(wW, W, q))))      1D: fma(wR, R, fma(wL, L, q))
// and the Jacobi-scaled residual D^{-1}(b - Ax) = (the same chain in double) - x.
struct Wt2 {
  double w, e, s, n;
  double om;  // multigrid smoother damping (reading c24), T-rounded; 1 = undamped
};
__device__ __forceinline__ double gupd2(double ww, double we, double ws, double wn, double W,
                                        double E, double S, double N, double q) {
  return __fma_rn(wn, N, __fma_rn(ws, S, __fma_rn(we, E, __fma_rn(ww, W, q))));
}
__device__ __forceinline__ float gupd2(float ww, float we, float ws, float wn, float W, float E,
                                       float S, float N, float q) {
  return __fmaf_rn(wn, N, __fmaf_rn(ws, S, __fmaf_rn(we, E, __fmaf_rn(ww, W, q))));
}
__device__ __forceinline__ double gres2(double ww, double we, double ws, double wn, double x,
                                        double W, double E, double S, double N, double q) {
  return __dsub_rn(gupd2(ww, we, ws, wn, W, E, S, N, q), x);
}
__device__ __forceinline__ double gupd1(double wl, double wr, double L, double R, double q) {
  return __fma_rn(wr, R, __fma_rn(wl, L, q));
}
__device__ __forceinline__ float gupd1(float wl, float wr, float L, float R, float q) {
  return __fmaf_rn(wr, R, __fmaf_rn(wl, L, q));
}
__device__ __forceinline__ double gres1(double wl, double wr, double x, double L, double R, double q) {
  return __dsub_rn(gupd1(wl, wr, L, R, q), x);
}

// Correctly rounded T arithmetic that the compiler may not contract (reading c24 fixes the order).
template <typename T>
__device__ __forceinline__ T add_t(T a, T b) {
  if constexpr (sizeof(T) == 8) return __dadd_rn(a, b);
  else return __fadd_rn(a, b);
}
template <typename T>
__device__ __forceinline__ T mul_t(T a, T b) {
  if constexpr (sizeof(T) == 8) return __dmul_rn(a, b);
  else return __fmul_rn(a, b);
}
// (Bi)linear interpolation of the coarse iterate at the fine ringed interior point (i, j) (coarse
// ringed point I sits on fine 2I; the coarse ring is zero): DESIGN.md reading c24.
template <typename T, typename F>
__device__ __forceinline__ T mg_interp_f(F&& E, long long i, long long j) {
  const bool ci = (i & 1) == 0, cj = (j & 1) == 0;
  if (ci && cj) return E(i / 2, j / 2);
  if (cj) return mul_t(T(0.5), add_t(E((i - 1) / 2, j / 2), E((i + 1) / 2, j / 2)));
  if (ci) return mul_t(T(0.5), add_t(E(i / 2, (j - 1) / 2), E(i / 2, (j + 1) / 2)));
  return mul_t(T(0.25), add_t(add_t(E((i - 1) / 2, (j - 1) / 2), E((i + 1) / 2, (j - 1) / 2)),
                              add_t(E((i - 1) / 2, (j + 1) / 2), E((i + 1) / 2, (j + 1) / 2))));
}
template <typename T>
__device__ __forceinline__ T mg_interp(const T* __restrict__ e, long long ep, long long i, long long j) {
  constexpr int COL0 = 16 / sizeof(T);
  return mg_interp_f<T>([&](long long I, long long J) { return e[J * ep + (COL0 - 1) + I]; }, i, j);
}

// Damped Jacobi (multigrid smoother, reading c24): x + omega (u - x) as ONE fma in T.
__device__ __forceinline__ double damp(double om, double x, double u) {
  return __fma_rn(om, __dsub_rn(u, x), x);
}
__device__ __forceinline__ float damp(float om, float x, float u) {
  return __fmaf_rn(om, __fsub_rn(u, x), x);
}

// The stopping test of DESIGN.md §3 (c1, c14) for S_c = the summed h^2-scaled squared residual of
// x_c (h2 = Geom::rdiv): history, S_0, convergence / max_cycles / non-finite; otherwise c + 1.
// Shared by the engine's finalize_kernel and the resident solvers (one thread).
__device__ __forceinline__ void hj_decide(Ctrl* ctrl, double S, double* hist, long long hist_cap, double h2,
                                          double tol, int tol_mode, double ref_residual, long long max_cycles) {
  const long long c = ctrl->c;
  if (hist && c < hist_cap) hist[c] = sqrt(S) / h2;
  ctrl->S_last = S;
  if (c == 0) {
    ctrl->S0 = S;
    ctrl->sqrtS0 = ref_residual > 0.0 ? ref_residual * h2 : sqrt(S);
  }
  if (!isfinite(S)) {
    ctrl->status = HJ_ERR_NUMERIC;
    ctrl->done = 1;
    ctrl->c_done = c;
    return;
  }
  const double sq = sqrt(S);
  const bool test = tol_mode == 0 ? (sq <= tol * ctrl->sqrtS0) : (sq / h2 <= tol);
  bool conv;
  if (c == 0) conv = (S == 0.0) || ((ref_residual > 0.0 || tol_mode == 1) && test);
  else conv = test;
  if (conv) {
    ctrl->done = 1;
    ctrl->converged = 1;
    ctrl->status = HJ_OK;
    ctrl->c_done = c;
  } else if (c >= max_cycles) {
    ctrl->done = 1;
    ctrl->converged = 0;
    ctrl->status = HJ_NOT_CONVERGED;
    ctrl->c_done = c;
  } else {
    ctrl->c = c + 1;
  }
}

// Grid-wide barrier of a co-resident (cooperatively launched) grid: bar[0] = arrival count,
// bar[1] = generation.  Stores before the barrier are visible to loads after it (__threadfence +
// acquire/release on the generation; readers of other CTAs' data use L2 loads, __ldcg).
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int g;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
    } else {
      unsigned int v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar + 1) : "memory");
      } while (v == g);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
#endif

}  // namespace hj
