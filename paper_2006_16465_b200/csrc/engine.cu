// Host engine and C-ABI of libhj.so (include/hj.h).
//
// A plan owns: two padded iterate buffers X[0], X[1] (snapshot semantics, DESIGN.md §3 c6),
// H2F = T(h^2 f), per-tile residual partials, per-row-group sums, the residual history and a
// device control block.  One cycle = cycle kernel (reads X[p], writes X[p^1], reduces the
// residual of X[p]) -> rowsum -> finalize (history, stopping test).  The stopping test runs on
// the device; cycles after convergence are no-ops, so the host captures G cycles in a CUDA
// graph and polls the control block once per graph launch.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "hj_internal.cuh"
#include "hj_plan.h"

namespace hj {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

// NVTX ranges around the host-side phases (plan build, runs, solves, graph capture) so one nsys trace
// shows them next to the kernels and the NCCL streams.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

long long history_limit() {
  static const long long lim = [] {
    const char* e = std::getenv("HJ_HIST_CAP");
    const long long v = e ? std::atoll(e) : 0;
    return v > 0 && v < HIST_CAP ? v : HIST_CAP;
  }();
  return lim;
}

cudaError_t configure_2d();
cudaError_t configure_1d();

namespace {

// ------------------------------------------------------------------ kernels --

// Fill a padded iterate buffer: ring from bc, interior from x0 (or zero), pads zero.
// dist: rows [0, R+1] of the slab; global row of local row r is gy0 + r (0 = south ring).
template <typename T>
__global__ void init_x_kernel(T* __restrict__ X, long long pitch, long long rows, int dim, long long nx,
                              long long ny_global, long long gy0, long long ny_local,
                              const double* __restrict__ bc, const double* __restrict__ x0,
                              int with_interior, int col0) {
  const long long n = pitch * rows;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const long long r = q / pitch, cc = q % pitch;
    const long long i = cc - (col0 - 1);  // padded x index: 0 = west ring, nx+1 = east ring
    T v = T(0);
    if (dim == 1) {  // row r = independent problem r (its own Dirichlet ends)
      if (i == 0) v = bc ? (T)bc[2 * r] : T(0);
      else if (i == nx + 1) v = bc ? (T)bc[2 * r + 1] : T(0);
      else if (i >= 1 && i <= nx && with_interior && x0) v = (T)x0[r * nx + i - 1];
    } else if (i >= 0 && i <= nx + 1 && r <= ny_local + 1) {
      const long long gj = gy0 + r;  // global padded row
      const bool iin = i >= 1 && i <= nx;
      if (gj == 0) {
        if (iin && bc) v = (T)bc[i - 1];
      } else if (gj == ny_global + 1) {
        if (iin && bc) v = (T)bc[nx + i - 1];
      } else if (r >= 1 && r <= ny_local) {
        if (i == 0) v = bc ? (T)bc[2 * nx + gj - 1] : T(0);
        else if (i == nx + 1) v = bc ? (T)bc[2 * nx + ny_global + gj - 1] : T(0);
        else if (with_interior && x0) v = (T)x0[(r - 1) * nx + (i - 1)];
      }
    }
    X[q] = v;
  }
}

// Q = scale * T(h^2 f), scale = 1/diag of the h^2-scaled stencil (0.5 in 1D, 0.25 in 2D): the
// rhs term of the Jacobi update pre-divided by the diagonal.  Scaling by a
// power of two is exact, so h^2 f = Q / scale exactly (the residual recovers it).
template <typename T>
__global__ void init_q_kernel(T* __restrict__ Q, long long fpitch, long long frows, long long nx,
                              long long ny, const double* __restrict__ f, double h2, T scale) {
  const long long n = fpitch * frows;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const long long j = q / fpitch, i = q % fpitch;
    Q[q] = (i < nx && j < ny) ? scale * (T)(h2 * f[j * nx + i]) : T(0);
  }
}

// General coefficients (reading c23): Q = T(b/d) with d a constant (2D, Eq. 10) or,
// in 1D (Eq. 4), per point from the stencil planes [a | d | c] together with WL = T(-a_i/d_i)
// and WR = T(-c_i/d_i).  Padding entries are 0.
template <typename T>
__global__ void init_gen_kernel(T* __restrict__ Q, T* __restrict__ WL, T* __restrict__ WR,
                                long long fpitch, long long frows, long long nx, long long ny,
                                const double* __restrict__ f, const double* __restrict__ st,
                                double d2) {
  const long long n = fpitch * frows, nt = nx * ny;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const long long j = q / fpitch, i = q % fpitch;
    const bool in = i < nx && j < ny;
    const long long g = j * nx + i;
    if (WL) {
      const double d = in ? st[nt + g] : 1.0;
      Q[q] = in ? (T)(f[g] / d) : T(0);
      WL[q] = in ? (T)(-st[g] / d) : T(0);
      WR[q] = in ? (T)(-st[2 * nt + g] / d) : T(0);
    } else {
      Q[q] = in ? (T)(f[g] / d2) : T(0);
    }
  }
}

// Count of invalid coefficients: non-finite anywhere, or a zero diagonal (1D: plane d).
__global__ void check_stencil_kernel(const double* __restrict__ st, long long n, long long d_lo,
                                     long long d_hi, unsigned long long* __restrict__ bad) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const double v = st[q];
    if (!isfinite(v) || (q >= d_lo && q < d_hi && v == 0.0)) atomicAdd(bad, 1ULL);
  }
}

// Extract the interior of X into a dense double array (row-major).
template <typename T>
__global__ void extract_kernel(const T* __restrict__ X, long long pitch, int dim, long long nx,
                               long long ny, int col0, double* __restrict__ out) {
  const long long n = nx * ny;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const long long j = q / nx, i = q % nx;
    out[q] = (double)X[(dim == 1 ? j : j + 1) * pitch + col0 + i];
  }
}

// R[rg_offset + g] = sum_{p < ppr} part[g*ppr + p], fixed order (lane-strided, then an xor tree).
// Peer transport (d.n > 0): the sum goes to slot rg_offset + g of EVERY rank's vector (remote
// stores), fenced at system scope before the finalize signal publishes it.  The vector is double
// buffered by cycle parity (offset (c & 1) * rp_stride): a rank signals cycle c before it reads
// its vector, so a faster rank may already store cycle c+1's sums — into the other half.
__global__ void rowsum_kernel(const double* __restrict__ part, long long ppr, long long nrg,
                              long long rg_offset, double* __restrict__ R, const Ctrl* __restrict__ ctrl,
                              PeerDsts d, long long rp_stride) {
  if (ctrl->done) return;
  rg_offset += (ctrl->c & 1) * rp_stride;
  const long long g = blockIdx.x * (long long)(blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (g >= nrg) return;
  double s = 0.0;
  for (long long p = lane; p < ppr; p += 32) s += part[g * ppr + p];
  s = warp_sum(s);
  if (d.n == 0) {
    if (lane == 0) R[rg_offset + g] = s;
    return;
  }
  for (int r = lane; r < d.n; r += 32) d.p[r][rg_offset + g] = s;
  __threadfence_system();
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// S_c = sum of R (fixed order); history; the stopping test of DESIGN.md §3 (c1, c14):
// c = 0: converged iff S_0 == 0 (or the test holds with an explicit r_0 / absolute mode);
// c >= 1: converged iff sqrt(S_c) <= tol * sqrt(S_0)  (absolute: sqrt(S_c)/h^2 <= tol).
// h2 here is Geom::rdiv (h^2 for the Poisson problem; DESIGN.md c3, c23).
// Peer transport (ps.n > 0): first signal every rank and wait until all nranks signals of this
// cycle arrived (their halo and rowsum stores are then visible), then read R from L2 (__ldcg).
__global__ void finalize_kernel(const double* __restrict__ R, long long nrg, Ctrl* __restrict__ ctrl,
                                double* __restrict__ hist, long long hist_cap, double h2, double tol,
                                int tol_mode, double ref_residual, long long max_cycles, PeerSync ps,
                                long long rp_stride) {
  if (ctrl->done) return;
  R += (ctrl->c & 1) * rp_stride;
  __shared__ double ws[32];
  if (ps.n > 0) {
    __shared__ int timed_out;
    if (threadIdx.x == 0) {
      __threadfence_system();
      for (int r = 0; r < ps.n; ++r) atomicAdd_system(ps.flag[r], 1ULL);
      const unsigned long long want = ctrl->sig0 + (unsigned long long)ps.n * (unsigned long long)(ctrl->c + 1);
      const unsigned long long t0 = gtimer();
      timed_out = 0;
      for (;;) {
        unsigned long long v;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(ps.own) : "memory");
        if (v >= want) break;
        if ((long long)(gtimer() - t0) > ps.timeout_ns) { timed_out = 1; break; }
        __nanosleep(200);
      }
      if (timed_out) {
        ctrl->status = HJ_ERR_PEER;
        ctrl->done = 1;
        ctrl->c_done = ctrl->c;
      }
    }
    __syncthreads();
    if (timed_out) return;
  }
  double s = 0.0;
  for (long long p = threadIdx.x; p < nrg; p += blockDim.x) s += __ldcg(R + p);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x != 0) return;
  double S = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) S += ws[w];
  hj_decide(ctrl, S, hist, hist_cap, h2, tol, tol_mode, ref_residual, max_cycles);
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

hj_status make_tmap(CUtensorMap* tm, const void* base, int dtype, uint64_t d0, uint64_t d1,
                    uint64_t stride_bytes, uint32_t b0, uint32_t b1) {
  auto enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return HJ_ERR_CUDA;
  }
  cuuint64_t dims[2] = {d0, d1};
  cuuint64_t strides[1] = {stride_bytes};
  cuuint32_t box[2] = {b0, b1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(tm, dtype == HJ_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                   2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return HJ_ERR_CUDA;
  }
  return HJ_OK;
}

long long round_up(long long a, long long b) { return (a + b - 1) / b * b; }

// Per device: the SM count and the large-dynamic-shared-memory opt-ins (cudaFuncSetAttribute is
// per device), done once for each device a plan is created on.
hj_status ensure_configured(int* nsm) {
  constexpr int MAXDEV = 64;
  static std::mutex mu;
  static bool done[MAXDEV] = {};
  static cudaError_t err[MAXDEV] = {};
  static int sms[MAXDEV] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess && (dev < 0 || dev >= MAXDEV)) e = cudaErrorInvalidDevice;
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(mu);
    if (!done[dev]) {
      cudaDeviceProp prop;
      cudaError_t r = cudaGetDeviceProperties(&prop, dev);
      if (r == cudaSuccess && prop.major < 10) r = cudaErrorInvalidDevice;
      if (r == cudaSuccess) sms[dev] = prop.multiProcessorCount;
      if (r == cudaSuccess) r = configure_2d();
      if (r == cudaSuccess) r = configure_1d();
      if (r == cudaSuccess) r = configure_2dt();
      err[dev] = r;
      done[dev] = true;
    }
    e = err[dev];
  }
  if (e != cudaSuccess) {
    set_error(std::string("libhj: no usable sm_100 device: ") + cudaGetErrorString(e));
    return HJ_ERR_CUDA;
  }
  *nsm = sms[dev];
  return HJ_OK;
}

}  // namespace

// ------------------------------------------------------------- validation ---
hj_status validate(const hj_problem* pb, const hj_params* pr, bool need_f) {
  if (!pb || !pr) { set_error("NULL problem or params"); return HJ_ERR_INVALID_ARG; }
  if (pb->dim != 1 && pb->dim != 2) { set_error("dim must be 1 or 2"); return HJ_ERR_INVALID_ARG; }
  if (pb->nx < 1 || pb->ny < 1) {
    set_error("nx, ny must be >= 1");
    return HJ_ERR_INVALID_ARG;
  }
  if (!pb->stencil && (!(pb->h > 0.0) || !std::isfinite(pb->h))) { set_error("h must be finite and > 0"); return HJ_ERR_INVALID_ARG; }
  if (need_f && !pb->f) { set_error("f is NULL"); return HJ_ERR_INVALID_ARG; }
  if (pb->nx > (1LL << 30) || pb->ny > (1LL << 30)) { set_error("grid too large"); return HJ_ERR_INVALID_ARG; }
  if (pr->mode != HJ_HIERARCHICAL && pr->mode != HJ_CLASSIC && pr->mode != HJ_MULTIGRID) {
    set_error("bad mode");
    return HJ_ERR_INVALID_CONFIG;
  }
  if (pr->mode == HJ_MULTIGRID) {  // reading c24
    if (pb->stencil) { set_error("multigrid: Poisson problems only (stencil must be NULL)"); return HJ_ERR_INVALID_CONFIG; }
    if (pr->overlap != 0 || (pb->dim == 2 && pr->overlap_y > 0)) {
      set_error("multigrid: overlap must be 0");
      return HJ_ERR_INVALID_CONFIG;
    }
    if (pb->nx < 3 || (pb->nx % 2) == 0 || (pb->dim == 2 && (pb->ny < 3 || (pb->ny % 2) == 0))) {
      set_error("multigrid: nx (and ny in 2D) must be odd and >= 3 (vertex-centred coarsening)");
      return HJ_ERR_INVALID_CONFIG;
    }
    if (pb->dim == 1 && pb->ny > 65535) { set_error("multigrid: at most 65535 1D problems"); return HJ_ERR_INVALID_CONFIG; }
    if (pr->mg_nu1 < 0 || pr->mg_nu2 < 0 || pr->mg_coarse_cycles < 0 || pr->mg_levels < 0 ||
        pr->mg_levels == 1 || !(pr->mg_omega >= 0.0) || pr->mg_omega > 1.0) {
      set_error("multigrid: nu1, nu2, coarse_cycles >= 0, levels 0 or >= 2, 0 <= omega <= 1");
      return HJ_ERR_INVALID_CONFIG;
    }
  }
  if (pr->dtype != HJ_F64 && pr->dtype != HJ_F32) { set_error("bad dtype"); return HJ_ERR_INVALID_CONFIG; }
  if (pr->mode == HJ_HIERARCHICAL) {
    const int ox = pr->overlap, oy = pb->dim == 2 ? (pr->overlap_y < 0 ? pr->overlap : pr->overlap_y) : 0;
    if (ox < 0 || (ox & 1) || ox >= pr->tile_x || oy < 0 || (oy & 1) || (pb->dim == 2 && oy >= pr->tile_y)) {
      set_error("overlap must be even and in [0, tile) (PAPER.md:249)");
      return HJ_ERR_INVALID_CONFIG;
    }
  }
  if (std::isnan(pr->tol) || pr->tol < 0.0 || (pr->tol_mode == HJ_TOL_RELATIVE && pr->tol >= 1.0)) {
    set_error("tol must be in [0, 1) (relative) or >= 0 (absolute)");
    return HJ_ERR_INVALID_CONFIG;
  }
  if (pr->tol_mode != HJ_TOL_RELATIVE && pr->tol_mode != HJ_TOL_ABSOLUTE) { set_error("bad tol_mode"); return HJ_ERR_INVALID_CONFIG; }
  if (pr->max_cycles < 0) { set_error("max_cycles must be >= 0"); return HJ_ERR_INVALID_CONFIG; }
  if (!(pr->ref_residual >= 0.0) || !std::isfinite(pr->ref_residual)) { set_error("bad ref_residual"); return HJ_ERR_INVALID_CONFIG; }
  if (pr->kernel != HJ_KERNEL_AUTO && pr->kernel != HJ_KERNEL_SMEM) { set_error("bad kernel"); return HJ_ERR_INVALID_CONFIG; }
  if (pr->mode == HJ_CLASSIC) {
    if (pr->k != 1) { set_error("classic mode needs k == 1"); return HJ_ERR_INVALID_CONFIG; }
    return HJ_OK;
  }
  if (pr->k < 1) { set_error("k must be >= 1"); return HJ_ERR_INVALID_CONFIG; }
  const bool mg = pr->mode == HJ_MULTIGRID;  // multigrid clips the tile to every level (c24)
  if (pr->tile_x < 1 || (!mg && pr->tile_x > pb->nx)) { set_error("tile_x must be in [1, nx]"); return HJ_ERR_INVALID_CONFIG; }
  if (pb->dim == 1 && pr->tile_y != 1) { set_error("dim 1 needs tile_y == 1"); return HJ_ERR_INVALID_CONFIG; }
  if (pb->dim == 2 && (pr->tile_y < 1 || (!mg && pr->tile_y > pb->ny))) { set_error("tile_y must be in [1, ny]"); return HJ_ERR_INVALID_CONFIG; }
  return HJ_OK;
}

// Choose the kernel and check it can run the tile shape.
static hj_status choose_kernel(const hj_problem* pb, const hj_params* pr, int* kind) {
  const size_t esz = pr->dtype == HJ_F64 ? 8 : 4;
  if (pr->mode == HJ_CLASSIC) { *kind = pb->dim == 2 ? K_CLASSIC2D : K_CLASSIC1D; return HJ_OK; }
  if (pb->dim == 2) {
    // TMA box origins must be 16-byte aligned along x: with overlapping blocks every block start
    // b*(32-o) and the shifted last start nx-32 must be a multiple of 16/sizeof(T) elements.
    const long long al = 16 / (long long)esz;
    const int ox = pr->overlap, oy = pr->overlap_y < 0 ? pr->overlap : pr->overlap_y;
    const bool aligned = ox == 0 || ((32 - ox) % al == 0 && (pb->nx - 32) % al == 0);
    // with overlap on either axis the register kernel runs EVERY block as a full 32x32 tile, so an
    // axis without overlap must have no ragged tile (its ragged tiles would need the edge kernel)
    const bool full = (ox == 0 && oy == 0) || ((ox > 0 || pb->nx % 32 == 0) && (oy > 0 || pb->ny % 32 == 0));
    if (pr->kernel == HJ_KERNEL_AUTO && pr->tile_x == 32 && pr->tile_y == 32 && aligned && full) {
      *kind = K_REG2D;
      return HJ_OK;
    }
    // other tile shapes in registers (kernels_2dt.cu): Poisson, no overlap, whole 32x32 blocks / tiles
    const long long bx = std::max(pr->tile_x, 32), by = std::max(pr->tile_y, 32);
    if (pr->kernel == HJ_KERNEL_AUTO && pr->mode == HJ_HIERARCHICAL && !pb->stencil && ox == 0 && oy == 0 &&
        regt_shape(pr->tile_x, pr->tile_y) && pb->nx % bx == 0 && pb->ny % by == 0) {
      *kind = K_REGT;
      return HJ_OK;
    }
    const size_t smem = esz * (2 * size_t(pr->tile_x + 2) * (pr->tile_y + 2) + size_t(pr->tile_x) * pr->tile_y);
    if ((long long)pr->tile_x * pr->tile_y > 1024 || smem > 200 * 1024) {
      set_error("tile does not fit one CTA (tile_x*tile_y <= 1024 and paper smem <= 200 KiB)");
      return HJ_ERR_INVALID_CONFIG;
    }
    *kind = K_SMEM2D;
    return HJ_OK;
  }
  const int t = pr->tile_x;
  // general coefficients keep x, q, wL, wR of a lane in registers: tiles up to 256 points
  if (pr->kernel == HJ_KERNEL_AUTO && pr->overlap == 0 && t % 32 == 0 && t <= (pb->stencil ? 256 : 1024) &&
      ((t / 32) & (t / 32 - 1)) == 0) {
    *kind = K_REG1D;
    return HJ_OK;
  }
  if (t > 1024) { set_error("1D tile must be <= 1024"); return HJ_ERR_INVALID_CONFIG; }
  *kind = K_SMEM1D;
  return HJ_OK;
}

// ------------------------------------------------------------- multigrid ---
// Reading c24: level l+1 halves every axis of level l (n -> (n-1)/2 while n is odd >= 3; 2D both
// axes, 1D the x axis of every independent problem), spacing 2h.  The coarse levels are internal
// hierarchical plans (tile clipped to the level, the same k); their right-hand sides are written
// by the restriction kernel every V-cycle, so they are built from a zero f and never reset.
static hj_status mg_build(hj_plan* P, const hj_params* pr) {
  const Geom& g = P->g;
  P->mg_nu1 = pr->mg_nu1;
  P->mg_nu2 = pr->mg_nu2;
  if (P->mg_nu1 == 0 && P->mg_nu2 == 0) P->mg_nu1 = P->mg_nu2 = 1;
  P->mg_coarse = pr->mg_coarse_cycles > 0 ? pr->mg_coarse_cycles : 1;
  const double om = pr->mg_omega > 0.0 ? pr->mg_omega : (g.dim == 2 ? 0.8 : 2.0 / 3.0);
  const double omT = g.dtype == HJ_F64 ? om : (double)(float)om;  // rounded to the iterate type
  P->g.omega = omT;
  std::vector<long long> sx{g.nx}, sy{g.ny};
  auto odd3 = [](long long n) { return n >= 3 && (n % 2) == 1; };
  while ((pr->mg_levels == 0 || (int)sx.size() < pr->mg_levels) && odd3(sx.back()) &&
         (g.dim == 1 || odd3(sy.back()))) {
    sx.push_back((sx.back() - 1) / 2);
    sy.push_back(g.dim == 2 ? (sy.back() - 1) / 2 : g.ny);
  }
  double* zf = nullptr;
  HJ_CUDA(cudaMalloc(&zf, sizeof(double) * size_t(sx[1]) * size_t(sy[1])));
  hj_status s = HJ_OK;
  cudaError_t e = cudaMemsetAsync(zf, 0, sizeof(double) * size_t(sx[1]) * size_t(sy[1]), P->stream);
  if (e != cudaSuccess) { cudaFree(zf); set_error("multigrid setup: memset"); return HJ_ERR_CUDA; }
  for (size_t l = 1; l < sx.size() && s == HJ_OK; ++l) {
    hj_problem q{};
    q.dim = g.dim;
    q.nx = sx[l];
    q.ny = sy[l];
    q.h = g.h * (double)(1LL << l);
    q.f = zf;
    hj_params r{};
    r.mode = HJ_HIERARCHICAL;
    r.dtype = pr->dtype;
    r.tile_x = (int32_t)std::min<long long>(pr->tile_x, sx[l]);
    r.tile_y = g.dim == 2 ? (int32_t)std::min<long long>(pr->tile_y, sy[l]) : 1;
    r.k = pr->k;
    r.overlap = 0;
    r.overlap_y = 0;
    r.tol = 0.0;
    r.tol_mode = HJ_TOL_RELATIVE;
    r.max_cycles = 1;
    r.kernel = pr->kernel;
    hj_plan* C = nullptr;
    s = plan_build(&q, &r, P->stream, nullptr, &C);
    if (s != HJ_OK) break;
    C->g.omega = (l + 1 == sx.size()) ? 1.0 : omT;   // coarsest: plain cycles
    if (g.dim == 2) {  // TMA boxes of the coarse patch under a fine 32x32 tile + halo (fused correction)
      const size_t esz = g.dtype == HJ_F64 ? 8 : 4;
      for (int b = 0; b < 2 && s == HJ_OK; ++b)
        s = make_tmap(&C->tmE[b], C->X[b], C->g.dtype, (uint64_t)C->g.pitch, (uint64_t)C->g.rows,
                      (uint64_t)C->g.pitch * esz, esz == 8 ? 20 : 24, 18);  // R2<T>::EW x EH
    }
    cudaFree(C->x0_d);                               // coarse levels are never reset
    C->x0_d = nullptr;
    P->mg.push_back(C);
  }
  cudaFree(zf);
  return s;
}

static int kernels_per_smooth(const hj_plan* L) {
  const Geom& g = L->g;
  if (g.kernel_kind != K_REG2D) return 1;
  const long long nfull = (g.nx / 32) * (g.ny / 32);
  return (nfull > 0 ? 1 : 0) + (g.ntiles > nfull ? 1 : 0);
}

// ------------------------------------------------------------------ plans ---
hj_status plan_build(const hj_problem* pb, const hj_params* pr, cudaStream_t st, const DistInfo* di,
                     hj_plan** out) {
  NvtxRange nv("hj_plan_build");
  hj_params prc;
  if (pr && pb && pr->mode == HJ_MULTIGRID) {  // reading c24: every level, the finest included, uses
    prc = *pr;                                 // tile = min(tile, n_level)
    if (prc.tile_x > pb->nx) prc.tile_x = (int32_t)pb->nx;
    if (pb->dim == 2 && prc.tile_y > pb->ny) prc.tile_y = (int32_t)pb->ny;
    pr = &prc;
  }
  HJ_TRY(validate(pb, pr, true));
  int nsm = 0;
  HJ_TRY(ensure_configured(&nsm));
  if (di && pr->mode == HJ_MULTIGRID) {
    set_error("multigrid is not supported with row slabs");
    return HJ_ERR_INVALID_CONFIG;
  }
  hj_plan* P = new hj_plan();
  P->prm = *pr;
  Geom& g = P->g;
  g.dim = pb->dim;
  g.dtype = pr->dtype;
  g.mode = pr->mode;
  g.h = pb->h;
  g.h2 = pb->h * pb->h;
  g.gen = pb->stencil != nullptr;
  g.rdiv = g.h2;
  g.nx = pb->nx;
  const long long ny_global = pb->ny;
  g.ny = di ? (di->row_end - di->row_begin) : pb->ny;
  g.tx = pr->mode == HJ_CLASSIC ? 1 : pr->tile_x;
  g.ty = pr->mode == HJ_CLASSIC ? 1 : pr->tile_y;
  g.k = pr->mode == HJ_CLASSIC ? 1 : pr->k;
  hj_status s = choose_kernel(pb, pr, &g.kernel_kind);
  if (s != HJ_OK) { delete P; return s; }
  P->nsm = nsm;
  const size_t esz = pr->dtype == HJ_F64 ? 8 : 4;
  g.col0 = 16 / esz;
  // tiles / partial layout
  const long long gy0 = di ? di->row_begin : 0;
  g.ox = pr->mode == HJ_HIERARCHICAL ? pr->overlap : 0;
  g.oy = (pr->mode == HJ_HIERARCHICAL && pb->dim == 2) ? (pr->overlap_y < 0 ? pr->overlap : pr->overlap_y) : 0;
  if (di && (g.ox || g.oy)) {
    delete P;
    set_error("overlapping subdomains are not supported with row slabs");
    return HJ_ERR_INVALID_CONFIG;
  }
  if (g.kernel_kind == K_REGT && g.ny % std::max(g.ty, 32) != 0) g.kernel_kind = K_SMEM2D;  // slab rows
  switch (g.kernel_kind) {
    case K_REG2D: case K_SMEM2D: case K_REGT:
      g.ax = make_axis((int)g.nx, g.tx, g.ox);
      g.ay = make_axis((int)g.ny, g.ty, g.oy);
      g.ntx = g.ax.nb;
      g.nty = g.ay.nb;
      g.nrg_global = (ny_global + g.ty - 1) / g.ty;
      g.rg_offset = gy0 / g.ty;
      if (!di) g.nrg_global = g.nty;
      break;
    case K_CLASSIC2D:
      g.ntx = (g.nx + CLASSIC2D_COLS - 1) / CLASSIC2D_COLS;
      g.nty = (g.ny + CLASSIC2D_ROWS - 1) / CLASSIC2D_ROWS;
      g.nrg_global = (ny_global + CLASSIC2D_ROWS - 1) / CLASSIC2D_ROWS;
      g.rg_offset = gy0 / CLASSIC2D_ROWS;
      break;
    case K_REG1D: case K_SMEM1D:  // one row (= row group) per independent problem
      g.ax = make_axis((int)g.nx, g.tx, g.ox);
      g.ntx = g.ax.nb; g.nty = g.ny; g.nrg_global = g.ny; g.rg_offset = 0;
      break;
    default:
      g.ntx = (g.nx + CLASSIC1D_CELLS - 1) / CLASSIC1D_CELLS; g.nty = g.ny; g.nrg_global = g.ny; g.rg_offset = 0;
  }
  g.ntiles = g.ntx * g.nty;
  g.parts_per_row = g.kernel_kind == K_CLASSIC2D ? 4 * g.ntx
                   : g.kernel_kind == K_REGT    ? g.ntx * regt_warps_per_tile(g.tx, g.ty)
                                                : g.ntx;
  g.nparts = g.parts_per_row * g.nty;
  g.nrg_local = g.nty;
  // buffer geometry
  if (g.dim == 2) {
    g.pitch = round_up(g.nx + 2 * g.col0 + 2, 256 / esz);  // 256-B rows
    g.rows = g.ny + 2;
    g.fpitch = round_up(g.nx, 128 / esz);
    g.frows = g.ny;
  } else {
    const long long span = g.ntx * (long long)(g.kernel_kind == K_CLASSIC1D ? CLASSIC1D_CELLS : g.tx);
    g.pitch = round_up(span + 4 * g.col0 + 64, 256 / esz);
    g.rows = g.ny;   // independent problems
    g.fpitch = round_up(span + 64, 128 / esz);
    g.frows = g.ny;
  }
  if (st == nullptr) {
    // The legacy default stream cannot be captured into graphs: run the plan on its own
    // stream, ordered after all prior work on the device (inputs may still be in flight).
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      set_error(std::string("plan stream: ") + cudaGetErrorString(e));
      delete P;
      return HJ_ERR_CUDA;
    }
    P->own_stream = true;
  }
  P->stream = st;
  P->ny_global = ny_global;
  P->gy0 = gy0;
  P->hist_cap = history_capacity(pr->max_cycles);
  const size_t xbytes = size_t(g.pitch) * g.rows * esz;
  const size_t fbytes = size_t(g.fpitch) * g.frows * esz;
  auto fail = [&](hj_status e) { plan_free(P); return e; };
#define PCK(call)                                                                          \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      set_error(std::string(#call) + ": " + cudaGetErrorString(e_));                      \
      return fail(e_ == cudaErrorMemoryAllocation ? HJ_ERR_OOM : HJ_ERR_CUDA);             \
    }                                                                                      \
  } while (0)
  PCK(cudaMalloc(&P->X[0], xbytes));
  PCK(cudaMalloc(&P->X[1], xbytes));
  PCK(cudaMalloc(&P->H2F, fbytes));
  if (g.gen && g.dim == 1) {
    PCK(cudaMalloc(&P->WL, fbytes));
    PCK(cudaMalloc(&P->WR, fbytes));
  }
  PCK(cudaMalloc(&P->part, sizeof(double) * (g.nparts + 1)));
  const bool peer = di && di->transport == 1;
  P->rp_stride = peer ? g.nrg_global + 1 : 0;   // peer: two halves, by cycle parity
  PCK(cudaMalloc(&P->rowpart, sizeof(double) * (g.nrg_global + 1) * (peer ? 2 : 1)));
  P->rowsum_dst = P->rowpart;
  if (di) {
    PCK(cudaMalloc(&P->rowpart_local, sizeof(double) * (g.nrg_global + 1)));
    PCK(cudaMemsetAsync(P->rowpart_local, 0, sizeof(double) * (g.nrg_global + 1), st));
    P->rowsum_dst = P->rowpart_local;
    if (di->transport == 1) {
      P->rowsum_dst = P->rowpart;   // peer: rowsum stores into every rank's rowpart itself
      s = peer_create(P, di);
    } else {
      s = dist_create(P, di);
    }
    if (s != HJ_OK) return fail(s);
  }
  PCK(cudaMalloc(&P->hist, sizeof(double) * P->hist_cap));
  PCK(cudaMalloc(&P->ctrl, sizeof(Ctrl)));
  PCK(cudaMallocHost(&P->ctrl_h, sizeof(Ctrl)));
  PCK(cudaEventCreate(&P->ev0));
  PCK(cudaEventCreate(&P->ev1));
  // keep device copies of x0 / bc so that hj_plan_reset can re-initialise
  const long long nloc = g.nx * g.ny;
  const long long nbc = g.dim == 1 ? 2 * g.ny : 2 * g.nx + 2 * ny_global;
  PCK(cudaMalloc(&P->bc_d, sizeof(double) * nbc));
  if (pb->bc) PCK(cudaMemcpyAsync(P->bc_d, pb->bc, sizeof(double) * nbc, cudaMemcpyDefault, st));
  else PCK(cudaMemsetAsync(P->bc_d, 0, sizeof(double) * nbc, st));
  PCK(cudaMalloc(&P->x0_d, sizeof(double) * nloc));
  if (pb->x0) PCK(cudaMemcpyAsync(P->x0_d, pb->x0, sizeof(double) * nloc, cudaMemcpyDefault, st));
  else PCK(cudaMemsetAsync(P->x0_d, 0, sizeof(double) * nloc, st));
  PCK(cudaMemsetAsync(P->rowpart, 0, sizeof(double) * (g.nrg_global + 1) * (peer ? 2 : 1), st));
  PCK(cudaMemsetAsync(P->part, 0, sizeof(double) * (g.nparts + 1), st));
  if (g.gen) {
    // general coefficients (c23): device copy of the stencil (host or device pointer), checked on
    // the device (finite, non-zero diagonal), then Q / weights
    const long long ns = g.dim == 1 ? 3 * nloc : 5;
    double* st_d = nullptr;
    unsigned long long* bad_d = nullptr;
    unsigned long long bad = 0;
    double st5[5] = {0, 0, 0, 0, 1};
    PCK(cudaMalloc(&st_d, sizeof(double) * ns + sizeof(unsigned long long)));
    bad_d = reinterpret_cast<unsigned long long*>(st_d + ns);
    cudaError_t e = cudaMemcpyAsync(st_d, pb->stencil, sizeof(double) * ns, cudaMemcpyDefault, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(bad_d, 0, sizeof(unsigned long long), st);
    if (e == cudaSuccess) {
      check_stencil_kernel<<<4 * nsm, 256, 0, st>>>(st_d, ns, g.dim == 1 ? nloc : 4, g.dim == 1 ? 2 * nloc : 5, bad_d);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(&bad, bad_d, sizeof(bad), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && g.dim == 2) e = cudaMemcpyAsync(st5, st_d, sizeof(st5), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess && bad == 0) {
      if (g.dim == 2) {
        for (int q = 0; q < 4; ++q)  // T-rounded weights, exact in double
          g.wt[q] = esz == 8 ? -st5[q] / st5[4] : (double)(float)(-st5[q] / st5[4]);
        g.rdiv = 1.0 / std::fabs(st5[4]);
      } else {
        g.rdiv = 1.0;
      }
      if (esz == 8)
        init_gen_kernel<double><<<4 * nsm, 256, 0, st>>>((double*)P->H2F, (double*)P->WL, (double*)P->WR,
                                                         g.fpitch, g.frows, g.nx, g.ny, pb->f, st_d, st5[4]);
      else
        init_gen_kernel<float><<<4 * nsm, 256, 0, st>>>((float*)P->H2F, (float*)P->WL, (float*)P->WR,
                                                        g.fpitch, g.frows, g.nx, g.ny, pb->f, st_d, st5[4]);
      e = cudaGetLastError();
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    }
    cudaFree(st_d);
    if (e != cudaSuccess) {
      set_error(std::string("stencil setup: ") + cudaGetErrorString(e));
      return fail(HJ_ERR_CUDA);
    }
    if (bad) {
      set_error("stencil: non-finite coefficient or zero diagonal");
      return fail(HJ_ERR_INVALID_ARG);
    }
  } else {
    const int blocks = 4 * nsm;
    const double scale = g.dim == 2 ? 0.25 : 0.5;
    if (esz == 8)
      init_q_kernel<double><<<blocks, 256, 0, st>>>((double*)P->H2F, g.fpitch, g.frows, g.nx, g.ny, pb->f, g.h2, scale);
    else
      init_q_kernel<float><<<blocks, 256, 0, st>>>((float*)P->H2F, g.fpitch, g.frows, g.nx, g.ny, pb->f, g.h2, (float)scale);
    PCK(cudaGetLastError());
  }
  if (g.kernel_kind == K_REG2D || g.kernel_kind == K_REGT) {
    using u64 = uint64_t;
    const uint32_t bw = (uint32_t)((((g.col0 + 33) * esz + 15) / 16) * 16 / esz);
    for (int b = 0; b < 2; ++b) {
      s = make_tmap(&P->tmX[b], P->X[b], g.dtype, (u64)g.pitch, (u64)g.rows, (u64)g.pitch * esz, bw, 34);
      if (s != HJ_OK) return fail(s);
      s = make_tmap(&P->tmXs[b], P->X[b], g.dtype, (u64)g.pitch, (u64)g.rows, (u64)g.pitch * esz, 32, 32);
      if (s != HJ_OK) return fail(s);
    }
    s = make_tmap(&P->tmF, P->H2F, g.dtype, (u64)g.fpitch, (u64)g.frows, (u64)g.fpitch * esz, 32, 32);
    if (s != HJ_OK) return fail(s);
  }
  if (pr->mode == HJ_MULTIGRID) {
    s = mg_build(P, pr);
    if (s != HJ_OK) return fail(s);
  }
  s = plan_reset(P);
  if (s != HJ_OK) return fail(s);
#undef PCK
  *out = P;
  return HJ_OK;
}

hj_status plan_reset(hj_plan* P) {
  NvtxRange nv("hj_plan_reset");
  const Geom& g = P->g;
  cudaStream_t st = P->stream;
  const int blocks = 4 * P->nsm;
  for (int b = 0; b < 2; ++b) {
    if (g.dtype == HJ_F64)
      init_x_kernel<double><<<blocks, 256, 0, st>>>((double*)P->X[b], g.pitch, g.rows, g.dim, g.nx,
                                                     P->ny_global, P->gy0, g.ny, P->bc_d, P->x0_d,
                                                     b == 0, (int)g.col0);
    else
      init_x_kernel<float><<<blocks, 256, 0, st>>>((float*)P->X[b], g.pitch, g.rows, g.dim, g.nx,
                                                    P->ny_global, P->gy0, g.ny, P->bc_d, P->x0_d,
                                                    b == 0, (int)g.col0);
    HJ_CUDA(cudaGetLastError());
  }
  Ctrl c0;
  std::memset(&c0, 0, sizeof(c0));
  *P->ctrl_h = c0;
  HJ_CUDA(cudaMemcpyAsync(P->ctrl, P->ctrl_h, sizeof(Ctrl), cudaMemcpyHostToDevice, st));
  if (P->dist) HJ_TRY(dist_initial_exchange(P));
  if (P->peer) HJ_TRY(peer_reset(P));
  HJ_CUDA(cudaStreamSynchronize(st));
  P->c_host = 0;
  return HJ_OK;
}

int launches_per_cycle(const hj_plan* P) {
  const Geom& g = P->g;
  if (!P->mg.empty()) {  // one V-cycle (see launch_vcycle): smoothing, rowsum + finalize,
                         // restriction, correction (unless fused into the post-smoothing)
    const bool fuse2d = g.dim == 2 && P->mg_nu2 > 0;
    const bool fine_fused = fuse2d && ((P->mg_nu1 + P->mg_nu2) & 1) == 0;
    int n = (P->mg_nu1 > 0 ? P->mg_nu1 : 1) * kernels_per_smooth(P) + 2 + P->mg_nu2 * kernels_per_smooth(P) +
            1 + (fine_fused ? 0 : 1);
    for (size_t l = 0; l < P->mg.size(); ++l) {
      const hj_plan* L = P->mg[l];
      if (l + 1 == P->mg.size()) n += P->mg_coarse * kernels_per_smooth(L);
      else n += (P->mg_nu1 + P->mg_nu2) * kernels_per_smooth(L) + 1 + (fuse2d ? 0 : 1);
    }
    return n;
  }
  int n = 3;  // cycle kernel + rowsum + finalize
  if (g.kernel_kind == K_REG2D) {
    const long long nfull = (g.nx / 32) * (g.ny / 32);
    n = (nfull > 0 ? 1 : 0) + (g.ntiles > nfull ? 1 : 0) + 2;
  }
  if (P->peer && g.kernel_kind != K_REG2D && peer_halo_launches(P)) n += 1;  // peer_halo_kernel
  return n;
}

// One hierarchical cycle of level plan L (X[in] -> X[in^1]) as a multigrid smoother; ctrl is the
// fine plan's (done check); maxc = LLONG_MAX for the internal cycles, -1 for a residual-only pass.
static hj_status mg_smooth(hj_plan* L, int in, long long maxc, const Ctrl* ctrl,
                           const hj_plan* cor = nullptr, int cor_buf = 0, bool zero_x = false) {
  CycleArgs a;
  a.zero_x = zero_x;
  if (cor) {  // fused coarse-grid correction (2D): the snapshot is x + P e, e = cor->X[cor_buf]
    a.cor_e = cor->X[cor_buf];
    a.cor_pitch = cor->g.pitch;
    a.tm_cor = &cor->tmE[cor_buf];
  }
  a.xin = L->X[in];
  a.xout = L->X[in ^ 1];
  a.h2f = L->H2F;
  a.wl = nullptr;
  a.wr = nullptr;
  a.tm_in = &L->tmX[in];
  a.tm_f = &L->tmF;
  a.tm_out = &L->tmXs[in ^ 1];
  a.part = L->part;
  a.ctrl = ctrl;
  a.max_cycles = maxc;
  cudaError_t e = L->g.dim == 2 ? launch_cycle_2d(L->g, a, L->nsm, L->stream)
                                : launch_cycle_1d(L->g, a, L->nsm, L->stream);
  if (e != cudaSuccess) { set_error(std::string("smoother launch: ") + cudaGetErrorString(e)); return HJ_ERR_CUDA; }
  return HJ_OK;
}

static hj_status mg_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) { set_error(std::string(what) + ": " + cudaGetErrorString(e)); return HJ_ERR_CUDA; }
  return HJ_OK;
}

// Coarse level l >= 1 (P->mg[l-1]) of the V-cycle; its iterate starts at zero in X[0] (written by
// the restriction); *out = the buffer holding its result.
// 2D coarse levels start from zero without reading it: the first cycle runs in zero-start mode
// and the restriction does not write the zeros (unless that level's first step is not a cycle).
static bool mg_zero_start(const hj_plan* P, size_t l) {  // level l >= 1
  if (P->g.dim != 2) return false;
  return l == P->mg.size() ? P->mg_coarse > 0 : P->mg_nu1 > 0;
}

static hj_status mg_level(hj_plan* P, size_t l, int* out) {
  hj_plan* L = P->mg[l - 1];
  const long long INF = LLONG_MAX;
  const bool z = mg_zero_start(P, l);
  int cur = 0;
  if (l == P->mg.size()) {  // coarsest grid: plain cycles from zero
    for (int c = 0; c < P->mg_coarse; ++c, cur ^= 1)
      HJ_TRY(mg_smooth(L, cur, INF, P->ctrl, nullptr, 0, z && c == 0));
    *out = cur;
    return HJ_OK;
  }
  hj_plan* N = P->mg[l];
  for (int c = 0; c < P->mg_nu1; ++c, cur ^= 1) HJ_TRY(mg_smooth(L, cur, INF, P->ctrl, nullptr, 0, z && c == 0));
  HJ_TRY(mg_check(launch_mg_restrict(L->g, L->X[cur], L->H2F, N->g, N->H2F, N->X[0], !mg_zero_start(P, l + 1),
                                     P->ctrl, P->stream), "restrict"));
  int ec = 0;
  HJ_TRY(mg_level(P, l + 1, &ec));
  int c = 0;
  if (L->g.dim == 2 && P->mg_nu2 > 0) {  // correction fused into the first post-smoothing cycle
    HJ_TRY(mg_smooth(L, cur, INF, P->ctrl, N, ec));
    cur ^= 1;
    c = 1;
  } else {
    HJ_TRY(mg_check(launch_mg_correct(L->g, L->X[cur], L->X[cur], N->g, N->X[ec], P->ctrl, P->stream), "correct"));
  }
  for (; c < P->mg_nu2; ++c, cur ^= 1) HJ_TRY(mg_smooth(L, cur, INF, P->ctrl));
  *out = cur;
  return HJ_OK;
}

// One V-cycle of the multigrid plan: x_c in X[0] -> x_{c+1} in X[0].  The first fine smoothing
// cycle (or a residual-only pass when nu1 = 0) carries the fused residual of x_c, reduced and
// tested right after it, so a converged solve skips the rest of this V-cycle (every later kernel
// checks Ctrl::done) and x_c stays intact in X[0].  The fine correction is written out of place
// when nu1 + nu2 is odd so that every V-cycle ends in X[0].
static hj_status launch_vcycle(hj_plan* P, bool timed) {
  const Geom& g = P->g;
  cudaStream_t st = P->stream;
  const long long INF = LLONG_MAX;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (timed) {
    while (P->evpool.size() < 2 * size_t(P->evused + 1)) {
      cudaEvent_t ev;
      HJ_CUDA(cudaEventCreate(&ev));
      P->evpool.push_back(ev);
    }
    e0 = P->evpool[2 * P->evused];
    e1 = P->evpool[2 * P->evused + 1];
    P->evused++;
    HJ_CUDA(cudaEventRecord(e0, st));
  }
  int cur = 0;
  if (P->mg_nu1 > 0) {
    HJ_TRY(mg_smooth(P, 0, P->prm.max_cycles, P->ctrl));
    cur = 1;
  } else {
    HJ_TRY(mg_smooth(P, 0, -1, P->ctrl));  // residual of x_c only
  }
  const int wpb = 8;
  rowsum_kernel<<<(unsigned)((g.nrg_local + wpb - 1) / wpb), 32 * wpb, 0, st>>>(
      P->part, g.parts_per_row, g.nrg_local, g.rg_offset, P->rowsum_dst, P->ctrl, PeerDsts{}, 0);
  HJ_CUDA(cudaGetLastError());
  finalize_kernel<<<1, 1024, 0, st>>>(P->rowpart, g.nrg_global, P->ctrl, P->hist, P->hist_cap, g.rdiv,
                                      P->prm.tol, (int)P->prm.tol_mode, P->prm.ref_residual,
                                      P->prm.max_cycles, PeerSync{}, 0);
  HJ_CUDA(cudaGetLastError());
  for (int c = 1; c < P->mg_nu1; ++c, cur ^= 1) HJ_TRY(mg_smooth(P, cur, INF, P->ctrl));
  hj_plan* N = P->mg[0];
  HJ_TRY(mg_check(launch_mg_restrict(g, P->X[cur], P->H2F, N->g, N->H2F, N->X[0], !mg_zero_start(P, 1),
                                     P->ctrl, st), "restrict"));
  int ec = 0;
  HJ_TRY(mg_level(P, 1, &ec));
  const int flip = (P->mg_nu1 + P->mg_nu2) & 1;
  int c2 = 0;
  if (g.dim == 2 && P->mg_nu2 > 0 && !flip) {  // correction fused into the first post-smoothing cycle
    HJ_TRY(mg_smooth(P, cur, INF, P->ctrl, N, ec));
    cur ^= 1;
    c2 = 1;
  } else {
    HJ_TRY(mg_check(launch_mg_correct(g, P->X[cur], P->X[cur ^ flip], N->g, N->X[ec], P->ctrl, st), "correct"));
    cur ^= flip;
  }
  for (; c2 < P->mg_nu2; ++c2, cur ^= 1) HJ_TRY(mg_smooth(P, cur, INF, P->ctrl));
  if (cur != 0) { set_error("internal: V-cycle parity"); return HJ_ERR_CUDA; }
  if (timed) HJ_CUDA(cudaEventRecord(e1, st));
  return HJ_OK;
}

// One cycle with static parity p: X[p] -> X[p^1].
hj_status launch_cycle(hj_plan* P, int p, bool timed, float* acc_ms) {
  if (!P->mg.empty()) return launch_vcycle(P, timed);
  const Geom& g = P->g;
  cudaStream_t st = P->stream;
  CycleArgs a;
  a.xin = P->X[p];
  a.xout = P->X[p ^ 1];
  a.h2f = P->H2F;
  a.wl = P->WL;
  a.wr = P->WR;
  a.tm_in = &P->tmX[p];
  a.tm_f = &P->tmF;
  a.tm_out = &P->tmXs[p ^ 1];
  a.part = P->part;
  a.ctrl = P->ctrl;
  a.max_cycles = P->prm.max_cycles;
  if (P->peer && g.kernel_kind == K_REG2D) peer_halo_ptrs(P, p ^ 1, &a.peer_lo, &a.peer_hi);
  (void)acc_ms;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (timed) {
    while (P->evpool.size() < 2 * size_t(P->evused + 1)) {
      cudaEvent_t ev;
      HJ_CUDA(cudaEventCreate(&ev));
      P->evpool.push_back(ev);
    }
    e0 = P->evpool[2 * P->evused];
    e1 = P->evpool[2 * P->evused + 1];
    P->evused++;
    HJ_CUDA(cudaEventRecord(e0, st));
  }
  const bool ovl = dist_overlap(P);
  // HJ_SPLIT_CYCLE=1 (tests): the overlapped transport's split launch order (boundary tile rows,
  // then interior tile rows) on any REG2D plan without edge tiles, so its kernel path is exercised
  // where NCCL cannot run with several ranks (one GPU)
  static const bool split_env = [] { const char* e = std::getenv("HJ_SPLIT_CYCLE"); return e && e[0] == '1'; }();
  const bool split = ovl || (split_env && g.dim == 2 && g.kernel_kind == K_REG2D && !g.ox && !g.oy &&
                             g.nx % 32 == 0 && g.ny % 32 == 0 && g.ny / 32 >= 3 && !a.cor_e && !a.zero_x);
  cudaError_t e;
  if (split) {
    // overlapped NCCL transport: the slab's boundary tile rows first, their rows sent
    // on the comm stream while the interior tile rows run, joined before the next cycle
    const int nty = (int)(g.ny / 32);
    a.ty0 = 0; a.tys = nty - 1; a.nty_run = 2;
    e = launch_cycle_2d(g, a, P->nsm, st);
    if (e == cudaSuccess) {
      if (ovl) HJ_TRY(dist_halo_fork(P, p ^ 1));
      a.ty0 = 1; a.tys = 1; a.nty_run = nty - 2;
      e = launch_cycle_2d(g, a, P->nsm, st);
    }
  } else {
    e = g.dim == 2 ? launch_cycle_2d(g, a, P->nsm, st) : launch_cycle_1d(g, a, P->nsm, st);
  }
  if (e != cudaSuccess) {
    set_error(std::string("cycle kernel launch: ") + cudaGetErrorString(e));
    return HJ_ERR_CUDA;
  }
  if (timed) HJ_CUDA(cudaEventRecord(e1, st));
  if (P->dist && !ovl) HJ_TRY(dist_halo_exchange(P, p ^ 1));
  PeerDsts pd{};
  PeerSync ps{};
  if (P->peer) {
    if (g.kernel_kind != K_REG2D) HJ_TRY(peer_halo(P, p ^ 1));  // REG2D: fused into the cycle kernel
    peer_cycle_args(P, &pd, &ps);
  }
  const int wpb = 8;
  rowsum_kernel<<<(unsigned)((g.nrg_local + wpb - 1) / wpb), 32 * wpb, 0, st>>>(
      P->part, g.parts_per_row, g.nrg_local, g.rg_offset, P->rowsum_dst, P->ctrl, pd, P->rp_stride);
  HJ_CUDA(cudaGetLastError());
  if (P->dist) HJ_TRY(dist_allreduce(P));
  finalize_kernel<<<1, 1024, 0, st>>>(P->rowpart, g.nrg_global, P->ctrl, P->hist, P->hist_cap, g.rdiv,
                                      P->prm.tol, (int)P->prm.tol_mode, P->prm.ref_residual,
                                      P->prm.max_cycles, ps, P->rp_stride);
  HJ_CUDA(cudaGetLastError());
  if (ovl) HJ_TRY(dist_halo_join(P));
  return HJ_OK;
}

static hj_status drain_events(hj_plan* P, float* acc) {
  if (P->evused == 0) return HJ_OK;
  HJ_CUDA(cudaEventSynchronize(P->evpool[2 * P->evused - 1]));
  for (int i = 0; i < P->evused; ++i) {
    float ms = 0.f;
    HJ_CUDA(cudaEventElapsedTime(&ms, P->evpool[2 * i], P->evpool[2 * i + 1]));
    *acc += ms;
  }
  P->evused = 0;
  return HJ_OK;
}

static hj_status get_graph(hj_plan* P, int G, cudaGraphExec_t* out) {
  auto it = P->graphs.find(G);
  if (it != P->graphs.end()) { *out = it->second; return HJ_OK; }
  NvtxRange nv("hj_graph_capture");
  cudaGraph_t graph;
  HJ_CUDA(cudaStreamBeginCapture(P->stream, cudaStreamCaptureModeThreadLocal));
  hj_status s = HJ_OK;
  for (int i = 0; i < G && s == HJ_OK; ++i) s = launch_cycle(P, i & 1, false, nullptr);
  cudaError_t e = cudaStreamEndCapture(P->stream, &graph);
  if (s != HJ_OK) return s;
  if (e != cudaSuccess) { set_error(std::string("graph capture: ") + cudaGetErrorString(e)); return HJ_ERR_CUDA; }
  cudaGraphExec_t ex;
  e = cudaGraphInstantiate(&ex, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) { set_error(std::string("graph instantiate: ") + cudaGetErrorString(e)); return HJ_ERR_CUDA; }
  P->graphs[G] = ex;
  *out = ex;
  return HJ_OK;
}

hj_status plan_run(hj_plan* P, long long ncycles, float* kernel_ms) {
  NvtxRange nv("hj_plan_run");
  if (ncycles < 0) { set_error("ncycles must be >= 0"); return HJ_ERR_INVALID_ARG; }
  if (P->peer && !peer_attached(P)) { set_error("peer plan used before hj_plan_peer_attach"); return HJ_ERR_PEER; }
  if (kernel_ms) {
    // eager launches, CUDA events around every cycle kernel, one synchronisation at the end
    *kernel_ms = 0.f;
    P->evused = 0;
    for (long long i = 0; i < ncycles; ++i) {
      HJ_TRY(launch_cycle(P, (int)(P->c_host & 1), true, kernel_ms));
      P->c_host++;
      if (P->evused == 4096) HJ_TRY(drain_events(P, kernel_ms));
    }
    HJ_TRY(drain_events(P, kernel_ms));
    if (P->dist) HJ_TRY(dist_check(P));
    return HJ_OK;
  }
  long long left = ncycles;
  if (left > 0 && (P->c_host & 1)) {  // graphs start at even parity
    HJ_TRY(launch_cycle(P, 1, false, nullptr));
    P->c_host++;
    left--;
  }
  while (left >= 2) {
    const int G = left >= 64 ? 64 : (int)(left & ~1LL);
    cudaGraphExec_t ex;
    HJ_TRY(get_graph(P, G, &ex));
    HJ_CUDA(cudaGraphLaunch(ex, P->stream));
    P->c_host += G;
    left -= G;
  }
  if (left == 1) {
    HJ_TRY(launch_cycle(P, 0, false, nullptr));
    P->c_host++;
  }
  return HJ_OK;
}

// The resident solver applies to single-GPU hierarchical 2D plans whose 32x32 tiles fit one per
// warp of one co-resident wave (8 warps x #SMs): no overlap, nx and ny multiples of 32, Poisson or
// general coefficients.  HJ_RESIDENT=0 disables it (the per-cycle path, HBM tile loads each cycle).
static bool resident_ok(const hj_plan* P) {
  const Geom& g = P->g;
  if (P->dist || P->peer || !P->mg.empty() || g.omega != 1.0) return false;
  if (const char* e = std::getenv("HJ_RESIDENT")) if (e[0] == '0') return false;
  if (g.dim == 1) {  // register 1D plans (tiles of 32..1024 points), no ragged tile
    if (g.kernel_kind != K_REG1D || g.gen || g.ox != 0 || g.nx % g.tx) return false;
    const long long nt = (g.nx / g.tx) * g.ny;
    if (nt <= 8LL * P->nsm && g.ny <= 1024) return true;            // one tile per warp (res1d)
    return g.tx == 32 && nt <= 8LL * 32 * P->nsm && nt < (1LL << 31);  // up to 32 tiles per warp (res1dm)
  }
  // hierarchical register plans only: the classic comparison stays the paper's global-memory sweep
  if (!(g.kernel_kind == K_REG2D && g.tx == 32 && g.ty == 32 && g.ox == 0 && g.oy == 0)) return false;
  if (g.nx % 32 || g.ny % 32) return false;
  return (g.nx / 32) * (g.ny / 32) <= std::min(8LL * P->nsm, 1184LL);
}

static hj_status run_resident(hj_plan* P, bool* used) {
  const Geom& g = P->g;
  *used = false;
  const long long ntiles = g.dim == 2 ? (g.nx / 32) * (g.ny / 32) : (g.nx / g.tx) * g.ny;
  const bool many = g.dim == 1 && !(ntiles <= 8LL * P->nsm && g.ny <= 1024);
  if (many && !P->res_R) HJ_CUDA(cudaMalloc(&P->res_R, sizeof(double) * 2 * g.ny));
  if (!P->res_part) {
    HJ_CUDA(cudaMalloc(&P->res_part, sizeof(double) * 2 * ntiles));
    HJ_CUDA(cudaMalloc(&P->res_bar, 2 * sizeof(unsigned int)));
    HJ_CUDA(cudaMemsetAsync(P->res_bar, 0, 2 * sizeof(unsigned int), P->stream));
  }
  const int k = g.k;
  cudaError_t e;
  int rc_c = 0, rc_d = 0;
  if (res1c_ok(g, &rc_c, &rc_d)) {
    // one small 1D problem: the whole solve in one CTA (res1c_kernel)
    e = launch_resident_1c(g, rc_c, rc_d, P->X[0], P->X[1], P->H2F, P->ctrl, P->hist, P->hist_cap, P->prm.tol,
                           (int)P->prm.tol_mode, P->prm.ref_residual, P->prm.max_cycles, k, P->stream);
    HJ_CUDA(e);
    *used = true;
    return HJ_OK;
  }
  if (res1w_ok(g) && !(std::getenv("HJ_RES1W") && std::getenv("HJ_RES1W")[0] == '0')) {
    // one small 1D problem: the whole solve in one warp (res1w_kernel)
    e = launch_resident_1w(g, P->X[0], P->X[1], P->H2F, P->ctrl, P->hist, P->hist_cap, P->prm.tol,
                           (int)P->prm.tol_mode, P->prm.ref_residual, P->prm.max_cycles, k, P->stream);
    HJ_CUDA(e);
    *used = true;
    return HJ_OK;
  }
  if (many) {
    // M <= 16: two CTAs per SM (<= 128 registers), M = 32: one
    int M = 2;
    while (M < 32 && ntiles > 8LL * M * (M <= 16 ? 2 : 1) * P->nsm) M *= 2;
    e = launch_resident_1dm(g, M, P->X[0], P->X[1], P->H2F, P->res_part, P->res_R, P->ctrl, P->hist, P->hist_cap,
                            P->prm.tol, (int)P->prm.tol_mode, P->prm.ref_residual, P->prm.max_cycles, k,
                            P->res_bar, P->stream);
  } else {
    e = (g.dim == 2 ? launch_resident_2d : launch_resident_1d)(
        g, P->X[0], P->X[1], P->H2F, P->res_part, P->ctrl, P->hist, P->hist_cap, P->prm.tol,
        (int)P->prm.tol_mode, P->prm.ref_residual, P->prm.max_cycles, k, P->res_bar, P->stream);
  }
  if (e == cudaErrorCooperativeLaunchTooLarge) {  // not co-resident here: the per-cycle path
    (void)cudaGetLastError();
    return HJ_OK;
  }
  HJ_CUDA(e);
  *used = true;
  return HJ_OK;
}

hj_status plan_solve(hj_plan* P, hj_result* res, double* x_dev, double* hist_dev) {
  NvtxRange nv("hj_plan_solve");
  const Geom& g = P->g;
  if (P->peer && !peer_attached(P)) { set_error("peer plan used before hj_plan_peer_attach"); return HJ_ERR_PEER; }
  cudaStream_t st = P->stream;
  HJ_CUDA(cudaEventRecord(P->ev0, st));
  bool resident = false;
  if (resident_ok(P)) HJ_TRY(run_resident(P, &resident));
  if (resident) {
    HJ_CUDA(cudaMemcpyAsync(P->ctrl_h, P->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
    HJ_CUDA(cudaStreamSynchronize(st));
    P->c_host = P->ctrl_h->c;
  } else {
    if (P->c_host & 1) {  // graphs start at even parity
      HJ_TRY(launch_cycle(P, 1, false, nullptr));
      P->c_host++;
    }
    int G = 2;
    for (;;) {
      cudaGraphExec_t ex;
      HJ_TRY(get_graph(P, G, &ex));
      HJ_CUDA(cudaGraphLaunch(ex, st));
      P->c_host += G;
      HJ_CUDA(cudaMemcpyAsync(P->ctrl_h, P->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
      HJ_CUDA(cudaStreamSynchronize(st));
      if (P->dist) HJ_TRY(dist_check(P));
      if (P->ctrl_h->done) break;
      if (G < 256) G *= 2;
    }
  }
  HJ_CUDA(cudaEventRecord(P->ev1, st));
  HJ_CUDA(cudaEventSynchronize(P->ev1));
  float ms = 0.f;
  HJ_CUDA(cudaEventElapsedTime(&ms, P->ev0, P->ev1));
  const Ctrl c = *P->ctrl_h;
  const long long cd = c.c_done;
  if (x_dev) {
    const void* X = P->X[P->mg.empty() ? (cd & 1) : 0];  // multigrid: every V-cycle ends in X[0]
    const int blocks = 4 * P->nsm;
    if (g.dtype == HJ_F64)
      extract_kernel<double><<<blocks, 256, 0, st>>>((const double*)X, g.pitch, g.dim, g.nx, g.ny, (int)g.col0, x_dev);
    else
      extract_kernel<float><<<blocks, 256, 0, st>>>((const float*)X, g.pitch, g.dim, g.nx, g.ny, (int)g.col0, x_dev);
    HJ_CUDA(cudaGetLastError());
  }
  // the history holds min(cycles + 1, hist_cap) entries (truncated past the cap, never beyond it)
  if (hist_dev)
    HJ_CUDA(cudaMemcpyAsync(hist_dev, P->hist, sizeof(double) * lmin(cd + 1, P->hist_cap), cudaMemcpyDeviceToDevice, st));
  HJ_CUDA(cudaStreamSynchronize(st));
  res->cycles = cd;
  res->converged = c.converged;
  res->initial_residual = std::sqrt(c.S0) / g.rdiv;
  res->final_residual = std::sqrt(c.S_last) / g.rdiv;
  res->seconds_solve = ms * 1e-3;
  // the plan is now "used": reset before another solve
  return (hj_status)c.status;
}

void plan_free(hj_plan* P) {
  if (!P) return;
  for (hj_plan* C : P->mg) plan_free(C);
  P->mg.clear();
  for (auto& kv : P->graphs) cudaGraphExecDestroy(kv.second);
  if (P->dist) dist_free(P);
  if (P->peer) peer_free(P);
  cudaFree(P->res_part);
  cudaFree(P->res_R);
  cudaFree(P->res_bar);
  cudaFree(P->X[0]);
  cudaFree(P->X[1]);
  cudaFree(P->H2F);
  cudaFree(P->WL);
  cudaFree(P->WR);
  cudaFree(P->part);
  cudaFree(P->rowpart);
  cudaFree(P->rowpart_local);
  cudaFree(P->hist);
  cudaFree(P->ctrl);
  cudaFree(P->bc_d);
  cudaFree(P->x0_d);
  if (P->ctrl_h) cudaFreeHost(P->ctrl_h);
  for (auto ev : P->evpool) cudaEventDestroy(ev);
  if (P->own_stream) {
    cudaStreamSynchronize(P->stream);
    cudaStreamDestroy(P->stream);
  }
  if (P->ev0) cudaEventDestroy(P->ev0);
  if (P->ev1) cudaEventDestroy(P->ev1);
  delete P;
}

}  // namespace hj

// ==================================================================== C-ABI ==
using namespace hj;

extern "C" {

const char* hj_last_error(void) { return g_last_error.c_str(); }

hj_status hj_resource_figures(const hj_problem* pb, const hj_params* pr, int64_t* tiles,
                              int64_t* threads, int64_t* smem) {
  if (!tiles || !threads || !smem) { set_error("NULL output"); return HJ_ERR_INVALID_ARG; }
  HJ_TRY(validate(pb, pr, false));
  const long long esz = pr->dtype == HJ_F64 ? 8 : 4;
  if (pr->mode == HJ_CLASSIC) {
    *tiles = 0; *threads = pb->nx * pb->ny; *smem = 0;
    return HJ_OK;
  }
  const long long tx = pr->tile_x, ty = pb->dim == 2 ? pr->tile_y : 1;
  const int oy = pb->dim == 2 ? (pr->overlap_y < 0 ? pr->overlap : pr->overlap_y) : 0;
  const long long ntx = axis_nb((int)pb->nx, (int)tx, pr->overlap);
  const long long nty = pb->dim == 2 ? axis_nb((int)pb->ny, (int)ty, oy) : pb->ny;  // 1D: per problem
  *tiles = ntx * nty;
  *threads = *tiles * tx * ty;
  *smem = pb->dim == 1 ? esz * (2 * (tx + 2) + tx) : esz * (2 * (tx + 2) * (ty + 2) + tx * ty);
  return HJ_OK;
}

hj_status hj_plan_create(const hj_problem* pb, const hj_params* pr, void* stream, hj_plan** plan) {
  if (!plan) { set_error("NULL plan"); return HJ_ERR_INVALID_ARG; }
  return plan_build(pb, pr, (cudaStream_t)stream, nullptr, plan);
}
hj_status hj_plan_create_dist(const hj_problem* pb, const hj_params* pr, const hj_dist* dist,
                              void* stream, hj_plan** plan) {
  if (!plan || !dist || !dist->nccl_id) { set_error("NULL argument"); return HJ_ERR_INVALID_ARG; }
  HJ_TRY(validate_dist(pb, pr, dist));
  DistInfo di{dist->rank, dist->nranks, dist->row_begin, dist->row_end, dist->nccl_id};
  return plan_build(pb, pr, (cudaStream_t)stream, &di, plan);
}
hj_status hj_plan_reset(hj_plan* P) {
  if (!P) { set_error("NULL plan"); return HJ_ERR_INVALID_ARG; }
  return plan_reset(P);
}
hj_status hj_plan_run(hj_plan* P, int64_t ncycles, float* kernel_ms) {
  if (!P) { set_error("NULL plan"); return HJ_ERR_INVALID_ARG; }
  return plan_run(P, ncycles, kernel_ms);
}
hj_status hj_plan_solve(hj_plan* P, hj_result* res) {
  if (!P || !res) { set_error("NULL argument"); return HJ_ERR_INVALID_ARG; }
  return plan_solve(P, res, res->x, res->history);
}
int64_t hj_history_capacity(const hj_params* pr) { return pr ? history_capacity(pr->max_cycles) : 0; }
int32_t hj_plan_launches_per_cycle(const hj_plan* P) { return P ? launches_per_cycle(P) : 0; }
int32_t hj_plan_kernel_kind(const hj_plan* P) { return P ? P->g.kernel_kind : -1; }
hj_status hj_plan_destroy(hj_plan* P) {
  plan_free(P);
  return HJ_OK;
}

hj_status jacobi_solve_device(const hj_problem* pb, const hj_params* pr, hj_result* res, void* stream) {
  if (!res) { set_error("NULL result"); return HJ_ERR_INVALID_ARG; }
  if (res->history && pr && history_capacity(pr->max_cycles) < pr->max_cycles + 1) {
    set_error("history is limited to 2^24 cycles (HJ_HIST_CAP); pass history = NULL");
    return HJ_ERR_INVALID_CONFIG;
  }
  auto t0 = std::chrono::steady_clock::now();
  hj_plan* P = nullptr;
  HJ_TRY(plan_build(pb, pr, (cudaStream_t)stream, nullptr, &P));
  hj_status s = plan_solve(P, res, res->x, res->history);
  plan_free(P);
  res->seconds_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return s;
}

hj_status jacobi_solve(const hj_problem* pb, const hj_params* pr, hj_result* res) {
  if (!res || !res->x) { set_error("NULL result or result->x"); return HJ_ERR_INVALID_ARG; }
  HJ_TRY(validate(pb, pr, true));
  if (res->history && history_capacity(pr->max_cycles) < pr->max_cycles + 1) {
    set_error("history is limited to 2^24 cycles (HJ_HIST_CAP); pass history = NULL");
    return HJ_ERR_INVALID_CONFIG;
  }
  auto t0 = std::chrono::steady_clock::now();
  const long long n = pb->nx * pb->ny;
  const long long nbc = pb->dim == 1 ? 2 * pb->ny : 2 * pb->nx + 2 * pb->ny;
  double *f = nullptr, *bc = nullptr, *x0 = nullptr, *x = nullptr, *hist = nullptr;
  cudaStream_t st;
  HJ_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  hj_status s = HJ_OK;
  auto cleanup = [&]() {
    cudaFree(f); cudaFree(bc); cudaFree(x0); cudaFree(x); cudaFree(hist);
    cudaStreamDestroy(st);
  };
#define SCK(call)                                                                          \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      set_error(std::string(#call) + ": " + cudaGetErrorString(e_));                      \
      cleanup();                                                                           \
      return e_ == cudaErrorMemoryAllocation ? HJ_ERR_OOM : HJ_ERR_CUDA;                   \
    }                                                                                      \
  } while (0)
  SCK(cudaMalloc(&f, sizeof(double) * n));
  SCK(cudaMemcpyAsync(f, pb->f, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  if (pb->bc) {
    SCK(cudaMalloc(&bc, sizeof(double) * nbc));
    SCK(cudaMemcpyAsync(bc, pb->bc, sizeof(double) * nbc, cudaMemcpyHostToDevice, st));
  }
  if (pb->x0) {
    SCK(cudaMalloc(&x0, sizeof(double) * n));
    SCK(cudaMemcpyAsync(x0, pb->x0, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  }
  SCK(cudaMalloc(&x, sizeof(double) * n));
  if (res->history) SCK(cudaMalloc(&hist, sizeof(double) * history_capacity(pr->max_cycles)));
  hj_problem dp = *pb;
  dp.f = f;
  dp.bc = bc;
  dp.x0 = x0;
  hj_plan* P = nullptr;
  s = plan_build(&dp, pr, st, nullptr, &P);
  if (s != HJ_OK) { cleanup(); return s; }
  double* hx = res->x;
  double* hh = res->history;
  s = plan_solve(P, res, x, hist);
  res->x = hx;
  res->history = hh;
  plan_free(P);
  if (s == HJ_OK || s == HJ_NOT_CONVERGED || s == HJ_ERR_NUMERIC) {
    SCK(cudaMemcpyAsync(hx, x, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    if (hh) SCK(cudaMemcpyAsync(hh, hist, sizeof(double) * lmin(res->cycles + 1, history_capacity(pr->max_cycles)), cudaMemcpyDeviceToHost, st));
    SCK(cudaStreamSynchronize(st));
  }
#undef SCK
  cleanup();
  res->seconds_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return s;
}

}  // extern "C"
