// Peer-memory transport for row slabs (north star multi-GPU): the per-cycle
// exchange of the hierarchical Jacobi path done by the library's own kernels through CUDA IPC
// mappings of the neighbours' buffers (NVLink / NVSwitch loads and stores between GPUs; also
// valid between processes sharing one GPU), instead of NCCL calls.
//
// Per cycle c (all on the plan's stream, captured in the cycle graph):
//   cycle kernel        X[p] -> X[p^1] (local), per-tile residual partials
//   peer_halo_kernel    row 1 of X[p^1] -> ghost row R+1 of rank-1's X[p^1];
//                       row R          -> ghost row 0   of rank+1's X[p^1]      (remote stores)
//   rowsum_kernel       this rank's row-group sums -> every rank's rowpart      (remote stores)
//   finalize_kernel     signal: fence.sys + atomicAdd_system on every rank's flag; wait:
//                       ld.acquire.sys on the own flag until all nranks signals of cycle c
//                       arrived (bounded spin, HJ_ERR_PEER on timeout); then the usual
//                       fixed-order sum of rowpart and stopping test.
// Every rank sums the same vector in the same order, so histories, counts and iterates are
// bitwise equal to the single-GPU solve (DESIGN.md c18).
//
// Hazards (why one flag wait per cycle suffices): a rank starts cycle c+1 only after every rank
// signalled cycle c, i.e. after every rank's cycle kernel c finished reading X[p] and every halo /
// rowsum store of cycle c was fenced.  Cycle c+1 writes the neighbours' X[p] ghost rows, which
// nobody reads until cycle c+2.
//
// Reset (collective): local init -> barrier B1 -> record the own signal count (sig0) -> push the
// initial ghost rows of X[0] -> barrier B2.  Barriers are a second monotonic counter per rank.
#include <cstdlib>
#include <cstring>
#include <string>

#include "hj_internal.cuh"
#include "hj_plan.h"

namespace {

constexpr uint32_t PEER_MAGIC = 0x524a4850u;  // "HJPR"

// The exported description of one rank's window (HJ_PEER_HANDLE_BYTES).
struct PeerBlob {
  uint32_t magic, version;
  int32_t rank, nranks, dtype, pad;
  int64_t nx, pitch, col0, rows_local, row_begin, nrg_global;
  cudaIpcMemHandle_t h_x0, h_x1, h_rowpart, h_flags;
};
static_assert(sizeof(PeerBlob) <= HJ_PEER_HANDLE_BYTES, "peer blob size");

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Increment every rank's counter (release), then wait until the own counter reaches want.
__device__ int signal_and_wait(unsigned long long* const* flags, int n, unsigned long long* own,
                               unsigned long long want, long long timeout_ns) {
  __threadfence_system();
  for (int r = 0; r < n; ++r) atomicAdd_system(flags[r], 1ULL);
  const unsigned long long t0 = globaltimer();
  while (ld_acquire_sys(own) < want) {
    if ((long long)(globaltimer() - t0) > timeout_ns) return 1;
    __nanosleep(200);
  }
  return 0;
}

__global__ void peer_barrier_kernel(hj::PeerSync bar, unsigned long long want, int* err) {
  if (threadIdx.x == 0 && signal_and_wait(bar.flag, bar.n, bar.own, want, bar.timeout_ns)) *err = 1;
}

__global__ void peer_sig0_kernel(hj::Ctrl* ctrl, const unsigned long long* own_sig) {
  if (threadIdx.x == 0) ctrl->sig0 = ld_acquire_sys(own_sig);
}

// Rows 1 and R of the local X[buf] into the neighbours' ghost rows (remote stores), then a
// system fence so that the finalize signal that follows publishes them.
template <typename T>
__global__ void peer_halo_kernel(const T* __restrict__ X, long long pitch, long long col0,
                                 long long nx, long long R, T* lo, T* hi,
                                 const hj::Ctrl* __restrict__ ctrl) {
  if (ctrl && ctrl->done) return;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nx;
       i += (long long)gridDim.x * blockDim.x) {
    if (lo) lo[i] = X[pitch + col0 + i];
    if (hi) hi[i] = X[R * pitch + col0 + i];
  }
  __threadfence_system();
}

}  // namespace

struct PeerState {
  int rank = 0, nranks = 1;
  long long row_begin = 0;
  unsigned long long* flags = nullptr;  // own window: [0] = cycle signals, [1] = barrier count
  bool attached = false;
  long long bar_epoch = 0;
  long long timeout_ns = 30LL * 1000 * 1000 * 1000;
  void* opened[hj::HJ_MAX_RANKS][4] = {};  // IPC mappings to close (x0, x1, rowpart, flags)
  hj::PeerDsts dsts{};                     // every rank's rowpart
  hj::PeerSync sig{}, bar{};               // every rank's signal / barrier counter
  void* lo[2] = {nullptr, nullptr};        // rank-1's ghost row R_{r-1}+1 in X[0] / X[1]
  void* hi[2] = {nullptr, nullptr};        // rank+1's ghost row 0 in X[0] / X[1]
  int* err_d = nullptr;
};

namespace hj {

hj_status peer_create(hj_plan* P, const DistInfo* di) {
  PeerState* ps = new PeerState();
  P->peer = ps;
  ps->rank = di->rank;
  ps->nranks = di->nranks;
  ps->row_begin = di->row_begin;
  if (di->nranks > HJ_MAX_RANKS) { set_error("peer transport: at most 64 ranks"); return HJ_ERR_INVALID_CONFIG; }
  if (const char* t = std::getenv("HJ_PEER_TIMEOUT_S")) ps->timeout_ns = (long long)(std::atof(t) * 1e9);
  HJ_CUDA(cudaMalloc(&ps->flags, 256));
  HJ_CUDA(cudaMemset(ps->flags, 0, 256));
  HJ_CUDA(cudaMalloc(&ps->err_d, sizeof(int)));
  HJ_CUDA(cudaMemset(ps->err_d, 0, sizeof(int)));
  HJ_CUDA(cudaDeviceSynchronize());
  return HJ_OK;
}

bool peer_attached(const hj_plan* P) { return P->peer && P->peer->attached; }
int peer_halo_launches(const hj_plan* P) { return (P->peer->lo[0] || P->peer->hi[0]) ? 1 : 0; }

static hj_status peer_barrier(hj_plan* P) {
  PeerState* ps = P->peer;
  ps->bar_epoch++;
  peer_barrier_kernel<<<1, 32, 0, P->stream>>>(ps->bar, (unsigned long long)ps->nranks * ps->bar_epoch,
                                               ps->err_d);
  HJ_CUDA(cudaGetLastError());
  return HJ_OK;
}

static hj_status launch_halo(hj_plan* P, int buf, const Ctrl* ctrl) {
  PeerState* ps = P->peer;
  const Geom& g = P->g;
  if (!ps->lo[buf] && !ps->hi[buf]) return HJ_OK;
  const int blocks = (int)((g.nx + 255) / 256 < 4 * P->nsm ? (g.nx + 255) / 256 : 4 * P->nsm);
  if (g.dtype == HJ_F64)
    peer_halo_kernel<double><<<blocks, 256, 0, P->stream>>>((const double*)P->X[buf], g.pitch, g.col0, g.nx,
                                                            g.ny, (double*)ps->lo[buf], (double*)ps->hi[buf], ctrl);
  else
    peer_halo_kernel<float><<<blocks, 256, 0, P->stream>>>((const float*)P->X[buf], g.pitch, g.col0, g.nx,
                                                           g.ny, (float*)ps->lo[buf], (float*)ps->hi[buf], ctrl);
  HJ_CUDA(cudaGetLastError());
  return HJ_OK;
}

hj_status peer_halo(hj_plan* P, int buf) { return launch_halo(P, buf, P->ctrl); }

void peer_halo_ptrs(const hj_plan* P, int buf, void** lo, void** hi) {
  *lo = P->peer->lo[buf];
  *hi = P->peer->hi[buf];
}

hj_status peer_reset(hj_plan* P) {
  PeerState* ps = P->peer;
  if (!ps->attached) return HJ_OK;  // hj_plan_peer_attach runs it
  HJ_CUDA(cudaMemsetAsync(ps->err_d, 0, sizeof(int), P->stream));
  HJ_TRY(peer_barrier(P));                       // B1: every rank initialised its buffers
  peer_sig0_kernel<<<1, 32, 0, P->stream>>>(P->ctrl, ps->flags);
  HJ_CUDA(cudaGetLastError());
  HJ_TRY(launch_halo(P, 0, nullptr));            // initial ghost rows of X[0]
  HJ_TRY(peer_barrier(P));                       // B2: every ghost row of X[0] has arrived
  int err = 0;
  HJ_CUDA(cudaMemcpyAsync(&err, ps->err_d, sizeof(int), cudaMemcpyDeviceToHost, P->stream));
  HJ_CUDA(cudaStreamSynchronize(P->stream));
  if (err) { set_error("peer barrier timed out (a rank did not reset / attach)"); return HJ_ERR_PEER; }
  return HJ_OK;
}

void peer_cycle_args(const hj_plan* P, PeerDsts* d, PeerSync* s) {
  *d = P->peer->dsts;
  *s = P->peer->sig;
}

void peer_free(hj_plan* P) {
  PeerState* ps = P->peer;
  if (!ps) return;
  for (int r = 0; r < HJ_MAX_RANKS; ++r)
    for (int b = 0; b < 4; ++b)
      if (ps->opened[r][b]) cudaIpcCloseMemHandle(ps->opened[r][b]);
  cudaFree(ps->flags);
  cudaFree(ps->err_d);
  delete ps;
  P->peer = nullptr;
}

}  // namespace hj

using namespace hj;

extern "C" {

hj_status hj_plan_create_peer(const hj_problem* pb, const hj_params* pr, const hj_dist* dist,
                              void* stream, hj_plan** plan) {
  if (!plan || !dist) { set_error("NULL argument"); return HJ_ERR_INVALID_ARG; }
  HJ_TRY(validate_dist(pb, pr, dist));
  DistInfo di{dist->rank, dist->nranks, dist->row_begin, dist->row_end, nullptr, 1};
  return plan_build(pb, pr, (cudaStream_t)stream, &di, plan);
}

hj_status hj_plan_peer_export(const hj_plan* P, void* out) {
  if (!P || !out || !P->peer) { set_error("not a peer plan"); return HJ_ERR_INVALID_ARG; }
  const PeerState* ps = P->peer;
  PeerBlob b;
  std::memset(&b, 0, sizeof(b));
  b.magic = PEER_MAGIC;
  b.version = 1;
  b.rank = ps->rank;
  b.nranks = ps->nranks;
  b.dtype = P->g.dtype;
  b.nx = P->g.nx;
  b.pitch = P->g.pitch;
  b.col0 = P->g.col0;
  b.rows_local = P->g.ny;
  b.row_begin = ps->row_begin;
  b.nrg_global = P->g.nrg_global;
  HJ_CUDA(cudaIpcGetMemHandle(&b.h_x0, P->X[0]));
  HJ_CUDA(cudaIpcGetMemHandle(&b.h_x1, P->X[1]));
  HJ_CUDA(cudaIpcGetMemHandle(&b.h_rowpart, P->rowpart));
  HJ_CUDA(cudaIpcGetMemHandle(&b.h_flags, ps->flags));
  std::memset(out, 0, HJ_PEER_HANDLE_BYTES);
  std::memcpy(out, &b, sizeof(b));
  return HJ_OK;
}

hj_status hj_plan_peer_attach(hj_plan* P, const void* all) {
  if (!P || !all || !P->peer) { set_error("not a peer plan"); return HJ_ERR_INVALID_ARG; }
  PeerState* ps = P->peer;
  if (ps->attached) { set_error("peer plan already attached"); return HJ_ERR_INVALID_ARG; }
  const int n = ps->nranks, me = ps->rank;
  const Geom& g = P->g;
  PeerBlob b[HJ_MAX_RANKS];
  for (int r = 0; r < n; ++r) {
    std::memcpy(&b[r], static_cast<const char*>(all) + size_t(r) * HJ_PEER_HANDLE_BYTES, sizeof(PeerBlob));
    const bool ok = b[r].magic == PEER_MAGIC && b[r].version == 1 && b[r].rank == r && b[r].nranks == n &&
                    b[r].dtype == g.dtype && b[r].nx == g.nx && b[r].pitch == g.pitch &&
                    b[r].col0 == g.col0 && b[r].nrg_global == g.nrg_global &&
                    (r == 0 || b[r].row_begin == b[r - 1].row_begin + b[r - 1].rows_local);
    if (!ok) { set_error("peer handles inconsistent (rank order, geometry or slabs)"); return HJ_ERR_INVALID_ARG; }
  }
  const size_t esz = g.dtype == HJ_F64 ? 8 : 4;
  auto open = [&](int r, int slot, const cudaIpcMemHandle_t& h, void** ptr) -> hj_status {
    HJ_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    ps->opened[r][slot] = *ptr;
    return HJ_OK;
  };
  ps->dsts.n = n;
  ps->sig.n = n;
  ps->bar.n = n;
  ps->sig.timeout_ns = ps->bar.timeout_ns = ps->timeout_ns;
  ps->sig.own = ps->flags;
  ps->bar.own = ps->flags + 1;
  for (int r = 0; r < n; ++r) {
    double* rp;
    unsigned long long* fl;
    if (r == me) {
      rp = P->rowpart;
      fl = ps->flags;
    } else {
      void *a = nullptr, *f = nullptr;
      HJ_TRY(open(r, 2, b[r].h_rowpart, &a));
      HJ_TRY(open(r, 3, b[r].h_flags, &f));
      rp = static_cast<double*>(a);
      fl = static_cast<unsigned long long*>(f);
    }
    ps->dsts.p[r] = rp;
    ps->sig.flag[r] = fl;
    ps->bar.flag[r] = fl + 1;
  }
  for (int side = 0; side < 2; ++side) {  // 0: rank-1 (its ghost row R+1), 1: rank+1 (ghost row 0)
    const int r = side == 0 ? me - 1 : me + 1;
    if (r < 0 || r >= n) continue;
    const long long row = side == 0 ? b[r].rows_local + 1 : 0;
    for (int buf = 0; buf < 2; ++buf) {
      void* base = nullptr;
      HJ_TRY(open(r, buf, buf == 0 ? b[r].h_x0 : b[r].h_x1, &base));
      void* ghost = static_cast<char*>(base) + (size_t(row) * g.pitch + g.col0) * esz;
      (side == 0 ? ps->lo : ps->hi)[buf] = ghost;
    }
  }
  ps->attached = true;
  return plan_reset(P);
}

}  // extern "C"
