// Multi-GPU row slabs (north star; the paper itself is single-GPU).
//
// Rank r owns interior rows [row_begin, row_end) of the global grid, stored as a local grid of
// R = row_end - row_begin rows plus ghost rows 0 and R+1.  Slab boundaries fall on tile-row
// boundaries, so every tile — and therefore the iteration — is the same as on one GPU
// (DESIGN.md §3 c18): iterates and cycle counts are bitwise identical for any number of ranks.
// Per cycle, after the cycle kernel wrote X[p^1]:
//   halo:      ncclSend(row 1 -> rank-1), ncclRecv(row 0 <- rank-1),
//              ncclSend(row R -> rank+1), ncclRecv(row R+1 <- rank+1)   (one group)
//   residual:  ncclAllReduce(sum) of the per-tile-row partial vector; each rank contributes only
//              its own tile rows (zeros elsewhere), so the sum is exact and order-independent.
// All calls are on the plan's stream and are captured in the cycle graph.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "hj_internal.cuh"
#include "hj_plan.h"

// NCCL is resolved at run time (dlopen) rather than linked: the process may already hold (or
// later load) torch's bundled libnccl.so.2, and binding another copy first would break it.
// Order: $HJ_NCCL_LIB (the Python binding points it at torch's wheel), an already-loaded
// libnccl.so.2, then the default search path.
namespace {
struct NcclApi {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  decltype(&ncclCommGetAsyncError) CommGetAsyncError = nullptr;
  bool ok = false;
  std::string err;
};
const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    if (const char* path = std::getenv("HJ_NCCL_LIB")) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) { api.err = dlerror(); return; }
#define HJ_SYM(name) api.name = reinterpret_cast<decltype(api.name)>(dlsym(h, "nccl" #name)); if (!api.name) { api.err = "missing nccl" #name; return; }
    HJ_SYM(GetUniqueId) HJ_SYM(CommInitRank) HJ_SYM(CommDestroy) HJ_SYM(Send) HJ_SYM(Recv)
    HJ_SYM(GroupStart) HJ_SYM(GroupEnd) HJ_SYM(AllReduce) HJ_SYM(GetErrorString) HJ_SYM(CommGetAsyncError)
#undef HJ_SYM
    api.ok = true;
  });
  return api;
}
}  // namespace

struct DistState {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  // overlapped exchange (REG2D plans without edge tiles, nranks > 1): the halo group runs on its
  // own stream, forked after the boundary tile rows and joined before the next cycle
  bool overlap = false;
  cudaStream_t cs = nullptr;
  cudaEvent_t ev_bnd = nullptr, ev_halo = nullptr;
};

namespace hj {

#define HJ_NCCL(call)                                                                     \
  do {                                                                                    \
    if (!nccl().ok) {                                                                     \
      set_error("libnccl.so.2 unavailable: " + nccl().err);                             \
      return HJ_ERR_NCCL;                                                                 \
    }                                                                                     \
    ncclResult_t r_ = (nccl().call);                                                      \
    if (r_ != ncclSuccess) {                                                              \
      set_error(std::string(#call) + ": " + nccl().GetErrorString(r_));                  \
      return HJ_ERR_NCCL;                                                                 \
    }                                                                                     \
  } while (0)

hj_status validate_dist(const hj_problem* pb, const hj_params* pr, const hj_dist* dist) {
  HJ_TRY(validate(pb, pr, true));
  if (pb->dim != 2) { set_error("row slabs need dim == 2"); return HJ_ERR_INVALID_CONFIG; }
  const long long rb = dist->row_begin, re = dist->row_end;
  const long long unit = pr->mode == HJ_CLASSIC ? CLASSIC2D_ROWS : pr->tile_y;
  if (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks || rb < 0 || re <= rb ||
      re > pb->ny || (dist->rank == 0 && rb != 0) || (dist->rank == dist->nranks - 1 && re != pb->ny)) {
    set_error("bad slab");
    return HJ_ERR_INVALID_CONFIG;
  }
  if (rb % unit != 0 || (re % unit != 0 && re != pb->ny)) {
    set_error("slab rows must be whole tile rows");
    return HJ_ERR_INVALID_CONFIG;
  }
  if (pr->mode == HJ_HIERARCHICAL && pr->tile_y > re - rb) {
    set_error("slab thinner than a tile row");
    return HJ_ERR_INVALID_CONFIG;
  }
  return HJ_OK;
}

hj_status dist_create(hj_plan* P, const DistInfo* di) {
  DistState* d = new DistState();
  d->rank = di->rank;
  d->nranks = di->nranks;
  P->dist = d;
  ncclUniqueId id;
  std::memcpy(&id, di->nccl_id, sizeof(id));
  HJ_NCCL(CommInitRank(&d->comm, di->nranks, id, di->rank));
  const Geom& g = P->g;
  const char* env = std::getenv("HJ_NCCL_OVERLAP");
  d->overlap = d->nranks > 1 && g.kernel_kind == K_REG2D && !g.ox && !g.oy && g.nx % 32 == 0 &&
               g.ny % 32 == 0 && g.ny / 32 >= 3 && !(env && env[0] == '0');
  if (d->overlap) {
    HJ_CUDA(cudaStreamCreateWithFlags(&d->cs, cudaStreamNonBlocking));
    HJ_CUDA(cudaEventCreateWithFlags(&d->ev_bnd, cudaEventDisableTiming));
    HJ_CUDA(cudaEventCreateWithFlags(&d->ev_halo, cudaEventDisableTiming));
  }
  return HJ_OK;
}

bool dist_overlap(const hj_plan* P) { return P->dist && P->dist->overlap; }

// Surface an asynchronous NCCL failure (a peer died, a network error) as HJ_ERR_NCCL instead of a
// hang: polled by the host between cycle graphs.
hj_status dist_check(hj_plan* P) {
  DistState* d = P->dist;
  if (!d || !d->comm || d->nranks == 1) return HJ_OK;
  ncclResult_t ae = ncclSuccess;
  HJ_NCCL(CommGetAsyncError(d->comm, &ae));
  if (ae != ncclSuccess && ae != ncclInProgress) {
    set_error(std::string("NCCL asynchronous error: ") + nccl().GetErrorString(ae));
    return HJ_ERR_NCCL;
  }
  return HJ_OK;
}

hj_status dist_halo_exchange(hj_plan* P, int buf) {
  DistState* d = P->dist;
  if (d->nranks == 1) return HJ_OK;
  const Geom& g = P->g;
  const size_t esz = g.dtype == HJ_F64 ? 8 : 4;
  const ncclDataType_t ty = g.dtype == HJ_F64 ? ncclFloat64 : ncclFloat32;
  char* X = static_cast<char*>(P->X[buf]);
  auto row = [&](long long r) { return X + (size_t(r) * g.pitch + g.col0) * esz; };
  const long long R = g.ny;
  HJ_NCCL(GroupStart());
  if (d->rank > 0) {
    HJ_NCCL(Send(row(1), g.nx, ty, d->rank - 1, d->comm, P->stream));
    HJ_NCCL(Recv(row(0), g.nx, ty, d->rank - 1, d->comm, P->stream));
  }
  if (d->rank < d->nranks - 1) {
    HJ_NCCL(Send(row(R), g.nx, ty, d->rank + 1, d->comm, P->stream));
    HJ_NCCL(Recv(row(R + 1), g.nx, ty, d->rank + 1, d->comm, P->stream));
  }
  HJ_NCCL(GroupEnd());
  return HJ_OK;
}

// Overlapped form: fork the halo group onto the comm stream once the boundary tile rows (the only
// writers of rows 1 and R) are done; join_halo makes the plan's stream wait for it (before anything
// reads the ghost rows: the next cycle).  Both are graph-capturable (event fork / join).
hj_status dist_halo_fork(hj_plan* P, int buf) {
  DistState* d = P->dist;
  HJ_CUDA(cudaEventRecord(d->ev_bnd, P->stream));
  HJ_CUDA(cudaStreamWaitEvent(d->cs, d->ev_bnd, 0));
  cudaStream_t main = P->stream;
  P->stream = d->cs;
  const hj_status s = dist_halo_exchange(P, buf);
  P->stream = main;
  HJ_TRY(s);
  HJ_CUDA(cudaEventRecord(d->ev_halo, d->cs));
  return HJ_OK;
}
hj_status dist_halo_join(hj_plan* P) {
  HJ_CUDA(cudaStreamWaitEvent(P->stream, P->dist->ev_halo, 0));
  return HJ_OK;
}

hj_status dist_initial_exchange(hj_plan* P) { return dist_halo_exchange(P, 0); }

hj_status dist_allreduce(hj_plan* P) {
  DistState* d = P->dist;
  if (d->nranks == 1) {
    HJ_CUDA(cudaMemcpyAsync(P->rowpart, P->rowpart_local, sizeof(double) * P->g.nrg_global,
                            cudaMemcpyDeviceToDevice, P->stream));
    return HJ_OK;
  }
  HJ_NCCL(AllReduce(P->rowpart_local, P->rowpart, P->g.nrg_global, ncclFloat64, ncclSum, d->comm,
                        P->stream));
  return HJ_OK;
}

void dist_free(hj_plan* P) {
  if (!P->dist) return;
  if (P->dist->cs) {
    cudaStreamSynchronize(P->dist->cs);
    cudaStreamDestroy(P->dist->cs);
  }
  if (P->dist->ev_bnd) cudaEventDestroy(P->dist->ev_bnd);
  if (P->dist->ev_halo) cudaEventDestroy(P->dist->ev_halo);
  if (P->dist->comm && nccl().ok) nccl().CommDestroy(P->dist->comm);
  delete P->dist;
  P->dist = nullptr;
}

}  // namespace hj

using namespace hj;

extern "C" {

hj_status hj_nccl_unique_id(char out[128]) {
  if (!out) { set_error("NULL out"); return HJ_ERR_INVALID_ARG; }
  ncclUniqueId id;
  HJ_NCCL(GetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out, &id, 128);
  return HJ_OK;
}

hj_status jacobi_solve_dist(const hj_problem* pb, const hj_params* pr, hj_result* res,
                            const hj_dist* dist) {
  if (!dist || !res || !res->x || !dist->nccl_id) { set_error("NULL argument"); return HJ_ERR_INVALID_ARG; }
  HJ_TRY(validate_dist(pb, pr, dist));
  const long long rb = dist->row_begin, re = dist->row_end;
  if (res->history && history_capacity(pr->max_cycles) < pr->max_cycles + 1) {
    set_error("history is limited to 2^24 cycles (HJ_HIST_CAP); pass history = NULL");
    return HJ_ERR_INVALID_CONFIG;
  }
  const long long nloc = pb->nx * (re - rb);
  const long long nbc = 2 * pb->nx + 2 * pb->ny;
  double *f = nullptr, *bc = nullptr, *x0 = nullptr, *x = nullptr, *hist = nullptr;
  cudaStream_t st;
  HJ_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  auto cleanup = [&]() {
    cudaFree(f); cudaFree(bc); cudaFree(x0); cudaFree(x); cudaFree(hist);
    cudaStreamDestroy(st);
  };
#define DCK(call)                                                                          \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      set_error(std::string(#call) + ": " + cudaGetErrorString(e_));                      \
      cleanup();                                                                           \
      return HJ_ERR_CUDA;                                                                  \
    }                                                                                      \
  } while (0)
  DCK(cudaMalloc(&f, sizeof(double) * nloc));
  DCK(cudaMemcpyAsync(f, pb->f, sizeof(double) * nloc, cudaMemcpyHostToDevice, st));
  if (pb->bc) {
    DCK(cudaMalloc(&bc, sizeof(double) * nbc));
    DCK(cudaMemcpyAsync(bc, pb->bc, sizeof(double) * nbc, cudaMemcpyHostToDevice, st));
  }
  if (pb->x0) {
    DCK(cudaMalloc(&x0, sizeof(double) * nloc));
    DCK(cudaMemcpyAsync(x0, pb->x0, sizeof(double) * nloc, cudaMemcpyHostToDevice, st));
  }
  DCK(cudaMalloc(&x, sizeof(double) * nloc));
  if (res->history) DCK(cudaMalloc(&hist, sizeof(double) * history_capacity(pr->max_cycles)));
  hj_problem dp = *pb;
  dp.f = f;
  dp.bc = bc;
  dp.x0 = x0;
  DistInfo di{dist->rank, dist->nranks, rb, re, dist->nccl_id};
  hj_plan* P = nullptr;
  hj_status s = plan_build(&dp, pr, st, &di, &P);
  if (s != HJ_OK) { cleanup(); return s; }
  double* hx = res->x;
  double* hh = res->history;
  s = plan_solve(P, res, x, hist);
  res->x = hx;
  res->history = hh;
  plan_free(P);
  if (s == HJ_OK || s == HJ_NOT_CONVERGED || s == HJ_ERR_NUMERIC) {
    DCK(cudaMemcpyAsync(hx, x, sizeof(double) * nloc, cudaMemcpyDeviceToHost, st));
    if (hh) DCK(cudaMemcpyAsync(hh, hist, sizeof(double) * lmin(res->cycles + 1, history_capacity(pr->max_cycles)), cudaMemcpyDeviceToHost, st));
    DCK(cudaStreamSynchronize(st));
  }
#undef DCK
  cleanup();
  return s;
}

}  // extern "C"
