// The plan object behind hj_plan* (engine.cu) and the distributed hooks (dist.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <map>
#include <vector>

#include "hj_internal.cuh"

struct DistState;  // dist.cu
struct PeerState;  // peer.cu

namespace hj {

struct DistInfo {
  int rank, nranks;
  long long row_begin, row_end;
  const char* nccl_id;  // 128 bytes (NCCL transport)
  int transport;        // 0: NCCL (dist.cu), 1: peer memory over CUDA IPC (peer.cu)
};

// Peer transport (peer.cu): every rank's residual-row vector and signal flags, as kernel params.
constexpr int HJ_MAX_RANKS = 64;
struct PeerDsts {   // rowsum writes its row-group sums into every rank's rowpart
  double* p[HJ_MAX_RANKS];
  int n;            // 0: single destination (the rowsum_kernel R argument)
};
struct PeerSync {   // finalize: signal every rank, then wait for all signals of this cycle
  unsigned long long* flag[HJ_MAX_RANKS];
  unsigned long long* own;
  int n;            // 0: no synchronisation (one GPU / NCCL)
  long long timeout_ns;
};

}  // namespace hj

struct hj_plan {
  hj::Geom g{};
  hj_params prm{};
  int nsm = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;           // created because the caller passed the NULL stream
  long long ny_global = 0, gy0 = 0;
  void* X[2] = {nullptr, nullptr};
  void* H2F = nullptr;
  void* WL = nullptr;               // 1D general coefficients: T(-a_i/d_i), layout of H2F
  void* WR = nullptr;               //                          T(-c_i/d_i)
  double* part = nullptr;
  double* rowpart = nullptr;        // per row group sums, global length (input of finalize)
  long long rp_stride = 0;          // peer transport: rowpart has two halves (cycle parity)
  double* rowpart_local = nullptr;  // dist: this rank's row groups, zeros elsewhere
  double* rowsum_dst = nullptr;     // where rowsum writes (rowpart, or rowpart_local in dist)
  double* hist = nullptr;
  long long hist_cap = 0;
  hj::Ctrl* ctrl = nullptr;
  hj::Ctrl* ctrl_h = nullptr;
  double* bc_d = nullptr;
  double* x0_d = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  CUtensorMap tmX[2];   // loads: 34-row box with halo
  CUtensorMap tmXs[2];  // stores: 32x32 interior box
  CUtensorMap tmF;
  CUtensorMap tmE[2];   // multigrid coarse level (2D): patch boxes for the fused correction
  std::map<int, cudaGraphExec_t> graphs;
  long long c_host = 0;
  std::vector<cudaEvent_t> evpool;  // timed runs: (start, end) per cycle kernel
  int evused = 0;
  DistState* dist = nullptr;
  PeerState* peer = nullptr;
  // HJ_MULTIGRID (reading c24): the coarse grids 1..L-1 as internal hierarchical plans (their own
  // buffers, Geom and omega; they share this plan's stream and Ctrl for the done check)
  std::vector<hj_plan*> mg;
  int mg_nu1 = 0, mg_nu2 = 0, mg_coarse = 0;
  // resident solver (launch_resident_2d): residual partials (2 x tiles) and the grid-barrier words
  double* res_part = nullptr;
  double* res_R = nullptr;           // many-tile 1D variant: row sums (2 x rows)
  unsigned int* res_bar = nullptr;
};

namespace hj {

constexpr long long HIST_CAP = 1LL << 24;
// Entries of the residual history a plan keeps: 2^24, or HJ_HIST_CAP from the environment (tests
// lower it to cross the cap in a few hundred cycles).  history_capacity(max_cycles) =
// min(max_cycles + 1, limit) without overflow.
long long history_limit();
inline long long history_capacity(long long max_cycles) {
  const long long lim = history_limit();
  return max_cycles >= lim - 1 ? lim : max_cycles + 1;
}

hj_status validate(const hj_problem* pb, const hj_params* pr, bool need_f);
hj_status validate_dist(const hj_problem* pb, const hj_params* pr, const hj_dist* dist);
hj_status plan_build(const hj_problem* pb, const hj_params* pr, cudaStream_t st, const DistInfo* di,
                     hj_plan** out);
hj_status plan_reset(hj_plan* P);
hj_status plan_run(hj_plan* P, long long ncycles, float* kernel_ms);
hj_status plan_solve(hj_plan* P, hj_result* res, double* x_dev, double* hist_dev);
void plan_free(hj_plan* P);
int launches_per_cycle(const hj_plan* P);

// dist.cu
hj_status dist_create(hj_plan* P, const DistInfo* di);
hj_status dist_initial_exchange(hj_plan* P);
hj_status dist_halo_exchange(hj_plan* P, int buf);
hj_status dist_allreduce(hj_plan* P);
bool dist_overlap(const hj_plan* P);
hj_status dist_halo_fork(hj_plan* P, int buf);
hj_status dist_halo_join(hj_plan* P);
hj_status dist_check(hj_plan* P);
void dist_free(hj_plan* P);

// peer.cu
hj_status peer_create(hj_plan* P, const DistInfo* di);
bool peer_attached(const hj_plan* P);
int peer_halo_launches(const hj_plan* P);       // 1 if this rank has a neighbour, else 0
hj_status peer_reset(hj_plan* P);                 // collective: device barriers + initial halos
hj_status peer_halo(hj_plan* P, int buf);          // push rows 1 and R of X[buf] to the neighbours
void peer_halo_ptrs(const hj_plan* P, int buf, void** lo, void** hi);  // the neighbours' ghost rows
void peer_cycle_args(const hj_plan* P, PeerDsts* d, PeerSync* s);
void peer_free(hj_plan* P);
}  // namespace hj
