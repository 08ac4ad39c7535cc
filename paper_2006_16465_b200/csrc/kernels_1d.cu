// 1D kernels of libhj.so: one hierarchical cycle (two designs) and one classic sweep.
//
// PAPER.md:161-166 (§3.3) and Appendix A (:532-575): each block copies its subdomain plus one
// point left and right to on-chip memory, performs k sub-iterations of the update
// x_i <- (b_i dx^2 + x_{i-1} + x_{i+1})/2 with the two halo points frozen, and
// writes the interior back.  Residual of the snapshot fused: s = h2f - (2x - (L+R)).
// GEN = true: the general tridiagonal update of Eq. 4 with per-point weights
// wL = T(-a_i/d_i), wR = T(-c_i/d_i) stored like Q (= T(b_i/d_i)); update / residual gupd1 / gres1
// (reading c23).  The kernels take SK (stencil kind): 0 the paper's Poisson update,
// 1 the general coefficients (GEN), 2 the Poisson update damped by omega (damp(): the multigrid
// smoother of reading c24).
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "hj_internal.cuh"

namespace hj {

namespace {

constexpr unsigned FULL = 0xffffffffu;

// =============================================================================
// REG1D — warp per tile of T = 32*C points; lane l holds points C*l..C*l+C-1 in registers,
// neighbours across lanes by one shuffle each way per sub-iteration; tile + halo staged in
// shared memory by the TMA bulk-copy engine (cp.async.bulk), double-buffered per warp.
// =============================================================================
template <typename T, int C, bool GEN = false>
struct R1 {
  static constexpr int TILE = 32 * C;
  static constexpr int COL0 = 16 / sizeof(T);
  static constexpr int XN = TILE + 2 * COL0;                  // elements copied for x (16-B multiple)
  static constexpr int XBYTES = XN * sizeof(T);
  static constexpr int XSLOT = (XBYTES + 127) / 128 * 128;
  static constexpr int FBYTES = TILE * sizeof(T);
  static constexpr int FSLOT = (FBYTES + 127) / 128 * 128;
  static constexpr int NF = GEN ? 3 : 1;                      // q (+ wL, wR)
  static constexpr int SLOT = XSLOT + NF * FSLOT;
  static constexpr int WARPS = 4;
  static constexpr size_t SMEM = 128 + 128 + size_t(WARPS) * 2 * SLOT;
  static_assert(SMEM <= 232448, "shared memory budget");
};

// Source pointers of one tile: x (with halo), q and, for GEN, the weight arrays.
template <typename T>
struct Src1 {
  const T *x, *q, *wl, *wr;
};

template <typename T, int C, bool RAGGED, int SK>
__device__ __forceinline__ void reg1d_tile(const unsigned char* __restrict__ sl,
                                           T* __restrict__ xrow, long long t, int w, int lane,
                                           int kk, double* __restrict__ part, long long u,
                                           uint64_t* bar, const Src1<T>* nxt, unsigned char* slot,
                                           T om) {
  constexpr bool GEN = SK == 1;
  using P = R1<T, C, GEN>;
  const T* sx = reinterpret_cast<const T*>(sl);
  const T* sf = reinterpret_cast<const T*>(sl + P::XSLOT);
  T x[C], q[C], wl[GEN ? C : 1], wr[GEN ? C : 1];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    x[c] = sx[P::COL0 + C * lane + c];
    q[c] = sf[C * lane + c];
    if constexpr (GEN) {
      wl[c] = sf[P::FSLOT / sizeof(T) + C * lane + c];
      wr[c] = sf[2 * P::FSLOT / sizeof(T) + C * lane + c];
    }
  }
  const T hl = sx[P::COL0 - 1];       // frozen left halo (used by lane 0)
  const T hr = sx[P::COL0 + P::TILE]; // frozen right halo (used by lane 31) — for a ragged
                                      // tile the right halo is x[w] (the ring), kept frozen below
  uint32_t act = 0xffffffffu;
  if (RAGGED) {
    act = 0;
#pragma unroll
    for (int c = 0; c < C; ++c)
      if (C * lane + c < w) act |= 1u << c;
  }
  // fused residual of the snapshot
  double acc = 0.0;
  {
    T l = __shfl_up_sync(FULL, x[C - 1], 1);
    T r = __shfl_down_sync(FULL, x[0], 1);
    if (lane == 0) l = hl;
    if (lane == 31) r = hr;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const T L = c == 0 ? l : x[c - 1];
      const T R = c == C - 1 ? r : x[c + 1];
      double s;
      if constexpr (GEN) s = gres1((double)wl[c], (double)wr[c], (double)x[c], (double)L, (double)R, (double)q[c]);
      else s = res1((double)x[c], (double)L, (double)R, (double)(T(2) * q[c]));
      if ((act >> c) & 1u) acc = __fma_rn(s, s, acc);
    }
  }
  acc = warp_sum(acc);
  if (lane == 0) part[u] = acc;
  __syncwarp();
  if (lane == 0 && nxt) {  // the slot is free: prefetch this warp's next tile into it
    fence_proxy_async();
    mbar_arrive_expect_tx(bar, P::XBYTES + P::NF * P::FBYTES);
    bulk_load(slot, nxt->x, P::XBYTES, bar);
    bulk_load(slot + P::XSLOT, nxt->q, P::FBYTES, bar);
    if constexpr (GEN) {
      bulk_load(slot + P::XSLOT + P::FSLOT, nxt->wl, P::FBYTES, bar);
      bulk_load(slot + P::XSLOT + 2 * P::FSLOT, nxt->wr, P::FBYTES, bar);
    }
  }
#pragma unroll 1
  for (int s = 0; s < kk; ++s) {
    T l = __shfl_up_sync(FULL, x[C - 1], 1);
    T r = __shfl_down_sync(FULL, x[0], 1);
    if (lane == 0) l = hl;
    if (lane == 31) r = hr;
    T prev = l;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const T R = c == C - 1 ? r : x[c + 1];
      T nv;
      if constexpr (GEN) nv = gupd1(wl[c], wr[c], prev, R, q[c]);
      else nv = upd1(prev, R, q[c]);
      if constexpr (SK == 2) nv = damp(om, x[c], nv);
      prev = x[c];
      if (!RAGGED || ((act >> c) & 1u)) x[c] = nv;
    }
  }
  if (kk == 0) return;
#pragma unroll
  for (int c = 0; c < C; ++c)
    if (!RAGGED || ((act >> c) & 1u)) xrow[P::COL0 + t * P::TILE + C * lane + c] = x[c];
}

// Rows of the padded arrays are independent problems (batched 1D); tile u of the
// launch is tile (u % ntpr) of problem (u / ntpr), and its residual partial is part[u].
template <typename T, int C, int SK>
__global__ void __launch_bounds__(R1<T, C, SK == 1>::WARPS * 32)
reg1d_kernel(const T* __restrict__ xin, T* __restrict__ xout, const T* __restrict__ h2f,
             const T* __restrict__ wla, const T* __restrict__ wra, int nx, long long pitch,
             long long fpitch, int ntpr, long long ntiles, double* __restrict__ part,
             const Ctrl* __restrict__ ctrl, int k, long long max_cycles, double omd) {
  constexpr bool GEN = SK == 1;
  using P = R1<T, C, GEN>;
  const T om = (T)omd;
  if (ctrl->done) return;
  const int kk = (ctrl->c >= max_cycles) ? 0 : k;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(base) + 2 * warp;
  unsigned char* slot0 = base + 128 + size_t(warp) * 2 * P::SLOT;
  unsigned char* slot1 = slot0 + P::SLOT;
  const long long gw = (long long)blockIdx.x * P::WARPS + warp;
  const long long nw = (long long)gridDim.x * P::WARPS;
  if (gw >= ntiles) return;
  auto src = [&](long long u) {
    const long long fo = (u / ntpr) * fpitch + (u % ntpr) * P::TILE;
    return Src1<T>{xin + (u / ntpr) * pitch + (u % ntpr) * P::TILE, h2f + fo,
                   GEN ? wla + fo : nullptr, GEN ? wra + fo : nullptr};
  };
  if (lane == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    for (int s = 0; s < 2; ++s) {
      const long long u = gw + s * nw;
      if (u < ntiles) {
        unsigned char* sl = s ? slot1 : slot0;
        const Src1<T> sr = src(u);
        mbar_arrive_expect_tx(&bars[s], P::XBYTES + P::NF * P::FBYTES);
        bulk_load(sl, sr.x, P::XBYTES, &bars[s]);
        bulk_load(sl + P::XSLOT, sr.q, P::FBYTES, &bars[s]);
        if constexpr (GEN) {
          bulk_load(sl + P::XSLOT + P::FSLOT, sr.wl, P::FBYTES, &bars[s]);
          bulk_load(sl + P::XSLOT + 2 * P::FSLOT, sr.wr, P::FBYTES, &bars[s]);
        }
      }
    }
  }
  __syncwarp();
  int it = 0;
  for (long long u = gw; u < ntiles; u += nw, ++it) {
    const int s = it & 1;
    unsigned char* sl = s ? slot1 : slot0;
    mbar_wait(&bars[s], (it >> 1) & 1);
    const long long t = u % ntpr;
    const int w = (int)lmin(P::TILE, nx - t * P::TILE);
    const long long un = u + 2 * nw;
    const Src1<T> nsr = un < ntiles ? src(un) : Src1<T>{nullptr, nullptr, nullptr, nullptr};
    const Src1<T>* nxt = un < ntiles ? &nsr : nullptr;
    T* xrow = xout + (u / ntpr) * pitch;
    if (w == P::TILE)
      reg1d_tile<T, C, false, SK>(sl, xrow, t, w, lane, kk, part, u, &bars[s], nxt, sl, om);
    else
      reg1d_tile<T, C, true, SK>(sl, xrow, t, w, lane, kk, part, u, &bars[s], nxt, sl, om);
  }
}

// =============================================================================
// RES1D — the resident 1D solver (see res2d_kernel in kernels_2d.cu): one warp per tile of 32*C
// points for the whole solve, the tile's points and q in registers across cycles, per cycle only
// the two frozen halo values of x_c are read (L2) and x_{c+1} written (snapshot semantics); one
// grid barrier per cycle (a CTA barrier when the grid is one CTA); every CTA reduces the partials
// in exactly the rowsum_kernel + finalize_kernel order and takes the same stopping decision.
// Poisson (SK 0) and damped (SK 2) updates, no ragged tiles, rows = independent problems.
// =============================================================================
constexpr int RES1D_WARPS = 8;
template <typename T, int C, int SK>
__global__ void __launch_bounds__(RES1D_WARPS * 32, 1)
res1d_kernel(T* __restrict__ X0, T* __restrict__ X1, const T* __restrict__ Q, long long pitch,
             long long fpitch, int ntpr, int rows, double* __restrict__ part, Ctrl* __restrict__ ctrl,
             double* __restrict__ hist, long long hist_cap, double rdiv, double tol, int tol_mode,
             double ref_residual, long long max_cycles, int k, double omd, unsigned int* bar) {
  constexpr int COL0 = 16 / sizeof(T);
  constexpr int TILE = 32 * C;
  __shared__ Ctrl cs;
  __shared__ int s_done;
  __shared__ double rsum[1024];   // per-problem residual sums (rows <= 1024)
  // one-CTA grids: the tiles' boundary values and partials stay in shared memory
  __shared__ T bnd_l[RES1D_WARPS], bnd_r[RES1D_WARPS];
  __shared__ double spart[RES1D_WARPS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long ntiles = (long long)ntpr * rows;
  const long long t = (long long)blockIdx.x * RES1D_WARPS + warp;
  const bool active = t < ntiles;
  const T om = (T)omd;
  if (threadIdx.x == 0) {
    cs = *ctrl;
    s_done = cs.done;
  }
  __syncthreads();
  if (s_done) return;
  const long long row = active ? t / ntpr : 0, x0 = active ? (t % ntpr) * (long long)TILE : 0;
  T x[C], q[C];
  int p = (int)(cs.c & 1);
  const bool one = gridDim.x == 1;
  const long long tr = t % ntpr;  // tile within its row
  T ring_l = T(0), ring_r = T(0);
  if (active) {
    const T* Xc = (p ? X1 : X0) + row * pitch + COL0 + x0 + C * lane;
    const T* Qr = Q + row * fpitch + x0 + C * lane;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      x[c] = Xc[c];
      q[c] = Qr[c];
    }
    const T* Xr = X0 + row * pitch + COL0;  // the Dirichlet ring (both buffers hold it)
    ring_l = Xr[-1];
    ring_r = Xr[(long long)ntpr * TILE];
    if (one) {
      if (lane == 0) bnd_l[warp] = x[0];
      if (lane == 31) bnd_r[warp] = x[C - 1];
    }
  }
  if (one) __syncthreads();
  for (;;) {
    const T* Xc = (p ? X1 : X0) + row * pitch + COL0;   // interior point i at Xc[i]; rings at -1, nx
    T* Xn = (p ? X0 : X1) + row * pitch + COL0;
    const long long c = cs.c;
    const int kk = c >= max_cycles ? 0 : k;
    double* pc = part + (c & 1) * ntiles;
    if (active) {
      T hl, hr;  // frozen halo of x_c
      if (one) {
        hl = tr == 0 ? ring_l : bnd_r[warp - 1];
        hr = tr == ntpr - 1 ? ring_r : bnd_l[warp + 1];
      } else {
        hl = __ldcg(Xc + x0 - 1);
        hr = __ldcg(Xc + x0 + TILE);
      }
      double acc = 0.0;
      {
        T l = __shfl_up_sync(FULL, x[C - 1], 1);
        T r = __shfl_down_sync(FULL, x[0], 1);
        if (lane == 0) l = hl;
        if (lane == 31) r = hr;
#pragma unroll
        for (int cc = 0; cc < C; ++cc) {
          const T L = cc == 0 ? l : x[cc - 1];
          const T R = cc == C - 1 ? r : x[cc + 1];
          const double s = res1((double)x[cc], (double)L, (double)R, (double)(T(2) * q[cc]));
          acc = __fma_rn(s, s, acc);
        }
      }
#pragma unroll 1
      for (int s = 0; s < kk; ++s) {
        T l = __shfl_up_sync(FULL, x[C - 1], 1);
        T r = __shfl_down_sync(FULL, x[0], 1);
        if (lane == 0) l = hl;
        if (lane == 31) r = hr;
        T prev = l;
#pragma unroll
        for (int cc = 0; cc < C; ++cc) {
          const T R = cc == C - 1 ? r : x[cc + 1];
          T nv = upd1(prev, R, q[cc]);
          if constexpr (SK == 2) nv = damp(om, x[cc], nv);
          prev = x[cc];
          x[cc] = nv;
        }
      }
      if (kk > 0) {
#pragma unroll
        for (int cc = 0; cc < C; ++cc) Xn[x0 + C * lane + cc] = x[cc];
      }
      acc = warp_sum(acc);
      if (!one && lane == 0) pc[t] = acc;
      if (one) {
        __syncthreads();   // every warp has read this cycle's boundary values
        if (lane == 0) { spart[warp] = acc; bnd_l[warp] = x[0]; }
        if (lane == 31) bnd_r[warp] = x[C - 1];
      }
    } else if (one) {
      __syncthreads();
    }
    if (one) __syncthreads();
    else grid_barrier(bar, gridDim.x);
    // rowsum_kernel + finalize_kernel order (see res2d_kernel): row sums by the CTA's warps, then
    // finalize's per-warp xor trees over rows 32w .. 32w+31 (rows <= 1024: one row per thread)
    for (int g = warp; g < rows; g += RES1D_WARPS) {
      double v = 0.0;
      for (int qq = lane; qq < ntpr; qq += 32) v += one ? spart[g * ntpr + qq] : __ldcg(pc + (long long)g * ntpr + qq);
      v = warp_sum(v);
      if (lane == 0) rsum[g] = v;
    }
    __syncthreads();
    if (warp == 0) {
      double S = 0.0;
      for (int w = 0; w < 32 && 32 * w < rows; ++w) {  // empty warps add +0.0: S unchanged
        const int g = 32 * w + lane;
        S += warp_sum(g < rows ? rsum[g] : 0.0);
      }
      if (lane == 0) {
        hj_decide(&cs, S, blockIdx.x == 0 ? hist : nullptr, hist_cap, rdiv, tol, tol_mode, ref_residual,
                  max_cycles);
        s_done = cs.done;
      }
    }
    __syncthreads();
    if (s_done) break;
    p ^= 1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *ctrl = cs;
}

// =============================================================================
// RES1W — the resident solver for ONE small 1D problem (nx = 32 C <= 1024 points, e.g. BASELINE config
// 1: N = 256, 8 tiles of 32, k = 16, tol 1e-8): the whole problem in ONE warp, C consecutive points
// per lane, every tile a run of tx / C lanes.  No CTA barrier, no shared memory, no per-cycle global
// traffic.  The cycle is a chain of dependent sub-iterations, so its time is the latency of that chain:
//  * sub-iterations run in PAIRS with one exchange per pair: a lane also keeps the two points on each
//    side of its own C (ghosts; the neighbouring lanes' points, their q preloaded), updates its C
//    points and the inner ghost on each side in the pair's first sub-iteration and its C points in
//    the second — one shuffle latency per two sub-iterations; the ghost updates are the same
//    expression of the same values as in the neighbour (bitwise the same iterate); at a tile edge the
//    ghost is the frozen halo of x_c and is not updated;
//  * the residual of x_c is folded into the first sub-iteration (fp64) and its warp reduction is
//    spread over the following pairs (one butterfly step per pair), so only the stopping decision
//    (hj_decide on the broadcast sum, the same on every lane) is left at the end of the cycle;
//  * x_c is kept beside x_{c+1} (registers for C < 16, else stored each cycle) so a converged solve
//    returns the snapshot it tested.
// Same per-point arithmetic as every other 1D kernel (bitwise iterates); the residual sum is one warp
// tree (history within the 1e-12 bar of the oracle, not bitwise equal to the multi-warp paths).
// =============================================================================
template <typename T, int C, int U = 2>
__global__ void __launch_bounds__(32, 1)
res1w_kernel(T* __restrict__ X0, T* __restrict__ X1, const T* __restrict__ Q, int tpl, Ctrl* __restrict__ ctrl,
             double* __restrict__ hist, long long hist_cap, double rdiv, double tol, int tol_mode,
             double ref_residual, long long max_cycles, int k) {
  constexpr int COL0 = 16 / sizeof(T);
  constexpr bool FOLD = sizeof(T) == 8;
  const int lane = threadIdx.x;
  Ctrl cs = *ctrl;  // every lane keeps an identical copy (same inputs, same decisions)
  if (cs.done) return;
  const T* Xc = ((cs.c & 1) ? X1 : X0) + COL0;
  T x[C], q[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    x[c] = Xc[C * lane + c];
    q[c] = Q[C * lane + c];
  }
  const T ring_l = X0[COL0 - 1], ring_r = X0[COL0 + 32 * C];
  const bool t0 = lane % tpl == 0, t1 = lane % tpl == tpl - 1;  // first / last lane of a tile
  const long long c_first = cs.c;
  double thr = tol * cs.sqrtS0, lo2, hi2;  // the relative stopping threshold (set at c = 0 or on resume)
  {
    const double t2 = thr * thr;
    lo2 = t2 * (1.0 - 0x1p-49);
    hi2 = t2 * (1.0 + 0x1p-49);
  }
  // q of the inner ghosts (the neighbours' edge points): constant for the whole solve
  const T qgl = __shfl_up_sync(FULL, q[C - 1], 1), qgr = __shfl_down_sync(FULL, q[0], 1);
  // PIPE (C >= 4): the exchange is software-pipelined — the shuffles a pair needs (the neighbours'
  // two edge points each side) are issued at the END of the previous pair, in the same basic block
  // as its interior updates, so their latency overlaps arithmetic instead of heading the next pair
  // (ncu of the unpipelined loop: the shuffle -> first-DADD wait and the butterfly's shuffle -> DADD
  // wait were the top stalls, in-order issue blocking the warp behind each); the shuffles issued
  // after a cycle's last pair are the next cycle's first exchange AND its frozen halo.
  constexpr bool PIPE = C >= 4;
  T sg1, sg2, sh0, sh1;  // pending: left lane's x[C-1], x[C-2]; right lane's x[0], x[1]
  auto issue = [&] {
    sg1 = __shfl_up_sync(FULL, x[C - 1], 1);
    sg2 = __shfl_up_sync(FULL, x[C >= 2 ? C - 2 : 0], 1);
    sh0 = __shfl_down_sync(FULL, x[0], 1);
    sh1 = __shfl_down_sync(FULL, x[C >= 2 ? 1 : 0], 1);
  };
  if constexpr (PIPE) issue();
  for (;;) {
    const long long cyc = cs.c;
    const int kk = cyc >= max_cycles ? 0 : k;
    // frozen halo of x_c (the neighbouring tiles' edge points; the ring at the ends)
    T hl, hr;
    if constexpr (PIPE) {
      hl = sg1;
      hr = sh0;
    } else {
      hl = __shfl_up_sync(FULL, x[C - 1], 1);
      hr = __shfl_down_sync(FULL, x[0], 1);
    }
    if (lane == 0) hl = ring_l;
    if (lane == 31) hr = ring_r;
    // the snapshot x_c: in registers (C < 16), else written to X[c & 1] every cycle
    constexpr bool SNAP_REG = C < 16;
    T xs[SNAP_REG ? C : 1];
    if constexpr (SNAP_REG) {
#pragma unroll
      for (int c = 0; c < C; ++c) xs[c] = x[c];
    } else {
      T* Xd = ((cyc & 1) ? X1 : X0) + COL0;
#pragma unroll
      for (int c = 0; c < C; ++c) Xd[C * lane + c] = x[c];
    }
    double acc = 0.0;
    if (!FOLD || kk == 0) {  // separate residual pass of x_c (fp32, residual-only cycle)
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const T L = c == 0 ? hl : x[c - 1];
        const T R = c == C - 1 ? hr : x[c + 1];
        const double sv = res1((double)x[c], (double)L, (double)R, (double)(T(2) * q[c]));
        acc = __fma_rn(sv, sv, acc);
      }
    }
    // one sub-iteration of the own points, neighbours L (left of point 0) and R (right of point C-1);
    // RES: fold the residual of the current values (x_c) in
    auto sweep1 = [&](T L, T R, auto res) {
      T prev = L;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const T Rc = c == C - 1 ? R : x[c + 1];
        if constexpr (decltype(res)::value) {
          const double sum = __dadd_rn(prev, Rc);
          const double t = __fma_rn(2.0, x[c], -sum);
          const double rr = __fma_rn(2.0, q[c], -t);
          acc = __fma_rn(rr, rr, acc);
          prev = x[c];
          x[c] = __fma_rn(0.5, sum, q[c]);
        } else {
          const T nv = upd1(prev, Rc, q[c]);
          prev = x[c];
          x[c] = nv;
        }
      }
    };
    // two sub-iterations with one exchange: ghosts at -2, -1 (left) and C, C+1 (right)
    // (C >= 2: the inner ghost's other neighbour is in the same lane, hence in the same tile; C == 1
    // runs single sub-iterations with one exchange each)
    auto pair = [&](auto res) {
      if constexpr (!PIPE) issue();
      T g1 = sg1, g2 = sg2, h0 = sh0, h1 = sh1;
      g1 = t0 ? hl : g1;
      h0 = t1 ? hr : h0;
      if constexpr (C >= 2) {
        // first sub-iteration: the inner ghosts too (not at a tile edge, where they are the frozen halo)
        const T gn = t0 ? hl : upd1(g2, x[0], qgl);
        const T hn = t1 ? hr : upd1(x[C - 1], h1, qgr);
        sweep1(g1, h0, res);
        sweep1(gn, hn, std::false_type{});
        if constexpr (PIPE) issue();  // the next pair's exchange (or the next cycle's halo)
      } else {
        sweep1(g1, h0, res);
        T l = __shfl_up_sync(FULL, x[0], 1), r = __shfl_down_sync(FULL, x[0], 1);
        l = t0 ? hl : l;
        r = t1 ? hr : r;
        sweep1(l, r, std::false_type{});
      }
    };
    int s = 0;
    if (kk & 1) {  // an odd count: one single sub-iteration first (the fold, fp64)
      if constexpr (FOLD) sweep1(hl, hr, std::true_type{});
      else sweep1(hl, hr, std::false_type{});
      if constexpr (PIPE) issue();
      s = 1;
    } else if (kk > 0) {
      if constexpr (FOLD) pair(std::true_type{});
      else pair(std::false_type{});
      s = 2;
    }
    int step = 16;  // butterfly of acc, one step per following pair: its shuffle issued before the
                    // pair and its add predicated after it (no branch, no wait inside the pair);
                    // two pairs per loop body so ptxas sees one pair's shuffles feed the next
#pragma unroll U
    for (; s < kk; s += 2) {
      const double pb = __shfl_xor_sync(FULL, acc, step ? step : 16);
      pair(std::false_type{});
      acc = step ? acc + pb : acc;
      step >>= 1;
    }
    for (; step; step >>= 1) acc += __shfl_xor_sync(FULL, acc, step);
    const double S = __shfl_sync(FULL, acc, 0);  // one value for every lane
    // the history gets S itself now and sqrt(S) / rdiv after the loop (the same value hj_decide would
    // write), keeping the square root and the division off the per-cycle chain
    if (lane == 0 && hist && cyc < hist_cap) hist[cyc] = S;
    if (cyc == 0 || tol_mode != 0) {
      hj_decide(&cs, S, nullptr, hist_cap, rdiv, tol, tol_mode, ref_residual, max_cycles);
      thr = tol * cs.sqrtS0;
      const double t2 = thr * thr;
      lo2 = t2 * (1.0 - 0x1p-49);
      hi2 = t2 * (1.0 + 0x1p-49);
    } else {
      // relative test sqrt(S) <= thr (hj_decide, reading c1) decided without the square root unless S is
      // within a few ulps of thr^2: S < lo2 implies sqrt(S) < thr exactly, S > hi2 implies RN(sqrt(S)) > thr
      cs.S_last = S;
      const bool conv = S < lo2 ? true : (S > hi2 ? false : sqrt(S) <= thr);
      if (!isfinite(S)) {
        cs.status = HJ_ERR_NUMERIC;
        cs.done = 1;
        cs.c_done = cyc;
      } else if (conv) {
        cs.done = 1;
        cs.converged = 1;
        cs.status = HJ_OK;
        cs.c_done = cyc;
      } else if (cyc >= max_cycles) {
        cs.done = 1;
        cs.converged = 0;
        cs.status = HJ_NOT_CONVERGED;
        cs.c_done = cyc;
      } else {
        cs.c = cyc + 1;
      }
    }
    if (cs.done) {  // x_c is the answer: into X[c & 1], where the engine extracts it
      if constexpr (SNAP_REG) {
        T* Xd = ((cyc & 1) ? X1 : X0) + COL0;
#pragma unroll
        for (int c = 0; c < C; ++c) Xd[C * lane + c] = xs[c];
      }
      break;
    }
  }
  if (hist) {  // S -> sqrt(S) / rdiv for the entries this launch wrote
    __syncwarp();
    const long long last = cs.c_done < hist_cap - 1 ? cs.c_done : hist_cap - 1;
    for (long long i = c_first + lane; i <= last; i += 32) hist[i] = sqrt(hist[i]) / rdiv;
  }
  if (lane == 0) *ctrl = cs;
}

// =============================================================================
// RES1C — the resident solver for ONE small 1D problem spread over one CTA: W = nx / (32 C) <= 8 warps
// (one per scheduler for W = 4), C consecutive points per lane, every tile a run of tpl = tx / C lanes
// inside one warp.  Same cycle as RES1W (§4.1: frozen halo of x_c, k sub-iterations,
// the residual of x_c folded into the first), but the k-long chain of dependent sub-iterations runs
// on W schedulers instead of one, and the exchange between lanes happens once per GROUP of D
// sub-iterations: a lane keeps D ghost points on each side (the neighbouring lanes' points, their q
// preloaded) and in the group's j-th sub-iteration updates its C points and the D - j inner ghosts
// on each side — the ghost updates are the neighbour's own expression on the same values, so the
// iterate is bitwise that of every other 1D kernel.  A ghost that is the tile's frozen halo (ghost
// -m with m == p C + 1 for the lane at position p of its tile) keeps its value; ghosts beyond it
// carry values of the next tile that never reach the tile (the frozen ghost separates them).
// Between warps: each cycle every warp publishes its edge points of x_{c+1} and its residual partial
// in shared memory (slots by cycle parity), ONE __syncthreads, then every thread sums the W partials
// in warp order and takes the same decision (the history within the 1e-12 bar of the oracle).
// =============================================================================
template <typename T, int C, int D>
__global__ void __launch_bounds__(256, 1)
res1c_kernel(T* __restrict__ X0, T* __restrict__ X1, const T* __restrict__ Q, int nx, int tpl,
             Ctrl* __restrict__ ctrl, double* __restrict__ hist, long long hist_cap, double rdiv, double tol,
             int tol_mode, double ref_residual, long long max_cycles, int k) {
  constexpr int COL0 = 16 / sizeof(T);
  constexpr bool FOLD = sizeof(T) == 8;
  __shared__ T s_e[2][8][2];    // [cycle parity][warp][first, last point] of the iterate entering the cycle
  __shared__ double s_p[2][8];  // [cycle parity][warp] residual partial
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
  Ctrl cs = *ctrl;  // every thread keeps an identical copy (same inputs, same decisions)
  if (cs.done) return;
  const T* Xc = ((cs.c & 1) ? X1 : X0) + COL0;
  T x[C], q[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    x[c] = Xc[C * threadIdx.x + c];
    q[c] = Q[C * threadIdx.x + c];
  }
  const T ring_l = X0[COL0 - 1], ring_r = X0[COL0 + nx];
  const int p = lane % tpl, tf = lane - p, tl = tf + tpl - 1;  // position in the tile, its first / last lane
  bool fl[D], fr[D];  // ghost m (1-based) is the tile's frozen left / right halo
  T qgl[D], qgr[D];   // q at the ghosts (constant for the whole solve)
#pragma unroll
  for (int m = 1; m <= D; ++m) {
    fl[m - 1] = m == p * C + 1;
    fr[m - 1] = m == (tpl - 1 - p) * C + 1;
    qgl[m - 1] = __shfl_up_sync(FULL, q[C - 1 - (m - 1) % C], (m - 1) / C + 1);
    qgr[m - 1] = __shfl_down_sync(FULL, q[(m - 1) % C], (m - 1) / C + 1);
  }
  const long long c_first = cs.c;
  double thr = tol * cs.sqrtS0, lo2, hi2;  // the relative stopping threshold (set at c = 0 or on resume)
  {
    const double t2 = thr * thr;
    lo2 = t2 * (1.0 - 0x1p-49);
    hi2 = t2 * (1.0 + 0x1p-49);
  }
  if (lane == 0) s_e[cs.c & 1][w][0] = x[0];
  if (lane == 31) s_e[cs.c & 1][w][1] = x[C - 1];
  __syncthreads();
  T gl[D], gr[D];  // ghosts: gl[m-1] = point -m, gr[m-1] = point C-1+m
  // software-pipelined exchange (as RES1W): the shuffles a group needs are issued at the end of the
  // previous group, in the same basic block as its last sub-iteration, into pa / pb; a group only
  // applies the frozen-halo selects to them
  T pa[D], pb[D];
  auto issue = [&] {
#pragma unroll
    for (int m = 1; m <= D; ++m) {
      pa[m - 1] = __shfl_up_sync(FULL, x[C - 1 - (m - 1) % C], (m - 1) / C + 1);
      pb[m - 1] = __shfl_down_sync(FULL, x[(m - 1) % C], (m - 1) / C + 1);
    }
  };
  issue();
  for (;;) {
    const long long cyc = cs.c;
    const int par = (int)(cyc & 1);
    const int kk = cyc >= max_cycles ? 0 : k;
    // the tiles' frozen halo of x_c: the neighbouring tile's edge point (another warp's: shared memory)
    T hl = __shfl_sync(FULL, x[C - 1], (tf - 1) & 31);
    T hr = __shfl_sync(FULL, x[0], (tl + 1) & 31);
    if (tf == 0) hl = w > 0 ? s_e[par][w - 1][1] : ring_l;
    if (tl == 31) hr = w < W - 1 ? s_e[par][w + 1][0] : ring_r;
    T xs[C];  // the snapshot x_c (returned if the cycle's test stops the solve)
#pragma unroll
    for (int c = 0; c < C; ++c) xs[c] = x[c];
    // ghosts of depth d from the neighbouring lanes (shuffled by the last issue()); the frozen ones
    // take the halo
    auto exch = [&](auto dd) {
      constexpr int d = decltype(dd)::value;
#pragma unroll
      for (int m = 1; m <= d; ++m) {
        gl[m - 1] = fl[m - 1] ? hl : pa[m - 1];
        gr[m - 1] = fr[m - 1] ? hr : pb[m - 1];
      }
    };
    double acc = 0.0;
    if (!FOLD || kk == 0) {  // separate residual pass of x_c (fp32, residual-only cycle)
      exch(std::integral_constant<int, 1>{});
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const T L = c == 0 ? gl[0] : x[c - 1];
        const T R = c == C - 1 ? gr[0] : x[c + 1];
        const double sv = res1((double)x[c], (double)L, (double)R, (double)(T(2) * q[c]));
        acc = __fma_rn(sv, sv, acc);
      }
    }
    // a group of d sub-iterations after one exchange; RES: fold the residual of x_c into the first
    auto group = [&](auto dd, auto res) {
      constexpr int d = decltype(dd)::value;
      exch(dd);
#pragma unroll
      for (int j = 1; j <= d; ++j) {
        const int e = d - j;  // ghosts still valid after this sub-iteration
        T ngl[D > 1 ? D - 1 : 1], ngr[D > 1 ? D - 1 : 1], nv[C];
#pragma unroll
        for (int m = 1; m <= e; ++m) {
          ngl[m - 1] = fl[m - 1] ? gl[m - 1] : upd1(gl[m], m == 1 ? x[0] : gl[m - 2], qgl[m - 1]);
          ngr[m - 1] = fr[m - 1] ? gr[m - 1] : upd1(m == 1 ? x[C - 1] : gr[m - 2], gr[m], qgr[m - 1]);
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const T L = c == 0 ? gl[0] : x[c - 1];
          const T R = c == C - 1 ? gr[0] : x[c + 1];
          if constexpr (decltype(res)::value) {
            if (j == 1) {
              const double sum = __dadd_rn(L, R);
              const double t = __fma_rn(2.0, x[c], -sum);
              const double rr = __fma_rn(2.0, q[c], -t);
              acc = __fma_rn(rr, rr, acc);
              nv[c] = __fma_rn(0.5, sum, q[c]);
              continue;
            }
          }
          nv[c] = upd1(L, R, q[c]);
        }
#pragma unroll
        for (int c = 0; c < C; ++c) x[c] = nv[c];
#pragma unroll
        for (int m = 1; m <= e; ++m) {
          gl[m - 1] = ngl[m - 1];
          gr[m - 1] = ngr[m - 1];
        }
      }
      issue();  // the next group's exchange (or the next cycle's first)
    };
    using I1 = std::integral_constant<int, 1>;
    using ID = std::integral_constant<int, D>;
    int s = 0;
    const int rem = kk % D;
    if (rem) {  // k not a multiple of D: single sub-iterations first (the first one folds)
      if constexpr (FOLD) group(I1{}, std::true_type{});
      else group(I1{}, std::false_type{});
      for (s = 1; s < rem; ++s) group(I1{}, std::false_type{});
    } else if (kk > 0) {
      if constexpr (FOLD) group(ID{}, std::true_type{});
      else group(ID{}, std::false_type{});
      s = D;
    }
    int step = 16;  // butterfly of acc, one step per following group (shuffle before, predicated add after)
#pragma unroll 2
    for (; s < kk; s += D) {
      const double pbf = __shfl_xor_sync(FULL, acc, step ? step : 16);
      group(ID{}, std::false_type{});
      acc = step ? acc + pbf : acc;
      step >>= 1;
    }
    for (; step; step >>= 1) acc += __shfl_xor_sync(FULL, acc, step);
    if (lane == 0) {
      s_p[par][w] = acc;
      s_e[par ^ 1][w][0] = x[0];
    }
    if (lane == 31) s_e[par ^ 1][w][1] = x[C - 1];
    __syncthreads();
    double S = s_p[par][0];
    for (int v = 1; v < W; ++v) S += s_p[par][v];
    if (threadIdx.x == 0 && hist && cyc < hist_cap) hist[cyc] = S;
    if (cyc == 0 || tol_mode != 0) {
      hj_decide(&cs, S, nullptr, hist_cap, rdiv, tol, tol_mode, ref_residual, max_cycles);
      thr = tol * cs.sqrtS0;
      const double t2 = thr * thr;
      lo2 = t2 * (1.0 - 0x1p-49);
      hi2 = t2 * (1.0 + 0x1p-49);
    } else {  // as RES1W: the relative test without the square root away from the threshold
      cs.S_last = S;
      const bool conv = S < lo2 ? true : (S > hi2 ? false : sqrt(S) <= thr);
      if (!isfinite(S)) {
        cs.status = HJ_ERR_NUMERIC;
        cs.done = 1;
        cs.c_done = cyc;
      } else if (conv) {
        cs.done = 1;
        cs.converged = 1;
        cs.status = HJ_OK;
        cs.c_done = cyc;
      } else if (cyc >= max_cycles) {
        cs.done = 1;
        cs.converged = 0;
        cs.status = HJ_NOT_CONVERGED;
        cs.c_done = cyc;
      } else {
        cs.c = cyc + 1;
      }
    }
    if (cs.done) {  // x_c is the answer: into X[c & 1], where the engine extracts it
      T* Xd = ((cyc & 1) ? X1 : X0) + COL0;
#pragma unroll
      for (int c = 0; c < C; ++c) Xd[C * threadIdx.x + c] = xs[c];
      break;
    }
  }
  if (hist) {  // S -> sqrt(S) / rdiv for the entries this launch wrote
    __syncthreads();
    const long long last = cs.c_done < hist_cap - 1 ? cs.c_done : hist_cap - 1;
    for (long long i = c_first + threadIdx.x; i <= last; i += blockDim.x) hist[i] = sqrt(hist[i]) / rdiv;
  }
  if (threadIdx.x == 0) *ctrl = cs;
}

// =============================================================================
// RES1DM — the resident 1D solver for MANY small tiles (tiles of 32 points, e.g. the paper's
// 1024 copies of N = 1024 with T = 32: 32,768 tiles): each warp owns M consecutive tiles for the
// whole solve, lane l holding point l of each, so a sub-iteration is M independent shuffle+update
// chains (latency hidden by ILP across tiles).  Per cycle: the tiles' frozen halo values (lane 0:
// left, lane 31: right; L2 loads), fused residual, k sub-iterations, x_{c+1} stored, per-tile
// partials; grid barrier; the row sums of rowsum_kernel, distributed over the CTAs; grid
// barrier; every CTA replays finalize_kernel's reduction (warps in parallel, the 32 warp sums in
// order) and takes the same hj_decide decision.  Bitwise the per-cycle path's iterates and
// histories.
// =============================================================================
template <typename T, int M, int SK>
__global__ void __launch_bounds__(256, (M <= 16 ? 2 : 1))
res1dm_kernel(T* __restrict__ X0, T* __restrict__ X1, const T* __restrict__ Q, long long pitch,
              long long fpitch, int ntpr, int rows, double* __restrict__ part, double* __restrict__ R,
              Ctrl* __restrict__ ctrl, double* __restrict__ hist, long long hist_cap, double rdiv, double tol,
              int tol_mode, double ref_residual, long long max_cycles, int k, double omd, unsigned int* bar) {
  constexpr int COL0 = 16 / sizeof(T);
  __shared__ Ctrl cs;
  __shared__ int s_done;
  __shared__ double ws[32];
  __shared__ long long s_off[8][M];       // interior point 0 of each of my tiles in X
  __shared__ T s_h[8][M][2];              // the tiles' frozen halo values (left, right)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = ntpr * rows;
  const int tb = (blockIdx.x * 8 + warp) * M;  // my first tile
  const T om = (T)omd;
  if (threadIdx.x == 0) {
    cs = *ctrl;
    s_done = cs.done;
  }
  for (int m = lane; m < M; m += 32) {
    const int t = tb + m < ntiles ? tb + m : 0;
    s_off[warp][m] = (long long)(t / ntpr) * pitch + COL0 + (long long)(t % ntpr) * 32;
  }
  __syncthreads();
  if (s_done) return;
  T x[M], q[M];
  int p = (int)(cs.c & 1);
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int t = tb + m;
    const long long o = s_off[warp][m];
    const long long qo = (long long)((t < ntiles ? t : 0) / ntpr) * fpitch + (long long)((t < ntiles ? t : 0) % ntpr) * 32;
    x[m] = (t < ntiles) ? (p ? X1 : X0)[o + lane] : T(0);
    q[m] = (t < ntiles) ? Q[qo + lane] : T(0);
  }
  for (;;) {
    const T* Xc = p ? X1 : X0;
    T* Xn = p ? X0 : X1;
    const long long c = cs.c;
    const int kk = c >= max_cycles ? 0 : k;
    double* pc = part + (c & 1) * (long long)ntiles;
    double* Rc = R + (c & 1) * (long long)rows;
    // frozen halos of x_c: lane m of the warp fetches tile m's two values (L2)
    for (int m = lane; m < M; m += 32) {
      if (tb + m < ntiles) {
        const long long o = s_off[warp][m];
        s_h[warp][m][0] = __ldcg(Xc + o - 1);
        s_h[warp][m][1] = __ldcg(Xc + o + 32);
      }
    }
    __syncwarp();
    // fused residual of the snapshot (reg1d_tile's expression), per-tile partials
#pragma unroll
    for (int m = 0; m < M; ++m) {
      T l = __shfl_up_sync(FULL, x[m], 1);
      T r = __shfl_down_sync(FULL, x[m], 1);
      if (lane == 0) l = s_h[warp][m][0];
      if (lane == 31) r = s_h[warp][m][1];
      const double s = res1((double)x[m], (double)l, (double)r, (double)(T(2) * q[m]));
      const double v = warp_sum(__fma_rn(s, s, 0.0));
      if (lane == 0 && tb + m < ntiles) pc[tb + m] = v;
    }
#pragma unroll 1
    for (int s = 0; s < kk; ++s) {
      constexpr int G = M < 4 ? M : 4;  // tiles per group: all shuffles of a group issued first
#pragma unroll
      for (int m0 = 0; m0 < M; m0 += G) {
        T l[G], r[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          l[g] = __shfl_up_sync(FULL, x[m0 + g], 1);
          r[g] = __shfl_down_sync(FULL, x[m0 + g], 1);
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const T hv = s_h[warp][m0 + g][lane == 31 ? 1 : 0];
          if (lane == 0) l[g] = hv;
          if (lane == 31) r[g] = hv;
          T nv = upd1(l[g], r[g], q[m0 + g]);
          if constexpr (SK == 2) nv = damp(om, x[m0 + g], nv);
          x[m0 + g] = nv;
        }
      }
    }
    if (kk > 0) {
#pragma unroll
      for (int m = 0; m < M; ++m)
        if (tb + m < ntiles) Xn[s_off[warp][m] + lane] = x[m];
    }
    grid_barrier(bar, gridDim.x);
    // rowsum_kernel's row sums, rows spread over the grid's warps
    for (int g = blockIdx.x * 8 + warp; g < rows; g += gridDim.x * 8) {
      double v = 0.0;
      for (int qq = lane; qq < ntpr; qq += 32) v += __ldcg(pc + (long long)g * ntpr + qq);
      v = warp_sum(v);
      if (lane == 0) Rc[g] = v;
    }
    grid_barrier(bar, gridDim.x);
    // finalize_kernel's reduction: warp w of its 1024 threads sums rows 32w + lane (+1024 ...)
    for (int w = warp; w < 32; w += 8) {
      double v = 0.0;
      for (int i = 32 * w + lane; i < rows; i += 1024) v += __ldcg(Rc + i);
      v = warp_sum(v);
      if (lane == 0) ws[w] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double S = 0.0;
      for (int w = 0; w < 32; ++w) S += ws[w];
      hj_decide(&cs, S, blockIdx.x == 0 ? hist : nullptr, hist_cap, rdiv, tol, tol_mode, ref_residual,
                max_cycles);
      s_done = cs.done;
    }
    __syncthreads();
    if (s_done) break;
    p ^= 1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *ctrl = cs;
}

// =============================================================================
// SMEM1D — the paper's Appendix A design: blockDim.x = T threads, shared memory
// [container 0 (T+2) | container 1 (T+2) | rhs (T)], __syncthreads per
// sub-iteration, write-back of the latest container (reading c8), into the other global
// buffer (reading c6), rhs of the updated point (reading c7).
// =============================================================================
template <typename T, int SK>
__global__ void smem1d_kernel(const T* __restrict__ xin_all, T* __restrict__ xout_all,
                              const T* __restrict__ h2f_all, const T* __restrict__ wla,
                              const T* __restrict__ wra, int nx, long long pitch,
                              long long fpitch, Axis ax, double* __restrict__ part,
                              const Ctrl* __restrict__ ctrl, int k, long long max_cycles, double omd) {
  constexpr bool GEN = SK == 1;
  // block = (problem row, subdomain): rows of the padded arrays are independent problems
  const long long row = blockIdx.x / ax.nb;
  const T* __restrict__ xin = xin_all + row * pitch;
  T* __restrict__ xout = xout_all + row * pitch;
  const T* __restrict__ h2f = h2f_all + row * fpitch;
  if (ctrl->done) return;
  const int kk = (ctrl->c >= max_cycles) ? 0 : k;
  constexpr int COL0 = 16 / sizeof(T);
  const int Tn = blockDim.x, L = Tn + 2;
  extern __shared__ unsigned char smem_raw[];
  T* A = reinterpret_cast<T*>(smem_raw);
  T* B = A + L;
  T* rhs = B + L;
  __shared__ double wsum[32];
  const long long t = blockIdx.x % ax.nb;
  const long long i0 = axis_start(ax, (int)t);     // interior origin (§3.3, §3.5)
  const int w = axis_width(ax, (int)t);
  const int o0 = axis_own_lo(ax, (int)t) - (int)i0, o1 = axis_own_hi(ax, (int)t) - (int)i0;
  const int a = threadIdx.x;
  for (int q = a; q < L; q += Tn) {
    const long long gi = i0 + q;  // padded index, 0 = left ring
    const T v = gi <= nx + 1 ? xin[COL0 - 1 + gi] : T(0);
    A[q] = v;
    B[q] = v;
  }
  const bool active = a < w;
  const bool owned = a >= o0 && a <= o1;   // overlapping blocks write only what they own
  if (active) rhs[a] = h2f[i0 + a];
  T wl = T(0), wr = T(0);   // GEN: this point's weights (registers; the paper keeps b only)
  if (GEN && active) {
    wl = wla[row * fpitch + i0 + a];
    wr = wra[row * fpitch + i0 + a];
  }
  __syncthreads();
  double s2 = 0.0;
  if (owned) {
    const double s =
        GEN ? gres1((double)wl, (double)wr, (double)A[a + 1], (double)A[a], (double)A[a + 2], (double)rhs[a])
            : res1((double)A[a + 1], (double)A[a], (double)A[a + 2], (double)(T(2) * rhs[a]));
    s2 = s * s;
  }
  s2 = warp_sum(s2);
  if ((a & 31) == 0) wsum[a >> 5] = s2;
  __syncthreads();
  if (a == 0) {
    double acc = 0.0;
    for (int q = 0; q < (Tn + 31) / 32; ++q) acc += wsum[q];
    part[blockIdx.x] = acc;
  }
  const T q2 = active ? rhs[a] : T(0);
  T* cur = A;
  T* nxt = B;
  for (int s = 0; s < kk; ++s) {
    if (active) {
      T u = GEN ? gupd1(wl, wr, cur[a], cur[a + 2], q2) : upd1(cur[a], cur[a + 2], q2);
      if constexpr (SK == 2) u = damp((T)omd, cur[a + 1], u);  // multigrid smoother (c24)
      nxt[a + 1] = u;
    }
    __syncthreads();
    T* tmp = cur; cur = nxt; nxt = tmp;
  }
  if (kk > 0 && owned) xout[COL0 + i0 + a] = cur[a + 1];
}

// =============================================================================
// CLASSIC1D — one sweep; 256 threads x 8 consecutive points per CTA (128-bit loads),
// neighbours by shuffle, fused residual, one partial per CTA.
// =============================================================================
template <typename T, bool GEN>
__global__ void __launch_bounds__(256)
classic1d_kernel(const T* __restrict__ xin_all, T* __restrict__ xout_all,
                 const T* __restrict__ h2f_all, const T* __restrict__ wla, const T* __restrict__ wra,
                 int nx, long long pitch, long long fpitch, int ncb,
                 double* __restrict__ part, const Ctrl* __restrict__ ctrl, long long max_cycles) {
  const long long row = blockIdx.x / ncb;  // independent problem
  const T* __restrict__ xin = xin_all + row * pitch;
  T* __restrict__ xout = xout_all + row * pitch;
  const T* __restrict__ h2f = h2f_all + row * fpitch;
  if (ctrl->done) return;
  const bool write = ctrl->c < max_cycles;
  constexpr int COL0 = 16 / sizeof(T);
  constexpr int V = 8;
  __shared__ double wsum[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long i0 = (long long)(blockIdx.x % ncb) * CLASSIC1D_CELLS + (long long)threadIdx.x * V;
  T x[V], f[V];
#pragma unroll
  for (int c = 0; c < V; ++c) {
    const long long i = i0 + c;
    x[c] = i <= nx ? xin[COL0 + i] : T(0);   // interior or right ring
    f[c] = i < nx ? h2f[i] : T(0);
  }
  T l = __shfl_up_sync(FULL, x[V - 1], 1);
  T r = __shfl_down_sync(FULL, x[0], 1);
  if (lane == 0 && i0 <= nx + 1) l = xin[COL0 + i0 - 1];
  if (lane == 31 && i0 + V <= nx) r = xin[COL0 + i0 + V];
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < V; ++c) {
    const long long i = i0 + c;
    const T L = c == 0 ? l : x[c - 1];
    const T R = c == V - 1 ? r : x[c + 1];
    if (i < nx) {
      if constexpr (GEN) {
        const T wl = wla[row * fpitch + i], wr = wra[row * fpitch + i];
        const double s = gres1((double)wl, (double)wr, (double)x[c], (double)L, (double)R, (double)f[c]);
        acc = __fma_rn(s, s, acc);
        if (write) xout[COL0 + i] = gupd1(wl, wr, L, R, f[c]);
      } else {
        const double s = res1((double)x[c], (double)L, (double)R, (double)(T(2) * f[c]));
        acc = __fma_rn(s, s, acc);
        if (write) xout[COL0 + i] = upd1(L, R, f[c]);
      }
    }
  }
  acc = warp_sum(acc);
  if (lane == 0) wsum[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < 8; ++q) s += wsum[q];
    part[blockIdx.x] = s;
  }
}

template <typename T, int C, int SK>
void launch_reg1d(const Geom& g, const CycleArgs& a, int grid_hint, cudaStream_t st) {
  using P = R1<T, C, SK == 1>;
  long long ctas = (g.ntiles + P::WARPS - 1) / P::WARPS;
  if (ctas > grid_hint) ctas = grid_hint;
  reg1d_kernel<T, C, SK><<<(unsigned)ctas, P::WARPS * 32, P::SMEM, st>>>(
      (const T*)a.xin, (T*)a.xout, (const T*)a.h2f, (const T*)a.wl, (const T*)a.wr, (int)g.nx,
      g.pitch, g.fpitch, (int)g.ntx, g.ntiles, a.part, a.ctrl, g.k, a.max_cycles, g.omega);
}

template <typename T, int SK>
cudaError_t launch_1d_t(const Geom& g, const CycleArgs& a, int grid_hint, cudaStream_t st) {
  constexpr bool GEN = SK == 1;
  constexpr int SKB = GEN ? 0 : SK;  // tiles 512/1024 exist for the Poisson kinds only
  if (g.kernel_kind == K_REG1D) {
    switch (g.tx / 32) {   // GEN: tiles <= 256 (x, q, wL, wR of a lane in registers)
      case 1: launch_reg1d<T, 1, SK>(g, a, grid_hint * 8, st); break;
      case 2: launch_reg1d<T, 2, SK>(g, a, grid_hint * 8, st); break;
      case 4: launch_reg1d<T, 4, SK>(g, a, grid_hint * 4, st); break;
      case 8: launch_reg1d<T, 8, SK>(g, a, grid_hint * 4, st); break;
      case 16: if (GEN) return cudaErrorInvalidValue; launch_reg1d<T, 16, SKB>(g, a, grid_hint * 2, st); break;
      case 32: if (GEN) return cudaErrorInvalidValue; launch_reg1d<T, 32, SKB>(g, a, grid_hint, st); break;
      default: return cudaErrorInvalidValue;
    }
  } else if (g.kernel_kind == K_SMEM1D) {
    const size_t smem = sizeof(T) * (2 * size_t(g.tx + 2) + size_t(g.tx));
    smem1d_kernel<T, SK><<<(unsigned)g.ntiles, g.tx, smem, st>>>(
        (const T*)a.xin, (T*)a.xout, (const T*)a.h2f, (const T*)a.wl, (const T*)a.wr, (int)g.nx,
        g.pitch, g.fpitch, g.ax, a.part, a.ctrl, g.k, a.max_cycles, g.omega);
  } else {
    classic1d_kernel<T, GEN><<<(unsigned)g.ntiles, 256, 0, st>>>(
        (const T*)a.xin, (T*)a.xout, (const T*)a.h2f, (const T*)a.wl, (const T*)a.wr, (int)g.nx,
        g.pitch, g.fpitch, (int)g.ntx, a.part, a.ctrl, a.max_cycles);
  }
  return cudaGetLastError();
}

template <typename T, int C, int SK = 0>
cudaError_t cfg1() {
  return cudaFuncSetAttribute(reg1d_kernel<T, C, SK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)R1<T, C, SK == 1>::SMEM);
}

}  // namespace

size_t reg1d_smem_bytes(int dtype, int tile) {
  (void)tile;
  return dtype == HJ_F64 ? R1<double, 32>::SMEM : R1<float, 32>::SMEM;
}
int reg1d_warps_per_cta(int, int) { return 4; }

cudaError_t configure_1d() {
  cudaError_t e = cudaSuccess;
#define HJ_CFG(T)                                                                              \
  if ((e = cfg1<T, 1>()) != cudaSuccess || (e = cfg1<T, 2>()) != cudaSuccess ||                \
      (e = cfg1<T, 4>()) != cudaSuccess || (e = cfg1<T, 8>()) != cudaSuccess ||                \
      (e = cfg1<T, 16>()) != cudaSuccess || (e = cfg1<T, 32>()) != cudaSuccess ||              \
      (e = cfg1<T, 1, 1>()) != cudaSuccess || (e = cfg1<T, 2, 1>()) != cudaSuccess ||          \
      (e = cfg1<T, 4, 1>()) != cudaSuccess || (e = cfg1<T, 8, 1>()) != cudaSuccess ||          \
      (e = cfg1<T, 1, 2>()) != cudaSuccess || (e = cfg1<T, 2, 2>()) != cudaSuccess ||          \
      (e = cfg1<T, 4, 2>()) != cudaSuccess || (e = cfg1<T, 8, 2>()) != cudaSuccess ||          \
      (e = cfg1<T, 16, 2>()) != cudaSuccess || (e = cfg1<T, 32, 2>()) != cudaSuccess)          \
    return e;
  HJ_CFG(double)
  HJ_CFG(float)
#undef HJ_CFG
  return cudaSuccess;
}

// Many-tile variant (tiles of 32 points, M tiles per warp); R: 2 x rows doubles.
cudaError_t launch_resident_1dm(const Geom& g, int M, void* X0, void* X1, const void* Q, double* part, double* R,
                                Ctrl* ctrl, double* hist, long long hist_cap, double tol, int tol_mode,
                                double ref_residual, long long max_cycles, int k, unsigned int* bar, cudaStream_t st) {
  int ntpr = (int)(g.nx / 32), rows = (int)g.ny;
  long long pitch = g.pitch, fpitch = g.fpitch;
  double rdiv = g.rdiv, om = g.omega;
  void* args[] = {&X0, &X1, &Q, &pitch, &fpitch, &ntpr, &rows, &part, &R, &ctrl, &hist, &hist_cap, &rdiv, &tol,
                  &tol_mode, &ref_residual, &max_cycles, &k, &om, &bar};
  const long long ntiles = (long long)ntpr * rows;
  const dim3 grid((unsigned)((ntiles + 8LL * M - 1) / (8LL * M))), block(256);
  const bool f64 = g.dtype == HJ_F64;
  const void* fn = nullptr;
#define HJ_RM(MM)                                                                                  \
  case MM:                                                                                         \
    fn = f64 ? (const void*)res1dm_kernel<double, MM, 0> : (const void*)res1dm_kernel<float, MM, 0>; \
    break;
  switch (M) {
    HJ_RM(2) HJ_RM(4) HJ_RM(8) HJ_RM(16) HJ_RM(32)
    default: return cudaErrorInvalidValue;
  }
#undef HJ_RM
  return cudaLaunchCooperativeKernel(fn, grid, block, args, 0, st);
}

// One small problem in one warp (res1w_kernel): ny == 1, nx = 32 C (C = 1..32), whole tiles of C-multiples.
bool res1w_ok(const Geom& g) {
  const long long C = g.nx / 32;
  return g.dim == 1 && g.ny == 1 && !g.gen && g.omega == 1.0 && g.ox == 0 && g.nx % 32 == 0 && C >= 1 &&
         C <= 32 && (C & (C - 1)) == 0 && g.tx % C == 0 && g.nx % g.tx == 0;
}

cudaError_t launch_resident_1w(const Geom& g, void* X0, void* X1, const void* Q, Ctrl* ctrl, double* hist,
                               long long hist_cap, double tol, int tol_mode, double ref_residual,
                               long long max_cycles, int k, cudaStream_t st) {
  const int C = (int)(g.nx / 32), tpl = g.tx / C;
  const bool f64 = g.dtype == HJ_F64;
  // HJ_RES1W_UNROLL=1: the pair loop not unrolled (A/B of the software-pipelined exchange)
  static const bool u1 = [] { const char* e = std::getenv("HJ_RES1W_UNROLL"); return e && e[0] == '1'; }();
#define HJ_RW(CC)                                                                                    \
  case CC:                                                                                           \
    if (f64) {                                                                                       \
      auto fn = u1 ? res1w_kernel<double, CC, 1> : res1w_kernel<double, CC, 2>;                      \
      fn<<<1, 32, 0, st>>>((double*)X0, (double*)X1, (const double*)Q, tpl, ctrl, hist, hist_cap,    \
                           g.rdiv, tol, tol_mode, ref_residual, max_cycles, k);                       \
    } else {                                                                                         \
      auto fn = u1 ? res1w_kernel<float, CC, 1> : res1w_kernel<float, CC, 2>;                        \
      fn<<<1, 32, 0, st>>>((float*)X0, (float*)X1, (const float*)Q, tpl, ctrl, hist, hist_cap,       \
                           g.rdiv, tol, tol_mode, ref_residual, max_cycles, k);                       \
    }                                                                                                \
    break;
  switch (C) {
    HJ_RW(1) HJ_RW(2) HJ_RW(4) HJ_RW(8) HJ_RW(16) HJ_RW(32)
    default: return cudaErrorInvalidValue;
  }
#undef HJ_RW
  return cudaGetLastError();
}

// One small problem in one CTA (res1c_kernel): C points per lane, W = nx / (32 C) <= 8 warps, tiles of
// tpl = tx / C lanes inside a warp (tpl a power of two <= 32).  *C / *D: the layout (RES1C_C, RES1C_D
// defaults, HJ_RES1C="C,D" overrides, HJ_RES1C=0 disables).
bool res1c_ok(const Geom& g, int* C, int* D) {
  int c = RES1C_C, d = RES1C_D;
  bool forced = false;
  if (const char* s = std::getenv("HJ_RES1C")) {
    if (s[0] == '0') return false;
    if (std::sscanf(s, "%d,%d", &c, &d) != 2) return false;
    forced = true;
  }
  // by default only where res1w would hold >= 16 points per lane (nx >= 512): measured faster there
  // (1D N = 1024: 1.38 vs 2.42 us per cycle), slower at config 1 (N = 256: 1.20 vs 1.14 us)
  if (!forced && g.nx < 512) return false;
  if (!(c == 1 || c == 2 || c == 4 || c == 8) || !(d == 1 || d == 2 || d == 4)) return false;
  if (!(g.dim == 1 && g.ny == 1 && !g.gen && g.omega == 1.0 && g.ox == 0)) return false;
  if (g.nx % (32LL * c) || g.nx / (32LL * c) > 8 || g.tx % c || g.nx % g.tx) return false;
  const long long tpl = g.tx / c;
  if (tpl > 32 || (tpl & (tpl - 1))) return false;
  *C = c;
  *D = d;
  return true;
}

cudaError_t launch_resident_1c(const Geom& g, int C, int D, void* X0, void* X1, const void* Q, Ctrl* ctrl,
                               double* hist, long long hist_cap, double tol, int tol_mode, double ref_residual,
                               long long max_cycles, int k, cudaStream_t st) {
  const int nx = (int)g.nx, tpl = (int)g.tx / C, threads = nx / C;
  const bool f64 = g.dtype == HJ_F64;
  double rdiv = g.rdiv;
#define HJ_RC(CC, DD)                                                                                  \
  if (C == CC && D == DD) {                                                                            \
    if (f64)                                                                                           \
      res1c_kernel<double, CC, DD><<<1, threads, 0, st>>>((double*)X0, (double*)X1, (const double*)Q,  \
                                                          nx, tpl, ctrl, hist, hist_cap, rdiv, tol,    \
                                                          tol_mode, ref_residual, max_cycles, k);      \
    else                                                                                               \
      res1c_kernel<float, CC, DD><<<1, threads, 0, st>>>((float*)X0, (float*)X1, (const float*)Q, nx,  \
                                                         tpl, ctrl, hist, hist_cap, rdiv, tol,         \
                                                         tol_mode, ref_residual, max_cycles, k);       \
    return cudaGetLastError();                                                                         \
  }
  HJ_RC(1, 1) HJ_RC(1, 2) HJ_RC(1, 4) HJ_RC(2, 1) HJ_RC(2, 2) HJ_RC(2, 4)
  HJ_RC(4, 1) HJ_RC(4, 2) HJ_RC(4, 4) HJ_RC(8, 1) HJ_RC(8, 2) HJ_RC(8, 4)
#undef HJ_RC
  return cudaErrorInvalidValue;
}

cudaError_t launch_resident_1d(const Geom& g, void* X0, void* X1, const void* Q, double* part, Ctrl* ctrl,
                               double* hist, long long hist_cap, double tol, int tol_mode, double ref_residual,
                               long long max_cycles, int k, unsigned int* bar, cudaStream_t st) {
  int ntpr = (int)(g.nx / g.tx), rows = (int)g.ny;
  long long pitch = g.pitch, fpitch = g.fpitch;
  double rdiv = g.rdiv, om = g.omega;
  void* args[] = {&X0, &X1, &Q, &pitch, &fpitch, &ntpr, &rows, &part, &ctrl, &hist, &hist_cap, &rdiv, &tol,
                  &tol_mode, &ref_residual, &max_cycles, &k, &om, &bar};
  const dim3 grid((unsigned)(((long long)ntpr * rows + RES1D_WARPS - 1) / RES1D_WARPS)), block(RES1D_WARPS * 32);
  const bool f64 = g.dtype == HJ_F64, wgt = g.omega != 1.0;
  const void* fn = nullptr;
#define HJ_R1(CC)                                                                                       \
  case CC:                                                                                              \
    fn = f64 ? (wgt ? (const void*)res1d_kernel<double, CC, 2> : (const void*)res1d_kernel<double, CC, 0>) \
             : (wgt ? (const void*)res1d_kernel<float, CC, 2> : (const void*)res1d_kernel<float, CC, 0>);   \
    break;
  switch (g.tx / 32) {
    HJ_R1(1) HJ_R1(2) HJ_R1(4) HJ_R1(8) HJ_R1(16) HJ_R1(32)
    default: return cudaErrorInvalidValue;
  }
#undef HJ_R1
  return cudaLaunchCooperativeKernel(fn, grid, block, args, 0, st);
}

cudaError_t launch_cycle_1d(const Geom& g, const CycleArgs& a, int grid_hint, cudaStream_t st) {
  if (g.gen)
    return g.dtype == HJ_F64 ? launch_1d_t<double, 1>(g, a, grid_hint, st)
                             : launch_1d_t<float, 1>(g, a, grid_hint, st);
  if (g.omega != 1.0)  // damped sub-iterations: the multigrid smoother (reading c24)
    return g.dtype == HJ_F64 ? launch_1d_t<double, 2>(g, a, grid_hint, st)
                             : launch_1d_t<float, 2>(g, a, grid_hint, st);
  return g.dtype == HJ_F64 ? launch_1d_t<double, 0>(g, a, grid_hint, st)
                           : launch_1d_t<float, 0>(g, a, grid_hint, st);
}

}  // namespace hj
