// Scratch micro-benchmark (not part of libhj.so): throughput of the in-register sub-iteration loop
// of a 32x32 tile (one warp per tile, lane = 8 rows x 4 columns), with the frozen halo in shared
// memory and NO HBM traffic (tiles re-read from a small L2-resident buffer), for several loop
// designs.  Reports cell-updates/s and the fraction of the FP64 issue limit (64 DP ops/clk/SM at the
// measured SM clock; 4 FP64 ops per update).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o loopbench scripts/loopbench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cstdint>

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ double upd2(double w, double e, double s, double n, double q) {
  return __fma_rn(0.25, __dadd_rn(__dadd_rn(w, e), __dadd_rn(s, n)), q);
}

// ---- A: the round-1 kernel's sweep (middle-out rows, up/dn shuffled at the sweep start) ----
struct TileA {
  double x[8][4], q[8][4];
  const double* hxp;
  const double* hyp;
  __device__ __forceinline__ void exchange_ns(int ly, double (&up)[4], double (&dn)[4]) const {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      up[c] = __shfl_down_sync(FULL, x[0][c], 8);
      dn[c] = __shfl_up_sync(FULL, x[7][c], 8);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double hv = hyp[c];
      up[c] = ly == 3 ? hv : up[c];
      dn[c] = ly == 0 ? hv : dn[c];
    }
  }
  __device__ __forceinline__ void exchange_we(int lx, int i, double& w, double& e) const {
    w = __shfl_up_sync(FULL, x[i][3], 1, 8);
    e = __shfl_down_sync(FULL, x[i][0], 1, 8);
    const double hv = hxp[i];
    w = lx == 0 ? hv : w;
    e = lx == 7 ? hv : e;
  }
  __device__ __forceinline__ void sweep(int lx, int ly) {
    double up[4], dn[4];
    exchange_ns(ly, up, dn);
    double olo[4], ohi[4];
#pragma unroll
    for (int step = 0; step < 8; ++step) {
      const int i = step == 0 ? 3 : (step & 1) ? 3 + (step + 1) / 2 : 3 - step / 2;
      const bool hi_side = step > 0 && (step & 1);
      double w, e;
      exchange_we(lx, i, w, e);
      double nw[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double W = c == 0 ? w : x[i][c - 1];
        const double E = c == 3 ? e : x[i][c + 1];
        const double S = (i == 0) ? dn[c] : (step > 0 && hi_side ? ohi[c] : x[i - 1][c]);
        const double N = (i == 7) ? up[c] : (step > 0 && !hi_side ? olo[c] : x[i + 1][c]);
        nw[c] = upd2(W, E, S, N, q[i][c]);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (step == 0) { olo[c] = x[i][c]; ohi[c] = x[i][c]; }
        else if (hi_side) ohi[c] = x[i][c];
        else olo[c] = x[i][c];
        x[i][c] = nw[c];
      }
    }
  }
};

// ---- B: row-sequential sweep, minimal live temporaries (for 3 warps per scheduler) ----
struct TileB {
  double x[8][4], q[8][4];
  const double* hxp;
  const double* hyp;
  __device__ __forceinline__ void sweep(int lx, int ly) {
    double up[4], prev[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double hv = hyp[c];
      const double u = __shfl_down_sync(FULL, x[0][c], 8);
      const double d = __shfl_up_sync(FULL, x[7][c], 8);
      up[c] = ly == 3 ? hv : u;
      prev[c] = ly == 0 ? hv : d;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double w = __shfl_up_sync(FULL, x[i][3], 1, 8);
      double e = __shfl_down_sync(FULL, x[i][0], 1, 8);
      const double hv = hxp[i];
      w = lx == 0 ? hv : w;
      e = lx == 7 ? hv : e;
      double nw[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double W = c == 0 ? w : x[i][c - 1];
        const double E = c == 3 ? e : x[i][c + 1];
        const double N = i == 7 ? up[c] : x[i + 1][c];
        nw[c] = upd2(W, E, prev[c], N, q[i][c]);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        prev[c] = x[i][c];
        x[i][c] = nw[c];
      }
    }
  }
};


// ---- TMEM helpers (tcgen05; per-warp lane quadrant = 32 * (warp % 4)) ----
__device__ __forceinline__ void tm_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tm_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---- C: x in registers, q in TMEM (row of 4 doubles = 8 columns per tcgen05.ld) ----
struct TileC {
  double x[8][4];
  uint32_t tq;  // TMEM address of this warp's q (lane quadrant | column base)
  const double* hxp;
  const double* hyp;
  __device__ __forceinline__ void load_q(const double (&q)[8][4]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t r[8];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        r[2 * c] = __double2loint(q[i][c]);
        r[2 * c + 1] = __double2hiint(q[i][c]);
      }
      tm_st8(tq + 8 * i, r);
    }
    tm_wait_st();
  }
  __device__ __forceinline__ void sweep(int lx, int ly) {
    double up[4], prev[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double hv = hyp[c];
      const double u = __shfl_down_sync(FULL, x[0][c], 8);
      const double d = __shfl_up_sync(FULL, x[7][c], 8);
      up[c] = ly == 3 ? hv : u;
      prev[c] = ly == 0 ? hv : d;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t r[8];
      tm_ld8(tq + 8 * i, r);
      double w = __shfl_up_sync(FULL, x[i][3], 1, 8);
      double e = __shfl_down_sync(FULL, x[i][0], 1, 8);
      const double hv = hxp[i];
      w = lx == 0 ? hv : w;
      e = lx == 7 ? hv : e;
      double sum[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double W = c == 0 ? w : x[i][c - 1];
        const double E = c == 3 ? e : x[i][c + 1];
        const double N = i == 7 ? up[c] : x[i + 1][c];
        sum[c] = __dadd_rn(__dadd_rn(W, E), __dadd_rn(prev[c], N));
      }
      tm_wait_ld();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        prev[c] = x[i][c];
        x[i][c] = __fma_rn(0.25, sum[c], __hiloint2double(r[2 * c + 1], r[2 * c]));
      }
    }
  }
};

// ---- D: x in registers, q in shared memory (two 128-bit loads per row) ----
struct TileD {
  double x[8][4];
  const double* qs;  // this lane's q: row i at qs + 32 * i (4 doubles)
  const double* hxp;
  const double* hyp;
  __device__ __forceinline__ void sweep(int lx, int ly) {
    double up[4], prev[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double hv = hyp[c];
      const double u = __shfl_down_sync(FULL, x[0][c], 8);
      const double d = __shfl_up_sync(FULL, x[7][c], 8);
      up[c] = ly == 3 ? hv : u;
      prev[c] = ly == 0 ? hv : d;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double2 qa = reinterpret_cast<const double2*>(qs + 128 * i)[0];
      const double2 qb = reinterpret_cast<const double2*>(qs + 128 * i)[1];
      const double qq[4] = {qa.x, qa.y, qb.x, qb.y};
      double w = __shfl_up_sync(FULL, x[i][3], 1, 8);
      double e = __shfl_down_sync(FULL, x[i][0], 1, 8);
      const double hv = hxp[i];
      w = lx == 0 ? hv : w;
      e = lx == 7 ? hv : e;
      double nw[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double W = c == 0 ? w : x[i][c - 1];
        const double E = c == 3 ? e : x[i][c + 1];
        const double N = i == 7 ? up[c] : x[i + 1][c];
        nw[c] = upd2(W, E, prev[c], N, qq[c]);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        prev[c] = x[i][c];
        x[i][c] = nw[c];
      }
    }
  }
};

// ---- A2: A with a conflict-free halo layout (one 8-B load per use, 8 / 16 distinct words per load) ----
//   hb[0..63]:  W/E halo, word (i * 8 + 2 * ly + isE)   (row i = 8 ly + i of the tile)
//   hb[64..127]: S/N halo, word (c * 16 + 2 * lx + isN)  (column 4 lx + c)
struct TileA2 : TileA {
  const double* hx2;  // hb + 2 * ly + (lx == 7)       (lx == 0 reads W, others E: only lx 0 / 7 use it)
  const double* hy2;  // hb + 64 + 2 * lx + (ly == 3)
  __device__ __forceinline__ void exchange_ns2(int ly, double (&up)[4], double (&dn)[4]) const {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      up[c] = __shfl_down_sync(FULL, x[0][c], 8);
      dn[c] = __shfl_up_sync(FULL, x[7][c], 8);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double hv = hy2[16 * c];
      up[c] = ly == 3 ? hv : up[c];
      dn[c] = ly == 0 ? hv : dn[c];
    }
  }
  __device__ __forceinline__ void sweep2(int lx, int ly) {
    double up[4], dn[4];
    exchange_ns2(ly, up, dn);
    double olo[4], ohi[4];
#pragma unroll
    for (int step = 0; step < 8; ++step) {
      const int i = step == 0 ? 3 : (step & 1) ? 3 + (step + 1) / 2 : 3 - step / 2;
      const bool hi_side = step > 0 && (step & 1);
      double w = __shfl_up_sync(FULL, x[i][3], 1, 8);
      double e = __shfl_down_sync(FULL, x[i][0], 1, 8);
      const double hv = hx2[8 * i];
      w = lx == 0 ? hv : w;
      e = lx == 7 ? hv : e;
      double nw[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double W = c == 0 ? w : x[i][c - 1];
        const double E = c == 3 ? e : x[i][c + 1];
        const double S = (i == 0) ? dn[c] : (step > 0 && hi_side ? ohi[c] : x[i - 1][c]);
        const double N = (i == 7) ? up[c] : (step > 0 && !hi_side ? olo[c] : x[i + 1][c]);
        nw[c] = upd2(W, E, S, N, q[i][c]);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (step == 0) { olo[c] = x[i][c]; ohi[c] = x[i][c]; }
        else if (hi_side) ohi[c] = x[i][c];
        else olo[c] = x[i][c];
        x[i][c] = nw[c];
      }
    }
  }
};

// ---- experiments: A with parts removed (WRONG results; they only locate the cost) ----
//   F = 1: no halo selects (edge lanes use the shuffled value);  F = 2: no W/E shuffles (own values);
//   F = 3: neither;  F = 4: no N/S shuffles
template <int F>
struct TileX : TileA {
  __device__ __forceinline__ void sweepx(int lx, int ly) {
    double up[4], dn[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      up[c] = F == 4 ? x[0][c] : __shfl_down_sync(FULL, x[0][c], 8);
      dn[c] = F == 4 ? x[7][c] : __shfl_up_sync(FULL, x[7][c], 8);
    }
    if (F != 1 && F != 3) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double hv = hyp[c];
        up[c] = ly == 3 ? hv : up[c];
        dn[c] = ly == 0 ? hv : dn[c];
      }
    }
    double olo[4], ohi[4];
#pragma unroll
    for (int step = 0; step < 8; ++step) {
      const int i = step == 0 ? 3 : (step & 1) ? 3 + (step + 1) / 2 : 3 - step / 2;
      const bool hi_side = step > 0 && (step & 1);
      double w = (F == 2 || F == 3) ? x[i][3] : __shfl_up_sync(FULL, x[i][3], 1, 8);
      double e = (F == 2 || F == 3) ? x[i][0] : __shfl_down_sync(FULL, x[i][0], 1, 8);
      if (F != 1 && F != 3) {
        const double hv = hxp[i];
        w = lx == 0 ? hv : w;
        e = lx == 7 ? hv : e;
      }
      double nw[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double W = c == 0 ? w : x[i][c - 1];
        const double E = c == 3 ? e : x[i][c + 1];
        const double S = (i == 0) ? dn[c] : (step > 0 && hi_side ? ohi[c] : x[i - 1][c]);
        const double N = (i == 7) ? up[c] : (step > 0 && !hi_side ? olo[c] : x[i + 1][c]);
        nw[c] = upd2(W, E, S, N, q[i][c]);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (step == 0) { olo[c] = x[i][c]; ohi[c] = x[i][c]; }
        else if (hi_side) ohi[c] = x[i][c];
        else olo[c] = x[i][c];
        x[i][c] = nw[c];
      }
    }
  }
  __device__ __forceinline__ void sweep(int lx, int ly) { sweepx(lx, ly); }
};

// ---- P: A with the frozen halo written by PREDICATED shared loads into the shuffled registers
// (edge lanes only; no selects): 1 instruction per halo value instead of 1 load + 2 FSEL ----
__device__ __forceinline__ void ld_if(double& v, const double* p, bool pred) {
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.shared.f64 %0, [%1];\n}\n"
               : "+d"(v)
               : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"((int)pred));
}
struct TileP : TileA {
  __device__ __forceinline__ void sweep(int lx, int ly) {
    double up[4], dn[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      up[c] = __shfl_down_sync(FULL, x[0][c], 8);
      dn[c] = __shfl_up_sync(FULL, x[7][c], 8);
      ld_if(up[c], hyp + c, ly == 3);
      ld_if(dn[c], hyp + c, ly == 0);
    }
    double olo[4], ohi[4];
#pragma unroll
    for (int step = 0; step < 8; ++step) {
      const int i = step == 0 ? 3 : (step & 1) ? 3 + (step + 1) / 2 : 3 - step / 2;
      const bool hi_side = step > 0 && (step & 1);
      double w = __shfl_up_sync(FULL, x[i][3], 1, 8);
      double e = __shfl_down_sync(FULL, x[i][0], 1, 8);
      ld_if(w, hxp + i, lx == 0);
      ld_if(e, hxp + i, lx == 7);
      double nw[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double W = c == 0 ? w : x[i][c - 1];
        const double E = c == 3 ? e : x[i][c + 1];
        const double S = (i == 0) ? dn[c] : (step > 0 && hi_side ? ohi[c] : x[i - 1][c]);
        const double N = (i == 7) ? up[c] : (step > 0 && !hi_side ? olo[c] : x[i + 1][c]);
        nw[c] = upd2(W, E, S, N, q[i][c]);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (step == 0) { olo[c] = x[i][c]; ohi[c] = x[i][c]; }
        else if (hi_side) ohi[c] = x[i][c];
        else olo[c] = x[i][c];
        x[i][c] = nw[c];
      }
    }
  }
};

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1)
bench_a2(const double* __restrict__ X, const double* __restrict__ Q, double* __restrict__ out, int tiles_per_warp,
         int k, long long* clk) {
  __shared__ __align__(16) double hb_all[WARPS][128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, lx = lane & 7, ly = lane >> 3;
  double* hb = hb_all[warp];
  const long long gw = (long long)blockIdx.x * WARPS + warp;
  long long t0 = clock64();
  double acc = 0.0;
  for (int t = 0; t < tiles_per_warp; ++t) {
    const long long src = ((gw * 7 + t) & 255) * 2048;
    TileA2 tl;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        tl.x[i][c] = __ldcg(X + src + (8 * ly + i) * 32 + 4 * lx + c);
        tl.q[i][c] = __ldcg(Q + src + (8 * ly + i) * 32 + 4 * lx + c);
      }
    // lane = tile row r (W, E) / tile column r (S, N)
    {
      const int r = lane, rly = r >> 3, ri = r & 7;
      hb[ri * 8 + 2 * rly + 0] = __ldcg(X + src + 1024 + r);        // W of row r
      hb[ri * 8 + 2 * rly + 1] = __ldcg(X + src + 1024 + 32 + r);   // E of row r
      const int rlx = r >> 2, rc = r & 3;
      hb[64 + rc * 16 + 2 * rlx + 0] = __ldcg(X + src + 1024 + 64 + r);  // S of column r
      hb[64 + rc * 16 + 2 * rlx + 1] = __ldcg(X + src + 1024 + 96 + r);  // N of column r
    }
    __syncwarp();
    tl.hx2 = hb + 2 * ly + (lx == 7 ? 1 : 0);
    tl.hy2 = hb + 64 + 2 * lx + (ly == 3 ? 1 : 0);
#pragma unroll 1
    for (int s = 0; s < k; s += 2) {
      tl.sweep2(lx, ly);
      tl.sweep2(lx, ly);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc += tl.x[i][c];
    __syncwarp();
  }
  out[gw * 32 + lane] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = clock64() - t0;
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1)
bench_c(const double* __restrict__ X, const double* __restrict__ Q, double* __restrict__ out, int tiles_per_warp,
        int k, long long* clk) {
  __shared__ __align__(16) double hb_all[WARPS][128];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, lx = lane & 7, ly = lane >> 3;
  constexpr int COLS = WARPS / 4 * 64 <= 32 ? 32 : WARPS / 4 * 64 <= 64 ? 64 : WARPS / 4 * 64 <= 128 ? 128 : WARPS / 4 * 64 <= 256 ? 256 : 512;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tbase)), "n"(COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tbase;
  double* hb = hb_all[warp];
  const long long gw = (long long)blockIdx.x * WARPS + warp;
  long long t0 = clock64();
  double acc = 0.0;
  for (int t = 0; t < tiles_per_warp; ++t) {
    const long long src = ((gw * 7 + t) & 255) * 2048;
    TileC tl;
    double q[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        tl.x[i][c] = __ldcg(X + src + (8 * ly + i) * 32 + 4 * lx + c);
        q[i][c] = __ldcg(Q + src + (8 * ly + i) * 32 + 4 * lx + c);
      }
    tl.tq = tb + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));
    tl.load_q(q);
    hb[lane] = __ldcg(X + src + 1024 + lane);
    hb[32 + lane] = __ldcg(X + src + 1024 + 32 + lane);
    hb[64 + lane] = __ldcg(X + src + 1024 + 64 + lane);
    hb[96 + lane] = __ldcg(X + src + 1024 + 96 + lane);
    __syncwarp();
    tl.hxp = hb + (lx == 0 ? 0 : 32) + 8 * ly;
    tl.hyp = hb + (ly == 0 ? 64 : 96) + 4 * lx;
#pragma unroll 1
    for (int s = 0; s < k; ++s) tl.sweep(lx, ly);
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc += tl.x[i][c];
    __syncwarp();
  }
  out[gw * 32 + lane] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = clock64() - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(COLS));
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1)
bench_d(const double* __restrict__ X, const double* __restrict__ Q, double* __restrict__ out, int tiles_per_warp,
        int k, long long* clk) {
  __shared__ __align__(16) double hb_all[WARPS][128];
  extern __shared__ __align__(16) double qsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, lx = lane & 7, ly = lane >> 3;
  double* hb = hb_all[warp];
  double* qw = qsm + warp * 1024;
  const long long gw = (long long)blockIdx.x * WARPS + warp;
  long long t0 = clock64();
  double acc = 0.0;
  for (int t = 0; t < tiles_per_warp; ++t) {
    const long long src = ((gw * 7 + t) & 255) * 2048;
    TileD tl;
    // q layout: lane-major rows so that row i of all lanes is 32 consecutive 4-double chunks
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        tl.x[i][c] = __ldcg(X + src + (8 * ly + i) * 32 + 4 * lx + c);
        qw[128 * i + 4 * lane + c] = __ldcg(Q + src + (8 * ly + i) * 32 + 4 * lx + c);
      }
    hb[lane] = __ldcg(X + src + 1024 + lane);
    hb[32 + lane] = __ldcg(X + src + 1024 + 32 + lane);
    hb[64 + lane] = __ldcg(X + src + 1024 + 64 + lane);
    hb[96 + lane] = __ldcg(X + src + 1024 + 96 + lane);
    __syncwarp();
    tl.qs = qw + 4 * lane;
    tl.hxp = hb + (lx == 0 ? 0 : 32) + 8 * ly;
    tl.hyp = hb + (ly == 0 ? 64 : 96) + 4 * lx;
#pragma unroll 1
    for (int s = 0; s < k; ++s) tl.sweep(lx, ly);
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc += tl.x[i][c];
    __syncwarp();
  }
  out[gw * 32 + lane] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = clock64() - t0;
}

template <typename Tile, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB)
bench(const double* __restrict__ X, const double* __restrict__ Q, double* __restrict__ out, int tiles_per_warp,
      int k, long long* clk) {
  __shared__ __align__(16) double hb_all[WARPS][128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, lx = lane & 7, ly = lane >> 3;
  double* hb = hb_all[warp];
  const long long gw = (long long)blockIdx.x * WARPS + warp;
  long long t0 = clock64();
  double acc = 0.0;
  for (int t = 0; t < tiles_per_warp; ++t) {
    const long long src = ((gw * 7 + t) & 255) * 2048;  // 256 source tiles (4 MB): L2-resident
    Tile tl;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        tl.x[i][c] = __ldcg(X + src + (8 * ly + i) * 32 + 4 * lx + c);
        tl.q[i][c] = __ldcg(Q + src + (8 * ly + i) * 32 + 4 * lx + c);
      }
    hb[lane] = __ldcg(X + src + 1024 + lane);
    hb[32 + lane] = __ldcg(X + src + 1024 + 32 + lane);
    hb[64 + lane] = __ldcg(X + src + 1024 + 64 + lane);
    hb[96 + lane] = __ldcg(X + src + 1024 + 96 + lane);
    __syncwarp();
    tl.hxp = hb + (lx == 0 ? 0 : 32) + 8 * ly;
    tl.hyp = hb + (ly == 0 ? 64 : 96) + 4 * lx;
#pragma unroll 1
    for (int s = 0; s < k; s += 2) {
      tl.sweep(lx, ly);
      tl.sweep(lx, ly);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc += tl.x[i][c];
    __syncwarp();
  }
  out[gw * 32 + lane] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = clock64() - t0;
}

template <typename Tile, int WARPS, int MINB>
void run(const char* name, const double* X, const double* Q, double* out, long long* clk, int nsm, int k) {
  const int tpw = 64;
  auto kern = bench<Tile, WARPS, MINB>;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) kern<<<nsm, WARPS * 32>>>(X, Q, out, tpw, k, clk);
  cudaEventRecord(a);
  const int R = 5;
  for (int rep = 0; rep < R; ++rep) kern<<<nsm, WARPS * 32>>>(X, Q, out, tpw, k, clk);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long c;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  const double upd = (double)nsm * WARPS * tpw * 1024.0 * k * R;
  const double secs = ms * 1e-3;
  const double mhz = (double)c / (ms / R * 1e-3) / 1e6;  // SM clock over one launch (CTA 0's span)
  const double peak = nsm * 16.0 * mhz * 1e6;            // updates/s at 64 DP ops/clk/SM
  printf("%-28s warps/SM %2d regs %3d spill %4d  %.3e upd/s  clk %.0f MHz  FP64 frac %.3f\n", name, WARPS,
         fa.numRegs, (int)fa.localSizeBytes, upd / secs, mhz, upd / secs / peak);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("  error: %s\n", cudaGetErrorString(e));
}


template <typename K>
void run_k(const char* name, K kern, int warps, size_t dsmem, const double* X, const double* Q, double* out,
           long long* clk, int nsm, int k) {
  const int tpw = 64;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  if (dsmem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) kern<<<nsm, warps * 32, dsmem>>>(X, Q, out, tpw, k, clk);
  cudaEventRecord(a);
  const int R = 5;
  for (int rep = 0; rep < R; ++rep) kern<<<nsm, warps * 32, dsmem>>>(X, Q, out, tpw, k, clk);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long c;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  const double upd = (double)nsm * warps * tpw * 1024.0 * k * R;
  const double secs = ms * 1e-3;
  const double mhz = (double)c / (ms / R * 1e-3) / 1e6;
  const double peak = nsm * 16.0 * mhz * 1e6;
  printf("%-28s warps/SM %2d regs %3d spill %4d  %.3e upd/s  clk %.0f MHz  FP64 frac %.3f\n", name, warps,
         fa.numRegs, (int)fa.localSizeBytes, upd / secs, mhz, upd / secs / peak);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("  error: %s\n", cudaGetErrorString(e));
}

int main(int argc, char** argv) {
  const int k = argc > 1 ? atoi(argv[1]) : 64;
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t n = 256 * 2048 + 4096;
  double *X, *Q, *out;
  long long* clk;
  cudaMalloc(&X, n * 8);
  cudaMalloc(&Q, n * 8);
  cudaMalloc(&out, (size_t)nsm * 16 * 32 * 8);
  cudaMalloc(&clk, 8);
  double* h = (double*)malloc(n * 8);
  for (size_t i = 0; i < n; ++i) h[i] = (double)((i * 2654435761u) % 1000) / 1000.0;
  cudaMemcpy(X, h, n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(Q, h, n * 8, cudaMemcpyHostToDevice);
  printf("k = %d sub-iterations per tile\n", k);
  run<TileA, 8, 1>("A middle-out (r1)", X, Q, out, clk, nsm, k);
  run_k("A2 conflict-free halo", bench_a2<8>, 8, 0, X, Q, out, clk, nsm, k);
  run<TileP, 8, 1>("P predicated halo loads", X, Q, out, clk, nsm, k);
  run<TileX<1>, 8, 1>("X1 no halo selects", X, Q, out, clk, nsm, k);
  run<TileX<2>, 8, 1>("X2 no W/E shuffles", X, Q, out, clk, nsm, k);
  run<TileX<3>, 8, 1>("X3 no W/E shfl, no sel", X, Q, out, clk, nsm, k);
  run<TileX<4>, 8, 1>("X4 no N/S shuffles", X, Q, out, clk, nsm, k);
  if (argc > 2) return 0;
  run<TileB, 8, 1>("B sequential", X, Q, out, clk, nsm, k);
  run<TileB, 12, 1>("B sequential 12w", X, Q, out, clk, nsm, k);
  run<TileA, 12, 1>("A middle-out 12w", X, Q, out, clk, nsm, k);
  run_k("C q in TMEM 8w", bench_c<8>, 8, 0, X, Q, out, clk, nsm, k);
  run_k("C q in TMEM 12w", bench_c<12>, 12, 0, X, Q, out, clk, nsm, k);
  run_k("C q in TMEM 16w", bench_c<16>, 16, 0, X, Q, out, clk, nsm, k);
  run_k("D q in smem 12w", bench_d<12>, 12, 12 * 8192, X, Q, out, clk, nsm, k);
  run_k("D q in smem 16w", bench_d<16>, 16, 16 * 8192, X, Q, out, clk, nsm, k);
  return 0;
}
