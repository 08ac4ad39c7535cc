// Register-tile building blocks shared by the 2D cycle kernels (kernels_2d.cu: the 32x32 hot path;
// kernels_2dt.cu: other tile shapes).  PAPER.md:380-387 (§4.1): the k sub-iterations of one
// augmented subdomain with its halo frozen; here the subdomain lives in a warp's registers.
#pragma once
#include "hj_internal.cuh"

namespace hj {
namespace rt {

constexpr unsigned FULL = 0xffffffffu;

template <typename T> struct VecOf;
template <> struct VecOf<double> { using v2 = double2; };
template <> struct VecOf<float> { using v2 = float2; };

// =============================================================================
// REG2D — the B200 design for 32x32 tiles.  One warp owns one tile; the tile lives in
// registers: lane l holds rows 8*(l>>3)..+7 and columns 4*(l&7)..+3 of the interior
// (32 cells), so a sub-iteration is 4 FP64 ops per cell plus warp shuffles for the
// 4x8-lane block edges.  Per warp, shared memory holds ONE input slot (x box with halo + h2f
// box, filled by TMA and completed on an mbarrier), the frozen halo of the tile in flight and
// an output staging tile drained by a TMA tensor store.  Registers are the second buffer:
// as soon as a tile is in registers the slot is refilled with the warp's next tile, so its
// HBM traffic overlaps the k sub-iterations.  Persistent grid, 4 warps per SM sub-partition
// multiple (8 f64 / 12 f32 warps per CTA, one CTA per SM).
// =============================================================================
template <typename T, int WARPS_ = (sizeof(T) == 8 ? 8 : 12), bool TMA_STORE_ = false>
struct R2 {
  static constexpr int COL0 = 16 / sizeof(T);                          // interior column offset
  static constexpr int BW = ((COL0 + 33) + (16 / sizeof(T)) - 1) / (16 / sizeof(T)) * (16 / sizeof(T));
  static constexpr int BH = 34;
  static constexpr int XBYTES = BW * BH * sizeof(T);
  static constexpr int XSLOT = (XBYTES + 127) / 128 * 128;
  static constexpr int FBYTES = 32 * 32 * sizeof(T);
  static constexpr bool TMA_STORE = TMA_STORE_;
  static constexpr int OBYTES = TMA_STORE ? 32 * 32 * sizeof(T) : 0;   // output staging tile
  static constexpr int HALO = 128 * sizeof(T);                          // frozen halo W|E|S|N
  // multigrid fused correction: the 18 x 18 coarse patch under the tile + halo (TMA box).  TMA box
  // origins must be 16-B aligned along x, so the box starts COL0 - 1 elements before the patch's
  // first ringed column (at element x0/2 of the padded row) and is COL0 - 1 + 18 wide, rounded
  // up to a 16-B multiple.
  static constexpr int EW = sizeof(T) == 8 ? 20 : 24, EH = 18;
  static constexpr int EBYTES = EW * EH * sizeof(T);
  static constexpr int ESLOT = (EBYTES + 127) / 128 * 128;
  static constexpr int EOFF = XSLOT + FBYTES + OBYTES + HALO;
  static constexpr int WSMEM = EOFF + ESLOT;                            // per warp
  static constexpr int WARPS = WARPS_;
  static constexpr int BARS = 128;                                      // barrier region bytes
  static constexpr size_t SMEM = 128 + BARS + size_t(WARPS) * WSMEM;    // +128 for alignment
  static_assert(SMEM <= 232448, "shared memory budget");
};

// TXL / TYL: lanes per method tile along x / y inside the warp's 32x32 block (8 / 4: one tile per
// warp, the block's edges are the tile's edges; smaller: several tiles per warp, kernels_2dt.cu).
template <typename T, bool MASK, int SK, int TXL = 8, int TYL = 4>
struct Tile2 {
  static constexpr bool GEN = SK == 1;  // general coefficients (Eq. 10, reading c23)
  static constexpr bool WGT = SK == 2;  // damped Jacobi: the multigrid smoother (reading c24)
  T x[8][4];      // current iterate
  T q[8][4];      // 0.25 * h^2 f  (GEN: b / d)
  T cw[4];        // GEN: weights W, E, S, N
  T om;           // WGT: damping factor omega
  const T* hxp;   // per-warp smem: frozen W (lx == 0) / E (lx == 7) halo of my 8 rows
  const T* hyp;   // per-warp smem: frozen S (ly == 0) / N (ly == 3) halo of my 4 columns
  uint32_t own;   // MASK (overlapping blocks): bit 4*i+c set if this block owns cell (i, c)

  __device__ __forceinline__ bool on(int i, int c) const {
    return !MASK || ((own >> (4 * i + c)) & 1u);
  }
  __device__ __forceinline__ T upd(T W, T E, T S, T N, T qq) const {
    if constexpr (GEN) return gupd2(cw[0], cw[1], cw[2], cw[3], W, E, S, N, qq);
    else return upd2(W, E, S, N, qq);
  }

  // N/S neighbour rows across lane rows: row 0 of the lane below is my row 7's N, row 7 of the
  // lane above is my row 0's S; the edge lane rows take the frozen halo (predicated loads).
  __device__ __forceinline__ void exchange_ns(int ly, T (&up)[4], T (&dn)[4]) const {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      up[c] = __shfl_down_sync(FULL, x[0][c], 8);
      dn[c] = __shfl_up_sync(FULL, x[7][c], 8);
    }
    // every lane's halo pointer is valid, so the loads are unconditional and only the
    // choice is a select (no divergent branches in the sub-iteration loop)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const T hv = hyp[c];
      up[c] = eN(ly) ? hv : up[c];
      dn[c] = eS(ly) ? hv : dn[c];
    }
  }
  // the lane's block edge is a tile edge (frozen halo instead of the neighbouring lane's value)
  static __device__ __forceinline__ bool eW(int lx) { if constexpr (TXL == 8) return lx == 0; else return lx % TXL == 0; }
  static __device__ __forceinline__ bool eE(int lx) { if constexpr (TXL == 8) return lx == 7; else return lx % TXL == TXL - 1; }
  static __device__ __forceinline__ bool eS(int ly) { if constexpr (TYL == 4) return ly == 0; else return ly % TYL == 0; }
  static __device__ __forceinline__ bool eN(int ly) { if constexpr (TYL == 4) return ly == 3; else return ly % TYL == TYL - 1; }
  __device__ __forceinline__ void exchange_we(int lx, int i, T& w, T& e) const {
    w = __shfl_up_sync(FULL, x[i][3], 1, 8);
    e = __shfl_down_sync(FULL, x[i][0], 1, 8);
    const T hv = hxp[i];
    w = eW(lx) ? hv : w;
    e = eE(lx) ? hv : e;
  }

  // Residual of the snapshot, s^2 summed over my cells (double).
  __device__ __forceinline__ double residual(int lx, int ly) const {
    T up[4], dn[4];
    exchange_ns(ly, up, dn);
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      T w, e;
      exchange_we(lx, i, w, e);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const T W = c == 0 ? w : x[i][c - 1];
        const T E = c == 3 ? e : x[i][c + 1];
        const T S = i == 0 ? dn[c] : x[i - 1][c];
        const T N = i == 7 ? up[c] : x[i + 1][c];
        const double s =
            GEN ? gres2((double)cw[0], (double)cw[1], (double)cw[2], (double)cw[3], (double)x[i][c],
                        (double)W, (double)E, (double)S, (double)N, (double)q[i][c])
                : res2((double)x[i][c], (double)W, (double)E, (double)S, (double)N,
                       (double)(T(4) * q[i][c]));
        if (on(i, c)) acc = __fma_rn(s, s, acc);
      }
    }
    return acc;
  }

  // sweep_mo with exchange hooks for tiles spread over several warps (kernels_2dt.cu): the same
  // rows in the same middle-out order, split in two halves — rows 3,4,2,5 (A) and 1,6,0,7 (B).
  // h.wait_a() / h.wait_b() before each half (the neighbours' block edges of the previous
  // sub-iteration for that half have arrived), h.send_a(*this) / h.send_b(*this) after it (my new
  // block-edge values of that half to the neighbours); the N/S lane exchange moves to just before
  // row 0 so that it reads the halo rows only after wait_b.  Same values as sweep_mo.
  template <bool RES, typename H>
  __device__ __forceinline__ void sweep_h(int lx, int ly, double* acc, H& h) {
    T up[4], dn[4];
    T olo[4], ohi[4];
    h.wait_a();
#pragma unroll
    for (int step = 0; step < 8; ++step) {
      const int i = step == 0 ? 3 : (step & 1) ? 3 + (step + 1) / 2 : 3 - step / 2;  // 3,4,2,5,1,6,0,7
      const bool hi_side = step > 0 && (step & 1);
      if (step == 4) h.wait_b();
      if (step == 6) exchange_ns(ly, up, dn);   // rows 0 and 7 still hold the old values
      T w, e;
      exchange_we(lx, i, w, e);
      T nw[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const T W = c == 0 ? w : x[i][c - 1];
        const T E = c == 3 ? e : x[i][c + 1];
        const T S = (i == 0) ? dn[c] : (step > 0 && hi_side ? ohi[c] : x[i - 1][c]);
        const T N = (i == 7) ? up[c] : (step > 0 && !hi_side ? olo[c] : x[i + 1][c]);
        if constexpr (RES) {  // Poisson, T = double (the REGT fold)
          const double sum = __dadd_rn(__dadd_rn(W, E), __dadd_rn(S, N));
          nw[c] = __fma_rn(0.25, sum, q[i][c]);
          const double t = __fma_rn(4.0, x[i][c], -sum);
          const double r = __fma_rn(4.0, q[i][c], -t);
          acc[c] = __fma_rn(r, r, acc[c]);
        } else {
          nw[c] = upd(W, E, S, N, q[i][c]);
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (step == 0) { olo[c] = x[i][c]; ohi[c] = x[i][c]; }
        else if (hi_side) ohi[c] = x[i][c];
        else olo[c] = x[i][c];
        x[i][c] = nw[c];
      }
      if (step == 3) h.send_a(*this);
    }
    h.send_b(*this);
  }

  // One Jacobi sub-iteration in middle-out row order 3,4,2,5,1,6,0,7: every row's inputs from the
  // previous sub-iteration were produced >= 3 rows earlier, and the cross-lane N/S values (rows 0
  // and 7 of the neighbouring lane rows) are consumed last, so consecutive sub-iterations overlap
  // instead of draining the pipeline.  The computed rows form a growing block [lo, hi]; the old
  // values of its two edge rows are kept in olo / ohi.
  template <bool RES = false>
  __device__ __forceinline__ void sweep_mo(int lx, int ly, double* acc = nullptr) {
    T up[4], dn[4];
    exchange_ns(ly, up, dn);
    T olo[4], ohi[4];
#pragma unroll
    for (int step = 0; step < 8; ++step) {
      const int i = step == 0 ? 3 : (step & 1) ? 3 + (step + 1) / 2 : 3 - step / 2;  // 3,4,2,5,1,6,0,7
      const bool hi_side = step > 0 && (step & 1);
      T w, e;
      exchange_we(lx, i, w, e);
      T nw[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const T W = c == 0 ? w : x[i][c - 1];
        const T E = c == 3 ? e : x[i][c + 1];
        // S = old row i-1, N = old row i+1
        const T S = (i == 0) ? dn[c] : (step > 0 && hi_side ? ohi[c] : x[i - 1][c]);
        const T N = (i == 7) ? up[c] : (step > 0 && !hi_side ? olo[c] : x[i + 1][c]);
        if constexpr (RES && GEN) {  // T = double: the residual is the update minus x (c23)
          nw[c] = upd(W, E, S, N, q[i][c]);
          const double r = __dsub_rn(nw[c], x[i][c]);
          if (on(i, c)) acc[c] = __fma_rn(r, r, acc[c]);
        } else if constexpr (RES) {
          const double sum = __dadd_rn(__dadd_rn(W, E), __dadd_rn(S, N));
          nw[c] = __fma_rn(0.25, sum, q[i][c]);
          if constexpr (WGT) nw[c] = damp(om, x[i][c], nw[c]);
          const double t = __fma_rn(4.0, x[i][c], -sum);
          const double r = __fma_rn(4.0, q[i][c], -t);
          if (on(i, c)) acc[c] = __fma_rn(r, r, acc[c]);
        } else {
          nw[c] = upd(W, E, S, N, q[i][c]);
          if constexpr (WGT) nw[c] = damp(om, x[i][c], nw[c]);
        }
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


}  // namespace rt
}  // namespace hj
