// 2D kernels of libhj.so: one hierarchical cycle (two kernel designs) and one classic sweep.
//
// PAPER.md:380-387 (§4.1): a cycle copies every (Tx+2)x(Ty+2) augmented subdomain from global
// to on-chip memory, runs k Jacobi sub-iterations on the Tx x Ty interior with the halo frozen,
// and copies the interior back.  PAPER.md:114-133 (§3.2): the classic sweep.
// Every kernel also reduces the h^2-scaled residual of the snapshot it reads:
// s = h2f - (4x - ((W+E)+(S+N))), sum of s^2 per tile -> part[tile].
// SK (stencil kind) = 1: the general constant-coefficient stencil of Eq. 10 —
// the update and residual of hj_internal.cuh gupd2 / gres2 (reading c23) with the
// weights held as kernel parameters; SK = 2: the Poisson update damped by omega (damp(), the
// multigrid smoother of reading c24); SK = 0: the paper's Poisson update.  Everything else (tiles,
// halo, stores) is unchanged.
#include <cstdlib>
#include <type_traits>

#include "hj_internal.cuh"
#include "reg_tile.cuh"

namespace hj {

// HJ_TILE_STRIP=S: REG2D walks the tiles in column strips of S tiles (0 / unset: row-major)
static int tile_strip() {
  static const int sw = [] { const char* e = std::getenv("HJ_TILE_STRIP"); return e ? std::atoi(e) : 0; }();
  return sw;
}

namespace {

using namespace rt;

// One full 32x32 tile: smem slot -> registers, refill, fused residual, k sub-iterations, store.
// XM (x mode): 0 = the snapshot from the slot; 1 = COR, the snapshot plus the interpolated coarse
// correction (multigrid post-smoothing, c24); 2 = ZX, the snapshot is identically zero and was not
// loaded (the first smoothing cycle of a coarse multigrid level: its iterate starts at zero, c24).
template <typename T, typename C, bool MASK, int SK, int XM, typename Refill, typename Store>
__device__ __forceinline__ void reg2d_tile(const Wt2& wt, const T* __restrict__ sx, const T* __restrict__ sf,
                                           T* __restrict__ so, T* __restrict__ hb, int lane, int kk,
                                           double* __restrict__ part, long long t, Refill&& refill,
                                           Store&& store, T* __restrict__ gdst, long long pitch,
                                           int ox0, int ox1, int oy0, int oy1, const T* __restrict__ eb,
                                           int x0, int y0, int nx, int ny, T* plo, T* phi) {
  using V2 = typename VecOf<T>::v2;
  constexpr bool COR = XM == 1, ZX = XM == 2;
  const int lx = lane & 7, ly = lane >> 3;
  Tile2<T, MASK, SK> tl;
  if constexpr (SK == 1) {
    tl.cw[0] = (T)wt.w; tl.cw[1] = (T)wt.e; tl.cw[2] = (T)wt.s; tl.cw[3] = (T)wt.n;
  }
  if constexpr (SK == 2) tl.om = (T)wt.om;
#pragma unroll
  for (int i = 0; i < 8; ++i) {  // 128-bit shared loads
    const int r = 8 * ly + i;
    const V2* rowx = reinterpret_cast<const V2*>(sx + (r + 1) * C::BW + C::COL0 + 4 * lx);
    const V2* rowf = reinterpret_cast<const V2*>(sf + r * 32 + 4 * lx);
    const V2 a = ZX ? V2{T(0), T(0)} : rowx[0], b = ZX ? V2{T(0), T(0)} : rowx[1];
    const V2 fa = rowf[0], fb = rowf[1];
    tl.x[i][0] = a.x; tl.x[i][1] = a.y; tl.x[i][2] = b.x; tl.x[i][3] = b.y;
    tl.q[i][0] = fa.x; tl.q[i][1] = fa.y; tl.q[i][2] = fb.x; tl.q[i][3] = fb.y;
  }
  // frozen halo -> the warp's halo buffer [W(32) | E(32) | S(32) | N(32)]
  T hw = ZX ? T(0) : sx[(lane + 1) * C::BW + C::COL0 - 1];
  T he = ZX ? T(0) : sx[(lane + 1) * C::BW + C::COL0 + 32];
  T hs = ZX ? T(0) : sx[C::COL0 + lane];
  T hn = ZX ? T(0) : sx[33 * C::BW + C::COL0 + lane];
  if constexpr (COR) {
    // multigrid: correct the snapshot (tile and halo) by the interpolated coarse iterate before
    // anything reads it — the coarse-grid correction fused into this post-smoothing cycle (c24).
    // The coarse patch under tile + halo (ringed coarse rows y0/2 .., columns x0/2 ..) arrived
    // with the tile by TMA (eb, row stride EW); lane patch = rows 4ly .. +4, columns 2lx .. +2.
    T E[5][3];
#pragma unroll
    for (int r = 0; r < 5; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) E[r][c] = eb[(4 * ly + r) * C::EW + (C::COL0 - 1) + 2 * lx + c];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int a = i / 2, b = c / 2;  // fine row i / col c of the lane: odd ringed index when even
        T v;
        if ((i & 1) == 0 && (c & 1) == 0)
          v = mul_t(T(0.25), add_t(add_t(E[a][b], E[a][b + 1]), add_t(E[a + 1][b], E[a + 1][b + 1])));
        else if ((i & 1) == 0)
          v = mul_t(T(0.5), add_t(E[a][(c + 1) / 2], E[a + 1][(c + 1) / 2]));
        else if ((c & 1) == 0)
          v = mul_t(T(0.5), add_t(E[(i + 1) / 2][b], E[(i + 1) / 2][b + 1]));
        else
          v = E[(i + 1) / 2][(c + 1) / 2];
        tl.x[i][c] = add_t(tl.x[i][c], v);
      }
    // halo points inside the domain (the domain ring holds g and is never corrected); tile-local
    // ringed coordinates (a, b) in [0, 33] have the parity of the global ones (x0, y0 even)
    auto EB = [&](int I, int J) { return eb[J * C::EW + (C::COL0 - 1) + I]; };
    if (x0 > 0) hw = add_t(hw, mg_interp_f<T>(EB, 0, lane + 1));
    if (x0 + 32 < nx) he = add_t(he, mg_interp_f<T>(EB, 33, lane + 1));
    if (y0 > 0) hs = add_t(hs, mg_interp_f<T>(EB, lane + 1, 0));
    if (y0 + 32 < ny) hn = add_t(hn, mg_interp_f<T>(EB, lane + 1, 33));
  }
  hb[lane] = hw;
  hb[32 + lane] = he;
  hb[64 + lane] = hs;
  hb[96 + lane] = hn;
  tl.hxp = hb + (lx == 0 ? 0 : 32) + 8 * ly;
  tl.hyp = hb + (ly == 0 ? 64 : 96) + 4 * lx;
  tl.own = 0xffffffffu;
  if (MASK) {  // owned sub-range [ox0, ox1] x [oy0, oy1] of the block (tile-local, inclusive)
    tl.own = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int r = 8 * ly + i, q = 4 * lx + c;
        if (r >= oy0 && r <= oy1 && q >= ox0 && q <= ox1) tl.own |= 1u << (4 * i + c);
      }
  }
  __syncwarp();
  refill();  // every value of the slot is now in registers or the halo buffer
  // fused residual of the snapshot: a separate pass for fp32 (residual in double, reading
  // c16) and for residual-only cycles; fp64 folds it into the first sub-iteration below.
  constexpr bool FOLD = sizeof(T) == 8;
  double acc = 0.0;
  int s = 0;
  if (FOLD && kk >= 8 && ((kk - 1) & 1)) {
    // even k >= 8: the residual sweep and the next plain sweep in ONE basic block with the warp
    // reduction of the residual after both, so ptxas interleaves its dependent shuffle chain
    // with the plain sweep instead of exposing it (the same value: warp_sum of the same a4).
    // Below k = 8 the HBM-bound cycle measured faster in the old order.
    double a4[4] = {0.0, 0.0, 0.0, 0.0};  // four independent accumulation chains
    tl.template sweep_mo<true>(lx, ly, a4);
    tl.template sweep_mo<false>(lx, ly);
    acc = warp_sum((a4[0] + a4[1]) + (a4[2] + a4[3]));
    s = 2;
  } else {
    if (!FOLD || kk == 0) acc = tl.residual(lx, ly);
    if (FOLD && kk > 0) {
      double a4[4] = {0.0, 0.0, 0.0, 0.0};
      tl.template sweep_mo<true>(lx, ly, a4);
      acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
      s = 1;
    }
    acc = warp_sum(acc);
    if (s < kk && ((kk - s) & 1)) {
      tl.template sweep_mo<false>(lx, ly);
      ++s;
    }
  }
  if (lane == 0) part[t] = acc;
  // remaining sub-iterations (an even number), halo frozen
#pragma unroll 1
  for (; s < kk; s += 2) {
    tl.template sweep_mo<false>(lx, ly);
    tl.template sweep_mo<false>(lx, ly);
  }
  if (kk == 0) return;  // residual-only pass (after max_cycles)
  if constexpr (MASK) {
    // overlapping blocks: only the owned points are written
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (tl.on(i, c)) gdst[(8 * ly + i) * pitch + 4 * lx + c] = tl.x[i][c];
  } else if constexpr (C::TMA_STORE) {
    // registers -> staging tile -> TMA store into the NEXT iterate (snapshot semantics)
    if (lane == 0) bulk_wait_read_all();  // the previous tile's store has read the staging tile
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      V2* dst = reinterpret_cast<V2*>(so + (8 * ly + i) * 32 + 4 * lx);
      dst[0] = V2{tl.x[i][0], tl.x[i][1]};
      dst[1] = V2{tl.x[i][2], tl.x[i][3]};
    }
    fence_proxy_async();
    __syncwarp();
    store();
  } else {
    // registers -> global, 128-bit stores (gdst = interior origin of the tile in the NEXT iterate)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      V2* dst = reinterpret_cast<V2*>(gdst + (8 * ly + i) * pitch + 4 * lx);
      dst[0] = V2{tl.x[i][0], tl.x[i][1]};
      dst[1] = V2{tl.x[i][2], tl.x[i][3]};
    }
  }
  // peer transport (row slabs): a tile in the slab's first / last tile row also stores its first /
  // last row straight into the neighbour's ghost row (NVLink stores through the CUDA-IPC mapping),
  // so the halo exchange overlaps the cycle tile by tile; the fence orders them before the
  // finalize kernel's signal
  if (plo && ly == 0) {
    V2* d = reinterpret_cast<V2*>(plo + x0 + 4 * lx);
    d[0] = V2{tl.x[0][0], tl.x[0][1]};
    d[1] = V2{tl.x[0][2], tl.x[0][3]};
    __threadfence_system();
  }
  if (phi && ly == 3) {
    V2* d = reinterpret_cast<V2*>(phi + x0 + 4 * lx);
    d[0] = V2{tl.x[7][0], tl.x[7][1]};
    d[1] = V2{tl.x[7][2], tl.x[7][3]};
    __threadfence_system();
  }
}

// Persistent kernel over the FULL 32x32 tiles (ntx_full x nty_full of them; ragged edge tiles,
// if any, are done by smem2d_kernel in edge mode).  Warp w handles full tiles w, w+W, ...;
// partials are indexed by the global tile index ty*ntx + tx.
template <typename T, typename C, bool MASK, int SK, int XM = 0>
__global__ void __launch_bounds__(C::WARPS * 32, 1)
reg2d_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmF,
             const __grid_constant__ CUtensorMap tmO, T* __restrict__ xout, long long pitch,
             Axis ax, Axis ay, int ntx_full, long long nfull, int ntx, double* __restrict__ part,
             const Ctrl* __restrict__ ctrl, int k, long long max_cycles, Wt2 wt,
             const __grid_constant__ CUtensorMap tmE, T* peer_lo, T* peer_hi, int ty0, int tys, int sw) {
  if (ctrl->done) return;
  constexpr bool COR = XM == 1, ZX = XM == 2;
  const int kk = (ctrl->c >= max_cycles) ? 0 : k;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bar = reinterpret_cast<uint64_t*>(base) + warp;
  unsigned char* slot = base + C::BARS + size_t(warp) * C::WSMEM;
  const T* sx = reinterpret_cast<const T*>(slot);
  const T* sf = reinterpret_cast<const T*>(slot + C::XSLOT);
  T* so = reinterpret_cast<T*>(slot + C::XSLOT + C::FBYTES);
  T* hb = reinterpret_cast<T*>(slot + C::XSLOT + C::FBYTES + C::OBYTES);
  const T* eb = reinterpret_cast<const T*>(slot + C::EOFF);
  const long long gw = (long long)blockIdx.x * C::WARPS + warp;
  const long long nw = (long long)gridDim.x * C::WARPS;
  if (gw >= nfull) return;
  // u -> tile: row-major (sw == 0), or column strips of sw tiles walked row by row (sw > 0, sw divides
  // ntx_full; HJ_TILE_STRIP, an experiment on L2 / TLB locality)
  const long long nrows_t = nfull / ntx_full;
  auto tile_of = [&](long long u, int& tx, int& ty) {
    if (sw > 0) {
      const long long per = (long long)sw * nrows_t, st = u / per, r = u % per;
      tx = (int)(st * sw + r % sw);
      ty = ty0 + (int)(r / sw) * tys;
    } else {
      tx = (int)(u % ntx_full);
      ty = ty0 + (int)(u / ntx_full) * tys;
    }
  };
  auto issue = [&](long long u) {  // u: full-block index; box origin = block's interior origin
    int utx, uty;
    tile_of(u, utx, uty);
    const int cx = axis_start(ax, utx), cy = axis_start(ay, uty);
    mbar_arrive_expect_tx(bar, (ZX ? 0 : C::XBYTES) + C::FBYTES + (COR ? C::EBYTES : 0));
    if (!ZX) tma_load_2d(slot, &tmX, cx, cy, bar);    // x box: padded rows 32ty.., cols 32tx..
    tma_load_2d(slot + C::XSLOT, &tmF, cx, cy, bar);   // h2f box
    if (COR) tma_load_2d(slot + C::EOFF, &tmE, cx / 2, cy / 2, bar);  // coarse patch (16-B aligned start)
  };
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    prefetch_tensormap(&tmX);
    prefetch_tensormap(&tmF);
    prefetch_tensormap(&tmO);
    if (COR) prefetch_tensormap(&tmE);
    issue(gw);
  }
  __syncwarp();
  int it = 0;
  for (long long u = gw; u < nfull; u += nw, ++it) {
    mbar_wait(bar, it & 1);
    int tx, ty;
    tile_of(u, tx, ty);
    const int x0 = axis_start(ax, tx), y0 = axis_start(ay, ty);
    reg2d_tile<T, C, MASK, SK, XM>(
        wt, sx, sf, so, hb, lane, kk, part, (long long)ty * ntx + tx,
        [&] {
          if (lane == 0 && u + nw < nfull) {
            fence_proxy_async();  // generic reads of the slot before the TMA overwrite
            issue(u + nw);
          }
        },
        [&] {
          if (lane == 0) {
            tma_store_2d(&tmO, C::COL0 + x0, y0 + 1, so);
            bulk_commit();
          }
        },
        xout + ((long long)y0 + 1) * pitch + C::COL0 + x0, pitch, axis_own_lo(ax, tx) - x0,
        axis_own_hi(ax, tx) - x0, axis_own_lo(ay, ty) - y0, axis_own_hi(ay, ty) - y0, eb, x0, y0,
        ax.n, ay.n, ty == 0 ? peer_lo : nullptr, ty == ay.nb - 1 && y0 + 32 == ay.n ? peer_hi : nullptr);
  }
  if (C::TMA_STORE && lane == 0) bulk_wait_all();
}

// =============================================================================
// RES2D — the resident solver, for grids whose 32x32 tiles fit one per warp of a co-resident grid
// (ntiles <= 8 x #SMs, o = 0, nx and ny multiples of 32; BASELINE configs 1 and 3 sizes): the
// WHOLE solve in one cooperative launch.  Each warp keeps its tile's iterate and q in registers
// for the entire solve; per cycle it reads only the tile's frozen halo (128 values) of x_c from
// X[p] (L2), runs the fused residual and the k sub-iterations exactly as reg2d_tile does, writes
// x_{c+1} into X[p^1] (snapshot semantics: x_c survives a converged test) and its residual
// partial; one grid barrier; then every CTA sums the partials in the same fixed order and takes
// the same stopping decision (hj_decide; CTA 0 writes the history and the control block).  Same
// cycle, same arithmetic — bitwise the iterates of the per-cycle path — without the per-cycle
// launches and without re-reading the interior.  Classic mode uses it with k = 1 (a hierarchical
// cycle with k = 1 is the classic sweep, bit for bit: PAPER.md:177, pin P1).
// =============================================================================
constexpr int RES2D_MAX_ROWS = 1184;  // tile rows <= tiles <= 8 warps x 148 SMs
template <typename T, int SK>
__global__ void __launch_bounds__(256, 1)
res2d_kernel(T* __restrict__ X0, T* __restrict__ X1, const T* __restrict__ Q, long long pitch,
             long long fpitch, int ntx, int nty, double* __restrict__ part, Ctrl* __restrict__ ctrl,
             double* __restrict__ hist, long long hist_cap, double rdiv, double tol, int tol_mode,
             double ref_residual, long long max_cycles, int k, Wt2 wt, unsigned int* bar) {
  using V2 = typename VecOf<T>::v2;
  constexpr int COL0 = 16 / sizeof(T);
  __shared__ Ctrl cs;
  __shared__ int s_done;
  __shared__ __align__(16) T hbuf[8][128];
  __shared__ double rsum[RES2D_MAX_ROWS];   // tile-row sums of the residual partials
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, lx = lane & 7, ly = lane >> 3;
  const long long ntiles = (long long)ntx * nty;
  const long long t = (long long)blockIdx.x * 8 + warp;
  const bool active = t < ntiles;
  if (threadIdx.x == 0) {
    cs = *ctrl;
    s_done = cs.done;
  }
  __syncthreads();
  if (s_done) return;
  const int tx = active ? (int)(t % ntx) : 0, ty = active ? (int)(t / ntx) : 0;
  const long long x0 = 32LL * tx, y0 = 32LL * ty;
  Tile2<T, false, SK> tl;
  if constexpr (SK == 1) {
    tl.cw[0] = (T)wt.w; tl.cw[1] = (T)wt.e; tl.cw[2] = (T)wt.s; tl.cw[3] = (T)wt.n;
  }
  if constexpr (SK == 2) tl.om = (T)wt.om;
  tl.own = 0xffffffffu;
  T* hb = hbuf[warp];
  tl.hxp = hb + (lx == 0 ? 0 : 32) + 8 * ly;
  tl.hyp = hb + (ly == 0 ? 64 : 96) + 4 * lx;
  int p = (int)(cs.c & 1);
  if (active) {  // the tile's iterate x_c and q, once for the whole solve
    const T* Xc = p ? X1 : X0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const long long r = 8 * ly + i;
      const V2* rx = reinterpret_cast<const V2*>(Xc + (y0 + 1 + r) * pitch + COL0 + x0 + 4 * lx);
      const V2* rf = reinterpret_cast<const V2*>(Q + (y0 + r) * fpitch + x0 + 4 * lx);
      const V2 a = rx[0], b = rx[1], fa = rf[0], fb = rf[1];
      tl.x[i][0] = a.x; tl.x[i][1] = a.y; tl.x[i][2] = b.x; tl.x[i][3] = b.y;
      tl.q[i][0] = fa.x; tl.q[i][1] = fa.y; tl.q[i][2] = fb.x; tl.q[i][3] = fb.y;
    }
  }
  for (;;) {
    const T* Xc = p ? X1 : X0;
    T* Xn = p ? X0 : X1;
    const long long c = cs.c;
    const int kk = c >= max_cycles ? 0 : k;
    double* pc = part + (c & 1) * ntiles;   // double-buffered: a slow CTA may still read cycle c-1's
    if (active) {
      // frozen halo of x_c: the neighbours' boundary cells written last cycle (L2 loads)
      hb[lane] = __ldcg(Xc + (y0 + 1 + lane) * pitch + COL0 - 1 + x0);
      hb[32 + lane] = __ldcg(Xc + (y0 + 1 + lane) * pitch + COL0 + x0 + 32);
      hb[64 + lane] = __ldcg(Xc + y0 * pitch + COL0 + x0 + lane);
      hb[96 + lane] = __ldcg(Xc + (y0 + 33) * pitch + COL0 + x0 + lane);
      __syncwarp();
      constexpr bool FOLD = sizeof(T) == 8;
      double acc = 0.0;
      if (!FOLD || kk == 0) acc = tl.residual(lx, ly);
      int s = 0;
      if (FOLD && kk > 0) {
        double a4[4] = {0.0, 0.0, 0.0, 0.0};
        tl.template sweep_mo<true>(lx, ly, a4);
        acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
        s = 1;
      }
      if (s < kk && ((kk - s) & 1)) {
        tl.template sweep_mo<false>(lx, ly);
        ++s;
      }
#pragma unroll 1
      for (; s < kk; s += 2) {
        tl.template sweep_mo<false>(lx, ly);
        tl.template sweep_mo<false>(lx, ly);
      }
      if (kk > 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          V2* dst = reinterpret_cast<V2*>(Xn + (y0 + 1 + 8 * ly + i) * pitch + COL0 + x0 + 4 * lx);
          dst[0] = V2{tl.x[i][0], tl.x[i][1]};
          dst[1] = V2{tl.x[i][2], tl.x[i][3]};
        }
      }
      acc = warp_sum(acc);
      if (lane == 0) pc[t] = acc;
      __syncwarp();
    }
    grid_barrier(bar, gridDim.x);
    // every CTA: the total in EXACTLY the order of rowsum_kernel + finalize_kernel (so the history
    // is bitwise that of the per-cycle path): per tile row a lane-strided sum + xor tree, then the
    // 1024-thread finalize reduction (thread i sums rows i, i+1024, ...; xor tree per warp; the 32
    // warp sums in order).  Warps split the tile rows; warp 0 finishes.
    {
      double* R = rsum;
      for (int g0 = warp; g0 < nty; g0 += 8 * 4) {  // 4 rows per warp at a time: loads and trees overlap
        double v[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int g = g0 + 8 * r;
          v[r] = 0.0;
          if (g < nty)
            for (int q = lane; q < ntx; q += 32) v[r] += __ldcg(pc + (long long)g * ntx + q);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int r = 0; r < 4; ++r) v[r] += __shfl_xor_sync(0xffffffffu, v[r], o);
#pragma unroll
        for (int r = 0; r < 4; ++r)
          if (lane == 0 && g0 + 8 * r < nty) R[g0 + 8 * r] = v[r];
      }
      __syncthreads();
      if (warp == 0) {
        double S = 0.0;
        for (int w = 0; w < 32 && 32 * w < nty; ++w) {  // warps beyond nty add +0.0: S unchanged
          double v = 0.0;
          for (int q = 32 * w + lane; q < nty; q += 1024) v += R[q];
          S += warp_sum(v);
        }
        if (lane == 0) {
          hj_decide(&cs, S, blockIdx.x == 0 ? hist : nullptr, hist_cap, rdiv, tol, tol_mode, ref_residual,
                    max_cycles);
          s_done = cs.done;
        }
      }
    }
    __syncthreads();
    if (s_done) break;
    p ^= 1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *ctrl = cs;
}

// =============================================================================
// SMEM2D — the paper's design (App. A): one CTA per tile, one thread per
// DOF, two (Tx+2)(Ty+2) containers plus a Tx*Ty rhs array in shared memory (exactly the
// paper's byte formula), __syncthreads between sub-iterations.  Any tile shape with
// Tx*Ty <= 1024.  Used for tile shapes REG2D does not cover and as the in-tile baseline.
// =============================================================================
// edge != 0: only the ragged edge tiles — blocks [0, nty) are the last tile column (if nx is
// ragged), the following blocks the last tile row (if ny is ragged) — for REG2D grids.
template <typename T, int SK>
__global__ void smem2d_kernel(const T* __restrict__ xin, T* __restrict__ xout,
                              const T* __restrict__ h2f, long long pitch, long long fpitch, int nx,
                              int ny, Axis ax, Axis ay, int edge, double* __restrict__ part,
                              const Ctrl* __restrict__ ctrl, int k, long long max_cycles, Wt2 wt,
                              const T* __restrict__ ecor, long long ep, T* peer_lo, T* peer_hi,
                              int zero_x) {
  constexpr bool GEN = SK == 1;  // general coefficients (reading c23)
  const int ntx = ax.nb, nty = ay.nb;
  if (ctrl->done) return;
  const int kk = (ctrl->c >= max_cycles) ? 0 : k;
  constexpr int COL0 = 16 / sizeof(T);
  const int Tx = blockDim.x, Ty = blockDim.y, L = Tx + 2;
  extern __shared__ unsigned char smem_raw[];
  T* A = reinterpret_cast<T*>(smem_raw);
  T* B = A + L * (Ty + 2);
  T* rhs = B + L * (Ty + 2);
  __shared__ double wsum[32];
  long long tx, ty;
  if (!edge) {
    tx = blockIdx.x % ntx;
    ty = blockIdx.x / ntx;
  } else {
    const int ncol = (nx % Tx) ? nty : 0;  // ragged last column
    if ((int)blockIdx.x < ncol) { tx = ntx - 1; ty = blockIdx.x; }
    else { tx = blockIdx.x - ncol; ty = nty - 1; }
  }
  const long long t = ty * ntx + tx;
  const long long i0 = axis_start(ax, (int)tx), j0 = axis_start(ay, (int)ty);  // interior origin
  const int w = axis_width(ax, (int)tx), hgt = axis_width(ay, (int)ty);
  // owned sub-range (tile-local, inclusive): the whole tile unless blocks overlap
  const int ox0 = axis_own_lo(ax, (int)tx) - (int)i0, ox1 = axis_own_hi(ax, (int)tx) - (int)i0;
  const int oy0 = axis_own_lo(ay, (int)ty) - (int)j0, oy1 = axis_own_hi(ay, (int)ty) - (int)j0;
  const int tid = threadIdx.y * Tx + threadIdx.x, nth = Tx * Ty;
  // Step 1: augmented subdomain into both containers (App. A :549-556)
  for (int q = tid; q < L * (Ty + 2); q += nth) {
    const int a = q % L, b = q / L;          // a: 0..Tx+1, b: 0..Ty+1 (halo included)
    const long long gi = i0 + a, gj = j0 + b; // padded coordinates (ring at 0)
    T v = T(0);
    if (!zero_x && gi <= nx + 1 && gj <= ny + 1) v = xin[gj * pitch + (COL0 - 1) + gi];
    // multigrid: fused coarse-grid correction of the interior points (reading c24)
    if (ecor && gi >= 1 && gi <= nx && gj >= 1 && gj <= ny) v = add_t(v, mg_interp(ecor, ep, gi, gj));
    A[q] = v;
    B[q] = v;
  }
  const int a = threadIdx.x, b = threadIdx.y;
  const bool active = a < w && b < hgt;
  const bool owned = a >= ox0 && a <= ox1 && b >= oy0 && b <= oy1;
  if (active) rhs[b * Tx + a] = h2f[(j0 + b) * fpitch + i0 + a];
  __syncthreads();
  // fused residual of the snapshot
  double s2 = 0.0;
  const int c = (b + 1) * L + (a + 1);
  const T ww = (T)wt.w, we = (T)wt.e, ws = (T)wt.s, wn = (T)wt.n;
  if (owned) {
    const double s =
        GEN ? gres2((double)ww, (double)we, (double)ws, (double)wn, (double)A[c], (double)A[c - 1],
                    (double)A[c + 1], (double)A[c - L], (double)A[c + L], (double)rhs[b * Tx + a])
            : res2((double)A[c], (double)A[c - 1], (double)A[c + 1], (double)A[c - L],
                   (double)A[c + L], (double)(T(4) * rhs[b * Tx + a]));
    s2 = s * s;
  }
  s2 = warp_sum(s2);
  if ((tid & 31) == 0) wsum[tid >> 5] = s2;
  __syncthreads();
  if (tid == 0) {
    double acc = 0.0;
    for (int q = 0; q < (nth + 31) / 32; ++q) acc += wsum[q];
    part[t] = acc;
  }
  // Step 2: k sub-iterations, ping-pong between the containers, halo frozen
  const T q4 = active ? rhs[b * Tx + a] : T(0);
  T* cur = A;
  T* nxt = B;
  for (int s = 0; s < kk; ++s) {
    if (active) {
      T u = GEN ? gupd2(ww, we, ws, wn, cur[c - 1], cur[c + 1], cur[c - L], cur[c + L], q4)
                : upd2(cur[c - 1], cur[c + 1], cur[c - L], cur[c + L], q4);
      if constexpr (SK == 2) u = damp((T)wt.om, cur[c], u);  // multigrid smoother (c24)
      nxt[c] = u;
    }
    __syncthreads();
    T* tmp = cur; cur = nxt; nxt = tmp;
  }
  // Step 3: interior back to global (the next iterate)
  if (kk > 0 && owned) {
    xout[(j0 + b + 1) * pitch + COL0 + i0 + a] = cur[c];
    // peer transport: the slab's first / last interior row also into the neighbour's ghost row
    if (peer_lo && j0 + b == 0) { peer_lo[i0 + a] = cur[c]; __threadfence_system(); }
    if (peer_hi && j0 + b == ny - 1) { peer_hi[i0 + a] = cur[c]; __threadfence_system(); }
  }
}

// =============================================================================
// CLASSIC2D — one Jacobi sweep over the grid, HBM-bound (24 B/cell f64):
// a CTA of 128 threads covers 256 columns x CLASSIC2D_ROWS rows, each lane two adjacent columns
// with 128-bit loads/stores; W/E neighbours by warp shuffle, N/S from the rows held in
// registers.  Fused residual of the snapshot, one partial per WARP (no CTA barrier).
// =============================================================================
template <typename T, bool GEN>
__global__ void __launch_bounds__(128)
classic2d_kernel(const T* __restrict__ xin, T* __restrict__ xout, const T* __restrict__ qarr,
                 long long pitch, long long fpitch, int nx, int ny, int ncb,
                 double* __restrict__ part, const Ctrl* __restrict__ ctrl, long long max_cycles,
                 Wt2 wt) {
  if (ctrl->done) return;
  const bool write = ctrl->c < max_cycles;
  constexpr int COL0 = 16 / sizeof(T);
  constexpr int R = CLASSIC2D_ROWS;
  using V2 = typename VecOf<T>::v2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long cb = blockIdx.x % ncb, rb = blockIdx.x / ncb;
  const long long i = cb * CLASSIC2D_COLS + 2 * threadIdx.x;  // first of my two columns (0-based)
  const long long j0 = rb * R;                                  // first interior row (0-based)
  const bool v0 = i < nx, v1 = i + 1 < nx;          // my columns are interior
  const bool l0 = i <= nx, l1 = i + 1 <= nx;        // ... or interior / east ring (loadable)
  T x0[R + 2], x1[R + 2];
  T f0[R], f1[R];
#pragma unroll
  for (int r = 0; r < R + 2; ++r) {            // padded rows j0 .. j0+R+1
    const long long pj = j0 + r;
    x0[r] = x1[r] = T(0);
    if (pj <= ny + 1) {
      const T* p = xin + pj * pitch + COL0 + i;
      if (l1) {
        const V2 v = *reinterpret_cast<const V2*>(p);
        x0[r] = v.x;
        x1[r] = v.y;
      } else if (l0) {
        x0[r] = p[0];
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const long long j = j0 + r;
    f0[r] = f1[r] = T(0);
    if (j < ny && v0) {
      const T* p = qarr + j * fpitch + i;
      if (v1) {
        const V2 v = *reinterpret_cast<const V2*>(p);
        f0[r] = v.x;
        f1[r] = v.y;
      } else {
        f0[r] = p[0];
      }
    }
  }
  const T ww = (T)wt.w, we = (T)wt.e, ws = (T)wt.s, wn = (T)wt.n;
  auto res = [&](T xc, T W, T E, T S, T N, T q) -> double {
    return GEN ? gres2((double)ww, (double)we, (double)ws, (double)wn, (double)xc, (double)W,
                       (double)E, (double)S, (double)N, (double)q)
               : res2((double)xc, (double)W, (double)E, (double)S, (double)N, (double)(T(4) * q));
  };
  auto upd = [&](T W, T E, T S, T N, T q) -> T {
    if constexpr (GEN) return gupd2(ww, we, ws, wn, W, E, S, N, q);
    else return upd2(W, E, S, N, q);
  };
  double acc = 0.0;
#pragma unroll
  for (int r = 1; r <= R; ++r) {
    const long long j = j0 + r - 1;
    T w = __shfl_up_sync(FULL, x1[r], 1);
    T e = __shfl_down_sync(FULL, x0[r], 1);
    if (lane == 0 && j < ny && v0) w = xin[(j + 1) * pitch + COL0 + i - 1];
    if (lane == 31 && j < ny && v1) e = xin[(j + 1) * pitch + COL0 + i + 2];
    if (j < ny) {
      T n0 = T(0), n1 = T(0);
      if (v0) {
        const double s = res(x0[r], w, x1[r], x0[r - 1], x0[r + 1], f0[r - 1]);
        acc = __fma_rn(s, s, acc);
        n0 = upd(w, x1[r], x0[r - 1], x0[r + 1], f0[r - 1]);
      }
      if (v1) {
        const double s = res(x1[r], x0[r], e, x1[r - 1], x1[r + 1], f1[r - 1]);
        acc = __fma_rn(s, s, acc);
        n1 = upd(x0[r], e, x1[r - 1], x1[r + 1], f1[r - 1]);
      }
      if (write) {
        T* dst = xout + (j + 1) * pitch + COL0 + i;
        if (v1) *reinterpret_cast<V2*>(dst) = V2{n0, n1};
        else if (v0) dst[0] = n0;
      }
    }
  }
  acc = warp_sum(acc);
  if (lane == 0) part[(rb * ncb + cb) * 4 + warp] = acc;
}

template <typename T, int SK>
cudaError_t launch_2d_t(const Geom& g, const CycleArgs& a, int grid_hint, cudaStream_t st) {
  const Wt2 wt{g.wt[0], g.wt[1], g.wt[2], g.wt[3], g.omega};
  const size_t smem_paper = sizeof(T) * (2 * size_t(g.tx + 2) * (g.ty + 2) + size_t(g.tx) * g.ty);
  if (g.kernel_kind == K_REG2D) {
    // o = 0: the full 32x32 tiles here, ragged edge tiles by smem2d in edge mode;
    // o > 0: every block is a full 32x32 tile (the last one shifted), owned-point stores.
    const bool ovl = g.ox || g.oy;
    const long long ntx_full = ovl ? g.ntx : g.nx / 32, nty_full = ovl ? g.nty : g.ny / 32;
    const bool subset = a.nty_run >= 0;  // a subset of the tile rows (no edge tiles, checked below)
    if (subset && (ovl || g.nx % 32 || g.ny % 32 || a.ty0 + (long long)(a.nty_run - 1) * a.tys >= nty_full))
      return cudaErrorInvalidValue;
    const long long nfull = ntx_full * (subset ? a.nty_run : nty_full);
    if (nfull > 0) {
      auto go = [&](auto cfg, auto mask, auto cor) {
        using C = decltype(cfg);
        long long ctas = (nfull + C::WARPS - 1) / C::WARPS;
        if (ctas > grid_hint) ctas = grid_hint;
        reg2d_kernel<T, C, decltype(mask)::value, SK, decltype(cor)::value>
            <<<(unsigned)ctas, C::WARPS * 32, C::SMEM, st>>>(
                *a.tm_in, *a.tm_f, *a.tm_out, (T*)a.xout, g.pitch, g.ax, g.ay, (int)ntx_full, nfull,
                (int)g.ntx, a.part, a.ctrl, g.k, a.max_cycles, wt, a.tm_cor ? *a.tm_cor : *a.tm_in,
                (T*)a.peer_lo, (T*)a.peer_hi, subset ? a.ty0 : 0, subset ? a.tys : 1,
                (!subset && tile_strip() > 0 && ntx_full % tile_strip() == 0) ? tile_strip() : 0);
      };
      using X0 = std::integral_constant<int, 0>;
      using X1 = std::integral_constant<int, 1>;
      using X2 = std::integral_constant<int, 2>;
      if (a.cor_e || a.zero_x) {  // multigrid: fused correction / zero start (o = 0)
        if (ovl || (a.cor_e && !a.tm_cor)) return cudaErrorInvalidValue;
        if constexpr (SK == 2) {
          if (a.cor_e) go(R2<T>{}, std::false_type{}, X1{});
          else go(R2<T>{}, std::false_type{}, X2{});
        } else if constexpr (SK == 0) {
          if (a.cor_e) return cudaErrorInvalidValue;
          go(R2<T>{}, std::false_type{}, X2{});
        } else {
          return cudaErrorInvalidValue;
        }
      } else if (ovl) {
        go(R2<T>{}, std::true_type{}, X0{});
      } else {
        go(R2<T>{}, std::false_type{}, X0{});
      }
    }
    const long long nedge = subset ? 0 : g.ntiles - nfull;
    if (nedge > 0)
      smem2d_kernel<T, SK><<<(unsigned)nedge, dim3(32, 32), smem_paper, st>>>(
          (const T*)a.xin, (T*)a.xout, (const T*)a.h2f, g.pitch, g.fpitch, (int)g.nx, (int)g.ny,
          g.ax, g.ay, 1, a.part, a.ctrl, g.k, a.max_cycles, wt, (const T*)a.cor_e, a.cor_pitch,
          (T*)a.peer_lo, (T*)a.peer_hi, (int)a.zero_x);
  } else if (g.kernel_kind == K_SMEM2D) {
    smem2d_kernel<T, SK><<<(unsigned)g.ntiles, dim3(g.tx, g.ty), smem_paper, st>>>(
        (const T*)a.xin, (T*)a.xout, (const T*)a.h2f, g.pitch, g.fpitch, (int)g.nx, (int)g.ny,
        g.ax, g.ay, 0, a.part, a.ctrl, g.k, a.max_cycles, wt, (const T*)a.cor_e, a.cor_pitch,
        (T*)a.peer_lo, (T*)a.peer_hi, (int)a.zero_x);
  } else {
    classic2d_kernel<T, SK == 1><<<(unsigned)(g.ntx * g.nty), 128, 0, st>>>(
        (const T*)a.xin, (T*)a.xout, (const T*)a.h2f, g.pitch, g.fpitch, (int)g.nx, (int)g.ny,
        (int)g.ntx, a.part, a.ctrl, a.max_cycles, wt);
  }
  return cudaGetLastError();
}

}  // namespace


template <typename T, typename C, int SK>
cudaError_t cfg2() {
  cudaError_t e = cudaFuncSetAttribute(reg2d_kernel<T, C, false, SK>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(reg2d_kernel<T, C, true, SK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)C::SMEM);
  if (e != cudaSuccess) return e;
  if constexpr (SK == 2) {
    e = cudaFuncSetAttribute(reg2d_kernel<T, C, false, SK, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)C::SMEM);
    if (e != cudaSuccess) return e;
  }
  if constexpr (SK == 0 || SK == 2) {
    e = cudaFuncSetAttribute(reg2d_kernel<T, C, false, SK, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)C::SMEM);
    if (e != cudaSuccess) return e;
  }
  return cudaFuncSetAttribute(smem2d_kernel<T, SK>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

cudaError_t configure_2d() {
  cudaError_t e;
  if ((e = cfg2<double, R2<double>, 0>()) != cudaSuccess) return e;
  if ((e = cfg2<float, R2<float>, 0>()) != cudaSuccess) return e;
  if ((e = cfg2<double, R2<double>, 1>()) != cudaSuccess) return e;
  if ((e = cfg2<float, R2<float>, 1>()) != cudaSuccess) return e;
  if ((e = cfg2<double, R2<double>, 2>()) != cudaSuccess) return e;
  return cfg2<float, R2<float>, 2>();
}

// The resident solve (res2d_kernel), one cooperative launch; k overrides g.k (classic: 1).
cudaError_t launch_resident_2d(const Geom& g, void* X0, void* X1, const void* Q, double* part, Ctrl* ctrl,
                               double* hist, long long hist_cap, double tol, int tol_mode, double ref_residual,
                               long long max_cycles, int k, unsigned int* bar, cudaStream_t st) {
  int ntx = (int)(g.nx / 32), nty = (int)(g.ny / 32);
  Wt2 wt{g.wt[0], g.wt[1], g.wt[2], g.wt[3], g.omega};
  long long pitch = g.pitch, fpitch = g.fpitch;
  double rdiv = g.rdiv;
  void* args[] = {&X0, &X1, &Q, &pitch, &fpitch, &ntx, &nty, &part, &ctrl, &hist, &hist_cap, &rdiv, &tol,
                  &tol_mode, &ref_residual, &max_cycles, &k, &wt, &bar};
  const dim3 grid((unsigned)((ntx * nty + 7) / 8)), block(256);
  const void* fn;
  if (g.dtype == HJ_F64) fn = g.gen ? (const void*)res2d_kernel<double, 1> : (const void*)res2d_kernel<double, 0>;
  else fn = g.gen ? (const void*)res2d_kernel<float, 1> : (const void*)res2d_kernel<float, 0>;
  return cudaLaunchCooperativeKernel(fn, grid, block, args, 0, st);
}

cudaError_t launch_cycle_2d(const Geom& g, const CycleArgs& a, int grid_hint, cudaStream_t st) {
  if (g.kernel_kind == K_REGT) return launch_regt(g, a, grid_hint, st);
  if (g.gen)
    return g.dtype == HJ_F64 ? launch_2d_t<double, 1>(g, a, grid_hint, st)
                             : launch_2d_t<float, 1>(g, a, grid_hint, st);
  if (g.omega != 1.0)  // damped sub-iterations: the multigrid smoother (reading c24)
    return g.dtype == HJ_F64 ? launch_2d_t<double, 2>(g, a, grid_hint, st)
                             : launch_2d_t<float, 2>(g, a, grid_hint, st);
  return g.dtype == HJ_F64 ? launch_2d_t<double, 0>(g, a, grid_hint, st)
                           : launch_2d_t<float, 0>(g, a, grid_hint, st);
}

}  // namespace hj
