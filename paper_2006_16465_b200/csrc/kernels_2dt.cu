// 2D hierarchical cycle for tile shapes other than 32x32 (BASELINE config 5's tile sweep):
// REGT — the register design of kernels_2d.cu (REG2D) generalised.  PAPER.md:380-387 (§4.1): every
// Tx x Ty subdomain with its one-cell halo is copied on chip, k Jacobi sub-iterations run with the
// halo frozen, the interior is written back; the tile shape is the method's parameter
// (PAPER.md:382, the shared-memory formula :389; 32x32 there only because of Volta's 48 KB, :425).
//
// The unit of on-chip storage stays a 32x32 BLOCK per warp (lane = 8 rows x 4 columns in
// registers, TMA-staged like REG2D):
//  * small tiles (Tx, Ty <= 32; 16x16, 32x16, 16x32): one block holds (32/Tx) x (32/Ty) method
//    tiles; lanes on a tile edge inside the block take the tile's frozen halo (snapshot values of
//    the neighbouring tile, from the TMA box) instead of the neighbouring lane's value — the same
//    selects as REG2D, so the same instruction count per update; the residual partial of each tile
//    is a segmented warp reduction.
//  * large tiles (Tx, Ty >= 32; 64x32, 32x64, 64x64, 128x32): one tile = a group of
//    (Tx/32) x (Ty/32) warps of one CTA, each holding one block; after every sub-iteration the
//    warps of a tile write their block-edge rows / columns into the neighbouring warps' halo
//    buffers (double-buffered by sub-iteration parity, predicated stores) and meet at a named
//    barrier (exchange mode 2, the default; the half-sub-iteration mbarrier scheme, modes 0 / 3, is
//    kept for A/B: 5-12% slower at k = 4 and 16, profiles/r02_regt_xch.md); tile edges keep the
//    frozen halo.  The iterate is exactly the method's: every cell sees the previous
//    sub-iteration's values of its in-tile neighbours and the frozen snapshot outside the tile.
// Poisson, o = 0, nx and ny multiples of max(Tx, 32) / max(Ty, 32) (engine.cu choose_kernel);
// everything else runs on smem2d_kernel.
#include <cstdlib>

#include "hj_internal.cuh"
#include "reg_tile.cuh"

namespace hj {

namespace {

using namespace rt;

template <typename T, int TX, int TY>
struct RT {
  using C = R2<T>;  // slot layout (x box with halo, q box) shared with REG2D
  static constexpr bool BIG = TX >= 32 && TY >= 32;
  static_assert(BIG || (TX <= 32 && TY <= 32 && TX >= 8 && TY >= 16), "tile shape");
  static constexpr int SBX = BIG ? TX / 32 : 1, SBY = BIG ? TY / 32 : 1;   // blocks per tile
  static constexpr int WPT = SBX * SBY;                                    // warps per tile
  static constexpr int TXL = BIG ? 8 : TX / 4, TYL = BIG ? 4 : TY / 8;     // lanes per tile in a block
  static constexpr int TPX = BIG ? 1 : 32 / TX, TPY = BIG ? 1 : 32 / TY;   // tiles per block
  // halo buffer (per parity): HX = 8 lane-columns x 32 rows (the W or E column each lane-column
  // reads), HY = 4 lane-rows x 32 columns (the S or N row each lane-row reads)
  static constexpr int HX = 8 * 32, HY = 4 * 32;
  static constexpr int NPAR = WPT > 1 ? 2 : 1;
  static constexpr int HBYTES = ((HX + HY) * (int)sizeof(T) * NPAR + 127) / 128 * 128;
  static constexpr int WSMEM = C::XSLOT + C::FBYTES + HBYTES;
  static constexpr int WARPS = sizeof(T) == 8 ? 8 : (WPT == 1 ? 12 : 8);
  static_assert(WARPS % WPT == 0, "warps per CTA");
  static constexpr int GROUPS = WARPS / WPT;
  static constexpr int BARS = 512;  // TMA mbarriers [0, 16), halo mbarriers 16 + 4 * warp + 2 * parity + half
  static constexpr size_t SMEM = 128 + BARS + size_t(WARPS) * WSMEM;
  static_assert(SMEM <= 232448, "shared memory budget");
};

__device__ __forceinline__ void group_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Block-edge exchange of a tile spread over a warp group, one half-sweep at a time (Tile2::sweep_h):
// after computing rows 3,4,2,5 (half A) of sub-iteration s a warp stores their block-edge values into
// the W / E neighbours' halo buffers of parity (s+1)&1 and arrives on their half-A mbarrier; after
// rows 1,6,0,7 (half B) the same for those rows plus its first / last row for the S / N neighbours,
// arriving on every neighbour's half-B mbarrier.  A warp waits on its own half-A / half-B mbarrier
// just before the corresponding half of sub-iteration s+1, so neighbours are only ever half a
// sub-iteration apart — no group-wide barrier per sub-iteration.  Buffer reuse is safe: the
// parity-p half-A (half-B) buffer is rewritten only after its reader's half-A (half-B) arrival of
// the sub-iteration that read it.
__device__ __forceinline__ void sts2(uint32_t a, double x, double y) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ void sts2(uint32_t a, float x, float y) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(x), "f"(y) : "memory");
}
// predicated (branch-free) form: lanes with p == 0 issue nothing
__device__ __forceinline__ void sts2p(bool p, uint32_t a, double x, double y) {
  asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %3, 0;\n@q st.shared.v2.f64 [%0], {%1, %2};\n}" ::"r"(a), "d"(x),
               "d"(y), "r"((int)p)
               : "memory");
}
__device__ __forceinline__ void sts2p(bool p, uint32_t a, float x, float y) {
  asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %3, 0;\n@q st.shared.v2.f32 [%0], {%1, %2};\n}" ::"r"(a), "f"(x),
               "f"(y), "r"((int)p)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_u32(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
// All addresses are 32-bit shared-window addresses derived from the warp index (few live registers):
//   halo buffer of warp w, parity p:  hb0 + w * WSMEM + p * (HX + HY) * sizeof(T)
//   halo mbarrier (w, p, half):       mb0 + 8 * (4 w + 2 p + half)
// XCH (exchange mode of the large tiles): 0 — the mbarrier scheme above, sends as divergent branches;
// 2 — no mbarriers: the sends are predicated stores and the tile's warps meet at ONE named barrier
// (bar.sync, hardware, no polling loop) after every sub-iteration (the parity buffers make one
// barrier per sub-iteration enough: a buffer read in sub-iteration s is rewritten in s + 1 by a
// neighbour that has passed the barrier ending s); 3 — the mbarrier scheme with predicated sends.
template <typename T, typename R, int XCH = 0>
struct Exch {
  uint32_t hb0, mb0;      // shared addresses: halo buffer of warp 0, halo mbarrier (0, 0, 0)
  int warp, lx, ly, lane;
  int pw;                 // parity written this sub-iteration
  uint32_t wa, wb, wph;   // my half-A / half-B mbarriers of the parity read, their phase
  bool do_wait, do_send, hW, hE, hS, hN;
  __device__ __forceinline__ uint32_t halo(int w) const {
    return hb0 + (uint32_t)(w * R::WSMEM) + (uint32_t)(pw * (R::HX + R::HY) * (int)sizeof(T));
  }
  __device__ __forceinline__ uint32_t mbar(int w, int half) const { return mb0 + 8u * (4 * w + 2 * pw + half); }
  __device__ __forceinline__ void wait_a() const {
    if constexpr (XCH != 2)
      if (do_wait && (hW || hE)) mbar_wait_u32(wa, wph);
  }
  __device__ __forceinline__ void wait_b() const {
    if constexpr (XCH != 2)
      if (do_wait) mbar_wait_u32(wb, wph);
  }
  template <typename TL>
  __device__ __forceinline__ void send_a(const TL& t) const {
    if (!do_send) return;
    if constexpr (XCH != 0) {
      constexpr uint32_t E = sizeof(T);
      const bool pw_ = hW && lx == 0, pe_ = hE && lx == 7;
      const uint32_t qw = halo(warp - 1) + (7 * 32 + 8 * ly) * E, qe = halo(warp + 1) + (8 * ly) * E;
      sts2p(pw_, qw + 2 * E, t.x[2][0], t.x[3][0]);
      sts2p(pw_, qw + 4 * E, t.x[4][0], t.x[5][0]);
      sts2p(pe_, qe + 2 * E, t.x[2][3], t.x[3][3]);
      sts2p(pe_, qe + 4 * E, t.x[4][3], t.x[5][3]);
      if constexpr (XCH == 3) {
        __syncwarp();
        if (lane == 0) {
          if (hW) mbar_arrive_u32(mbar(warp - 1, 0));
          if (hE) mbar_arrive_u32(mbar(warp + 1, 0));
        }
      }
      return;
    }
    constexpr uint32_t E = sizeof(T);
    if (hW && lx == 0) {  // my column 0 -> W neighbour's E column (its lane-column 7)
      const uint32_t q = halo(warp - 1) + (7 * 32 + 8 * ly) * E;
      sts2(q + 2 * E, t.x[2][0], t.x[3][0]);
      sts2(q + 4 * E, t.x[4][0], t.x[5][0]);
    }
    if (hE && lx == 7) {  // my column 31 -> E neighbour's W column (its lane-column 0)
      const uint32_t q = halo(warp + 1) + (8 * ly) * E;
      sts2(q + 2 * E, t.x[2][3], t.x[3][3]);
      sts2(q + 4 * E, t.x[4][3], t.x[5][3]);
    }
    __syncwarp();
    if (lane == 0) {
      if (hW) mbar_arrive_u32(mbar(warp - 1, 0));
      if (hE) mbar_arrive_u32(mbar(warp + 1, 0));
    }
  }
  template <typename TL>
  __device__ __forceinline__ void send_b(const TL& t) const {
    if (!do_send) return;
    if constexpr (XCH != 0) {
      constexpr uint32_t E = sizeof(T);
      const bool pw_ = hW && lx == 0, pe_ = hE && lx == 7, ps_ = hS && ly == 0, pn_ = hN && ly == 3;
      const uint32_t qw = halo(warp - 1) + (7 * 32 + 8 * ly) * E, qe = halo(warp + 1) + (8 * ly) * E;
      const uint32_t qs = halo(warp - R::SBX) + (R::HX + 3 * 32 + 4 * lx) * E;
      const uint32_t qn = halo(warp + R::SBX) + (R::HX + 4 * lx) * E;
      sts2p(pw_, qw, t.x[0][0], t.x[1][0]);
      sts2p(pw_, qw + 6 * E, t.x[6][0], t.x[7][0]);
      sts2p(pe_, qe, t.x[0][3], t.x[1][3]);
      sts2p(pe_, qe + 6 * E, t.x[6][3], t.x[7][3]);
      sts2p(ps_, qs, t.x[0][0], t.x[0][1]);
      sts2p(ps_, qs + 2 * E, t.x[0][2], t.x[0][3]);
      sts2p(pn_, qn, t.x[7][0], t.x[7][1]);
      sts2p(pn_, qn + 2 * E, t.x[7][2], t.x[7][3]);
      if constexpr (XCH == 3) {
        __syncwarp();
        if (lane == 0) {
          if (hW) mbar_arrive_u32(mbar(warp - 1, 1));
          if (hE) mbar_arrive_u32(mbar(warp + 1, 1));
          if (hS) mbar_arrive_u32(mbar(warp - R::SBX, 1));
          if (hN) mbar_arrive_u32(mbar(warp + R::SBX, 1));
        }
      }
      return;
    }
    constexpr uint32_t E = sizeof(T);
    if (hW && lx == 0) {
      const uint32_t q = halo(warp - 1) + (7 * 32 + 8 * ly) * E;
      sts2(q, t.x[0][0], t.x[1][0]);
      sts2(q + 6 * E, t.x[6][0], t.x[7][0]);
    }
    if (hE && lx == 7) {
      const uint32_t q = halo(warp + 1) + (8 * ly) * E;
      sts2(q, t.x[0][3], t.x[1][3]);
      sts2(q + 6 * E, t.x[6][3], t.x[7][3]);
    }
    if (hS && ly == 0) {  // my row 0 -> S neighbour's N row (its lane-row 3)
      const uint32_t q = halo(warp - R::SBX) + (R::HX + 3 * 32 + 4 * lx) * E;
      sts2(q, t.x[0][0], t.x[0][1]);
      sts2(q + 2 * E, t.x[0][2], t.x[0][3]);
    }
    if (hN && ly == 3) {  // my row 31 -> N neighbour's S row (its lane-row 0)
      const uint32_t q = halo(warp + R::SBX) + (R::HX + 4 * lx) * E;
      sts2(q, t.x[7][0], t.x[7][1]);
      sts2(q + 2 * E, t.x[7][2], t.x[7][3]);
    }
    __syncwarp();
    if (lane == 0) {
      if (hW) mbar_arrive_u32(mbar(warp - 1, 1));
      if (hE) mbar_arrive_u32(mbar(warp + 1, 1));
      if (hS) mbar_arrive_u32(mbar(warp - R::SBX, 1));
      if (hN) mbar_arrive_u32(mbar(warp + R::SBX, 1));
    }
  }
};

template <typename T, int TX, int TY, int XCH = 0>
__global__ void __launch_bounds__(RT<T, TX, TY>::WARPS * 32, 1)
regt_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmF,
            T* __restrict__ xout, long long pitch, long long nunits, int units_x, double* __restrict__ part,
            long long ppr, const Ctrl* __restrict__ ctrl, int k, long long max_cycles, int sweep_bar) {
  using R = RT<T, TX, TY>;
  using C = typename R::C;
  using V2 = typename VecOf<T>::v2;
  if (ctrl->done) return;
  const int kk = (ctrl->c >= max_cycles) ? 0 : k;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, lx = lane & 7, ly = lane >> 3;
  const int grp = warp / R::WPT, wg = warp % R::WPT, sbx = wg % R::SBX, sby = wg / R::SBX;
  uint64_t* bar = reinterpret_cast<uint64_t*>(base) + warp;
  auto slot_of = [&](int w) { return base + R::BARS + size_t(w) * R::WSMEM; };
  unsigned char* slot = slot_of(warp);
  const T* sx = reinterpret_cast<const T*>(slot);
  const T* sf = reinterpret_cast<const T*>(slot + C::XSLOT);
  T* hb = reinterpret_cast<T*>(slot + C::XSLOT + C::FBYTES);          // [par][HX + HY]
  auto halo_of = [&](int w) { return reinterpret_cast<T*>(slot_of(w) + C::XSLOT + C::FBYTES); };
  const long long gg = (long long)blockIdx.x * R::GROUPS + grp;
  const long long ng = (long long)gridDim.x * R::GROUPS;
  // internal block edges of my tile (neighbouring warps of the group) and my halo mbarriers
  const bool hW = sbx > 0, hE = sbx < R::SBX - 1, hS = sby > 0, hN = sby < R::SBY - 1;
  const int nA = hW + hE, nB = nA + hS + hN;
  auto hmb = [&](int w, int par, int half) { return reinterpret_cast<uint64_t*>(base) + 16 + 4 * w + 2 * par + half; };
  if constexpr (R::WPT > 1) {
    if (lane == 0) {
      for (int p = 0; p < 2; ++p) {
        mbar_init(hmb(warp, p, 0), nA > 0 ? nA : 1);
        mbar_init(hmb(warp, p, 1), nB);
      }
      fence_mbar_init();
    }
    __syncthreads();  // every halo mbarrier is initialised before any neighbour arrives on it
  }
  if (gg >= nunits) return;  // the whole group leaves together (named barriers stay balanced)
  // unit u -> this warp's 32x32 block origin (0-based interior coordinates)
  auto origin = [&](long long u, int& x0, int& y0) {
    const int ux = (int)(u % units_x), uy = (int)(u / units_x);
    x0 = R::BIG ? ux * TX + 32 * sbx : 32 * ux;
    y0 = R::BIG ? uy * TY + 32 * sby : 32 * uy;
  };
  auto issue = [&](long long u) {
    int x0, y0;
    origin(u, x0, y0);
    mbar_arrive_expect_tx(bar, C::XBYTES + C::FBYTES);
    tma_load_2d(slot, &tmX, x0, y0, bar);
    tma_load_2d(slot + C::XSLOT, &tmF, x0, y0, bar);
  };
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    prefetch_tensormap(&tmX);
    prefetch_tensormap(&tmF);
    issue(gg);
  }
  __syncwarp();
  using TL = Tile2<T, false, 0, R::TXL, R::TYL>;
  // halo pointers: lane-column lx reads column (W edge ? 4lx-1 : 4lx+4) of its rows, lane-row ly
  // reads row (S edge ? 8ly-1 : 8ly+8) of its columns (block-local, -1 / 32 = the TMA box's ring)
  const int hxo = lx * 32 + 8 * ly, hyo = R::HX + ly * 32 + 4 * lx;
  const int bar_id = 1 + grp, bar_n = 32 * R::WPT;
  uint32_t ph = 0u;  // bit p: phase of my parity-p halo mbarriers
  int it = 0;
  for (long long u = gg; u < nunits; u += ng, ++it) {
    mbar_wait(bar, it & 1);
    int x0, y0;
    origin(u, x0, y0);
    TL tl;
#pragma unroll
    for (int i = 0; i < 8; ++i) {  // 128-bit shared loads
      const int r = 8 * ly + i;
      const V2* rowx = reinterpret_cast<const V2*>(sx + (r + 1) * C::BW + C::COL0 + 4 * lx);
      const V2* rowf = reinterpret_cast<const V2*>(sf + r * 32 + 4 * lx);
      const V2 a = rowx[0], b = rowx[1], fa = rowf[0], fb = rowf[1];
      tl.x[i][0] = a.x; tl.x[i][1] = a.y; tl.x[i][2] = b.x; tl.x[i][3] = b.y;
      tl.q[i][0] = fa.x; tl.q[i][1] = fa.y; tl.q[i][2] = fb.x; tl.q[i][3] = fb.y;
    }
    // frozen halo of the snapshot, for every lane-column / lane-row (both parities for tile groups:
    // the block edges inside a tile are overwritten by the neighbours after each sub-iteration)
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int col = TL::eW(c) ? 4 * c - 1 : 4 * c + 4;
      const T v = sx[(lane + 1) * C::BW + C::COL0 + col];
#pragma unroll
      for (int p = 0; p < R::NPAR; ++p) hb[p * (R::HX + R::HY) + c * 32 + lane] = v;
    }
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int row = TL::eS(l) ? 8 * l - 1 : 8 * l + 8;
      const T v = sx[(row + 1) * C::BW + C::COL0 + lane];
#pragma unroll
      for (int p = 0; p < R::NPAR; ++p) hb[p * (R::HX + R::HY) + R::HX + l * 32 + lane] = v;
    }
    tl.hxp = hb + hxo;
    tl.hyp = hb + hyo;
    tl.own = 0xffffffffu;
    __syncwarp();
    if (lane == 0 && u + ng < nunits) {  // the slot is in registers / the halo buffer: refill
      fence_proxy_async();
      issue(u + ng);
    }
    if constexpr (R::WPT > 1) group_bar(bar_id, bar_n);  // every warp of the tile filled its halo
    // fused residual of the snapshot folded into the first sub-iteration (f64); separate pass (f32)
    constexpr bool FOLD = sizeof(T) == 8;
    double acc = 0.0;
    if (!FOLD || kk == 0) acc = tl.residual(lx, ly);
    if constexpr (R::WPT == 1) {
      int s = 0;
      if constexpr (FOLD) {
        if (kk > 0) {
          double a4[4] = {0.0, 0.0, 0.0, 0.0};
          tl.template sweep_mo<true>(lx, ly, a4);
          acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
          s = 1;
        }
      }
#pragma unroll 1
      for (; s < kk; ++s) tl.template sweep_mo<false>(lx, ly);
    } else {
      Exch<T, R, XCH> ex;
      ex.hb0 = smem_u32(halo_of(0));
      ex.mb0 = smem_u32(hmb(0, 0, 0));
      ex.warp = warp; ex.lx = lx; ex.ly = ly; ex.lane = lane;
      ex.hW = hW; ex.hE = hE; ex.hS = hS; ex.hN = hN;
      auto setup = [&](int s) {  // sub-iteration s reads parity s&1 and writes parity (s+1)&1
        const int pr = s & 1;
        ex.pw = pr ^ 1;
        ex.do_wait = s > 0;
        ex.do_send = s + 1 < kk;
        ex.wa = ex.mb0 + 8u * (4 * warp + 2 * pr);
        ex.wb = ex.wa + 8u;
        ex.wph = (ph >> pr) & 1u;
        tl.hxp = hb + pr * (R::HX + R::HY) + hxo;
        tl.hyp = hb + pr * (R::HX + R::HY) + hyo;
      };
      int s = 0;
      if constexpr (FOLD) {
        if (kk > 0) {
          double a4[4] = {0.0, 0.0, 0.0, 0.0};
          setup(0);
          tl.template sweep_h<true>(lx, ly, a4, ex);
          if (XCH == 2 || sweep_bar) group_bar(bar_id, bar_n);
          acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
          s = 1;
        }
      }
#pragma unroll 1
      for (; s < kk; ++s) {
        setup(s);
        tl.template sweep_h<false>(lx, ly, nullptr, ex);
        if (s > 0) ph ^= 1u << (s & 1);  // this parity's mbarriers completed one more phase
        if (XCH == 2 || sweep_bar) group_bar(bar_id, bar_n);
      }
    }
    // residual partials: per tile (small tiles: segmented reduction over the tile's lanes)
    if constexpr (R::BIG) {
      acc = warp_sum(acc);
      if (lane == 0) {
        const long long ux = u % units_x, uy = u / units_x;
        part[uy * ppr + ux * R::WPT + wg] = acc;
      }
    } else {
#pragma unroll
      for (int o = 1; o < R::TXL; o <<= 1) acc += __shfl_xor_sync(FULL, acc, o);
#pragma unroll
      for (int o = 1; o < R::TYL; o <<= 1) acc += __shfl_xor_sync(FULL, acc, 8 * o);
      if (lx % R::TXL == 0 && ly % R::TYL == 0) {
        const long long tx = x0 / TX + lx / R::TXL, ty = y0 / TY + ly / R::TYL;
        part[ty * ppr + tx] = acc;
      }
    }
    if (kk > 0) {  // registers -> the NEXT iterate, 128-bit stores (snapshot semantics)
      T* g = xout + ((long long)y0 + 1) * pitch + C::COL0 + x0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        V2* dst = reinterpret_cast<V2*>(g + (8 * ly + i) * pitch + 4 * lx);
        dst[0] = V2{tl.x[i][0], tl.x[i][1]};
        dst[1] = V2{tl.x[i][2], tl.x[i][3]};
      }
    }
  }
}

// HJ_REGT_SWEEP_BARRIER=1 (diagnostics): a group barrier after every sub-iteration of a large tile, on top
// of the mbarrier exchange — the ordering racecheck models (it does not follow mbarrier arrive / wait
// between warps); same values, slower.
bool regt_sweep_barrier() {
  static const bool on = [] { const char* e = std::getenv("HJ_REGT_SWEEP_BARRIER"); return e && e[0] == '1'; }();
  return on;
}
// HJ_REGT_XCH = 0 / 2 / 3: the large tiles' exchange mode (Exch); default REGT_XCH
constexpr int REGT_XCH = 2;
int regt_xch() {
  static const int m = [] {
    const char* e = std::getenv("HJ_REGT_XCH");
    const int v = e ? std::atoi(e) : REGT_XCH;
    return (v == 2 || v == 3) ? v : 0;
  }();
  return m;
}

template <typename T, int TX, int TY>
cudaError_t launch_t(const Geom& g, const CycleArgs& a, int grid_hint, cudaStream_t st) {
  using R = RT<T, TX, TY>;
  const long long units_x = R::BIG ? g.nx / TX : g.nx / 32;
  const long long nunits = R::BIG ? units_x * (g.ny / TY) : units_x * (g.ny / 32);
  long long ctas = (nunits + R::GROUPS - 1) / R::GROUPS;
  if (ctas > grid_hint) ctas = grid_hint;
  const int xch = R::BIG && !regt_sweep_barrier() ? regt_xch() : 0;
  auto fn = xch == 2 ? regt_kernel<T, TX, TY, (R::BIG ? 2 : 0)>
                     : xch == 3 ? regt_kernel<T, TX, TY, (R::BIG ? 3 : 0)> : regt_kernel<T, TX, TY, 0>;
  fn<<<(unsigned)ctas, R::WARPS * 32, R::SMEM, st>>>(*a.tm_in, *a.tm_f, (T*)a.xout, g.pitch, nunits, (int)units_x,
                                                    a.part, g.parts_per_row, a.ctrl, g.k, a.max_cycles,
                                                    regt_sweep_barrier() ? 1 : 0);
  return cudaGetLastError();
}

template <typename T, int TX, int TY>
cudaError_t cfg_t() {
  constexpr bool BIG = RT<T, TX, TY>::BIG;
  cudaError_t e = cudaFuncSetAttribute(regt_kernel<T, TX, TY, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)RT<T, TX, TY>::SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(regt_kernel<T, TX, TY, (BIG ? 2 : 0)>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)RT<T, TX, TY>::SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(regt_kernel<T, TX, TY, (BIG ? 3 : 0)>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)RT<T, TX, TY>::SMEM);
  return e;
}

template <typename T>
cudaError_t launch_regt_T(const Geom& g, const CycleArgs& a, int grid_hint, cudaStream_t st) {
  const int tx = g.tx, ty = g.ty;
  if (tx == 16 && ty == 16) return launch_t<T, 16, 16>(g, a, grid_hint, st);
  if (tx == 32 && ty == 16) return launch_t<T, 32, 16>(g, a, grid_hint, st);
  if (tx == 16 && ty == 32) return launch_t<T, 16, 32>(g, a, grid_hint, st);
  if (tx == 64 && ty == 32) return launch_t<T, 64, 32>(g, a, grid_hint, st);
  if (tx == 32 && ty == 64) return launch_t<T, 32, 64>(g, a, grid_hint, st);
  if (tx == 64 && ty == 64) return launch_t<T, 64, 64>(g, a, grid_hint, st);
  if (tx == 128 && ty == 32) return launch_t<T, 128, 32>(g, a, grid_hint, st);
  return cudaErrorInvalidValue;
}

template <typename T>
cudaError_t cfg_T() {
  cudaError_t e;
  if ((e = cfg_t<T, 16, 16>()) != cudaSuccess) return e;
  if ((e = cfg_t<T, 32, 16>()) != cudaSuccess) return e;
  if ((e = cfg_t<T, 16, 32>()) != cudaSuccess) return e;
  if ((e = cfg_t<T, 64, 32>()) != cudaSuccess) return e;
  if ((e = cfg_t<T, 32, 64>()) != cudaSuccess) return e;
  if ((e = cfg_t<T, 64, 64>()) != cudaSuccess) return e;
  return cfg_t<T, 128, 32>();
}

}  // namespace

// The tile shapes REGT runs (the rest of engine.cu's choice is in choose_kernel).
bool regt_shape(int tx, int ty) {
  return (tx == 16 && ty == 16) || (tx == 32 && ty == 16) || (tx == 16 && ty == 32) || (tx == 64 && ty == 32) ||
         (tx == 32 && ty == 64) || (tx == 64 && ty == 64) || (tx == 128 && ty == 32);
}
int regt_warps_per_tile(int tx, int ty) { return tx >= 32 && ty >= 32 ? (tx / 32) * (ty / 32) : 1; }

cudaError_t launch_regt(const Geom& g, const CycleArgs& a, int grid_hint, cudaStream_t st) {
  return g.dtype == HJ_F64 ? launch_regt_T<double>(g, a, grid_hint, st) : launch_regt_T<float>(g, a, grid_hint, st);
}

cudaError_t configure_2dt() {
  cudaError_t e = cfg_T<double>();
  return e != cudaSuccess ? e : cfg_T<float>();
}

}  // namespace hj
