// Grid-transfer kernels of the multigrid solver: the hierarchical cycle
// as the smoother of a textbook V-cycle.  PAPER.md:17 (§1: stationary iterations "form the
// backbone of highly effective geometric and algebraic multigrid methods"), :530 (§5: the
// hierarchical solver "has the potential to accelerate multigrid solvers which utilize this
// approach as a smoother").  The paper defines no coarse-grid method; reading c24 fixes
// the operators and their evaluation order, which these kernels follow exactly:
//
//   restriction  coarse point I (ringed) sits on fine point 2I; the fine h^2-scaled residual
//                s = 4q - (4x - ((W+E)+(S+N)))            (2D, in double; q = Q of the level)
//                s = 2q - (2x - (L+R))                    (1D)
//                is full-weighted onto the coarse right-hand side, stored like every Q:
//                2D  Qc = T(0.0625 * ((4 s_C + 2 ((s_W+s_E) + (s_S+s_N))) + ((s_SW+s_SE) + (s_NW+s_NE))))
//                1D  Qc = T(0.5 * (2 s_C + (s_L + s_R)))
//                (= 1/diag * (2h)^2 * R(s / h^2); every factor a power of two), and the coarse
//                iterate's interior is zeroed (the coarse solve starts from 0).
//   correction   x += (bi)linear interpolation of the coarse iterate e (zero ring), in T:
//                on a coarse point e; between two e's T(0.5)*(eW+eE) (or (eS+eN)); between four
//                T(0.25)*((eSW+eSE)+(eNW+eNE)).
//
// Both are HBM-streaming kernels (restriction: read x and q once, 16 B per fine cell in f64, write
// 1/4 of that; correction: read + write x, 16 B per fine cell, plus the coarse iterate, 2 B).
#include <type_traits>

#include "hj_internal.cuh"

namespace hj {

namespace {

// Streaming restriction.  Lane I of the grid owns coarse column I and the fine column pair
// (2I+1, 2I+2) (ringed; one 2-wide vector load of x and of q per fine row, 16-B aligned), and walks
// down a strip of RB coarse rows keeping three fine rows of x and of residuals in registers.  The
// west neighbour x(2I) and the residual s(2I+3) come from the neighbouring lanes by shuffle; the
// warp's edge lanes load / compute them themselves.  HBM: x and q read once per fine cell (plus
// 3 x rows per strip of 2 RB), the coarse q written once.
template <typename T>
struct XRow {
  T w, a, b, e, e2;   // x at ringed columns 2I, 2I+1, 2I+2, 2I+3, 2I+4 of one fine row
  T qa, qb, qc;       // q at 2I+1, 2I+2 (and 2I+3 for the warp's last lane)
};

template <typename T>
__global__ void __launch_bounds__(128, 8)
mg_restrict2d_stream(const T* __restrict__ xf, const T* __restrict__ qf, long long pf, long long fpf,
                     int nx, int ny, T* __restrict__ qc, T* __restrict__ xc, long long pc, long long fpc,
                     int nxc, int nyc, int RB, int write_zero, const Ctrl* __restrict__ ctrl) {
  if (ctrl->done) return;
  using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int COL0 = 16 / sizeof(T);
  const int lane = threadIdx.x & 31;
  const int I = blockIdx.x * blockDim.x + threadIdx.x;  // 0-based coarse column
  const int J0 = blockIdx.y * RB;
  const bool live = I <= nxc;          // my pair (2I+1, 2I+2) lies inside [1, nx+1]
  const bool act = I < nxc;            // I am a coarse point
  const bool last = lane == 31;
  auto load = [&](long long j, XRow<T>& R) {
    R = XRow<T>{T(0), T(0), T(0), T(0), T(0), T(0), T(0), T(0)};
    const T* xr = xf + j * pf + (COL0 - 1);
    if (live) {
      const V2 v = *reinterpret_cast<const V2*>(xr + 2LL * I + 1);
      R.a = v.x;
      R.b = v.y;
      if (j >= 1 && j <= ny) {
        const V2 u = *reinterpret_cast<const V2*>(qf + (j - 1) * fpf + 2LL * I);
        R.qa = u.x;
        R.qb = u.y;
      }
    }
    if (lane == 0 && live) R.w = xr[2LL * I];
    if (last && act) {
      R.e = xr[2LL * I + 3];
      R.e2 = xr[2LL * I + 4];
      if (j >= 1 && j <= ny) R.qc = qf[(j - 1) * fpf + 2LL * I + 2];
    }
  };
  auto resid = [](T q, T xc_, T w, T e, T s, T n) {
    const double h2f = (double)(T(4) * q);
    return __dsub_rn(h2f, __dsub_rn(__dmul_rn(4.0, (double)xc_),
                                    __dadd_rn(__dadd_rn((double)w, (double)e), __dadd_rn((double)s, (double)n))));
  };
  // the lane neighbours' x of a loaded row
  auto nbr = [&](XRow<T>& R) {
    const T w = __shfl_up_sync(FULL, R.b, 1), e = __shfl_down_sync(FULL, R.a, 1);
    if (lane != 0) R.w = w;
    if (!last) R.e = e;
  };
  struct SRow { double a, b, c; };         // residuals at columns 2I+1, 2I+2, 2I+3 of one row
  auto srow = [&](const XRow<T>& S, const XRow<T>& C, const XRow<T>& N) {
    SRow r;
    r.a = resid(C.qa, C.a, C.w, C.b, S.a, N.a);
    r.b = resid(C.qb, C.b, C.a, C.e, S.b, N.b);
    r.c = __shfl_down_sync(FULL, r.a, 1);
    if (last) r.c = act ? resid(C.qc, C.e, C.b, C.e2, S.e, N.e) : 0.0;
    return r;
  };
  // prologue: x rows 2J0, 2J0+1, 2J0+2 and the residual row 2J0+1
  XRow<T> r0, p1, p2, n1, n2;
  load(2LL * J0, r0);
  load(2LL * J0 + 1, p1);
  load(2LL * J0 + 2, p2);
  nbr(r0);
  nbr(p1);
  nbr(p2);
  SRow sp = srow(r0, p1, p2);
  const int mmax = (int)lmin(RB, (long long)nyc - J0);
  for (int m = 0; m < mmax; ++m) {
    // coarse row J needs residual rows 2J+2 and 2J+3: x rows 2J+3 and 2J+4 (both loads in flight)
    const int J = J0 + m;
    load(2LL * J + 3, n1);
    load(2LL * J + 4, n2);
    nbr(n1);
    nbr(n2);
    const SRow sm = srow(p1, p2, n1);
    const SRow sn = srow(p2, n1, n2);
    if (act) {
      const double A = __dmul_rn(4.0, sm.b);
      const double B = __dmul_rn(2.0, __dadd_rn(__dadd_rn(sm.a, sm.c), __dadd_rn(sp.b, sn.b)));
      const double C = __dadd_rn(__dadd_rn(sp.a, sp.c), __dadd_rn(sn.a, sn.c));
      qc[(long long)J * fpc + I] = (T)__dmul_rn(0.0625, __dadd_rn(__dadd_rn(A, B), C));
      if (write_zero) xc[(long long)(J + 1) * pc + COL0 + I] = T(0);
    }
    p1 = n1;
    p2 = n2;
    sp = sn;
  }
}

// Vectorised correction: thread (Ir, Jr) (ringed coarse, 0..nxc x 0..nyc) updates the fine 2x2
// block at ringed (2Ir+1, 2Ir+2) x (2Jr+1, 2Jr+2) from the four coarse values around it, with one
// 2-wide vector load and store per fine row (interior column 2Ir is 16-B aligned in f64, 8-B in f32).
template <typename T>
__global__ void mg_correct2d_vec(const T* xin, T* xout, long long pf, int nx, int ny,
                                 const T* __restrict__ e, long long pc, int nxc, int nyc,
                                 const Ctrl* __restrict__ ctrl) {
  if (ctrl->done) return;
  using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
  constexpr int COL0 = 16 / sizeof(T);
  const int Ir = blockIdx.x * blockDim.x + threadIdx.x;
  const int Jr = blockIdx.y * blockDim.y + threadIdx.y;
  if (Ir > nxc || Jr > nyc) return;
  const T* ep = e + (long long)Jr * pc + (COL0 - 1) + Ir;
  const T sw = ep[0], se = ep[1], nw = ep[pc], ne = ep[pc + 1];
  const bool two = 2 * Ir + 2 <= nx;  // the east point of the pair is interior (not the ring)
  for (int h = 0; h < 2; ++h) {
    const long long j = 2LL * Jr + 1 + h;  // ringed fine row
    if (j > ny) break;
    T v0, v1;
    if (h == 0) {  // odd row: between coarse rows Jr and Jr+1
      v0 = mul_t(T(0.25), add_t(add_t(sw, se), add_t(nw, ne)));
      v1 = mul_t(T(0.5), add_t(se, ne));
    } else {       // even row: on coarse row Jr+1
      v0 = mul_t(T(0.5), add_t(nw, ne));
      v1 = ne;
    }
    const long long o = j * pf + (COL0 - 1) + 2LL * Ir + 1;
    if (two) {
      const V2 xv = *reinterpret_cast<const V2*>(xin + o);
      *reinterpret_cast<V2*>(xout + o) = V2{add_t(xv.x, v0), add_t(xv.y, v1)};
    } else {
      xout[o] = add_t(xin[o], v0);
    }
  }
}

// 1D: rows of the padded arrays are independent problems (the batch of NEXT #2).
template <typename T>
__global__ void mg_restrict1d_kernel(const T* __restrict__ xf, const T* __restrict__ qf, long long pf,
                                     long long fpf, T* __restrict__ qc, T* __restrict__ xc,
                                     long long pc, long long fpc, int nxc, int rows,
                                     const Ctrl* __restrict__ ctrl) {
  if (ctrl->done) return;
  constexpr int COL0 = 16 / sizeof(T);
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (I >= nxc || r >= rows) return;
  const T* x = xf + (long long)r * pf + (COL0 - 1);   // x[i], i ringed
  const T* q = qf + (long long)r * fpf;
  auto s = [&](long long i) {
    const double h2f = (double)(T(2) * q[i - 1]);
    return __dsub_rn(h2f, __dsub_rn(__dmul_rn(2.0, (double)x[i]), __dadd_rn((double)x[i - 1], (double)x[i + 1])));
  };
  const long long i = 2LL * (I + 1);
  const double v = __dadd_rn(__dmul_rn(2.0, s(i)), __dadd_rn(s(i - 1), s(i + 1)));
  qc[(long long)r * fpc + I] = (T)__dmul_rn(0.5, v);
  xc[(long long)r * pc + COL0 + I] = T(0);
}

template <typename T>
__global__ void mg_correct1d_kernel(const T* xin, T* xout, long long pf, int nx, int rows,
                                    const T* __restrict__ e, long long pc,
                                    const Ctrl* __restrict__ ctrl) {
  if (ctrl->done) return;
  constexpr int COL0 = 16 / sizeof(T);
  const int i0 = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (i0 >= nx || r >= rows) return;
  const long long i = i0 + 1;
  const T* er = e + (long long)r * pc + (COL0 - 1);
  const T v = (i & 1) == 0 ? er[i / 2] : mul_t(T(0.5), add_t(er[(i - 1) / 2], er[(i + 1) / 2]));
  const long long o = (long long)r * pf + (COL0 - 1) + i;
  xout[o] = add_t(xin[o], v);
}

template <typename T>
cudaError_t restrict_t(const Geom& gf, const void* xf, const void* qf, const Geom& gc, void* qc,
                       void* xc, bool write_zero, const Ctrl* ctrl, cudaStream_t st) {
  if (gf.dim == 2) {
    // strip height: long strips amortise the 3 re-read rows on big grids, short ones keep the
    // latency chain short (and the grid full) on small ones
    const int rb = gc.ny >= 4096 ? 16 : (gc.ny >= 1024 ? 8 : (gc.ny >= 128 ? 4 : 1));
    const dim3 b(128), g((unsigned)((gc.nx + 128) / 128), (unsigned)((gc.ny + rb - 1) / rb));
    mg_restrict2d_stream<T><<<g, b, 0, st>>>((const T*)xf, (const T*)qf, gf.pitch, gf.fpitch, (int)gf.nx,
                                             (int)gf.ny, (T*)qc, (T*)xc, gc.pitch, gc.fpitch, (int)gc.nx,
                                             (int)gc.ny, rb, (int)write_zero, ctrl);
  } else {
    const dim3 b(256), g((unsigned)((gc.nx + 255) / 256), (unsigned)gc.ny);
    mg_restrict1d_kernel<T><<<g, b, 0, st>>>((const T*)xf, (const T*)qf, gf.pitch, gf.fpitch, (T*)qc,
                                             (T*)xc, gc.pitch, gc.fpitch, (int)gc.nx, (int)gc.ny, ctrl);
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t correct_t(const Geom& gf, const void* xin, void* xout, const Geom& gc, const void* e,
                      const Ctrl* ctrl, cudaStream_t st) {
  if (gf.dim == 2) {
    const dim3 b(128, 2), g((unsigned)((gc.nx + 1 + 127) / 128), (unsigned)((gc.ny + 1 + 1) / 2));
    mg_correct2d_vec<T><<<g, b, 0, st>>>((const T*)xin, (T*)xout, gf.pitch, (int)gf.nx, (int)gf.ny,
                                         (const T*)e, gc.pitch, (int)gc.nx, (int)gc.ny, ctrl);
  } else {
    const dim3 b(256), g((unsigned)((gf.nx + 255) / 256), (unsigned)gf.ny);
    mg_correct1d_kernel<T><<<g, b, 0, st>>>((const T*)xin, (T*)xout, gf.pitch, (int)gf.nx, (int)gf.ny,
                                            (const T*)e, gc.pitch, ctrl);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_mg_restrict(const Geom& gf, const void* xf, const void* qf, const Geom& gc, void* qc,
                               void* xc, bool write_zero, const Ctrl* ctrl, cudaStream_t st) {
  return gf.dtype == HJ_F64 ? restrict_t<double>(gf, xf, qf, gc, qc, xc, write_zero, ctrl, st)
                            : restrict_t<float>(gf, xf, qf, gc, qc, xc, write_zero, ctrl, st);
}

cudaError_t launch_mg_correct(const Geom& gf, const void* xin, void* xout, const Geom& gc, const void* e,
                              const Ctrl* ctrl, cudaStream_t st) {
  return gf.dtype == HJ_F64 ? correct_t<double>(gf, xin, xout, gc, e, ctrl, st)
                            : correct_t<float>(gf, xin, xout, gc, e, ctrl, st);
}

}  // namespace hj
