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
// 1/4 of that; correction: read + write x, 16 B per fine cell, plus the coarse iterate).  The
// 9-point residual window of a coarse point is re-read through L1 by its neighbours.
#include "hj_internal.cuh"

namespace hj {

namespace {

template <typename T>
__device__ __forceinline__ double resid2_at(const T* __restrict__ X, const T* __restrict__ Q,
                                            long long pitch, long long fpitch, int col0, long long i,
                                            long long j) {
  // (i, j): 1-based ringed fine coordinates of an interior point
  const T* p = X + j * pitch + (col0 - 1) + i;
  const double x = (double)p[0], w = (double)p[-1], e = (double)p[1];
  const double s = (double)p[-pitch], n = (double)p[pitch];
  const double h2f = (double)(T(4) * Q[(j - 1) * fpitch + (i - 1)]);
  return __dsub_rn(h2f, __dsub_rn(__dmul_rn(4.0, x), __dadd_rn(__dadd_rn(w, e), __dadd_rn(s, n))));
}

template <typename T>
__global__ void mg_restrict2d_kernel(const T* __restrict__ xf, const T* __restrict__ qf, long long pf,
                                     long long fpf, T* __restrict__ qc, T* __restrict__ xc,
                                     long long pc, long long fpc, int nxc, int nyc,
                                     const Ctrl* __restrict__ ctrl) {
  if (ctrl->done) return;
  constexpr int COL0 = 16 / sizeof(T);
  const int I = blockIdx.x * blockDim.x + threadIdx.x;  // 0-based coarse interior
  const int J = blockIdx.y * blockDim.y + threadIdx.y;
  if (I >= nxc || J >= nyc) return;
  const long long i = 2LL * (I + 1), j = 2LL * (J + 1);  // ringed fine centre
  auto s = [&](long long a, long long b) { return resid2_at<T>(xf, qf, pf, fpf, COL0, a, b); };
  const double a = __dmul_rn(4.0, s(i, j));
  const double b = __dmul_rn(2.0, __dadd_rn(__dadd_rn(s(i - 1, j), s(i + 1, j)), __dadd_rn(s(i, j - 1), s(i, j + 1))));
  const double c = __dadd_rn(__dadd_rn(s(i - 1, j - 1), s(i + 1, j - 1)), __dadd_rn(s(i - 1, j + 1), s(i + 1, j + 1)));
  qc[(long long)J * fpc + I] = (T)__dmul_rn(0.0625, __dadd_rn(__dadd_rn(a, b), c));
  xc[(long long)(J + 1) * pc + COL0 + I] = T(0);
}

template <typename T>
__device__ __forceinline__ T add_t(T a, T b) {
  if constexpr (sizeof(T) == 8) return __dadd_rn(a, b);
  else return __fadd_rn(a, b);
}
template <typename T>
__device__ __forceinline__ T mul_t(T a, T b) {
  if constexpr (sizeof(T) == 8) return __dmul_rn(a, b);
  else return __fmul_rn(a, b);
}

// xout = xin + P e over the fine interior (xin == xout allowed: each point reads then writes itself).
template <typename T>
__global__ void mg_correct2d_kernel(const T* xin, T* xout, long long pf, int nx, int ny,
                                    const T* __restrict__ e, long long pc,
                                    const Ctrl* __restrict__ ctrl) {
  if (ctrl->done) return;
  constexpr int COL0 = 16 / sizeof(T);
  const int i0 = blockIdx.x * blockDim.x + threadIdx.x;  // 0-based fine interior
  const int j0 = blockIdx.y * blockDim.y + threadIdx.y;
  if (i0 >= nx || j0 >= ny) return;
  const long long i = i0 + 1, j = j0 + 1;  // ringed
  auto E = [&](long long I, long long J) { return e[J * pc + (COL0 - 1) + I]; };
  const bool ci = (i & 1) == 0, cj = (j & 1) == 0;
  T v;
  if (ci && cj) v = E(i / 2, j / 2);
  else if (cj) v = mul_t(T(0.5), add_t(E((i - 1) / 2, j / 2), E((i + 1) / 2, j / 2)));
  else if (ci) v = mul_t(T(0.5), add_t(E(i / 2, (j - 1) / 2), E(i / 2, (j + 1) / 2)));
  else
    v = mul_t(T(0.25), add_t(add_t(E((i - 1) / 2, (j - 1) / 2), E((i + 1) / 2, (j - 1) / 2)),
                             add_t(E((i - 1) / 2, (j + 1) / 2), E((i + 1) / 2, (j + 1) / 2))));
  const long long o = j * pf + (COL0 - 1) + i;
  xout[o] = add_t(xin[o], v);
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
                       void* xc, const Ctrl* ctrl, cudaStream_t st) {
  if (gf.dim == 2) {
    const dim3 b(32, 8), g((unsigned)((gc.nx + 31) / 32), (unsigned)((gc.ny + 7) / 8));
    mg_restrict2d_kernel<T><<<g, b, 0, st>>>((const T*)xf, (const T*)qf, gf.pitch, gf.fpitch, (T*)qc,
                                             (T*)xc, gc.pitch, gc.fpitch, (int)gc.nx, (int)gc.ny, ctrl);
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
    const dim3 b(64, 4), g((unsigned)((gf.nx + 63) / 64), (unsigned)((gf.ny + 3) / 4));
    mg_correct2d_kernel<T><<<g, b, 0, st>>>((const T*)xin, (T*)xout, gf.pitch, (int)gf.nx, (int)gf.ny,
                                            (const T*)e, gc.pitch, ctrl);
  } else {
    const dim3 b(256), g((unsigned)((gf.nx + 255) / 256), (unsigned)gf.ny);
    mg_correct1d_kernel<T><<<g, b, 0, st>>>((const T*)xin, (T*)xout, gf.pitch, (int)gf.nx, (int)gf.ny,
                                            (const T*)e, gc.pitch, ctrl);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_mg_restrict(const Geom& gf, const void* xf, const void* qf, const Geom& gc, void* qc,
                               void* xc, const Ctrl* ctrl, cudaStream_t st) {
  return gf.dtype == HJ_F64 ? restrict_t<double>(gf, xf, qf, gc, qc, xc, ctrl, st)
                            : restrict_t<float>(gf, xf, qf, gc, qc, xc, ctrl, st);
}

cudaError_t launch_mg_correct(const Geom& gf, const void* xin, void* xout, const Geom& gc, const void* e,
                              const Ctrl* ctrl, cudaStream_t st) {
  return gf.dtype == HJ_F64 ? correct_t<double>(gf, xin, xout, gc, e, ctrl, st)
                            : correct_t<float>(gf, xin, xout, gc, e, ctrl, st);
}

}  // namespace hj
