// oracle/hjo.cpp — CPU ORACLE. TEST INFRASTRUCTURE ONLY.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs may load this library.  The product path
// (paper_2006_16465_b200/) never links, imports or calls it, and shares no code,
// header, table or constant generator with it.
//
// What it computes: classic Jacobi and the paper's hierarchical ("shared-memory")
// Jacobi for the 1D 3-point and 2D 5-point Poisson problem, written as plain,
// slow, single-threaded loops that follow the paper step by step:
//   * Jacobi splitting / elemental update      PAPER.md:29-37  (§2.1, Eqs. 1-2)
//   * 1D Poisson system and update             PAPER.md:180-212 (§3.4, Eqs. 5-7)
//   * 2D Poisson system and update             PAPER.md:393-421 (§4.2)
//   * CPU approach (two arrays, swap)          PAPER.md:94-112  (§3.1 listing)
//   * hierarchical cycle: copy tile+halo, k sub-iterations with frozen halo,
//     write the interior back                  PAPER.md:161-166 (§3.3), :382-387 (§4.1),
//                                              Appendix A
//   * stopping rule: reduce the L2 residual of the initial solution by a factor
//     (relative test)
//   * resource figures (shared bytes, blocks)
//   * multigrid with the hierarchical cycle as smoother
//                                              PAPER.md:17 (§1), :530 (§5); the textbook V-cycle
//                                              of the tutorial the paper cites (reading c24,
//                                              see vcycle_2d below)
//
// Readings where the paper is silent/garbled are SURVEY.md §8(c) c1..c18, listed
// in DESIGN.md §3.  In particular:
//   c6  snapshot semantics: a cycle reads x_c and writes x_{c+1} into a second array
//       (Appendix A writes in place, a race — PAPER.md:549, :573);
//   c7  the rhs of the updated cell is used (Appendix A's rhs index is off by one);
//   c8  the write-back takes the values after exactly k sub-iterations (odd k too);
//   c10 ragged last tile when n is not a multiple of the tile;
//   c12 the Dirichlet ring may hold non-zero values g;
//   c21 overlapping subdomains: last block shifted left to end at n, half-split ownership with
//       the left block taking the odd extra point (see block_plan);
//   c3  the residual is computed in the h^2-scaled form
//       s = h^2 f - (2x - (x_{i-1}+x_{i+1}))            (1D)
//       s = h^2 f - (4x - ((xW+xE)+(xS+xN)))            (2D)
//       in double, ||b - Ax||_2 = sqrt(sum s^2) / h^2;
//   c16 fp32 iterates: h2f = float(h*h*f) (one rounding of the double product),
//       update in fp32 with the same expression; the residual is accumulated in
//       double from the iterate and that SAME rounded h2f widened to double, i.e.
//       it is the residual of the system the fp32 iteration actually solves
//       (c16: keeps fp32 at 12 B/cell; differs from the true rhs by
//       at most one fp32 rounding of h^2 f, far below the fp32 residual floor).
//
// General coefficients (reading c23): the tridiagonal update of
// Eq. 4 with per-point a_i, d_i, c_i and the pentadiagonal update of Eq. 10
// with constants a, c, e, f, d, evaluated as
//       1D: fma(wR, xR, fma(wL, xL, q))                       wL = T(-a_i/d_i), wR = T(-c_i/d_i)
//       2D: fma(wN, xN, fma(wS, xS, fma(wE, xE, fma(wW, xW, q))))   wW = T(-a/d), wE = T(-c/d),
//                                                              wS = T(-e/d), wN = T(-f/d)
//       q = T(b/d) (b = the f array, NOT scaled by h^2; h is unused)
// (the division of Eq. 4/10 distributed over the terms, each quotient rounded once to T).  The
// residual is the Jacobi-scaled s = D^{-1}(b - Ax) = (same chain in double) - x, summed as s^2;
// the reported norm is ||s|| * |d| in 2D (= ||b - Ax||, d constant) and ||s|| in 1D (d_i varies).
//
// Canonical arithmetic: the elemental update of
// PAPER.md:210 / :420 is evaluated exactly as
//       1D: T(0.5)  * ((xL + xR) + h2f)
//       2D: T(0.25) * (((xW + xE) + (xS + xN)) + h2f)
// Built with -O2 -ffp-contract=off (no FMA contraction, no fast-math).
//
// Layout: interior arrays are row-major, x fastest.
// Internally every grid carries its Dirichlet ring: (nx+2) x (ny+2) values,
// index (j)*(nx+2) + i with i = 0..nx+1 along x and j = 0..ny+1 along y
// (1D: nx+2 values).  Ring corners are never read by the 5-point stencil.
//
// Boundary-data layout ("bc"), shared with the ABI only by documentation:
//   1D: [g_left, g_right] per problem (batched: problem b at bc[2b], bc[2b+1])
//   2D: [south(nx) | north(nx) | west(ny) | east(ny)]   (south = row y=0)
//   NULL means homogeneous (the paper's u = 0).

#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>

namespace {

// ------------------------------------------------------------ block plan -----
// Subdomains along one dimension of n interior points (1-based), tile width T, overlap o.
//  o = 0: tiles [1 + t*T, min((t+1)*T, n)], ragged last tile (reading c10);
//        every tile owns its whole interior.
//  o > 0 (PAPER.md:243-258, §3.5; :454-458, §4.3): block b starts at 1 + b*(T - o) and spans T
//        points; the number of blocks is ceil((n - T)/(T - o)) + 1 (= (n - o)/(T - o) when it
//        divides, Eq. 8); if it does not divide, the last block is shifted left to
//        end at n (reading c21).  In each overlap between consecutive blocks the
//        left block owns the left half and the right block the right half, the left block
//        taking the extra point when the overlap is odd (reading c21).
struct BlockPlan {
  std::vector<int64_t> start, width, own_lo, own_hi;  // 1-based, inclusive
};

inline BlockPlan block_plan(int64_t n, int64_t T, int64_t o) {
  BlockPlan P;
  if (o == 0) {
    for (int64_t s = 1; s <= n; s += T) {
      const int64_t w = std::min(T, n - s + 1);
      P.start.push_back(s);
      P.width.push_back(w);
      P.own_lo.push_back(s);
      P.own_hi.push_back(s + w - 1);
    }
    return P;
  }
  const int64_t nb = (n - T + (T - o) - 1) / (T - o) + 1;
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t s = (b == nb - 1) ? n - T + 1 : 1 + b * (T - o);
    P.start.push_back(s);
    P.width.push_back(T);
  }
  P.own_lo.assign(nb, 1);
  P.own_hi.assign(nb, n);
  for (int64_t b = 0; b + 1 < nb; ++b) {
    const int64_t ov_lo = P.start[b + 1], ov_hi = P.start[b] + T - 1;  // overlap region
    const int64_t L = ov_hi - ov_lo + 1;
    const int64_t left_end = ov_lo + (L + 1) / 2 - 1;                  // left takes ceil(L/2)
    P.own_hi[b] = left_end;
    P.own_lo[b + 1] = left_end + 1;
  }
  return P;
}

// Damped (weighted) Jacobi, the multigrid smoother of SURVEY.md §8(f) NEXT #4 (reading c24):
// x <- x + omega (u - x) with u the plain Jacobi value, evaluated as ONE fused multiply-add in T,
// fma(omega, u - x, x).  Used only by the multigrid solver's smoothing cycles (omega != 1).
template <typename T>
inline T damp(T omega, T x, T u) {
  return std::fma(omega, u - x, x);
}

// ---------------------------------------------------------------- 1D ----------

// Elemental Jacobi update for -u'' = f, PAPER.md:210 (Eq. jacobi-stencil-1d-poisson):
//     x_i <- (b_i dx^2 + x_{i-1} + x_{i+1}) / 2
template <typename T>
inline T update1d(T left, T right, T h2f) {
  return T(0.5) * ((left + right) + h2f);
}

// Residual contribution in the h^2-scaled form (reading c3), always double.
inline double resid1d(double x, double left, double right, double h2f64) {
  return h2f64 - (2.0 * x - (left + right));
}

// General tridiagonal update, Eq. 4: x_i <- (b_i - a_i x_{i-1} - c_i x_{i+1}) / d_i
// with the division distributed (reading c23): q + wL x_{i-1} + wR x_{i+1}, two fused
// multiply-adds in T.
template <typename T>
inline T update1d_gen(T wl, T wr, T left, T right, T q) {
  return std::fma(wr, right, std::fma(wl, left, q));
}
// D^{-1}(b - Ax) at one point, in double from the T weights and q (reading c23).
inline double resid1d_gen(double wl, double wr, double x, double left, double right, double q) {
  return std::fma(wr, right, std::fma(wl, left, q)) - x;
}

template <typename T>
struct Problem1D {
  int64_t n;                 // interior points (paper's N)
  double h2;                 // h*h
  bool gen = false;          // general coefficients (Eq. 4) instead of -u'' = f
  std::vector<T> h2f;        // Poisson: T(h2*f_i), i = 0..n-1; general: q_i = T(b_i/d_i)
  std::vector<double> h2f64; // Poisson: double(h2f_i), rhs used by the residual (c16)
  std::vector<T> wl, wr;     // general: T(-a_i/d_i), T(-c_i/d_i)
  T gl, gr;                  // Dirichlet values at x=0 and x=1
  bool weighted = false;     // multigrid smoother (reading c24): damped sub-iterations
  T omega = T(1);
};

// x has n+2 entries: x[0] = g_left, x[1..n] interior, x[n+1] = g_right.
template <typename T>
double residual_sq_1d(const Problem1D<T>& p, const std::vector<T>& x) {
  double S = 0.0;
  for (int64_t i = 1; i <= p.n; ++i) {
    double s = p.gen ? resid1d_gen((double)p.wl[i - 1], (double)p.wr[i - 1], (double)x[i],
                                   (double)x[i - 1], (double)x[i + 1], (double)p.h2f[i - 1])
                     : resid1d((double)x[i], (double)x[i - 1], (double)x[i + 1], p.h2f64[i - 1]);
    S += s * s;
  }
  return S;
}

// §3.1 CPU approach: every DOF from the previous iterate.
template <typename T>
void classic_sweep_1d(const Problem1D<T>& p, const std::vector<T>& x0, std::vector<T>& x1) {
  for (int64_t i = 1; i <= p.n; ++i)
    x1[i] = p.gen ? update1d_gen<T>(p.wl[i - 1], p.wr[i - 1], x0[i - 1], x0[i + 1], p.h2f[i - 1])
                  : update1d<T>(x0[i - 1], x0[i + 1], p.h2f[i - 1]);
}

// §3.3 hierarchical cycle, 1D (Appendix A :548-573), blocks from block_plan.
// tile_order = 0: blocks in increasing order; 1: decreasing (used by the order-independence
// test — the result must not depend on it).
template <typename T>
void hier_cycle_1d(const Problem1D<T>& p, const BlockPlan& bp, int k, int tile_order,
                   const std::vector<T>& xc, std::vector<T>& xn) {
  const int64_t nb = (int64_t)bp.start.size();
  std::vector<T> A, B, rhs, wl, wr;
  for (int64_t tt = 0; tt < nb; ++tt) {
    const int64_t t = tile_order == 0 ? tt : nb - 1 - tt;
    const int64_t lo = bp.start[t];        // first interior point of the subdomain
    const int64_t w = bp.width[t];
    const int64_t hi = lo + w - 1;
    // Step 1: copy the augmented subdomain [lo-1, hi+1] into two containers,
    // and the rhs of the interior points.
    A.assign(xc.begin() + (lo - 1), xc.begin() + (hi + 2));
    B = A;
    rhs.assign(p.h2f.begin() + (lo - 1), p.h2f.begin() + hi);
    if (p.gen) {  // the block's coefficients travel with its rhs (reading c23)
      wl.assign(p.wl.begin() + (lo - 1), p.wl.begin() + hi);
      wr.assign(p.wr.begin() + (lo - 1), p.wr.begin() + hi);
    }
    // Step 2: k sub-iterations on the interior; the two halo points are never
    // written (frozen at snapshot values, reading c5).
    for (int q = 0; q < k; ++q) {
      for (int64_t i = 1; i <= w; ++i) {
        B[i] = p.gen ? update1d_gen<T>(wl[i - 1], wr[i - 1], A[i - 1], A[i + 1], rhs[i - 1])
                     : update1d<T>(A[i - 1], A[i + 1], rhs[i - 1]);
        if (p.weighted) B[i] = damp<T>(p.omega, A[i], B[i]);
      }
      std::swap(A, B);
    }
    // Step 3: write the latest values of the OWNED points into the NEXT global array
    // (snapshot semantics c6; latest values c8; ownership PAPER.md:249).
    for (int64_t g = bp.own_lo[t]; g <= bp.own_hi[t]; ++g) xn[g] = A[g - lo + 1];
  }
}

// ---------------------------------------------------------------- 2D ----------

// Elemental Jacobi update for -(u_xx + u_yy) = f with dx = dy = h,
// x_ij <- (b_ij h^2 + x_{i-1,j} + x_{i+1,j} + x_{i,j-1} + x_{i,j+1}) / 4
template <typename T>
inline T update2d(T w, T e, T s, T n, T h2f) {
  return T(0.25) * (((w + e) + (s + n)) + h2f);
}

inline double resid2d(double x, double w, double e, double s, double n, double h2f64) {
  return h2f64 - (4.0 * x - ((w + e) + (s + n)));
}

// General pentadiagonal update, Eq. 10:
//   x_ij <- (b_ij - a x_{i-1,j} - c x_{i+1,j} - e x_{i,j-1} - f x_{i,j+1}) / d
// with the division distributed (reading c23): four fused multiply-adds in T, W, E, S, N order.
template <typename T>
inline T update2d_gen(const T* wt, T w, T e, T s, T n, T q) {
  return std::fma(wt[3], n, std::fma(wt[2], s, std::fma(wt[1], e, std::fma(wt[0], w, q))));
}
template <typename T>
inline double resid2d_gen(const T* wt, double x, double w, double e, double s, double n, double q) {
  return std::fma((double)wt[3], n,
                  std::fma((double)wt[2], s, std::fma((double)wt[1], e, std::fma((double)wt[0], w, q)))) - x;
}

template <typename T>
struct Problem2D {
  int64_t nx, ny;
  double h2;
  bool gen = false;          // general constant coefficients (Eq. 10) instead of -Δu = f
  T wt[4] = {T(0), T(0), T(0), T(0)};  // general: T(-a/d), T(-c/d), T(-e/d), T(-f/d)  (W, E, S, N)
  std::vector<T> h2f;        // nx*ny, row-major: Poisson T(h2*f); general q = T(b/d)
  std::vector<double> h2f64; // nx*ny, double(h2f) (c16)
  bool weighted = false;     // multigrid smoother (reading c24): damped sub-iterations
  T omega = T(1);
  int64_t pitch() const { return nx + 2; }
  T upd(T w, T e, T s, T n, T q) const {
    return gen ? update2d_gen<T>(wt, w, e, s, n, q) : update2d<T>(w, e, s, n, q);
  }
};

// index of (i, j) in a ringed grid, i = 0..nx+1 (x), j = 0..ny+1 (y)
template <typename T>
inline int64_t at(const Problem2D<T>& p, int64_t i, int64_t j) { return j * p.pitch() + i; }

template <typename T>
double residual_sq_2d(const Problem2D<T>& p, const std::vector<T>& x) {
  double S = 0.0;
  for (int64_t j = 1; j <= p.ny; ++j)
    for (int64_t i = 1; i <= p.nx; ++i) {
      const double xc = (double)x[at(p, i, j)], w = (double)x[at(p, i - 1, j)],
                   e = (double)x[at(p, i + 1, j)], so = (double)x[at(p, i, j - 1)],
                   no = (double)x[at(p, i, j + 1)];
      double s = p.gen ? resid2d_gen<T>(p.wt, xc, w, e, so, no, (double)p.h2f[(j - 1) * p.nx + (i - 1)])
                       : resid2d(xc, w, e, so, no, p.h2f64[(j - 1) * p.nx + (i - 1)]);
      S += s * s;
    }
  return S;
}

template <typename T>
void classic_sweep_2d(const Problem2D<T>& p, const std::vector<T>& x0, std::vector<T>& x1) {
  for (int64_t j = 1; j <= p.ny; ++j)
    for (int64_t i = 1; i <= p.nx; ++i)
      x1[at(p, i, j)] = p.upd(x0[at(p, i - 1, j)], x0[at(p, i + 1, j)], x0[at(p, i, j - 1)],
                              x0[at(p, i, j + 1)], p.h2f[(j - 1) * p.nx + (i - 1)]);
}

// §4.1 hierarchical cycle, 2D.  Block (a, b) = x-block a of bx times y-block b
// of by; the augmented subdomain is (w+2) x (hgt+2); the halo is frozen.  A point
// is written by the block owning it in both x and y (§4.3).
template <typename T>
void hier_cycle_2d(const Problem2D<T>& p, const BlockPlan& bx, const BlockPlan& by, int k,
                   int tile_order, const std::vector<T>& xc, std::vector<T>& xn) {
  const int64_t ntx = (int64_t)bx.start.size(), nty = (int64_t)by.start.size();
  const int64_t ntiles = ntx * nty;
  std::vector<T> A, B, rhs;
  for (int64_t tt = 0; tt < ntiles; ++tt) {
    const int64_t t = tile_order == 0 ? tt : ntiles - 1 - tt;
    const int64_t a = t % ntx, b = t / ntx;
    const int64_t ilo = bx.start[a], w = bx.width[a];
    const int64_t jlo = by.start[b], hgt = by.width[b];
    const int64_t lp = w + 2;
    // Step 1: copy the augmented subdomain (two containers) and the local rhs.
    A.assign((size_t)(lp * (hgt + 2)), T(0));
    for (int64_t jj = 0; jj < hgt + 2; ++jj)
      for (int64_t ii = 0; ii < lp; ++ii) A[jj * lp + ii] = xc[at(p, ilo - 1 + ii, jlo - 1 + jj)];
    B = A;
    rhs.assign((size_t)(w * hgt), T(0));
    for (int64_t jj = 0; jj < hgt; ++jj)
      for (int64_t ii = 0; ii < w; ++ii)
        rhs[jj * w + ii] = p.h2f[(jlo - 1 + jj) * p.nx + (ilo - 1 + ii)];
    // Step 2: k sub-iterations on the interior, halo frozen.
    for (int q = 0; q < k; ++q) {
      for (int64_t jj = 1; jj <= hgt; ++jj)
        for (int64_t ii = 1; ii <= w; ++ii) {
          B[jj * lp + ii] = p.upd(A[jj * lp + ii - 1], A[jj * lp + ii + 1], A[(jj - 1) * lp + ii],
                                  A[(jj + 1) * lp + ii], rhs[(jj - 1) * w + (ii - 1)]);
          if (p.weighted) B[jj * lp + ii] = damp<T>(p.omega, A[jj * lp + ii], B[jj * lp + ii]);
        }
      std::swap(A, B);
    }
    // Step 3: write the owned points into the next global array.
    for (int64_t j = by.own_lo[b]; j <= by.own_hi[b]; ++j)
      for (int64_t i = bx.own_lo[a]; i <= bx.own_hi[a]; ++i)
        xn[at(p, i, j)] = A[(j - jlo + 1) * lp + (i - ilo + 1)];
  }
}

// ------------------------------------------------------------- driver ---------
// SURVEY.md §8(c) step 6.  S_0 = S(x_0) (or (ref_residual*rdiv)^2).  hist[0].
// If S_0 == 0 return c = 0.  For c = 1..max_cycles: x_c, S_c, hist[c];
// non-finite -> status 4; sqrt(S_c) <= tol*sqrt(S_0) -> converged at c.
// Absolute mode: sqrt(S_c)/rdiv <= tol.  rdiv converts the summed scaled residual into the
// reported norm: h^2 (Poisson, c3), 1/|d| (general 2D), 1 (general 1D) — reading c23.

enum { ST_OK = 0, ST_NOT_CONVERGED = 1, ST_INVALID = 2, ST_NUMERIC = 4 };

struct DriverOut {
  int64_t cycles = 0;
  int converged = 0;
  int status = ST_OK;
};

template <typename Cycle, typename Resid>
DriverOut drive(double rdiv, double tol, int tol_mode, double ref_residual, int64_t max_cycles,
                double* hist, Cycle&& cycle, Resid&& resid) {
  DriverOut out;
  double S0 = resid();
  double sqrtS0 = ref_residual > 0.0 ? ref_residual * rdiv : std::sqrt(S0);
  if (hist) hist[0] = std::sqrt(S0) / rdiv;
  if (!std::isfinite(S0)) { out.status = ST_NUMERIC; return out; }
  auto test = [&](double S) {
    return tol_mode == 0 ? (std::sqrt(S) <= tol * sqrtS0) : (std::sqrt(S) / rdiv <= tol);
  };
  if (S0 == 0.0 || (ref_residual > 0.0 && test(S0)) || (tol_mode == 1 && test(S0))) {
    out.converged = 1;
    out.cycles = 0;
    return out;
  }
  for (int64_t c = 1; c <= max_cycles; ++c) {
    cycle();
    double S = resid();
    if (hist) hist[c] = std::sqrt(S) / rdiv;
    out.cycles = c;
    if (!std::isfinite(S)) { out.status = ST_NUMERIC; return out; }
    if (test(S)) { out.converged = 1; return out; }
  }
  out.status = ST_NOT_CONVERGED;
  return out;
}

// B independent 1D problems (the paper's "1024 copies"):
// problem b has interior f[b*n .. b*n+n), ends bc[2b], bc[2b+1]; one cycle advances every problem;
// the stopping test uses the L2 norm of the stacked residual (sum over problems in order).
// stencil (general coefficients, Eq. 4) = NULL or three planes of n*batch doubles:
// [a (sub-diagonal) | d (diagonal) | c (super-diagonal)], point i of problem b at b*n + i.
template <typename T>
int solve1d(int64_t n, int64_t batch, double h, const double* f, const double* bc, const double* x0,
            const double* stencil, int mode, int64_t tile, int64_t overlap, int k, double tol,
            int tol_mode, double ref_residual, int64_t max_cycles, int tile_order, double* x_out,
            double* hist, int64_t* cycles, int* converged) {
  std::vector<Problem1D<T>> ps(batch);
  std::vector<std::vector<T>> xa(batch), xb(batch);
  const int64_t nt = n * batch;
  for (int64_t b = 0; b < batch; ++b) {
    Problem1D<T>& p = ps[b];
    p.n = n;
    p.h2 = h * h;
    p.gen = stencil != nullptr;
    p.h2f.resize(n);
    p.h2f64.resize(n);
    if (p.gen) {
      p.wl.resize(n);
      p.wr.resize(n);
    }
    for (int64_t i = 0; i < n; ++i) {
      const int64_t g = b * n + i;
      if (p.gen) {  // reading c23: q = T(b/d), wL = T(-a/d), wR = T(-c/d)
        const double a = stencil[g], d = stencil[nt + g], c = stencil[2 * nt + g];
        p.h2f[i] = (T)(f[g] / d);
        p.wl[i] = (T)(-a / d);
        p.wr[i] = (T)(-c / d);
      } else {
        p.h2f[i] = (T)(p.h2 * f[g]);
      }
      p.h2f64[i] = (double)p.h2f[i];  // reading c16: residual of the rounded system
    }
    xa[b].assign(n + 2, T(0));
    xa[b][0] = bc ? (T)bc[2 * b] : T(0);
    xa[b][n + 1] = bc ? (T)bc[2 * b + 1] : T(0);
    xb[b] = xa[b];
    for (int64_t i = 0; i < n; ++i) xa[b][i + 1] = x0 ? (T)x0[b * n + i] : T(0);
  }
  bool flip = false;  // false: current iterate in xa
  const BlockPlan bp = mode == 1 ? BlockPlan() : block_plan(n, tile, overlap);
  auto cycle = [&]() {
    for (int64_t b = 0; b < batch; ++b) {
      const std::vector<T>& cur = flip ? xb[b] : xa[b];
      std::vector<T>& nxt = flip ? xa[b] : xb[b];
      if (mode == 1) classic_sweep_1d(ps[b], cur, nxt);
      else hier_cycle_1d(ps[b], bp, k, tile_order, cur, nxt);
    }
    flip = !flip;
  };
  auto resid = [&]() {
    double S = 0.0;
    for (int64_t b = 0; b < batch; ++b) S += residual_sq_1d(ps[b], flip ? xb[b] : xa[b]);
    return S;
  };
  DriverOut o = drive(stencil ? 1.0 : h * h, tol, tol_mode, ref_residual, max_cycles, hist, cycle, resid);
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t i = 0; i < n; ++i) x_out[b * n + i] = (double)(flip ? xb[b] : xa[b])[i + 1];
  *cycles = o.cycles;
  *converged = o.converged;
  return o.status;
}

// stencil (general constant coefficients, Eq. 10) = NULL or {a, c, e, f, d}: the coefficients of
// x_{i-1,j} (west), x_{i+1,j} (east), x_{i,j-1} (south), x_{i,j+1} (north) and x_{ij}.
template <typename T>
int solve2d(int64_t nx, int64_t ny, double h, const double* f, const double* bc, const double* x0,
            const double* stencil, int mode, int64_t tx, int64_t ty, int64_t ox, int64_t oy, int k,
            double tol, int tol_mode, double ref_residual, int64_t max_cycles, int tile_order,
            double* x_out, double* hist, int64_t* cycles, int* converged) {
  Problem2D<T> p;
  p.nx = nx;
  p.ny = ny;
  p.h2 = h * h;
  p.gen = stencil != nullptr;
  p.h2f.resize(nx * ny);
  p.h2f64.resize(nx * ny);
  double rdiv = p.h2;
  if (p.gen) {  // reading c23
    const double d = stencil[4];
    for (int q = 0; q < 4; ++q) p.wt[q] = (T)(-stencil[q] / d);
    rdiv = 1.0 / std::fabs(d);
  }
  for (int64_t q = 0; q < nx * ny; ++q) {
    p.h2f[q] = p.gen ? (T)(f[q] / stencil[4]) : (T)(p.h2 * f[q]);
    p.h2f64[q] = (double)p.h2f[q];  // reading c16: residual of the rounded system
  }
  std::vector<T> xa((nx + 2) * (ny + 2), T(0));
  // Dirichlet ring (reading c12): south row j=0, north row j=ny+1, west col i=0, east col i=nx+1
  if (bc) {
    for (int64_t i = 1; i <= nx; ++i) {
      xa[at(p, i, 0)] = (T)bc[i - 1];
      xa[at(p, i, ny + 1)] = (T)bc[nx + i - 1];
    }
    for (int64_t j = 1; j <= ny; ++j) {
      xa[at(p, 0, j)] = (T)bc[2 * nx + j - 1];
      xa[at(p, nx + 1, j)] = (T)bc[2 * nx + ny + j - 1];
    }
  }
  std::vector<T> xb = xa;  // both arrays carry the ring
  for (int64_t j = 1; j <= ny; ++j)
    for (int64_t i = 1; i <= nx; ++i) xa[at(p, i, j)] = x0 ? (T)x0[(j - 1) * nx + (i - 1)] : T(0);
  std::vector<T>* cur = &xa;
  std::vector<T>* nxt = &xb;
  const BlockPlan bx = mode == 1 ? BlockPlan() : block_plan(nx, tx, ox);
  const BlockPlan by = mode == 1 ? BlockPlan() : block_plan(ny, ty, oy);
  auto cycle = [&]() {
    if (mode == 1) classic_sweep_2d(p, *cur, *nxt);
    else hier_cycle_2d(p, bx, by, k, tile_order, *cur, *nxt);
    std::swap(cur, nxt);
  };
  auto resid = [&]() { return residual_sq_2d(p, *cur); };
  DriverOut o = drive(rdiv, tol, tol_mode, ref_residual, max_cycles, hist, cycle, resid);
  for (int64_t j = 1; j <= ny; ++j)
    for (int64_t i = 1; i <= nx; ++i) x_out[(j - 1) * nx + (i - 1)] = (double)(*cur)[at(p, i, j)];
  *cycles = o.cycles;
  *converged = o.converged;
  return o.status;
}

// ===================================================== multigrid (NEXT #4) ====
// the hierarchical cycle as a multigrid smoother.  PAPER.md:17 (§1):
// Jacobi iteration and similar stationary methods "form the backbone of highly effective
// geometric and algebraic multigrid methods [Briggs2000]"; PAPER.md:530 (§5): the hierarchical
// solver "has the potential to accelerate multigrid solvers which utilize this approach as a
// smoother".  The paper gives no coarse-grid design, so reading c24 takes the
// textbook V-cycle of the tutorial it cites (Briggs, Henson & McCormick, "A Multigrid Tutorial",
// ch. 3-4), with the paper's hierarchical cycle as the smoother:
//   grids     level 0 = the problem (ringed, Dirichlet data g).  Level l+1 coarsens every
//             axis of level l that has an odd number n_l >= 3 of interior points to
//             (n_l - 1)/2 points with spacing 2 h_l (vertex-centred and nested: coarse ringed
//             point I is fine ringed point 2I); 2D coarsens x and y together and stops when
//             either is even or < 3; 1D (each of the ny independent problems) coarsens x.  At
//             most max_levels levels (0 = no limit).  Coarse rings are zero (error equation).
//   smoother  nu1 (pre) / nu2 (post) hierarchical cycles of DAMPED Jacobi (damp(), omega) with
//             the tile clipped to the level, k sub-iterations, halo frozen, snapshot semantics.
//             Undamped Jacobi does not smooth (its highest mode has eigenvalue -cos(pi h)), hence
//             the damping — the weighted Jacobi the paper's related work cites.
//   coarsest  coarse_cycles plain (undamped) hierarchical cycles from zero.
//   restrict  full weighting of the h^2-scaled residual s (reading c3) of the smoothed iterate.
//             The coarse equation is A_2h e = R r with r = s / h^2, i.e. coarse
//             h2f = (2h)^2 R r = 4 R s:
//               2D  T(0.25 * ((4 s_C + 2 ((s_W + s_E) + (s_S + s_N))) + ((s_SW + s_SE) + (s_NW + s_NE))))
//               1D  T(2 s_C + (s_L + s_R))
//             (s in double, reading c16; the power-of-two factors are exact).  The coarse
//             iterate starts at zero.
//   correct   (bi)linear interpolation of the coarse iterate e added to the fine iterate, in T:
//               fine on a coarse point            x + e
//               between two coarse points         x + T(0.5)  * (e_W + e_E)   (or (e_S + e_N))
//               between four (2D)                 x + T(0.25) * ((e_SW + e_SE) + (e_NW + e_NE))
//   solve     one solver cycle = one V-cycle on level 0; the relative/absolute stopping test of
//             the hierarchical solver (drive(), reading c1) after every V-cycle.
struct MgOpts {
  int k, nu1, nu2, coarse_cycles;
};

template <typename T>
struct MgLevel2D {
  Problem2D<T> p;
  BlockPlan bx, by;
  std::vector<T> x, y;  // iterate and the second (snapshot) array, both ringed
};

template <typename T>
void mg_smooth_2d(MgLevel2D<T>& L, int k, int cycles, bool weighted) {
  L.p.weighted = weighted;
  for (int c = 0; c < cycles; ++c) {
    hier_cycle_2d(L.p, L.bx, L.by, k, 0, L.x, L.y);
    std::swap(L.x, L.y);
  }
}

template <typename T>
void mg_restrict_2d(const MgLevel2D<T>& F, MgLevel2D<T>& C) {
  const Problem2D<T>& p = F.p;
  const std::vector<T>& x = F.x;
  auto s = [&](int64_t i, int64_t j) {
    return resid2d((double)x[at(p, i, j)], (double)x[at(p, i - 1, j)], (double)x[at(p, i + 1, j)],
                   (double)x[at(p, i, j - 1)], (double)x[at(p, i, j + 1)], p.h2f64[(j - 1) * p.nx + (i - 1)]);
  };
  for (int64_t J = 1; J <= C.p.ny; ++J)
    for (int64_t I = 1; I <= C.p.nx; ++I) {
      const int64_t i = 2 * I, j = 2 * J;
      const double a = 4.0 * s(i, j);
      const double b = 2.0 * ((s(i - 1, j) + s(i + 1, j)) + (s(i, j - 1) + s(i, j + 1)));
      const double c = (s(i - 1, j - 1) + s(i + 1, j - 1)) + (s(i - 1, j + 1) + s(i + 1, j + 1));
      const T v = (T)(0.25 * ((a + b) + c));
      C.p.h2f[(J - 1) * C.p.nx + (I - 1)] = v;
      C.p.h2f64[(J - 1) * C.p.nx + (I - 1)] = (double)v;
      C.x[at(C.p, I, J)] = T(0);
    }
}

template <typename T>
void mg_correct_2d(MgLevel2D<T>& F, const MgLevel2D<T>& C) {
  auto e = [&](int64_t I, int64_t J) { return C.x[at(C.p, I, J)]; };  // ring = 0
  for (int64_t j = 1; j <= F.p.ny; ++j)
    for (int64_t i = 1; i <= F.p.nx; ++i) {
      const bool ci = (i % 2) == 0, cj = (j % 2) == 0;  // on a coarse line
      T v;
      if (ci && cj) v = e(i / 2, j / 2);
      else if (cj) v = T(0.5) * (e((i - 1) / 2, j / 2) + e((i + 1) / 2, j / 2));
      else if (ci) v = T(0.5) * (e(i / 2, (j - 1) / 2) + e(i / 2, (j + 1) / 2));
      else
        v = T(0.25) * ((e((i - 1) / 2, (j - 1) / 2) + e((i + 1) / 2, (j - 1) / 2)) +
                       (e((i - 1) / 2, (j + 1) / 2) + e((i + 1) / 2, (j + 1) / 2)));
      T& xv = F.x[at(F.p, i, j)];
      xv = xv + v;
    }
}

template <typename T>
void vcycle_2d(std::vector<MgLevel2D<T>>& Ls, size_t l, const MgOpts& o) {
  MgLevel2D<T>& L = Ls[l];
  if (l + 1 == Ls.size()) {
    mg_smooth_2d(L, o.k, o.coarse_cycles, false);
    return;
  }
  mg_smooth_2d(L, o.k, o.nu1, true);
  mg_restrict_2d(L, Ls[l + 1]);
  vcycle_2d(Ls, l + 1, o);
  mg_correct_2d(L, Ls[l + 1]);
  mg_smooth_2d(L, o.k, o.nu2, true);
}

// Level sizes (reading c24): returns the interior sizes of every level.
inline std::vector<int64_t> mg_sizes(int64_t n, int max_levels) {
  std::vector<int64_t> v{n};
  while ((max_levels <= 0 || (int)v.size() < max_levels) && v.back() >= 3 && (v.back() % 2) == 1)
    v.push_back((v.back() - 1) / 2);
  return v;
}

template <typename T>
int solve_mg_2d(int64_t nx, int64_t ny, double h, const double* f, const double* bc, const double* x0,
                int64_t tx, int64_t ty, const MgOpts& o, double omega, int max_levels, double tol,
                int tol_mode, double ref_residual, int64_t max_cycles, double* x_out, double* hist,
                int64_t* cycles, int* converged, int* levels_out) {
  const std::vector<int64_t> sx = mg_sizes(nx, max_levels), sy = mg_sizes(ny, max_levels);
  const size_t L = std::min(sx.size(), sy.size());
  if (L < 2) return ST_INVALID;
  std::vector<MgLevel2D<T>> Ls(L);
  for (size_t l = 0; l < L; ++l) {
    MgLevel2D<T>& V = Ls[l];
    V.p.nx = sx[l];
    V.p.ny = sy[l];
    const double hl = h * (double)(int64_t(1) << l);
    V.p.h2 = hl * hl;
    V.p.omega = (T)omega;
    V.p.h2f.assign(V.p.nx * V.p.ny, T(0));
    V.p.h2f64.assign(V.p.nx * V.p.ny, 0.0);
    V.bx = block_plan(V.p.nx, std::min<int64_t>(tx, V.p.nx), 0);
    V.by = block_plan(V.p.ny, std::min<int64_t>(ty, V.p.ny), 0);
    V.x.assign((V.p.nx + 2) * (V.p.ny + 2), T(0));
  }
  Problem2D<T>& p = Ls[0].p;
  for (int64_t q = 0; q < nx * ny; ++q) {
    p.h2f[q] = (T)(p.h2 * f[q]);
    p.h2f64[q] = (double)p.h2f[q];
  }
  std::vector<T>& xa = Ls[0].x;
  if (bc) {
    for (int64_t i = 1; i <= nx; ++i) {
      xa[at(p, i, 0)] = (T)bc[i - 1];
      xa[at(p, i, ny + 1)] = (T)bc[nx + i - 1];
    }
    for (int64_t j = 1; j <= ny; ++j) {
      xa[at(p, 0, j)] = (T)bc[2 * nx + j - 1];
      xa[at(p, nx + 1, j)] = (T)bc[2 * nx + ny + j - 1];
    }
  }
  for (auto& V : Ls) V.y = V.x;  // both arrays carry the ring
  for (int64_t j = 1; j <= ny; ++j)
    for (int64_t i = 1; i <= nx; ++i) xa[at(p, i, j)] = x0 ? (T)x0[(j - 1) * nx + (i - 1)] : T(0);
  auto cycle = [&]() { vcycle_2d(Ls, 0, o); };
  auto resid = [&]() { return residual_sq_2d(Ls[0].p, Ls[0].x); };
  DriverOut d = drive(p.h2, tol, tol_mode, ref_residual, max_cycles, hist, cycle, resid);
  for (int64_t j = 1; j <= ny; ++j)
    for (int64_t i = 1; i <= nx; ++i) x_out[(j - 1) * nx + (i - 1)] = (double)Ls[0].x[at(p, i, j)];
  *cycles = d.cycles;
  *converged = d.converged;
  *levels_out = (int)L;
  return d.status;
}

template <typename T>
struct MgLevel1D {
  Problem1D<T> p;
  BlockPlan bp;
  std::vector<T> x, y;
};

template <typename T>
void mg_smooth_1d(MgLevel1D<T>& L, int k, int cycles, bool weighted) {
  L.p.weighted = weighted;
  for (int c = 0; c < cycles; ++c) {
    hier_cycle_1d(L.p, L.bp, k, 0, L.x, L.y);
    std::swap(L.x, L.y);
  }
}

template <typename T>
void mg_restrict_1d(const MgLevel1D<T>& F, MgLevel1D<T>& C) {
  const std::vector<T>& x = F.x;
  auto s = [&](int64_t i) {
    return resid1d((double)x[i], (double)x[i - 1], (double)x[i + 1], F.p.h2f64[i - 1]);
  };
  for (int64_t I = 1; I <= C.p.n; ++I) {
    const int64_t i = 2 * I;
    const T v = (T)(2.0 * s(i) + (s(i - 1) + s(i + 1)));
    C.p.h2f[I - 1] = v;
    C.p.h2f64[I - 1] = (double)v;
    C.x[I] = T(0);
  }
}

template <typename T>
void mg_correct_1d(MgLevel1D<T>& F, const MgLevel1D<T>& C) {
  for (int64_t i = 1; i <= F.p.n; ++i) {
    const T v = (i % 2) == 0 ? C.x[i / 2] : T(0.5) * (C.x[(i - 1) / 2] + C.x[(i + 1) / 2]);
    F.x[i] = F.x[i] + v;
  }
}

template <typename T>
void vcycle_1d(std::vector<MgLevel1D<T>>& Ls, size_t l, const MgOpts& o) {
  MgLevel1D<T>& L = Ls[l];
  if (l + 1 == Ls.size()) {
    mg_smooth_1d(L, o.k, o.coarse_cycles, false);
    return;
  }
  mg_smooth_1d(L, o.k, o.nu1, true);
  mg_restrict_1d(L, Ls[l + 1]);
  vcycle_1d(Ls, l + 1, o);
  mg_correct_1d(L, Ls[l + 1]);
  mg_smooth_1d(L, o.k, o.nu2, true);
}

// ny independent problems (the batch of NEXT #2), each with its own level hierarchy; one solver
// cycle = one V-cycle of every problem; the stopping test uses the stacked residual.
template <typename T>
int solve_mg_1d(int64_t n, int64_t batch, double h, const double* f, const double* bc, const double* x0,
                int64_t tile, const MgOpts& o, double omega, int max_levels, double tol, int tol_mode,
                double ref_residual, int64_t max_cycles, double* x_out, double* hist, int64_t* cycles,
                int* converged, int* levels_out) {
  const std::vector<int64_t> sz = mg_sizes(n, max_levels);
  const size_t L = sz.size();
  if (L < 2) return ST_INVALID;
  std::vector<std::vector<MgLevel1D<T>>> pb(batch, std::vector<MgLevel1D<T>>(L));
  for (int64_t b = 0; b < batch; ++b)
    for (size_t l = 0; l < L; ++l) {
      MgLevel1D<T>& V = pb[b][l];
      V.p.n = sz[l];
      const double hl = h * (double)(int64_t(1) << l);
      V.p.h2 = hl * hl;
      V.p.omega = (T)omega;
      V.p.h2f.assign(V.p.n, T(0));
      V.p.h2f64.assign(V.p.n, 0.0);
      V.bp = block_plan(V.p.n, std::min<int64_t>(tile, V.p.n), 0);
      V.x.assign(V.p.n + 2, T(0));
      if (l == 0) {
        for (int64_t i = 0; i < n; ++i) {
          V.p.h2f[i] = (T)(V.p.h2 * f[b * n + i]);
          V.p.h2f64[i] = (double)V.p.h2f[i];
        }
        V.x[0] = bc ? (T)bc[2 * b] : T(0);
        V.x[n + 1] = bc ? (T)bc[2 * b + 1] : T(0);
      }
      V.y = V.x;
      if (l == 0)
        for (int64_t i = 0; i < n; ++i) V.x[i + 1] = x0 ? (T)x0[b * n + i] : T(0);
    }
  auto cycle = [&]() {
    for (int64_t b = 0; b < batch; ++b) vcycle_1d(pb[b], 0, o);
  };
  auto resid = [&]() {
    double S = 0.0;
    for (int64_t b = 0; b < batch; ++b) S += residual_sq_1d(pb[b][0].p, pb[b][0].x);
    return S;
  };
  DriverOut d = drive(h * h, tol, tol_mode, ref_residual, max_cycles, hist, cycle, resid);
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t i = 0; i < n; ++i) x_out[b * n + i] = (double)pb[b][0].x[i + 1];
  *cycles = d.cycles;
  *converged = d.converged;
  *levels_out = (int)L;
  return d.status;
}

}  // namespace

extern "C" {

// Solve -Δu = f with classic (mode 1) or hierarchical (mode 0) Jacobi.
// dim 1: ny = number of independent problems (1 = a single problem), tile_y ignored;
// bc = [left_0, right_0, left_1, right_1, ...].  dtype 0 = double, 1 = float.
// x_out: nx*ny doubles.  hist: max_cycles+1 doubles or NULL.
// Returns 0 converged, 1 not converged, 2 invalid argument, 4 non-finite residual.
// overlap_x/overlap_y: the paper's o (even, 0 <= o < tile).
// stencil: NULL (Poisson) or the general coefficients (see solve1d / solve2d; reading c23);
// every d must be finite and non-zero.
int hjo_solve(int dim, int64_t nx, int64_t ny, double h, const double* f, const double* bc,
              const double* x0, const double* stencil, int mode, int dtype, int64_t tile_x,
              int64_t tile_y, int64_t overlap_x, int64_t overlap_y, int k, double tol, int tol_mode,
              double ref_residual, int64_t max_cycles, int tile_order, double* x_out, double* hist,
              int64_t* cycles, int* converged) {
  if (!f || !x_out || !cycles || !converged) return ST_INVALID;
  if (nx < 1 || ny < 1 || max_cycles < 0) return ST_INVALID;
  if (!stencil && (!(h > 0.0) || !std::isfinite(h))) return ST_INVALID;
  if (stencil) {
    const int64_t ns = dim == 1 ? 3 * nx * ny : 5;
    for (int64_t q = 0; q < ns; ++q)
      if (!std::isfinite(stencil[q])) return ST_INVALID;
    if (dim == 1) {
      for (int64_t q = 0; q < nx * ny; ++q)
        if (stencil[nx * ny + q] == 0.0) return ST_INVALID;
    } else if (stencil[4] == 0.0) {
      return ST_INVALID;
    }
  }
  if (mode != 0 && mode != 1) return ST_INVALID;
  if (mode == 0 && (k < 1 || tile_x < 1 || tile_x > nx)) return ST_INVALID;
  if (mode == 0 && (overlap_x < 0 || overlap_x % 2 != 0 || overlap_x >= tile_x)) return ST_INVALID;
  if (dim == 1) {  // ny = number of independent problems (batch)
    if (dtype == 0)
      return solve1d<double>(nx, ny, h, f, bc, x0, stencil, mode, tile_x, overlap_x, k, tol, tol_mode,
                             ref_residual, max_cycles, tile_order, x_out, hist, cycles, converged);
    return solve1d<float>(nx, ny, h, f, bc, x0, stencil, mode, tile_x, overlap_x, k, tol, tol_mode,
                          ref_residual, max_cycles, tile_order, x_out, hist, cycles, converged);
  }
  if (dim == 2) {
    if (mode == 0 && (tile_y < 1 || tile_y > ny)) return ST_INVALID;
    if (mode == 0 && (overlap_y < 0 || overlap_y % 2 != 0 || overlap_y >= tile_y)) return ST_INVALID;
    if (dtype == 0)
      return solve2d<double>(nx, ny, h, f, bc, x0, stencil, mode, tile_x, tile_y, overlap_x, overlap_y,
                             k, tol, tol_mode, ref_residual, max_cycles, tile_order, x_out, hist,
                             cycles, converged);
    return solve2d<float>(nx, ny, h, f, bc, x0, stencil, mode, tile_x, tile_y, overlap_x, overlap_y, k,
                          tol, tol_mode, ref_residual, max_cycles, tile_order, x_out, hist, cycles,
                          converged);
  }
  return ST_INVALID;
}

// The block plan of one dimension (1-based, inclusive ranges); returns the block count, fills
// at most cap entries of each output array.  -1 on invalid input.
int64_t hjo_block_plan(int64_t n, int64_t tile, int64_t overlap, int64_t cap, int64_t* start,
                       int64_t* width, int64_t* own_lo, int64_t* own_hi) {
  if (n < 1 || tile < 1 || tile > n || overlap < 0 || overlap % 2 != 0 || overlap >= tile) return -1;
  const BlockPlan P = block_plan(n, tile, overlap);
  const int64_t nb = (int64_t)P.start.size();
  for (int64_t b = 0; b < nb && b < cap; ++b) {
    start[b] = P.start[b];
    width[b] = P.width[b];
    own_lo[b] = P.own_lo[b];
    own_hi[b] = P.own_hi[b];
  }
  return nb;
}

// ||f - A x||_2 for interior x (double), A = (1/h^2) * stencil, ring from bc.
double hjo_residual(int dim, int64_t nx, int64_t ny, double h, const double* f, const double* bc,
                    const double* x) {
  const double h2 = h * h;
  if (dim == 1) {  // ny independent problems
    double S = 0.0;
    for (int64_t b = 0; b < ny; ++b) {
      Problem1D<double> p;
      p.n = nx;
      p.h2 = h2;
      p.h2f64.resize(nx);
      for (int64_t i = 0; i < nx; ++i) p.h2f64[i] = h2 * f[b * nx + i];
      std::vector<double> xx(nx + 2);
      xx[0] = bc ? bc[2 * b] : 0.0;
      xx[nx + 1] = bc ? bc[2 * b + 1] : 0.0;
      for (int64_t i = 0; i < nx; ++i) xx[i + 1] = x[b * nx + i];
      S += residual_sq_1d(p, xx);
    }
    return std::sqrt(S) / h2;
  }
  Problem2D<double> p;
  p.nx = nx;
  p.ny = ny;
  p.h2 = h2;
  p.h2f64.resize(nx * ny);
  for (int64_t q = 0; q < nx * ny; ++q) p.h2f64[q] = h2 * f[q];
  std::vector<double> xx((nx + 2) * (ny + 2), 0.0);
  if (bc) {
    for (int64_t i = 1; i <= nx; ++i) {
      xx[at(p, i, 0)] = bc[i - 1];
      xx[at(p, i, ny + 1)] = bc[nx + i - 1];
    }
    for (int64_t j = 1; j <= ny; ++j) {
      xx[at(p, 0, j)] = bc[2 * nx + j - 1];
      xx[at(p, nx + 1, j)] = bc[2 * nx + ny + j - 1];
    }
  }
  for (int64_t j = 1; j <= ny; ++j)
    for (int64_t i = 1; i <= nx; ++i) xx[at(p, i, j)] = x[(j - 1) * nx + (i - 1)];
  return std::sqrt(residual_sq_2d(p, xx)) / h2;
}

// The general-coefficient residual by its plain definition (reading c23), in double from the
// coefficients themselves (not the rounded weights): 2D ||b - Ax||_2 with
// (Ax)_ij = a x_{i-1,j} + c x_{i+1,j} + e x_{i,j-1} + f x_{i,j+1} + d x_ij (Eq. 10's matrix);
// 1D ||D^{-1}(b - Ax)||_2 with (Ax)_i = a_i x_{i-1} + d_i x_i + c_i x_{i+1} (Eq. 4's matrix),
// over ny independent problems.  Ring values from bc as in hjo_solve.
double hjo_residual_general(int dim, int64_t nx, int64_t ny, const double* f, const double* bc,
                            const double* x, const double* stencil) {
  double S = 0.0;
  if (dim == 1) {
    const int64_t nt = nx * ny;
    for (int64_t b = 0; b < ny; ++b)
      for (int64_t i = 0; i < nx; ++i) {
        const int64_t g = b * nx + i;
        const double xl = i > 0 ? x[g - 1] : (bc ? bc[2 * b] : 0.0);
        const double xr = i < nx - 1 ? x[g + 1] : (bc ? bc[2 * b + 1] : 0.0);
        const double ax = stencil[g] * xl + stencil[nt + g] * x[g] + stencil[2 * nt + g] * xr;
        const double r = (f[g] - ax) / stencil[nt + g];
        S += r * r;
      }
    return std::sqrt(S);
  }
  auto val = [&](int64_t i, int64_t j) -> double {  // 0-based interior, -1 / n = ring
    if (i >= 0 && i < nx && j >= 0 && j < ny) return x[j * nx + i];
    if (!bc) return 0.0;
    if (j < 0) return bc[i];
    if (j >= ny) return bc[nx + i];
    if (i < 0) return bc[2 * nx + j];
    return bc[2 * nx + ny + j];
  };
  for (int64_t j = 0; j < ny; ++j)
    for (int64_t i = 0; i < nx; ++i) {
      const double ax = stencil[0] * val(i - 1, j) + stencil[1] * val(i + 1, j) +
                        stencil[2] * val(i, j - 1) + stencil[3] * val(i, j + 1) +
                        stencil[4] * x[j * nx + i];
      const double r = f[j * nx + i] - ax;
      S += r * r;
    }
  return std::sqrt(S);
}

// Resource figures (o = 0):
//   tiles   = ceil(nx/Tx) [* ceil(ny/Ty)]            (Eq. 8/13 at o=0)
//   threads = tiles * Tx [* Ty]                       (Eq. 9/14 at o=0: one thread per DOF)
//   smem    = 8 * (2*(Tx+2) + Tx)            1D       (PAPER.md:175; 800 B at Tx=32, :215)
//           = 8 * (2*(Tx+2)*(Ty+2) + Tx*Ty)  2D       (PAPER.md:389; 26,688 B at 32x32, :425)
// bytes_per_value lets fp32 report 4-byte figures ("4 bytes for floats").
// With overlap o (PAPER.md:293-305, Eqs. 7-9; :491-508, Eqs. 12-14): operational blocks =
// (N - o)/(tpb - o) per dimension (ceiling when inexact = the plan's length), threads =
// blocks * tpb.
int hjo_resource_figures(int dim, int64_t nx, int64_t ny, int64_t tx, int64_t ty, int64_t ox,
                         int64_t oy, int64_t bytes_per_value, int64_t* tiles, int64_t* threads,
                         int64_t* smem) {
  if (tx < 1 || tx > nx || ox < 0 || ox % 2 != 0 || ox >= tx) return ST_INVALID;
  if (dim == 1) {  // ny independent problems: blocks for all of them
    *tiles = (int64_t)block_plan(nx, tx, ox).start.size() * ny;
    *threads = *tiles * tx;
    *smem = bytes_per_value * (2 * (tx + 2) + tx);
    return ST_OK;
  }
  if (dim != 2 || ty < 1 || ty > ny || oy < 0 || oy % 2 != 0 || oy >= ty) return ST_INVALID;
  *tiles = (int64_t)(block_plan(nx, tx, ox).start.size() * block_plan(ny, ty, oy).start.size());
  *threads = *tiles * tx * ty;
  *smem = bytes_per_value * (2 * (tx + 2) * (ty + 2) + tx * ty);
  return ST_OK;
}

// Multigrid with the hierarchical cycle as smoother (reading c24; see vcycle_2d / vcycle_1d).
// Poisson only (no stencil), overlap 0.  dim 1: ny independent problems.  Returns like
// hjo_solve; *levels_out = number of grid levels (>= 2, else ST_INVALID).
int hjo_solve_mg(int dim, int64_t nx, int64_t ny, double h, const double* f, const double* bc,
                 const double* x0, int dtype, int64_t tile_x, int64_t tile_y, int k, int nu1, int nu2,
                 double omega, int coarse_cycles, int max_levels, double tol, int tol_mode,
                 double ref_residual, int64_t max_cycles, double* x_out, double* hist, int64_t* cycles,
                 int* converged, int* levels_out) {
  if (!f || !x_out || !cycles || !converged || !levels_out) return ST_INVALID;
  if (nx < 1 || ny < 1 || max_cycles < 0 || !(h > 0.0) || !std::isfinite(h)) return ST_INVALID;
  if (k < 1 || nu1 < 0 || nu2 < 0 || nu1 + nu2 < 1 || coarse_cycles < 1) return ST_INVALID;
  if (!(omega > 0.0) || omega > 1.0 || tile_x < 1 || (dim == 2 && tile_y < 1)) return ST_INVALID;
  const MgOpts o{k, nu1, nu2, coarse_cycles};
  if (dim == 1) {
    if (dtype == 0)
      return solve_mg_1d<double>(nx, ny, h, f, bc, x0, tile_x, o, omega, max_levels, tol, tol_mode,
                                 ref_residual, max_cycles, x_out, hist, cycles, converged, levels_out);
    return solve_mg_1d<float>(nx, ny, h, f, bc, x0, tile_x, o, omega, max_levels, tol, tol_mode,
                              ref_residual, max_cycles, x_out, hist, cycles, converged, levels_out);
  }
  if (dim != 2) return ST_INVALID;
  if (dtype == 0)
    return solve_mg_2d<double>(nx, ny, h, f, bc, x0, tile_x, tile_y, o, omega, max_levels, tol, tol_mode,
                               ref_residual, max_cycles, x_out, hist, cycles, converged, levels_out);
  return solve_mg_2d<float>(nx, ny, h, f, bc, x0, tile_x, tile_y, o, omega, max_levels, tol, tol_mode,
                            ref_residual, max_cycles, x_out, hist, cycles, converged, levels_out);
}

// The two grid-transfer steps alone, in double (for the pins): op 0 = restriction — coarse
// h2f (nxc*nyc, or nxc per problem in 1D) of the fine iterate x (interior, nx*ny) with ring bc
// (NULL = 0) and rhs h2f = h^2 f (h = 1: f itself); op 1 = correction — x + P e for the coarse
// interior e.  Returns the number of values written to out, or -1.
int64_t hjo_mg_transfer(int dim, int op, int64_t nx, int64_t ny, const double* x, const double* bc,
                        const double* a, double* out) {
  if (nx < 3 || (nx % 2) == 0 || (dim == 2 && (ny < 3 || (ny % 2) == 0)) || ny < 1) return -1;
  const int64_t nxc = (nx - 1) / 2;
  if (dim == 1) {
    int64_t w = 0;
    for (int64_t b = 0; b < ny; ++b) {
      MgLevel1D<double> F, C;
      F.p.n = nx;
      F.p.h2 = 1.0;
      F.x.assign(nx + 2, 0.0);
      F.x[0] = bc ? bc[2 * b] : 0.0;
      F.x[nx + 1] = bc ? bc[2 * b + 1] : 0.0;
      for (int64_t i = 0; i < nx; ++i) F.x[i + 1] = x[b * nx + i];
      C.p.n = nxc;
      C.p.h2f.assign(nxc, 0.0);
      C.p.h2f64.assign(nxc, 0.0);
      C.x.assign(nxc + 2, 0.0);
      if (op == 0) {
        F.p.h2f64.assign(a + b * nx, a + (b + 1) * nx);
        mg_restrict_1d(F, C);
        for (int64_t I = 0; I < nxc; ++I) out[w++] = C.p.h2f64[I];
      } else {
        for (int64_t I = 0; I < nxc; ++I) C.x[I + 1] = a[b * nxc + I];
        mg_correct_1d(F, C);
        for (int64_t i = 0; i < nx; ++i) out[w++] = F.x[i + 1];
      }
    }
    return w;
  }
  const int64_t nyc = (ny - 1) / 2;
  MgLevel2D<double> F, C;
  F.p.nx = nx;
  F.p.ny = ny;
  F.p.h2 = 1.0;
  F.x.assign((nx + 2) * (ny + 2), 0.0);
  if (bc) {
    for (int64_t i = 1; i <= nx; ++i) {
      F.x[at(F.p, i, 0)] = bc[i - 1];
      F.x[at(F.p, i, ny + 1)] = bc[nx + i - 1];
    }
    for (int64_t j = 1; j <= ny; ++j) {
      F.x[at(F.p, 0, j)] = bc[2 * nx + j - 1];
      F.x[at(F.p, nx + 1, j)] = bc[2 * nx + ny + j - 1];
    }
  }
  for (int64_t j = 1; j <= ny; ++j)
    for (int64_t i = 1; i <= nx; ++i) F.x[at(F.p, i, j)] = x[(j - 1) * nx + (i - 1)];
  C.p.nx = nxc;
  C.p.ny = nyc;
  C.p.h2f.assign(nxc * nyc, 0.0);
  C.p.h2f64.assign(nxc * nyc, 0.0);
  C.x.assign((nxc + 2) * (nyc + 2), 0.0);
  if (op == 0) {
    F.p.h2f64.assign(a, a + nx * ny);
    mg_restrict_2d(F, C);
    std::copy(C.p.h2f64.begin(), C.p.h2f64.end(), out);
    return nxc * nyc;
  }
  for (int64_t J = 1; J <= nyc; ++J)
    for (int64_t I = 1; I <= nxc; ++I) C.x[at(C.p, I, J)] = a[(J - 1) * nxc + (I - 1)];
  mg_correct_2d(F, C);
  for (int64_t j = 1; j <= ny; ++j)
    for (int64_t i = 1; i <= nx; ++i) out[(j - 1) * nx + (i - 1)] = F.x[at(F.p, i, j)];
  return nx * ny;
}

}  // extern "C"
