// Scratch micro-benchmark (not part of libhj.so): dependent-chain latencies on one B200 warp — DADD,
// DFMA, the 1D update (DADD -> DFMA), 32-bit SHFL, a 64-bit shuffle (2 SHFL) feeding a DADD, and a
// 4-warp __syncthreads — the constants that bound the resident small-problem solvers (res1w / res1c,
// config 1: a cycle is a chain of k dependent sub-iterations).  Cycles per link, clock64 over 4096 links.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o latbench scripts/latbench.cu && ./latbench
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, int iters, double a, long long* clk) {
  double v = threadIdx.x * 1e-3 + 1.0;
  float f = (float)v;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (OP == 0) v = __dadd_rn(v, a);
    if (OP == 1) v = __fma_rn(v, 0.999, a);
    if (OP == 2) v = __fma_rn(0.5, __dadd_rn(v, a), a);                       // the 1D update
    if (OP == 3) f = __shfl_down_sync(0xffffffffu, f, 1) + 0.0f * it;          // SHFL (+ FADD)
    if (OP == 4) v = __dadd_rn(__shfl_down_sync(0xffffffffu, v, 1), a);        // 64-bit shuffle + DADD
    if (OP == 5) { v = __dadd_rn(v, a); __syncthreads(); }                     // DADD + CTA barrier
    if (OP == 6) f = __fadd_rn(f, (float)a);                                   // FADD
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *clk = t1 - t0;
  out[threadIdx.x] = v + f;
}

// res1w-like cycle (C = 8 points per lane, tiles of 4 lanes, k = 16 as 8 pairs, residual butterfly
// spread over the pairs, a uniform decision per cycle): cycles per solver cycle
__global__ void res1w_like(double* out, int cycles, long long* clk) {
  const unsigned F = 0xffffffffu;
  const int lane = threadIdx.x;
  double x[8], q[8];
  for (int c = 0; c < 8; ++c) { x[c] = 1.0 + lane * 8 + c; q[c] = 1e-3 * c; }
  const bool t0 = lane % 4 == 0, t1 = lane % 4 == 3;
  const double qgl = __shfl_up_sync(F, q[7], 1), qgr = __shfl_down_sync(F, q[0], 1);
  double tot = 0.0;
  long long t_0 = clock64();
  for (int cyc = 0; cyc < cycles; ++cyc) {
    double hl = __shfl_up_sync(F, x[7], 1), hr = __shfl_down_sync(F, x[0], 1);
    double acc = 0.0;
    int step = 16;
#pragma unroll 1
    for (int s = 0; s < 16; s += 2) {
      double g1 = __shfl_up_sync(F, x[7], 1), g2 = __shfl_up_sync(F, x[6], 1);
      double h0 = __shfl_down_sync(F, x[0], 1), h1 = __shfl_down_sync(F, x[1], 1);
      g1 = t0 ? hl : g1;
      h0 = t1 ? hr : h0;
      const double gn = t0 ? hl : __fma_rn(0.5, __dadd_rn(g2, x[0]), qgl);
      const double hn = t1 ? hr : __fma_rn(0.5, __dadd_rn(x[7], h1), qgr);
      for (int pass = 0; pass < 2; ++pass) {
        double prev = pass ? gn : g1;
        const double R = pass ? hn : h0;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const double Rc = c == 7 ? R : x[c + 1];
          const double nv = __fma_rn(0.5, __dadd_rn(prev, Rc), q[c]);
          if (s == 0 && pass == 0) acc = __fma_rn(nv, nv, acc);
          prev = x[c];
          x[c] = nv;
        }
      }
      if (step) { acc += __shfl_xor_sync(F, acc, step); step >>= 1; }
    }
    for (; step; step >>= 1) acc += __shfl_xor_sync(F, acc, step);
    const double S = __shfl_sync(F, acc, 0);
    tot += S;
    if (S < -1.0) break;  // uniform, never taken
  }
  long long t_1 = clock64();
  if (lane == 0) *clk = t_1 - t_0;
  out[lane] = tot + x[0];
}

int main() {
  double* out; long long* clk;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMalloc(&clk, sizeof(long long));
  const char* names[] = {"DADD", "DFMA", "DADD->DFMA (1D update)", "SHFL.32 (+FADD)", "SHFL.64->DADD",
                         "DADD + __syncthreads (128 thr)", "FADD"};
  const int iters = 4096;
  for (int op = 0; op < 7; ++op) {
    const int thr = op == 5 ? 128 : 32;
    long long c = 0;
    for (int rep = 0; rep < 3; ++rep) {
      switch (op) {
        case 0: chain<0><<<1, thr>>>(out, iters, 1e-9, clk); break;
        case 1: chain<1><<<1, thr>>>(out, iters, 1e-9, clk); break;
        case 2: chain<2><<<1, thr>>>(out, iters, 1e-9, clk); break;
        case 3: chain<3><<<1, thr>>>(out, iters, 1e-9, clk); break;
        case 4: chain<4><<<1, thr>>>(out, iters, 1e-9, clk); break;
        case 5: chain<5><<<1, thr>>>(out, iters, 1e-9, clk); break;
        case 6: chain<6><<<1, thr>>>(out, iters, 1e-9, clk); break;
      }
      cudaMemcpy(&c, clk, sizeof(c), cudaMemcpyDeviceToHost);
    }
    printf("%-32s %.2f cycles per link\n", names[op], (double)c / iters);
  }
  {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    long long c = 0;
    const int cycles = 20000;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      res1w_like<<<1, 32>>>(out, cycles, clk);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaMemcpy(&c, clk, sizeof(c), cudaMemcpyDeviceToHost);
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-32s %.1f cycles per solver cycle, %.3f us per solver cycle, effective SM clock %.0f MHz\n",
           "res1w-like cycle (C=8, k=16)", (double)c / cycles, ms * 1e3 / cycles, (double)c / (ms * 1e3));
  }
  return 0;
}
