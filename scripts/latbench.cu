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
  return 0;
}
