// Scratch micro-benchmark (not part of libhj.so): the achievable FP64 instruction rate of one B200 for
// the stencil's instruction mix (3 DADD : 1 DFMA, independent chains, operands in registers, no
// memory traffic), 8 / 12 / 16 warps per SM — the measured FP64 ceiling the cycle kernel's
// fp64_pipe_frac is read against.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64peak scripts/fp64peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH, int MIX>
__global__ void fp64mix(double* out, int iters, double a, long long* clk) {
  double v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = threadIdx.x * 1e-3 + c;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (MIX == 0) {               // 3 DADD + 1 DFMA per "update"
        v[c] = __dadd_rn(v[c], a);
        v[c] = __dadd_rn(v[c], a);
        v[c] = __dadd_rn(v[c], a);
        v[c] = __fma_rn(v[c], 0.25, a);
      } else {                      // DFMA only
        v[c] = __fma_rn(v[c], 0.999, a);
        v[c] = __fma_rn(v[c], 0.999, a);
        v[c] = __fma_rn(v[c], 0.999, a);
        v[c] = __fma_rn(v[c], 0.999, a);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = clock64() - t0;
}

template <int CH, int MIX>
void run(const char* name, int warps, double* out, long long* clk, int nsm) {
  const int iters = 4096;
  for (int r = 0; r < 2; ++r) fp64mix<CH, MIX><<<nsm, warps * 32>>>(out, iters, 1e-9, clk);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  fp64mix<CH, MIX><<<nsm, warps * 32>>>(out, iters, 1e-9, clk);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long c;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  const double ops = (double)nsm * warps * 32 * iters * CH * 4;
  const double mhz = c / (ms * 1e-3) / 1e6;
  printf("%-14s chains %2d warps/SM %2d: %.3e FP64 ops/s = %.1f ops/clk/SM at %.0f MHz (%.3f of 64)\n", name, CH,
         warps, ops / (ms * 1e-3), ops / (ms * 1e-3) / nsm / (mhz * 1e6), mhz,
         ops / (ms * 1e-3) / nsm / (mhz * 1e6) / 64.0);
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  long long* clk;
  cudaMalloc(&out, (size_t)nsm * 1024 * 8);
  cudaMalloc(&clk, 8);
  for (int w : {4, 8, 12, 16, 32}) {
    run<8, 0>("3dadd+1dfma", w, out, clk, nsm);
    run<16, 0>("3dadd+1dfma", w, out, clk, nsm);
    run<8, 1>("dfma", w, out, clk, nsm);
  }
  return 0;
}
