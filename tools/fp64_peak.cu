// tools/fp64_peak.cu — DFMA throughput microbenchmark (the FP64 roofline denominator).
// Each thread runs 8 independent FMA chains (enough ILP to cover the DFMA latency), the grid is
// a multiple of 148 SMs x full occupancy.  flops = 2 per DFMA.  Timed with CUDA events after
// warm-up; prints one JSON line.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_chains(double* out, long long iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-9, x2 = x0 + 2e-9, x3 = x0 + 3e-9;
  double x4 = x0 + 4e-9, x5 = x0 + 5e-9, x6 = x0 + 6e-9, x7 = x0 + 7e-9;
  for (long long i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[blockIdx.x] = s;  // keep the chains alive
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 1 << 20);
  const int threads = 256, blocks = sms * 8;
  const long long iters = 4000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) dfma_chains<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    dfma_chains<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
  printf("{\"fp64_tflops\": %.4f, \"sms\": %d, \"clock_mhz_attr\": %d, \"best_ms\": %.4f, \"how\": "
         "\"DFMA 8 independent chains/thread, %d x %d threads, best of 10, CUDA events\"}\n",
         flops / (best * 1e-3) / 1e12, sms, clk / 1000, best, blocks, threads);
  return 0;
}
