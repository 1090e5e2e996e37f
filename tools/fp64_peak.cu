// FP64 DFMA peak of this B200 (the ALU roofline denominator for the FP64 kernels).
// Each thread runs 16 independent FMA chains (enough ILP to cover the DFMA latency) for `iters`
// steps; grid = 148 SMs x 8 CTAs x 256 threads.  FLOPs = 2 per FMA.  CUDA events, best of 5.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 16; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 16; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;   // keeps the chains live
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 1 << 14, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int per : {4, 8}) {
    const int blocks = sms * per;
    k_dfma<<<blocks, threads>>>(out, 64, 0.999999, 1e-7);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double flops = 2.0 * 16 * (double)iters * threads * blocks;
    const double tf = flops / (best * 1e-3) / 1e12;
    printf("{\"ctas_per_sm\": %d, \"sms\": %d, \"ms\": %.4f, \"fp64_tflops\": %.3f, \"fma_per_clk_per_sm_at_max_clock\": %.2f, "
           "\"clock_rate_khz\": %d}\n",
           per, sms, best, tf, tf * 1e12 / 2 / sms / (clk * 1e3), clk);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
