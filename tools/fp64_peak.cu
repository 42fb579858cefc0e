// FP64 FMA throughput of one B200 (the roofline of the ALU-bound setup
// kernels).  Every thread runs 8 independent DFMA chains; grid = 4 x SM count x 1024
// threads.  Prints one JSON line: TFLOP/s (2 flops per FMA), measured with CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
         x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
  if (s == 12345.678) out[threadIdx.x] = s;   // keep the chains live
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  const int threads = 1024, blocks = 4 * sms, iters = 2048;
  k_dfma<<<blocks, threads>>>(out, 64, 0.999999, 1e-7);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double fmas = (double)blocks * threads * iters * 16 * 8;
  const double tflops = 2.0 * fmas / (best * 1e-3) / 1e12;
  printf("{\"fp64_fma_tflops\": %.3f, \"ms\": %.3f, \"sms\": %d, \"sm_clock_khz_attr\": %d, "
         "\"how\": \"tools/fp64_peak.cu: %d blocks x %d threads x 8 independent DFMA chains, best of 5\"}\n",
         tflops, best, sms, clk, blocks, threads);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
