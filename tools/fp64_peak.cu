// FP64 FMA throughput of this B200 (the FP64 roofline denominator for the
// face kernels, which MEASURED_PEAKS.json does not carry): 8 independent
// FMA chains per thread, 148 x 8 CTAs of 256 threads, best of 10 timed runs.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_fma(double* out, int iters, double a, double b) {
  double r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = fma(r[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += r[k];
  if (s == 12345.678) out[0] = s;  // keeps the chains live
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount, blocks = sms * 8, threads = 256, iters = 1 << 14;
  double* out;
  cudaMalloc(&out, sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 13; ++rep) {
    cudaEventRecord(e0);
    k_fma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep >= 3 && ms < best) best = ms;
  }
  const double flops = 2.0 * 8.0 * iters * (double)blocks * threads;
  printf("{\"fp64_tflops\": %.3f, \"sms\": %d, \"ms\": %.4f, \"how\": \"8 FMA chains/thread, %d x %d threads, best of 10\"}\n",
         flops / (best * 1e-3) / 1e12, sms, best, blocks, threads);
  return 0;
}
