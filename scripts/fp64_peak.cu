// FP64 DFMA throughput microbenchmark (roofline denominator for the FP64 pipe).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/fp64_peak.cu -o /tmp/fp64_peak && /tmp/fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, int iters, double s) {
  double a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-9 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], s, 1e-7);
  }
  double r = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) r += a[j];
  if (r == 12345.0) out[0] = r;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 1 << 16, blocks = sms * 8, threads = 256;
  k<<<blocks, threads>>>(out, 256, 0.999999);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k<<<blocks, threads>>>(out, iters, 0.999999);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  double flops = 2.0 * 8 * (double)iters * blocks * threads;
  printf("{\"fp64_dfma_tflops\": %.2f, \"sms\": %d, \"ms\": %.3f}\n", flops / best / 1e9, sms, best);
  return 0;
}
