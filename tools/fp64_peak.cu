// Microbenchmark: sustained fp64 DFMA throughput on all SMs (roofline denominator for fp64-bound kernels).
// Also prints device properties relevant to the design (SMs, L2, smem).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_chain(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3,
         x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("name=%s sms=%d l2=%d smem_per_block_optin=%zu smem_per_sm=%zu regs_per_sm=%d clock_khz=%d\n",
         p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin,
         p.sharedMemPerMultiprocessor, p.regsPerMultiprocessor, p.clockRate);
  double* d; cudaMalloc(&d, 8);
  int iters = 20000;
  for (int threads : {128, 256, 512}) for (int bps : {4, 8}) {
    int blocks = p.multiProcessorCount * bps * 256 / threads;
    dfma_chain<<<blocks, threads>>>(d, 100, 0.999999, 1e-7);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    dfma_chain<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("threads=%d blocks=%d time=%.3f ms  fp64=%.2f TFLOP/s\n", threads, blocks, ms, flops / ms / 1e9);
  }
  return 0;
}
