// Microbenchmark: fp64 tensor-core MMA (mma.sync.aligned.m8n8k4 f64, DMMA) vs the
// DFMA peak on this B200.  Each warp runs independent chains of m8n8k4 MMAs on register tiles;
// flops = 2*8*8*4 per MMA.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* sink, long long iters) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-6;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (long long it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* sink;
  cudaMalloc(&sink, 1 << 26);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const long long iters = 20000;
  for (int threads : {128, 256, 512}) {
    for (int blocks_per_sm : {1, 2, 4}) {
      const int blocks = 148 * blocks_per_sm;
      k<8><<<blocks, threads>>>(sink, 100);
      cudaEventRecord(e0);
      k<8><<<blocks, threads>>>(sink, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double flops = double(blocks) * (threads / 32) * iters * 8 * 2.0 * 8 * 8 * 4;
      printf("DMMA m8n8k4: threads=%d blocks=%d  %.2f TFLOP/s  (%s)\n", threads, blocks, flops / ms * 1e-9,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
