// DMMA m8n8k4 f64 latency and per-SMSP throughput vs chains per warp and warps per SM (one CTA per SM).
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* sink, long long iters, long long* cyc) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-6;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  long long t0 = clock64();
  for (long long it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int CH>
void run(int warps, double* sink, long long* cyc) {
  const long long iters = 4000;
  k<CH><<<148, warps * 32>>>(sink, 100, cyc);
  k<CH><<<148, warps * 32>>>(sink, iters, cyc);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double per = double(h) / (iters * CH);
  printf("chains=%d warps/SM=%2d: %.2f cycles per DMMA per warp (%.2f per DMMA per SMSP)\n", CH, warps, per,
         per / (warps >= 4 ? warps / 4.0 : 1.0));
}
int main() {
  double* sink;
  long long* cyc;
  cudaMalloc(&sink, 1 << 24);
  cudaMalloc(&cyc, 8);
  for (int w : {1, 4, 8, 16}) {
    run<1>(w, sink, cyc);
    run<2>(w, sink, cyc);
    run<4>(w, sink, cyc);
  }
  return 0;
}
