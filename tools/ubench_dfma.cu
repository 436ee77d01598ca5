// Microbenchmark: DFMA latency and per-warp issue rate on one SM (clock64 cycles per DFMA
// per warp) for K independent accumulation chains and W warps per CTA (1 CTA per SM).
#include <cstdio>
#include <cuda_runtime.h>
template <int K>
__global__ void kd(double* sink, long long* cyc, double x, int iters) {
  double a[K];
#pragma unroll
  for (int i = 0; i < K; ++i) a[i] = threadIdx.x * 1e-3 + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < K; ++i) a[i] = fma(a[i], x, 1e-9);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < K; ++i) s += a[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* sink;
  long long* cyc;
  cudaMalloc(&sink, 148 * 1024 * 8);
  cudaMalloc(&cyc, 148 * 8);
  long long h[148];
  const int iters = 256;
  for (int W : {1, 2, 4, 8, 16, 32}) {
    for (int K : {1, 2, 4, 8, 16}) {
      auto launch = [&](void) {
        switch (K) {
          case 1: kd<1><<<148, 32 * W>>>(sink, cyc, 0.999, iters); break;
          case 2: kd<2><<<148, 32 * W>>>(sink, cyc, 0.999, iters); break;
          case 4: kd<4><<<148, 32 * W>>>(sink, cyc, 0.999, iters); break;
          case 8: kd<8><<<148, 32 * W>>>(sink, cyc, 0.999, iters); break;
          default: kd<16><<<148, 32 * W>>>(sink, cyc, 0.999, iters); break;
        }
      };
      launch();
      launch();
      cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      double c = 0;
      for (int b = 0; b < 148; ++b) c += h[b];
      c /= 148;
      const double ndfma = double(iters) * 16 * K;  // per warp
      printf("warps/SM=%2d chains=%2d: %6.2f cycles per DFMA per warp, SM rate %5.1f FMA/clk\n", W, K, c / ndfma,
             32.0 * W * ndfma / c);
    }
  }
  return 0;
}
