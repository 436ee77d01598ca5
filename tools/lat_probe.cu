// Latency probes on the B200: dependent DFMA / DADD chains, LDS round trip (single warp, clock64).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(double* out, long long* cyc, double a, double b, int iters) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i * 1e-3;
  __syncthreads();
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  double y = threadIdx.x;
  for (int i = 0; i < iters; ++i) y = y * a + b;  // DMUL + DADD (may fuse)
  long long t2 = clock64();
  int idx = threadIdx.x & 7;
  double z = 0;
  for (int i = 0; i < iters; ++i) { z += sm[idx]; idx = (int)(z) & 7; }
  long long t3 = clock64();
  double w = threadIdx.x;
  for (int i = 0; i < iters; ++i) { w = w + a; }
  long long t4 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
  out[threadIdx.x] = x + y + z + w;
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 1024 * 8); cudaMalloc(&c, 64);
  int iters = 4096;
  probe<<<1, 32>>>(d, c, 0.999, 1e-3, iters);
  probe<<<1, 32>>>(d, c, 0.999, 1e-3, iters);
  long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.1f cycles\n", (double)h[0] / iters);
  printf("DMUL+DADD chain: %.1f cycles/iter\n", (double)h[1] / iters);
  printf("LDS dependent chain: %.1f cycles/iter\n", (double)h[2] / iters);
  printf("DADD dependent latency: %.1f cycles\n", (double)h[3] / iters);
  return 0;
}
