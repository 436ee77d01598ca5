// Microbenchmark: dependent-latency of shared-memory loads (LDS.64, LDS.128), of an
// LDS -> DFMA -> STS round trip, and of __syncwarp, on one warp (clock64 cycles per step).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(long long* out, double* sink) {
  __shared__ __align__(16) double sm[1024];
  __shared__ int idx[1024];
  const int lane = threadIdx.x;
  for (int i = lane; i < 1024; i += 32) { sm[i] = 1.0 + 1e-9 * i; idx[i] = (i * 7 + 3) & 1023; }
  __syncwarp();
  // 1) int pointer chase in smem (LDS.32 latency)
  int p = lane;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) p = idx[p];
  long long t1 = clock64();
  // 2) double chain: x = sm[f(x)] (LDS.64 + F2I-ish conversion avoided: use bits)
  double x = sm[lane];
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
    const int j = (__double2loint(x) & 511);
    x = sm[j] * 1.0000001;
  }
  long long t3 = clock64();
  // 3) LDS.128 broadcast then 4 dependent DFMA then STS then __syncwarp (one "operator step")
  double acc = 0.0;
  long long t4 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
    const double2 a = *reinterpret_cast<const double2*>(sm + 2 * (i & 63));
    acc = fma(a.x, acc, a.y);
    acc = fma(a.x, acc, a.y);
    acc = fma(a.x, acc, a.y);
    acc = fma(a.x, acc, a.y);
    if (lane == 0) sm[512 + (i & 63)] = acc;
    __syncwarp();
  }
  long long t5 = clock64();
  // 4) pure dependent DFMA
  double y = acc;
  long long t6 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { y = fma(y, 1.0000001, 1e-9); y = fma(y, 1.0000001, 1e-9); y = fma(y, 1.0000001, 1e-9); y = fma(y, 1.0000001, 1e-9); }
  long long t7 = clock64();
  // 5) dependent DADD
  double z = y;
  long long t8 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { z = z + 1e-9; z = z + 1e-9; z = z + 1e-9; z = z + 1e-9; }
  long long t9 = clock64();
  sink[lane] = x + acc + y + z + p;
  if (lane == 0) {
    out[0] = (t1 - t0) / 256; out[1] = (t3 - t2) / 256; out[2] = (t5 - t4) / 256; out[3] = (t7 - t6) / 1024;
    out[4] = (t9 - t8) / 1024;
  }
}
int main() {
  long long* o; double* s;
  cudaMalloc(&o, 64); cudaMalloc(&s, 4096);
  for (int r = 0; r < 2; ++r) {
    k<<<1, 32>>>(o, s);
    long long h[5];
    cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
    printf("LDS.32 chase %lld | LDS.64+DMUL chain %lld | LDS.128 + 4xDFMA + STS + syncwarp %lld | DFMA %lld | DADD %lld cycles\n",
           h[0], h[1], h[2], h[3], h[4]);
  }
  return 0;
}
