// Microbenchmark: latency of small fp64 operator applications on one SM, with the operator
// read from (a) __constant__ memory, (b) a __grid_constant__ kernel parameter, (c) shared
// memory.  Prints clock64 cycles per phase for a cold and a warm pass in the same CTA.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kM = 18;
__constant__ double cB[kM * kM];
struct P { double T[2][32][kM]; };

template <int MODE>
__device__ __forceinline__ double bval(const double* sB, int n, int k) {
  if (MODE == 0) return cB[n * kM + k];
  return sB[n * kM + k];
}
template <int MODE>
__device__ void m2m(const double* sB, const double* x0, const double* x1, double* out) {
  double acc[kM];
#pragma unroll
  for (int n = 0; n < kM; ++n) acc[n] = 0.0;
#pragma unroll
  for (int k = 0; k < kM; ++k) {
    const double zp = x0[k] + x1[k], zm = x0[k] - x1[k];
#pragma unroll
    for (int n = k; n < kM; ++n) acc[n] = fma(bval<MODE>(sB, n, k), ((n - k) & 1) ? zm : zp, acc[n]);
  }
#pragma unroll
  for (int n = 0; n < kM; ++n) out[n] = acc[n];
}
template <int MODE>
__global__ void k_m2m(const double* B, long long* cyc, double* sink) {
  __shared__ double sB[kM * kM];
  __shared__ double buf[2][128 * kM];
  for (int i = threadIdx.x; i < kM * kM; i += blockDim.x) sB[i] = B[i];
  for (int i = threadIdx.x; i < 128 * kM; i += blockDim.x) buf[0][i] = 1e-3 * i;
  __syncthreads();
  for (int rep = 0; rep < 2; ++rep) {
    long long t0 = clock64();
    int src = 0;
    for (int lp = 5; lp >= 0; --lp) {  // 6 levels: 64 .. 1 parents
      const int np = 1 << lp;
      if (threadIdx.x < np) m2m<MODE>(sB, buf[src] + 2 * threadIdx.x * kM, buf[src] + (2 * threadIdx.x + 1) * kM, buf[src ^ 1] + threadIdx.x * kM);
      __syncthreads();
      src ^= 1;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x * 2 + rep] = t1 - t0;
  }
  if (threadIdx.x == 0) sink[blockIdx.x] = buf[0][0];
}
template <int MODE>
__global__ void k_step1(const __grid_constant__ P p, const double* T, long long* cyc, double* sink) {
  __shared__ double sT[2 * 32 * kM];
  __shared__ double fs[64 * 66 + 64];
  for (int i = threadIdx.x; i < 2 * 32 * kM; i += blockDim.x) sT[i] = T[i];
  for (int i = threadIdx.x; i < 64 * 66 + 64; i += blockDim.x) fs[i] = 1e-3 * i;
  __syncthreads();
  double out = 0;
  for (int rep = 0; rep < 2; ++rep) {
    long long t0 = clock64();
    const int lf = threadIdx.x % 64, kg = threadIdx.x / 64;
    if (kg < 3) {
      const double* fp = fs + lf * 66;
      double a[6], b[6];
#pragma unroll
      for (int i = 0; i < 6; ++i) a[i] = b[i] = 0.0;
#pragma unroll
      for (int m = 0; m < 32; ++m) {
        const double2 f2 = *reinterpret_cast<const double2*>(fp + 2 * m);
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const int kk = 6 * (kg == 0 ? 0 : kg == 1 ? 1 : 2) + i;
          double t0v, t1v;
          if (MODE == 1) { t0v = p.T[0][m][kk]; t1v = p.T[1][m][kk]; }
          else { t0v = sT[(0 * 32 + m) * kM + kk]; t1v = sT[(1 * 32 + m) * kM + kk]; }
          a[i] = fma(f2.x, t0v, a[i]);
          b[i] = fma(f2.y, t1v, b[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < 6; ++i) out += a[i] + b[i];
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x * 2 + rep] = t1 - t0;
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = out;
}
int main() {
  double hB[kM * kM];
  for (int i = 0; i < kM * kM; ++i) hB[i] = 1.0 / (1 + i);
  cudaMemcpyToSymbol(cB, hB, sizeof(hB));
  double *dB, *dT, *sink;
  long long* cyc;
  P p;
  for (int i = 0; i < 2 * 32 * kM; ++i) (&p.T[0][0][0])[i] = 1.0 / (3 + i);
  cudaMalloc(&dB, sizeof(hB));
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  cudaMalloc(&dT, sizeof(p.T));
  cudaMemcpy(dT, p.T, sizeof(p.T), cudaMemcpyHostToDevice);
  cudaMalloc(&sink, 1 << 20);
  cudaMalloc(&cyc, 4096 * sizeof(long long));
  long long h[2 * 148];
  auto rep = [&](const char* name) {
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double c0 = 0, c1 = 0;
    for (int b = 0; b < 148; ++b) { c0 += h[2 * b]; c1 += h[2 * b + 1]; }
    printf("%-28s cold %8.0f cyc  warm %8.0f cyc (mean over 148 CTAs)  err=%s\n", name, c0 / 148, c1 / 148,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int it = 0; it < 2; ++it) {
    k_m2m<0><<<148, 64>>>(dB, cyc, sink); rep("m2m 6 levels, __constant__ B");
    k_m2m<1><<<148, 64>>>(dB, cyc, sink); rep("m2m 6 levels, smem B");
    k_step1<1><<<148, 192>>>(p, dT, cyc, sink); rep("step1 64 leaves, param T");
    k_step1<2><<<148, 192>>>(p, dT, cyc, sink); rep("step1 64 leaves, smem T");
  }
  return 0;
}
