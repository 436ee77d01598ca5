// Microbenchmark of the up kernel's subtree M2M (step 2, Alg. a.1) as compiled in lc_exec.cu:
// cycles per tree level for one CTA of 256 threads, 6 levels from 64 leaves (VT = 1).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kM = 18, kMM = kM * kM;
__constant__ double c_B0[kMM];
template <int R0, int R1>
__device__ __forceinline__ void m2m_rows(const double* __restrict__ x0, const double* __restrict__ x1,
                                         double* __restrict__ out) {
  constexpr int NR = R1 - R0;
  double zp[R1], zm[R1];
#pragma unroll
  for (int k = 0; k < R1; k += 2) {
    const double2 a2 = *reinterpret_cast<const double2*>(x0 + k);
    const double2 b2 = *reinterpret_cast<const double2*>(x1 + k);
    zp[k] = a2.x + b2.x;
    zm[k] = a2.x - b2.x;
    if (k + 1 < R1) {
      zp[k + 1] = a2.y + b2.y;
      zm[k + 1] = a2.y - b2.y;
    }
  }
  double acc[NR];
#pragma unroll
  for (int n = R0; n < R1; ++n) {
    double ae = 0.0, ao = 0.0;
#pragma unroll
    for (int k = 0; k <= n; k += 2) ae = fma(c_B0[n * kM + k], ((n - k) & 1) ? zm[k] : zp[k], ae);
#pragma unroll
    for (int k = 1; k <= n; k += 2) ao = fma(c_B0[n * kM + k], ((n - k) & 1) ? zm[k] : zp[k], ao);
    acc[n - R0] = ae + ao;
  }
#pragma unroll
  for (int i = 0; i < NR; ++i) out[R0 + i] = acc[i];
}
template <int VT>
__device__ __forceinline__ void m2m_level(const double* __restrict__ Bs, const double* __restrict__ ch,
                                          double* __restrict__ pa, int lp) {
  const int np = 1 << lp;
  const int per = 2 * np * VT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpr = (blockDim.x >> 5) / 3;
  if (warp >= 3 * wpr) return;
  const int rg = warp % 3;
  for (int r = (warp / 3) * 32 + lane; r < per; r += wpr * 32) {
    const int v = r % VT;
    const int sp = r / VT;
    const int P = sp & (np - 1);
    const int sg = sp >> lp;
    const double* x0 = ch + ((sg * 2 * np + 2 * P) * VT + v) * kM;
    double* o = pa + r * kM;
    if (rg == 0) m2m_rows<0, 10>(x0, x0 + VT * kM, o);
    else if (rg == 1) m2m_rows<10, 15>(x0, x0 + VT * kM, o);
    else m2m_rows<15, 18>(x0, x0 + VT * kM, o);
  }
}
// variant: only the FMA part with x in registers from a fixed location (no smem traffic) to isolate
__global__ void kfma(long long* cyc, double* sink) {
  double x[kM];
  for (int k = 0; k < kM; ++k) x[k] = threadIdx.x * 1e-3 + k;
  long long t0 = clock64();
  double acc[3];
#pragma unroll
  for (int n = 15; n < 18; ++n) {
    double ae = 0.0, ao = 0.0;
#pragma unroll
    for (int k = 0; k <= n; k += 2) ae = fma(c_B0[n * kM + k], x[k], ae);
#pragma unroll
    for (int k = 1; k <= n; k += 2) ao = fma(c_B0[n * kM + k], x[k], ao);
    acc[n - 15] = ae + ao;
  }
  long long t1 = clock64();
  sink[threadIdx.x] = acc[0] + acc[1] + acc[2];
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k(const double* B, long long* cyc, double* sink, int k_) {
  extern __shared__ double sm[];
  double* Bs = sm;
  double* tree = sm + kMM + 4;
  auto tree_off = [&](int j) { return ((1 << j) - 1) * 2 * kM; };
  for (int i = threadIdx.x; i < kMM; i += blockDim.x) Bs[i] = B[i];
  for (int i = threadIdx.x; i < (2 << k_) * 2 * kM; i += blockDim.x) tree[i] = 1e-3 * i;
  __syncthreads();
  for (int rep = 0; rep < 2; ++rep) {
    for (int j = k_; j >= 1; --j) {
      long long t0 = clock64();
      m2m_level<1>(Bs, tree + tree_off(j), tree + tree_off(j - 1), j - 1);
      __syncthreads();
      long long t1 = clock64();
      if (threadIdx.x == 0) cyc[(blockIdx.x * 2 + rep) * 8 + j] = t1 - t0;
    }
  }
  if (threadIdx.x == 0) sink[blockIdx.x] = tree[0];
}
int main() {
  double hB[kMM];
  for (int i = 0; i < kMM; ++i) hB[i] = 1.0 / (1 + i);
  double *dB, *sink;
  long long* cyc;
  cudaMalloc(&dB, sizeof(hB));
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  cudaMalloc(&sink, 1 << 20);
  cudaMalloc(&cyc, 148 * 16 * 8);
  cudaMemcpyToSymbol(c_B0, hB, sizeof(hB));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  for (int r = 0; r < 3; ++r) {
    kfma<<<1, 32>>>(cyc, sink);
    cudaDeviceSynchronize();
    long long hc;
    cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
    printf("fma-only rows 15..17 (51 DFMA, const B): %lld cycles\n", hc);
  }
  for (int blocks : {1, 148, 296}) {
    k<<<blocks, 256, 80000>>>(dB, cyc, sink, 6);
    cudaDeviceSynchronize();
    long long h[148 * 16];
    cudaMemcpy(h, cyc, sizeof(long long) * 16 * (blocks < 148 ? blocks : 148), cudaMemcpyDeviceToHost);
    printf("blocks=%d err=%s  cycles per level (j=6..1), warm rep of CTA 0:", blocks, cudaGetErrorString(cudaGetLastError()));
    for (int j = 6; j >= 1; --j) printf(" %lld", h[(0 * 2 + 1) * 8 + j]);
    printf("\n");
  }
  return 0;
}
