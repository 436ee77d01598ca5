// Microbenchmark of the down kernel's step-4 descent (warp-level B(p)^T, lane = mode) as in
// lc_exec.cu: cycles per subtree level for one CTA of 4 warps, kd = 4 levels, VT = 1.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kM = 18, kMM = kM * kM;
__constant__ double c_B0[kMM];
struct BCol { double v[kM]; };
__device__ __forceinline__ void load_bcol(BCol& c, int l) {
#pragma unroll
  for (int n = 0; n < kM; ++n) c.v[n] = (l < kM && n >= l) ? c_B0[n * kM + (l < kM ? l : 0)] : 0.0;
}
__device__ __forceinline__ void l2l_warp2(const BCol& cb, const double* __restrict__ c0, int p0,
                                          const double* __restrict__ c1, int p1, int l, double& r0, double& r1) {
  double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
  for (int n = 0; n < kM; n += 2) {
    const double2 x = *reinterpret_cast<const double2*>(c0 + n);
    const double2 y = *reinterpret_cast<const double2*>(c1 + n);
    a0 = fma(cb.v[n], x.x, a0);
    a1 = fma(cb.v[n + 1], x.y, a1);
    b0 = fma(cb.v[n], y.x, b0);
    b1 = fma(cb.v[n + 1], y.y, b1);
  }
  r0 = p0 ? a0 - a1 : a0 + a1;
  if (p0 && (l & 1)) r0 = -r0;
  r1 = p1 ? b0 - b1 : b0 + b1;
  if (p1 && (l & 1)) r1 = -r1;
}
// variant B: explicit register preload of both inputs, 4 partial chains per output
__device__ __forceinline__ void l2l_warp2b(const BCol& cb, const double* __restrict__ c0, int p0,
                                           const double* __restrict__ c1, int p1, int l, double& r0, double& r1) {
  double x[kM], y[kM];
#pragma unroll
  for (int n = 0; n < kM; n += 2) {
    const double2 a = *reinterpret_cast<const double2*>(c0 + n);
    const double2 b = *reinterpret_cast<const double2*>(c1 + n);
    x[n] = a.x; x[n + 1] = a.y; y[n] = b.x; y[n + 1] = b.y;
  }
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0, b0 = 0, b1 = 0, b2 = 0, b3 = 0;
#pragma unroll
  for (int n = 0; n < kM; n += 4) {
    a0 = fma(cb.v[n], x[n], a0); b0 = fma(cb.v[n], y[n], b0);
    a1 = fma(cb.v[n + 1], x[n + 1], a1); b1 = fma(cb.v[n + 1], y[n + 1], b1);
    if (n + 2 < kM) { a2 = fma(cb.v[n + 2], x[n + 2], a2); b2 = fma(cb.v[n + 2], y[n + 2], b2); }
    if (n + 3 < kM) { a3 = fma(cb.v[n + 3], x[n + 3], a3); b3 = fma(cb.v[n + 3], y[n + 3], b3); }
  }
  const double ae = a0 + a2, ao = a1 + a3, be = b0 + b2, bo = b1 + b3;
  r0 = p0 ? ae - ao : ae + ao;
  if (p0 && (l & 1)) r0 = -r0;
  r1 = p1 ? be - bo : be + bo;
  if (p1 && (l & 1)) r1 = -r1;
}
template <int VAR>
__global__ void k(long long* cyc, double* sink, int kd) {
  __shared__ double cm[64 * 2 * kM];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 64 * 2 * kM; i += blockDim.x) cm[i] = 1e-3 * i;
  BCol bc;
  load_bcol(bc, lane);
  __syncthreads();
  auto cm_lvl = [&](int j) { return cm + ((1 << j) - 1) * 2 * kM; };
  for (int rep = 0; rep < 2; ++rep) {
    for (int j = 1; j <= kd; ++j) {
      long long t0 = clock64();
      const int nodes = 1 << j;
      const double* par = cm_lvl(j - 1);
      double* cur = cm_lvl(j);
      const int items = 2 * nodes;
      for (int i0_ = warp * 2; i0_ < items; i0_ += 8) {
        const int it0 = i0_, it1 = i0_ + 1 < items ? i0_ + 1 : i0_;
        auto parent = [&](int it, int& p) {
          const int node = it & (nodes - 1);
          const int sg = it >> j;
          p = node & 1;
          return par + (sg * (nodes >> 1) + (node >> 1)) * kM;
        };
        int p0, p1;
        const double* c0 = parent(it0, p0);
        const double* c1 = parent(it1, p1);
        double r0, r1;
        if (VAR == 0) l2l_warp2(bc, c0, p0, c1, p1, lane, r0, r1);
        else l2l_warp2b(bc, c0, p0, c1, p1, lane, r0, r1);
        if (lane < kM) {
          cur[it0 * kM + lane] += r0;
          if (it1 != it0) cur[it1 * kM + lane] += r1;
        }
      }
      __syncthreads();
      long long t1 = clock64();
      if (tid == 0) cyc[(blockIdx.x * 2 + rep) * 8 + j] = t1 - t0;
    }
  }
  if (tid == 0) sink[blockIdx.x] = cm[100];
}
int main() {
  double hB[kMM];
  for (int i = 0; i < kMM; ++i) hB[i] = 1.0 / (1 + i);
  cudaMemcpyToSymbol(c_B0, hB, sizeof(hB));
  double* sink;
  long long* cyc;
  cudaMalloc(&sink, 1 << 20);
  cudaMalloc(&cyc, 1024 * 16 * 8);
  for (int var = 0; var < 2; ++var)
    for (int blocks : {1, 592}) {
      if (var == 0) k<0><<<blocks, 128>>>(cyc, sink, 4); else k<1><<<blocks, 128>>>(cyc, sink, 4);
      cudaDeviceSynchronize();
      long long h[16];
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      printf("var=%d blocks=%d err=%s cycles per level j=1..4 (warm):", var, blocks, cudaGetErrorString(cudaGetLastError()));
      for (int j = 1; j <= 4; ++j) printf(" %lld", h[8 + j]);
      printf("\n");
    }
  return 0;
}
