// Microbenchmark: per-item cycles of the warp-level step-4 operator (lane = mode) in a loop of
// independent items, for variants: A = lane<18 branch around the work, B = branch-free (store
// predicated), C = B with 2 items per iteration, D = B with 4 items per iteration.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kM = 18;
struct BReg { double b[kM]; };
__device__ __forceinline__ double l2l_lane(const BReg& br, const double* __restrict__ c, int p, int l) {
  double x[kM];
#pragma unroll
  for (int n = 0; n < kM; n += 2) {
    const double2 t = *reinterpret_cast<const double2*>(c + n);
    x[n] = t.x; x[n + 1] = t.y;
  }
  double e0 = 0.0, e1 = 0.0, o0 = 0.0, o1 = 0.0;
#pragma unroll
  for (int n = 0; n < kM; n += 4) {
    e0 = fma(br.b[n], x[n], e0);
    o0 = fma(br.b[n + 1], x[n + 1], o0);
    if (n + 2 < kM) e1 = fma(br.b[n + 2], x[n + 2], e1);
    if (n + 3 < kM) o1 = fma(br.b[n + 3], x[n + 3], o1);
  }
  const double e = e0 + e1, o = o0 + o1;
  const double r = p ? e - o : e + o;
  return (p && (l & 1)) ? -r : r;
}
template <int VAR>
__global__ void k(const double* B, long long* cyc, double* sink, int items) {
  __shared__ __align__(16) double par[64 * kM];
  __shared__ __align__(16) double cur[128 * kM];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * kM; i += blockDim.x) par[i] = 1e-3 * i;
  for (int i = threadIdx.x; i < 128 * kM; i += blockDim.x) cur[i] = 1e-4 * i;
  BReg br;
#pragma unroll
  for (int n = 0; n < kM; ++n) br.b[n] = (lane < kM && n >= lane) ? __ldg(B + n * kM + (lane < kM ? lane : 0)) : 0.0;
  __syncthreads();
  long long t0 = clock64();
  if (VAR == 0) {
    for (int it = warp; it < items; it += 8) {
      if (lane < kM) {
        const double own = cur[it * kM + lane];
        const double r = l2l_lane(br, par + (it >> 1) * kM, it & 1, lane);
        cur[it * kM + lane] = own + r;
      }
    }
  } else if (VAR == 1) {
    const int ll = lane < kM ? lane : 0;
    for (int it = warp; it < items; it += 8) {
      const double own = cur[it * kM + ll];
      const double r = l2l_lane(br, par + (it >> 1) * kM, it & 1, lane);
      if (lane < kM) cur[it * kM + lane] = own + r;
    }
  } else if (VAR == 2) {
    const int ll = lane < kM ? lane : 0;
    for (int it = warp * 2; it < items; it += 16) {
      const double own0 = cur[it * kM + ll], own1 = cur[(it + 1) * kM + ll];
      const double r0 = l2l_lane(br, par + (it >> 1) * kM, it & 1, lane);
      const double r1 = l2l_lane(br, par + ((it + 1) >> 1) * kM, (it + 1) & 1, lane);
      if (lane < kM) { cur[it * kM + lane] = own0 + r0; cur[(it + 1) * kM + lane] = own1 + r1; }
    }
  } else {
    const int ll = lane < kM ? lane : 0;
    for (int it = warp * 4; it < items; it += 32) {
      double own[4], r[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) own[q] = cur[(it + q) * kM + ll];
#pragma unroll
      for (int q = 0; q < 4; ++q) r[q] = l2l_lane(br, par + ((it + q) >> 1) * kM, (it + q) & 1, lane);
      if (lane < kM) {
#pragma unroll
        for (int q = 0; q < 4; ++q) cur[(it + q) * kM + lane] = own[q] + r[q];
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x] = cur[5];
}
int main() {
  double hB[kM * kM];
  for (int i = 0; i < kM * kM; ++i) hB[i] = 1.0 / (1 + i);
  double *dB, *sink; long long* cyc;
  cudaMalloc(&dB, sizeof(hB)); cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  cudaMalloc(&sink, 1 << 16); cudaMalloc(&cyc, 4096);
  for (int var = 0; var < 4; ++var)
    for (int blocks : {1, 296}) {
      for (int rep = 0; rep < 2; ++rep) {
        switch (var) {
          case 0: k<0><<<blocks, 256>>>(dB, cyc, sink, 128); break;
          case 1: k<1><<<blocks, 256>>>(dB, cyc, sink, 128); break;
          case 2: k<2><<<blocks, 256>>>(dB, cyc, sink, 128); break;
          default: k<3><<<blocks, 256>>>(dB, cyc, sink, 128); break;
        }
      }
      cudaDeviceSynchronize();
      long long h;
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("var %d blocks %d: 128 items over 8 warps: %lld cycles = %.0f per item-per-warp\n", var, blocks, h, h / 16.0);
    }
  return 0;
}
