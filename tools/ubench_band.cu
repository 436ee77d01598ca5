// Microbenchmark of the band loop of the streaming kernel (step 6, register-blocked sliding
// window): one CTA of 128 threads computes one band unit (16 leaf segments, s = 31, VT = 1) from
// shared-memory tiles; cycles per unit for variants of the inner loop.
//   A: as in lc_exec.cu (3 shared loads per column step, padded indices)
//   B: the next group's a, b, g values loaded into registers while the current group computes
#include <cstdio>
#include <cuda_runtime.h>
constexpr int R = 8;
__device__ __forceinline__ int pidx(int x) { return x + (x >> 4); }

template <int VAR>
__device__ void band_items(const double* ta, const double* tb, const double* gt, double* zst, int s, int nleaf,
                           int N, int btid) {
  const int seglen = 2 * s;
  const int ntb = (s + R - 1) / R;
  const int items = nleaf * 2 * ntb;
  for (int it = btid; it < items; it += 128) {
    int tb_i, sg, uu;
    if (VAR == 2) {  // segment fastest: the lanes of a warp share the row block (uniform trip count)
      uu = it % nleaf;
      const int r2 = it / nleaf;
      sg = r2 & 1;
      tb_i = r2 >> 1;
    } else {
      tb_i = it % ntb;
      int r_ = it / ntb;
      sg = r_ & 1;
      uu = r_ >> 1;
    }
    const int m0 = R * tb_i;
    const int ii = uu * seglen + sg + 2 * m0;
    const int je = seglen * (uu + 2) < N ? seglen * (uu + 2) : N;
    const int cmax = (je - ii - 1) >> 1;
    double acc[R], aw[R], bw[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      acc[r] = 0.0;
      aw[r] = 0.0;
      bw[r] = tb[pidx(ii + r)];
    }
    const int ngrp = (cmax + 1) / R;
    int c0 = 0;
    if (VAR != 1) {
      for (int gi = 0; gi < ngrp; ++gi, c0 += R) {
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int c = c0 + q;
          aw[q] = ta[c];
          const int xb = ii + R - 1 + c, xg = ii + 2 * c;
          bw[(q + R - 1) % R] = tb[pidx(xb)];
          const double gval = gt[pidx(xg)];
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r] = fma(aw[(q - r + R) % R] * bw[(r + q) % R], gval, acc[r]);
        }
      }
    } else {
      double na[R], nb[R], ng[R];
      auto load = [&](int cc) {
#pragma unroll
        for (int q = 0; q < R; ++q) {
          na[q] = ta[cc + q];
          nb[q] = tb[pidx(ii + R - 1 + cc + q)];
          ng[q] = gt[pidx(ii + 2 * (cc + q))];
        }
      };
      if (ngrp > 0) load(0);
      for (int gi = 0; gi < ngrp; ++gi, c0 += R) {
        double ca[R], cbv[R], cg[R];
#pragma unroll
        for (int q = 0; q < R; ++q) { ca[q] = na[q]; cbv[q] = nb[q]; cg[q] = ng[q]; }
        if (gi + 1 < ngrp) load(c0 + R);
#pragma unroll
        for (int q = 0; q < R; ++q) {
          aw[q] = ca[q];
          bw[(q + R - 1) % R] = cbv[q];
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r] = fma(aw[(q - r + R) % R] * bw[(r + q) % R], cg[q], acc[r]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int c = c0 + q;
      if (c <= cmax) {
        aw[q] = ta[c];
        bw[(q + R - 1) % R] = tb[pidx(ii + R - 1 + c)];
        const double gval = gt[pidx(ii + 2 * c)];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = fma(aw[(q - r + R) % R] * bw[(r + q) % R], gval, acc[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (m0 + r < s) zst[ii + 2 * r] = acc[r];
  }
}

template <int VAR>
__global__ void __launch_bounds__(128, 4) k(long long* cyc, double* sink, int s, int reps) {
  extern __shared__ double sm[];
  const int nleaf = 16, seglen = 2 * s;
  const int tcols = (nleaf + 2) * seglen;
  const int tp = pidx(tcols + 2 * R) + 2;
  double* ta = sm;
  double* tb = ta + 2 * s + 2 * R + 8;
  double* gt = tb + tp + 8;
  double* zst = gt + tp + 8;
  for (int i = threadIdx.x; i < 2 * s + 2 * R; i += 128) ta[i] = 1.0 / (1 + i);
  for (int i = threadIdx.x; i < tp; i += 128) { tb[i] = 1.0 / (2 + i); gt[i] = 1e-3 * (i % 97); }
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    band_items<VAR>(ta, tb, gt, zst, s, nleaf, 1 << 30, threadIdx.x);
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
  sink[blockIdx.x * 128 + threadIdx.x] = zst[threadIdx.x];
}
int main() {
  long long* cyc; double* sink;
  cudaMalloc(&cyc, 4096 * 8); cudaMalloc(&sink, 1 << 24);
  const int s = 31;
  const size_t smem = 40000;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  // fp64 ops per unit: sum over rows of (cmax+1) steps x 2 (DMUL + DFMA)
  long long ops = 0;
  for (int uu = 0; uu < 16; ++uu) for (int r = 0; r < 2 * s; ++r) { const int ii = uu * 2 * s + r; ops += 2 * (((2 * s * (uu + 2) - ii - 1) >> 1) + 1); }
  for (int var = 0; var < 3; ++var)
    for (int blocks : {1, 296, 592}) {
      for (int t = 0; t < 2; ++t) {
        if (var == 0) k<0><<<blocks, 128, smem>>>(cyc, sink, s, 20);
        else if (var == 1) k<1><<<blocks, 128, smem>>>(cyc, sink, s, 20);
        else k<2><<<blocks, 128, smem>>>(cyc, sink, s, 20);
      }
      cudaDeviceSynchronize();
      long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      const double per_sm = blocks >= 148 ? blocks / 148.0 : 1.0;
      printf("var %d blocks %d: %lld cycles per unit per CTA, %.1f fp64 ops/clk/SM (peak 64)  err=%s\n", var, blocks, h,
             ops * per_sm / double(h), cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
