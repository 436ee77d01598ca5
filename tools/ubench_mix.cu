// Microbenchmark: do DMMA (fp64 tensor MMA) and DFMA share the SM's fp64 datapath?  Warps [0, nd) of
// each CTA run DMMA chains, warps [nd, 8) DFMA chains, for fixed work per warp; if the pipes were
// separate, the mixed CTA would finish in about max(t_dmma, t_dfma) instead of their sum.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* sink, long long it_mma, long long it_fma, int nd) {
  const int warp = threadIdx.x >> 5;
  double a = 1.0 + threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-6;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  if (warp < nd) {
    for (long long it = 0; it < it_mma; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  } else {
    for (long long it = 0; it < it_fma; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(c[i][0]) : "d"(a), "d"(b));
        asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(c[i][1]) : "d"(a), "d"(b));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* sink;
  cudaMalloc(&sink, 1 << 26);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = 148 * 2, threads = 256;
  // per warp: it_mma x 8 DMMA (8 x 256 FMA each) vs it_fma x 16 DFMA (32 FMA each): equal FMA counts
  // when it_fma = 4 it_mma (8 x 256 = 2048 = 4 x 16 x 32)
  const long long im = 4000, ifm = 16000;
  struct Case { const char* name; long long m, f; int nd; } cases[] = {
      {"all DMMA (8 warps)", im, 0, 8}, {"all DFMA (8 warps)", 0, ifm, 0},
      {"4 DMMA warps only", im, 0, 4}, {"4 DFMA warps only (other 4 idle)", 0, ifm, 4 /*warps 4-7 DFMA*/},
      {"4 DMMA + 4 DFMA warps", im, ifm, 4}};
  for (auto& cs : cases) {
    for (int rep = 0; rep < 2; ++rep) {
      long long m = cs.m, f = cs.f;
      int nd = cs.nd;
      // "4 DFMA warps only": warps 0-3 get zero DMMA iterations
      if (cs.m == 0 && cs.nd == 4) m = 0;
      cudaEventRecord(e0);
      k<<<blocks, threads>>>(sink, m, f, nd);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("%-36s %.3f ms  (%s)\n", cs.name, ms, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
