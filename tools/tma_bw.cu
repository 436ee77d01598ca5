// Microbenchmark: achievable HBM read bandwidth of a cp.async.bulk (1-D TMA) + mbarrier ring,
// one producer lane per CTA, consumers only wait/release (no compute).  Sweeps chunk size,
// ring depth and CTAs per SM.  Reading 256 MB (> L2) per pass.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void ring(const char* src, size_t total, int chunk, int depth, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)(sm + (size_t)depth * chunk);
  uint64_t* empty = full + depth;
  const int tid = threadIdx.x;
  const size_t nchunks = total / chunk;
  const size_t mine = nchunks > blockIdx.x ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (tid == 0) {
    for (int i = 0; i < depth; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (tid == 0) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (size_t i = 0; i < mine; ++i) {
      const int slot = i % depth;
      if (i >= (size_t)depth) {
        uint32_t ok = 0, ph = ((i / depth) - 1) & 1;
        do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(sa(&empty[slot])), "r"(ph) : "memory"); } while (!ok);
      }
      const char* g = src + (blockIdx.x + i * gridDim.x) * (size_t)chunk;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[slot])), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(sa(sm + (size_t)slot * chunk)), "l"(g), "r"(chunk), "r"(sa(&full[slot])), "l"(pol) : "memory");
    }
  } else if (tid == 32) {
    unsigned long long acc = 0;
    for (size_t i = 0; i < mine; ++i) {
      const int slot = i % depth;
      uint32_t ok = 0, ph = (i / depth) & 1;
      do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(sa(&full[slot])), "r"(ph) : "memory"); } while (!ok);
      acc += sm[(size_t)slot * chunk + 7];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[slot])) : "memory");
    }
    if (acc == 0xdeadbeef) sink[0] = acc;
  }
}
int main() {
  const size_t total = 256ull << 20;
  char* d; cudaMalloc(&d, total); cudaMemset(d, 1, total);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  char* flush; cudaMalloc(&flush, 512ull << 20);
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(ring, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  int chunks[] = {8192, 16384, 23328, 32768, 49152};
  int depths[] = {2, 3, 4, 6, 8};
  int ctas[] = {1, 2, 3, 4};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int c : chunks) for (int dp : depths) for (int k : ctas) {
    size_t smem = (size_t)c * dp + 256;
    if (smem * k > 220 * 1024) continue;
    int grid = 148 * k;
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemsetAsync(flush, rep, 512ull << 20);
      cudaEventRecord(e0);
      ring<<<grid, 64, smem>>>(d, total / c * c, c, dp, sink);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    printf("chunk %6d depth %d ctas/SM %d inflight/SM %4zu KB : %7.1f GB/s %s\n", c, dp, k, (size_t)c * dp * k / 1024,
           (double)(total / c * c) / best / 1e6, err == cudaSuccess ? "" : cudaGetErrorString(err));
  }
  return 0;
}
