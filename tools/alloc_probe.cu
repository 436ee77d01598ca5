// Wall time of device allocations of the plan sizes: cudaMalloc, cudaMallocAsync from the default pool
// (release threshold 0: memory returns to the driver at each synchronisation) and from a pool that keeps
// freed memory (release threshold UINT64_MAX).  build: nvcc -O2 -o tools/alloc_probe tools/alloc_probe.cu
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
int main() {
  cudaFree(0);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const size_t sizes[] = {size_t(135) << 20, size_t(1350) << 20};
  for (size_t sz : sizes) {
    for (int rep = 0; rep < 3; ++rep) {
      void* p = nullptr;
      double t = now_ms();
      cudaMalloc(&p, sz);
      const double a = now_ms() - t;
      t = now_ms();
      cudaFree(p);
      const double b = now_ms() - t;
      t = now_ms();
      cudaMallocAsync(&p, sz, st);
      cudaStreamSynchronize(st);
      const double c = now_ms() - t;
      t = now_ms();
      cudaFreeAsync(p, st);
      cudaStreamSynchronize(st);
      const double d = now_ms() - t;
      std::printf("%5zu MB rep %d: cudaMalloc %.3f ms, cudaFree %.3f ms, cudaMallocAsync(default pool)+sync %.3f ms, cudaFreeAsync+sync %.3f ms\n",
                  sz >> 20, rep, a, b, c, d);
    }
  }
  cudaMemPool_t pool;
  cudaDeviceGetDefaultMemPool(&pool, 0);
  uint64_t thr = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  for (size_t sz : sizes) {
    for (int rep = 0; rep < 3; ++rep) {
      void* p = nullptr;
      double t = now_ms();
      cudaMallocAsync(&p, sz, st);
      cudaStreamSynchronize(st);
      const double c = now_ms() - t;
      t = now_ms();
      cudaFreeAsync(p, st);
      cudaStreamSynchronize(st);
      const double d = now_ms() - t;
      std::printf("%5zu MB rep %d: retaining pool: cudaMallocAsync+sync %.3f ms, cudaFreeAsync+sync %.3f ms\n", sz >> 20, rep, c, d);
    }
  }
  return 0;
}
