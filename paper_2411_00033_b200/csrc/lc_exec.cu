// lc_exec.cu -- execution stage (Alg. 4, alg:fastercomplete)
// as three sm_100a kernels per transform; both parities are processed together
// (the same A_hat serves sigma = 0 and 1, so it is streamed once).
//
//   lc_up_kernel     one CTA per subtree of 2^kup leaf segments x VT vectors:
//                    step 1 (eq:wMM, w = f^sigma T(sigma)) and step 2 (eq:wtk with
//                    Alg. a.1) inside the subtree; the last CTA
//                    of each group of 2^G sibling subtrees (atomic arrival counter)
//                    continues the upward pass G levels, up to level 0.  Writes
//                    w(g) of every level; raises readiness flags.
//   lc_stream_kernel persistent, warp-specialised.  One producer lane streams the
//                    level-major A_hat arena with TMA bulk copies (cp.async.bulk +
//                    mbarrier ring, L2 evict-first), finest level first, together
//                    with each chunk's w window; eight consumer warps apply
//                    step 3 (M2L) and, interleaved with it, the
//                    direct band of step 6 (Alg. 1 restricted to j < j_end(i)),
//                    which depends only on f and lambda: the fp64-heavy band runs
//                    in the shadow of the HBM-bound A_hat stream.
//   lc_down_kernel   one CTA per subtree of 2^k leaf row segments x VT vectors:
//                    step 4 ("faster downward spreading", B(p)^T)
//                    along the ancestor chain and down the subtree, step 5
//                    (eq:step5) added to the band result, step 7 (C^{-1}), store.
//
// Kernels are chained with programmatic dependent launch (griddepcontrol); the
// streaming kernel synchronises with the up kernel through release/acquire flags
// so that the band and the fine-level M2L overlap the end of the upward pass.
#include <algorithm>
#include <cstdio>

#include "lc_internal.h"

namespace lc {

// B(0) (App. A3) is a universal constant for M = 18: in constant memory the fully
// unrolled triangular products take it as a uniform DFMA operand.
__constant__ double c_B0[kMM];

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// 1-D TMA bulk copy global -> shared, completion signalled on an mbarrier (SASS: UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// cp.async (LDGSTS): per-element asynchronous global->shared copies for the small gathers
// whose shared destinations are padded or scattered; src_bytes = 0 zero-fills (the zero
// padding beyond n).
__device__ __forceinline__ void cp_async8(void* dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
// named barrier among the consumer warps of the streaming kernel (the producer warp does not join)
__device__ __forceinline__ void consumer_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");  // barrier 1: the band warps
}
// release/acquire helpers for the readiness flags (gpu scope)
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_flag(const int* p) {
  while (ld_acquire(p) == 0) __nanosleep(64);
}

// Phase timestamps for the debug build (-DLC_PHASE_TIMING): %globaltimer (ns) per CTA and phase.
#ifdef LC_PHASE_TIMING
__device__ unsigned long long g_lc_ts[3][1 << 20];
__device__ __forceinline__ void lc_ts(int kern, int slot) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned cta = blockIdx.y * gridDim.x + blockIdx.x;
    if (cta * 8 + slot < (1u << 20)) g_lc_ts[kern][cta * 8 + slot] = t;
  }
}
__device__ __forceinline__ void lc_ts_any(int kern, int slot) {  // any thread
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  const unsigned cta = blockIdx.y * gridDim.x + blockIdx.x;
  if (cta * 8 + slot < (1u << 20)) g_lc_ts[kern][cta * 8 + slot] = t;
}
#define LC_TS(k, s) lc_ts(k, s)
#else
#define LC_TS(k, s) ((void)0)
#endif

__device__ __forceinline__ int64_t vaddr(int layout, int64_t ld, int64_t v, int64_t j) {
  return layout == LC_VEC_CONTIGUOUS ? v * ld + j : j * ld + v;
}

// ---------------------------------------------------------------- transfer operators
// Alg. a.1 for one parent node:
// parent[n] = sum_{k<=n} b_nk (x0_k + (-1)^(n-k) x1_k)  (B(1) = B(0) with the odd diagonals
// negated, App. A3).  Children streamed from shared memory one mode at a time; 18 register
// accumulators; B(0) from constant memory.
__device__ __forceinline__ void m2m18(const double* __restrict__ x0, const double* __restrict__ x1,
                                      double* __restrict__ out) {
  double acc[kM];
#pragma unroll
  for (int n = 0; n < kM; ++n) acc[n] = 0.0;
#pragma unroll
  for (int k = 0; k < kM; ++k) {
    const double a = x0[k], b = x1[k];
    const double zp = a + b, zm = a - b;
#pragma unroll
    for (int n = k; n < kM; ++n) acc[n] = fma(c_B0[n * kM + k], ((n - k) & 1) ? zm : zp, acc[n]);
  }
#pragma unroll
  for (int n = 0; n < kM; n += 2) *reinterpret_cast<double2*>(out + n) = make_double2(acc[n], acc[n + 1]);
}

// Step 4: dst += B(p)^T src with (B(p)^T c)_k = sum_{n>=k} b_nk (-1)^{p(n-k)} c_n
// = (-1)^{pk} sum_n b_nk c'_n, c'_n = (-1)^{pn} c_n ("faster downward spreading",
// B(1) differs from B(0) only in the sign of the odd diagonals).
__device__ __forceinline__ void l2l18(const double* __restrict__ src, int p, double* __restrict__ dst) {
  double acc[kM];
#pragma unroll
  for (int k = 0; k < kM; ++k) acc[k] = 0.0;
#pragma unroll
  for (int n = 0; n < kM; ++n) {
    double cn = src[n];
    if ((n & 1) && p) cn = -cn;
#pragma unroll
    for (int k = 0; k <= n; ++k) acc[k] = fma(c_B0[n * kM + k], cn, acc[k]);
  }
#pragma unroll
  for (int k = 0; k < kM; ++k) dst[k] += ((k & 1) && p) ? -acc[k] : acc[k];
}

// Warp-level transfer operators: lane l < 18 owns output mode l and keeps its row (M2M) or
// column (L2L) of B(0) in registers; the input vector is read from shared memory by all lanes
// at once (broadcast), so one warp applies one 18 x 18 triangular operator in ~36 instructions.
struct BRow {  // brow[k] = b_{l k} (k <= l), 0 otherwise
  double v[kM];
};
struct BCol {  // bcol[n] = b_{n l} (n >= l), 0 otherwise
  double v[kM];
};
__device__ __forceinline__ void load_brow(BRow& r, const double* __restrict__ B, int l) {
#pragma unroll
  for (int k = 0; k < kM; ++k) r.v[k] = (l < kM && k <= l) ? __ldg(B + l * kM + k) : 0.0;
}
__device__ __forceinline__ void load_bcol(BCol& c, const double* __restrict__ B, int l) {
#pragma unroll
  for (int n = 0; n < kM; ++n) c.v[n] = (l < kM && n >= l) ? __ldg(B + n * kM + l) : 0.0;
}
// Alg. a.1: parent_l = sum_k b_lk x0_k + (-1)^l sum_k b_lk (-1)^k x1_k   (lane l; returns for l < 18)
__device__ __forceinline__ double m2m_warp(const BRow& r, const double* __restrict__ x0,
                                           const double* __restrict__ x1, int l) {
  double a0 = 0.0, a1 = 0.0;
#pragma unroll
  for (int k = 0; k < kM; ++k) {
    a0 = fma(r.v[k], x0[k], a0);
    a1 = fma(r.v[k], (k & 1) ? -x1[k] : x1[k], a1);
  }
  return (l & 1) ? a0 - a1 : a0 + a1;
}
// Step 4: (B(p)^T c)_l = (-1)^{pl} sum_n b_nl (-1)^{pn} c_n   (lane l)
__device__ __forceinline__ double l2l_warp(const BCol& cb, const double* __restrict__ c, int p, int l) {
  double a0 = 0.0, a1 = 0.0;
#pragma unroll
  for (int n = 0; n < kM; n += 2) {
    a0 = fma(cb.v[n], c[n], a0);
    a1 = fma(cb.v[n + 1], c[n + 1], a1);
  }
  // even n keep their sign; odd n flip when p = 1; then the lane sign (-1)^{pl}
  const double r = p ? a0 - a1 : a0 + a1;
  return (p && (l & 1)) ? -r : r;
}

// ---------------------------------------------------------------- parameters
// flags (workspace ints): [0] up main-phase arrivals, [1] fine levels of w ready,
// [2] finished level-0 continuations, [3] coarse levels of w ready, [4] finished
// streaming CTAs, [5] predecessor complete (input readable).  Self-resetting.
struct UpParams {
  const double* in;
  int64_t ld_in, n, N, batch;
  int layout, L, s, k, gr, G;
  const double* T;  // [2][s][M]
  const double* B;  // B(0) [M][M]
  double* w;
  int* cnt;
  int* flags;
  int64_t w_tile, cnt_tile;
};

struct StreamParams {
  const double* A;
  const double* w;
  double* c;
  const double* in;
  double* out;
  const double* tabA;
  const double* tabB;
  int* flags;
  int64_t w_tile;  // doubles per vector tile (w and c share the layout)
  int64_t ld_in, ld_out, n, N, batch;
  int64_t ntiles, nm2l, nband;
  int layout, L, s, cb, nst, kb, gr_up;
};

struct DownParams {
  double* out;
  int64_t ld_out, n, N, batch;
  int layout, L, s, k, gr;
  const double* Tt;  // [2][M][s]
  const double* B;   // B(0) [M][M]
  const double* c;   // c_m2l
  int64_t w_tile;
};

// ============================================================== up kernel
// one tree level in shared memory ([sigma][node][v][M]); item = (sigma, parent, v) handled by
// one warp (lane = output mode); nparent = 2^lp
template <int VT>
__device__ __forceinline__ void m2m_level(const double* __restrict__ ch, double* __restrict__ pa, int lp,
                                          const BRow& br) {
  const int nparent = 1 << lp;
  const int items = 2 * nparent * VT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int it = warp; it < items; it += nwarps) {
    const int v = it % VT;
    const int sp = it / VT;
    const int P = sp & (nparent - 1);
    const int sg = sp >> lp;
    const double* x0 = ch + ((sg * 2 * nparent + 2 * P) * VT + v) * kM;
    const double r = m2m_warp(br, x0, x0 + VT * kM, lane);
    if (lane < kM) pa[it * kM + lane] = r;
  }
}

template <int VT>
__global__ void __launch_bounds__(kThreads, 2) lc_up_kernel(const UpParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ int s_last;
  const int s = P.s, k = P.k;
  const int tid = threadIdx.x;
  double* Ts = reinterpret_cast<double*>(smem);
  double* fs = reinterpret_cast<double*>(smem + align_up(int64_t(2) * s * kM * 8, 128));
  const int nleaf = 1 << k;
  const int seglen = 2 * s;
  const int tlen = nleaf * seglen;
  double* tree = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(fs) + align_up(int64_t(VT) * tlen * 8, 128));
  auto tree_off = [&](int j) { return ((1 << j) - 1) * 2 * VT * kM; };

  const int64_t R = blockIdx.x;
  const int64_t tile = blockIdx.y;
  LC_TS(0, 0);
  BRow br;
  load_brow(br, P.B, tid & 31);
  for (int i = tid; i < s * kM; i += blockDim.x) cp_async16(Ts + 2 * i, P.T + 2 * i);
  cp_async_commit();
  griddep_wait();  // the input may be produced by the preceding kernel
  // Trigger the dependent (streaming) launch only now: every streaming CTA then starts after the
  // whole previous execution completed, so it can never observe flags of that execution.
  griddep_launch();
  if (tid == 0) st_release(&P.flags[5], 1);  // predecessor complete: the streaming kernel may read the input

  // stage the leaf range [R 2^k, (R+1) 2^k) of segments, zero padding beyond n
  const int64_t j0 = R * tlen;
  if (P.layout == LC_VEC_CONTIGUOUS) {
#pragma unroll 1
    for (int v = 0; v < VT; ++v) {
      const int64_t gv = tile * VT + v;
      const double* src = P.in + gv * P.ld_in + j0;
      const int64_t lim = gv < P.batch ? P.n - j0 : 0;  // valid elements of this vector in the tile
      for (int jj = tid; jj < tlen; jj += blockDim.x) {
        const bool ok = jj < lim;
        cp_async8(fs + v * tlen + jj, ok ? src + jj : P.in, ok ? 8u : 0u);
      }
    }
  } else {
    for (int idx = tid; idx < VT * tlen; idx += blockDim.x) {
      const int jj = idx / VT, v = idx - jj * VT;  // v fastest: coalesced in the batch layout
      const int64_t gv = tile * VT + v, j = j0 + jj;
      const bool ok = gv < P.batch && j < P.n;
      cp_async8(fs + v * tlen + jj, ok ? P.in + j * P.ld_in + gv : P.in, ok ? 8u : 0u);
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  LC_TS(0, 1);

  // step 1: w(L-1)[t][k] = sum_m f[2s t + 2m + sigma] T(sigma)[m][k]   (eq:wMM)
  // item = (v, seg, sigma, group of 6 modes); 3 lanes share each f value.
  {
    double* leaf = tree + tree_off(k);
    const int items = nleaf * 2 * VT * 3;
    for (int it = tid; it < items; it += blockDim.x) {
      const int kg = it % 3;
      int r = it / 3;
      const int sg = r & 1;
      r >>= 1;
      const int seg = r & (nleaf - 1);
      const int v = r >> k;
      const double* fp = fs + v * tlen + seg * seglen + sg;
      const double* tp = Ts + sg * s * kM + 6 * kg;
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0;
#pragma unroll 4
      for (int m = 0; m < s; ++m) {
        const double f = fp[2 * m];
        const double2 t01 = *reinterpret_cast<const double2*>(tp + m * kM);
        const double2 t23 = *reinterpret_cast<const double2*>(tp + m * kM + 2);
        const double2 t45 = *reinterpret_cast<const double2*>(tp + m * kM + 4);
        a0 = fma(f, t01.x, a0); a1 = fma(f, t01.y, a1);
        a2 = fma(f, t23.x, a2); a3 = fma(f, t23.y, a3);
        a4 = fma(f, t45.x, a4); a5 = fma(f, t45.y, a5);
      }
      double* o = leaf + ((sg * nleaf + seg) * VT + v) * kM + 6 * kg;
      *reinterpret_cast<double2*>(o) = make_double2(a0, a1);
      *reinterpret_cast<double2*>(o + 2) = make_double2(a2, a3);
      *reinterpret_cast<double2*>(o + 4) = make_double2(a4, a5);
    }
  }
  __syncthreads();
  LC_TS(0, 2);
  // step 2 inside the subtree
  for (int j = k; j >= 1; --j) {
    m2m_level<VT>(tree + tree_off(j), tree + tree_off(j - 1), j - 1, br);
    __syncthreads();
  }
  LC_TS(0, 3);
  double* wt = P.w + tile * P.w_tile;
  const int64_t VM = int64_t(VT) * kM;
  for (int j = 0; j <= k; ++j) {
    const int g = P.gr + j;
    const int cnt2 = int((int64_t(1) << j) * VM / 2);
    for (int sg = 0; sg < 2; ++sg) {
      double2* dst = reinterpret_cast<double2*>(wt + (w_level_offset_units(g) + sg * nseg(g) + (R << j)) * VM);
      const double2* src = reinterpret_cast<const double2*>(tree + tree_off(j) + sg * (int64_t(1) << j) * VM);
      for (int i = tid; i < cnt2; i += blockDim.x) dst[i] = src[i];
    }
  }
  // the fine levels (gr..L-1) of the whole batch are ready once every CTA got here
  __threadfence();
  __syncthreads();
  LC_TS(0, 4);
  if (tid == 0) {
    const int total = int(gridDim.x * gridDim.y);
    if (atomicAdd(&P.flags[0], 1) == total - 1) {
      atomicExch(&P.flags[0], 0);
      __threadfence();
      st_release(&P.flags[1], 1);
      if (P.gr == 0) st_release(&P.flags[3], 1);
    }
  }

  // upward continuation above the subtree roots: the last arriver of each
  // group of 2^G nodes merges them G levels up (threadfence-reduction pattern).
  int g = P.gr;
  int64_t node = R;
  while (g > 0) {
    const int ge = min(P.G, g);
    const int64_t grp = node >> ge;
    __syncthreads();
    if (tid == 0) {
      int* c = P.cnt + tile * P.cnt_tile + (nseg(g) - 4) + grp;
      const int old = atomicAdd(c, 1);
      const int last = (old == (1 << ge) - 1);
      if (last) atomicExch(c, 0);  // self-reset for the next launch
      s_last = last;
    }
    __syncthreads();
    if (!s_last) {
      LC_TS(0, 7);
      return;
    }
    LC_TS(0, 5);
    __threadfence();
    const int cnt2 = int((int64_t(1) << ge) * VM / 2);
    for (int sg = 0; sg < 2; ++sg) {
      const double2* src =
          reinterpret_cast<const double2*>(wt + (w_level_offset_units(g) + sg * nseg(g) + (grp << ge)) * VM);
      double2* dst = reinterpret_cast<double2*>(tree + tree_off(ge) + sg * 2 * cnt2);
      for (int i = tid; i < cnt2; i += blockDim.x) dst[i] = __ldcg(src + i);
    }
    __syncthreads();
    for (int j = ge; j >= 1; --j) {
      m2m_level<VT>(tree + tree_off(j), tree + tree_off(j - 1), j - 1, br);
      __syncthreads();
    }
    for (int j = 0; j < ge; ++j) {
      const int gg = g - ge + j;
      const int cj2 = int((int64_t(1) << j) * VM / 2);
      for (int sg = 0; sg < 2; ++sg) {
        double2* dst = reinterpret_cast<double2*>(wt + (w_level_offset_units(gg) + sg * nseg(gg) + (grp << j)) * VM);
        const double2* src = reinterpret_cast<const double2*>(tree + tree_off(j) + sg * 2 * cj2);
        for (int i = tid; i < cj2; i += blockDim.x) dst[i] = src[i];
      }
    }
    __threadfence();
    g -= ge;
    node = grp;
    LC_TS(0, 6);
  }
  if (P.gr > 0) {  // this CTA produced one of the 4 level-0 nodes of its vector tile
    __syncthreads();
    if (tid == 0) {
      const int total = 4 * int(gridDim.y);
      if (atomicAdd(&P.flags[2], 1) == total - 1) {
        atomicExch(&P.flags[2], 0);
        __threadfence();
        st_release(&P.flags[3], 1);
      }
    }
  }
  LC_TS(0, 7);
}

// ============================================================== streaming kernel
constexpr int kM2lWarps = 4;   // consumer warps applying M2L to the A_hat ring
constexpr int kBandWarps = 4;  // consumer warps computing the direct band (independent pipeline)
constexpr int kStreamThreads = 32 * (1 + kM2lWarps + kBandWarps);
constexpr int kBandThreads = 32 * kBandWarps;

// M2L unit q (< nm2l) = (chunk, tile): chunk = (level g, blocks [b0, b0+nb)), nb <= cb, the
// finest level first; tiles innermost so concurrent CTAs share A_hat in L2.
// cstart[o] = first chunk of level L-1-o (shared-memory table, 32-bit arithmetic only).
__device__ __forceinline__ void m2l_unit(int q, int ntiles, int L, int cb, const int* cstart, int& g, int& b0,
                                         int& nb, int& tile) {
  int ch = q;
  tile = 0;
  if (ntiles > 1) {
    ch = q / ntiles;
    tile = q - ch * ntiles;
  }
  int o = 0;
  while (o + 1 < L && cstart[o + 1] <= ch) ++o;
  g = L - 1 - o;
  b0 = (ch - cstart[o]) * cb;
  const int bg = (2 << g) - 1;
  nb = (bg - b0) < cb ? (bg - b0) : cb;
}

// Work units of the CTA: u = blockIdx.x + i * gridDim.x over [0, nband + nm2l); units below
// nband are band units (leaf range of 2^kb segments x vector tile), the rest M2L units.
template <int VT, int DIR>
__global__ void __launch_bounds__(kStreamThreads, 2) lc_stream_kernel(const StreamParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ int cstart[32];
  const int tid = threadIdx.x;
  const int s = P.s, cb = P.cb, nst = P.nst, kb = P.kb;
  const int64_t VM = int64_t(VT) * kM;
  const StreamSmem SL = stream_smem_layout(VT, cb, nst, kb, s);
  const int64_t a_bytes = align_up(int64_t(cb) * 3 * kMM * 8, 128);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SL.bars);
  uint64_t* empty = full + nst;
  double* ta = reinterpret_cast<double*>(smem + SL.ta);
  double* tb = reinterpret_cast<double*>(smem + SL.tb);
  double* gt = reinterpret_cast<double*>(smem + SL.gt);
  double* zst = reinterpret_cast<double*>(smem + SL.zst);
  const int tp = int(SL.tp);

  const int nband = int(P.nband), nm2l = int(P.nm2l);
  const int nunits = nband + nm2l;
  const int nmine = nunits > int(blockIdx.x) ? (nunits - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x) : 0;
  if (tid == 0) {
    int acc = 0;
    for (int o = 0; o < P.L && o < 32; ++o) {
      cstart[o] = acc;
      const int g = P.L - 1 - o;
      acc += ((2 << g) - 1 + cb - 1) / cb;
    }
    for (int i = 0; i < nst; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kM2lWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int ntiles = int(P.ntiles);
  LC_TS(1, 0);
  griddep_launch();

  if (tid < 32) {
    // ------------------------------------------------ producer warp: the A_hat / w stream
    if (tid == 0) {
      const uint64_t pol = policy_evict_first();
      bool fine_ok = false, coarse_ok = false;
      auto issue = [&](int q, int j, bool with_a, bool with_w) {  // M2L unit q, ring use j
        int g, nb, b0, tile;
        m2l_unit(q, ntiles, P.L, cb, cstart, g, b0, nb, tile);
        const int slot = j % nst;
        unsigned char* base = smem + SL.ring + slot * SL.slot;
        const uint32_t abytes = uint32_t(nb) * 3 * kMM * 8;
        const uint32_t wbytes = uint32_t(2 * nb * VM * 8);
        if (with_a) {
          fence_proxy_async();
          mbar_arrive_expect_tx(&full[slot], abytes + 2 * wbytes);
          bulk_g2s(base, P.A + (ahat_level_offset(g) + 3 * int64_t(b0)) * kMM, abytes, &full[slot], pol);
        }
        if (with_w) {
          // w of level g: fine levels after the up kernel's main phase, coarse ones after its continuation
          bool& ok = g >= P.gr_up ? fine_ok : coarse_ok;
          if (!ok) {
            wait_flag(&P.flags[g >= P.gr_up ? 1 : 3]);
            LC_TS(1, g >= P.gr_up ? 4 : 5);
            asm volatile("fence.proxy.async.global;" ::: "memory");  // order the bulk reads after the acquire
            ok = true;
          }
          double* wwin = reinterpret_cast<double*>(base + a_bytes);
          const double* wt = P.w + int64_t(tile) * P.w_tile;
          for (int sg = 0; sg < 2; ++sg)
            bulk_g2s(wwin + sg * 2 * cb * VM, wt + (w_level_offset_units(g) + sg * nseg(g) + 2 * int64_t(b0) + 2) * VM,
                     wbytes, &full[slot], pol);
        }
      };
      // the A_hat of the first nst M2L units is plan data: issue it before any dependency
      int j = 0;
      int firstq[8];
      for (int i = 0; i < nmine && j < nst && j < 8; ++i) {
        const int u = int(blockIdx.x) + i * int(gridDim.x);
        if (u < nband) continue;
        firstq[j] = u - nband;
        issue(firstq[j], j, true, false);
        ++j;
      }
      const int npre = j;
      for (int jj = 0; jj < npre; ++jj) issue(firstq[jj], jj, false, true);
      j = 0;
      for (int i = 0; i < nmine; ++i) {
        const int u = int(blockIdx.x) + i * int(gridDim.x);
        if (u < nband) continue;
        if (j >= npre) {
          mbar_wait(&empty[j % nst], uint32_t(((j / nst) - 1) & 1));
          issue(u - nband, j, true, true);
        }
        ++j;
      }
    }
  } else if (tid < 32 * (1 + kM2lWarps)) {
    // ------------------------------------------------ M2L consumer warps
    const int ctid = tid - 32;
    int j = 0;  // M2L ring use counter
    for (int i = 0; i < nmine; ++i) {
      const int u = int(blockIdx.x) + i * int(gridDim.x);
      if (u < nband) continue;
      {
        // ---------------- M2L unit: step 3 on a chunk of blocks of one level
          int g, nb, b0, tile;
          m2l_unit(u - nband, ntiles, P.L, cb, cstart, g, b0, nb, tile);
          const int slot = j % nst;
#ifdef LC_PHASE_TIMING
          if (j == 0 && ctid == 0) lc_ts_any(1, 2);
#endif
          mbar_wait(&full[slot], uint32_t((j / nst) & 1));
#ifdef LC_PHASE_TIMING
          if (j == 0 && ctid == 0) lc_ts_any(1, 3);
#endif
          const double* As = reinterpret_cast<const double*>(smem + SL.ring + slot * SL.slot);
          const double* wwin = reinterpret_cast<const double*>(smem + SL.ring + slot * SL.slot + a_bytes);
          double* ct = P.c + int64_t(tile) * P.w_tile + (w_level_offset_units(g) + 2 * int64_t(b0)) * VM;
          const int64_t sgstride = nseg(g) * VM;
          const int nrows = 2 * nb;
          for (int it = ctid; it < nrows * kM; it += 32 * kM2lWarps) {
            const int ri = it / kM, kk = it % kM;  // row u = 2 b0 + ri
            double acc[2][VT];
#pragma unroll
            for (int sg = 0; sg < 2; ++sg)
#pragma unroll
              for (int v = 0; v < VT; ++v) acc[sg][v] = 0.0;
            // even row (p=0): r=0 with column t=u+2 and r=1 with t=u+3; odd row (p=1): r=2 with t=u+2
            const int nmat = (ri & 1) ? 1 : 2;
            for (int mi = 0; mi < nmat; ++mi) {
              const int r = (ri & 1) ? 2 : mi;
              const int tloc = (ri & 1) ? ri : ri + mi;  // t - (2 b0 + 2)
              const double* arow = As + (3 * (ri >> 1) + r) * kMM + kk * kM;
              double ar[kM];
#pragma unroll
              for (int l = 0; l < kM; l += 2) {
                const double2 t2 = *reinterpret_cast<const double2*>(arow + l);
                ar[l] = t2.x;
                ar[l + 1] = t2.y;
              }
#pragma unroll
              for (int sg = 0; sg < 2; ++sg)
#pragma unroll
                for (int v = 0; v < VT; ++v) {
                  const double* wp = wwin + (sg * 2 * cb + tloc) * VM + v * kM;
                  double sacc = 0.0;
#pragma unroll
                  for (int l = 0; l < kM; ++l) sacc = fma(ar[l], wp[l], sacc);
                  acc[sg][v] += sacc;
                }
            }
#pragma unroll
            for (int sg = 0; sg < 2; ++sg)
#pragma unroll
              for (int v = 0; v < VT; ++v) ct[sg * sgstride + ri * VM + v * kM + kk] = acc[sg][v];
          }
          __syncwarp();
          if ((tid & 31) == 0) mbar_arrive(&empty[slot]);  // this warp is done with the slot
        ++j;
      }
    }
  } else {
    // ------------------------------------------------ band consumer warps
    const int btid = tid - 32 * (1 + kM2lWarps);
    bool input_ok = false;
    for (int x = btid; x < 2 * s + 2 * kBandR; x += kBandThreads) ta[x] = x < 2 * s ? P.tabA[x] : 0.0;
    for (int i = 0; i < nmine; ++i) {
      const int u = int(blockIdx.x) + i * int(gridDim.x);
      if (u >= nband) continue;
      {
        // ---------------- band unit: step 6 for rows of 2^kb leaf segments of one vector tile
        const int tile = ntiles > 1 ? u % ntiles : 0;
        const int lr = ntiles > 1 ? u / ntiles : u;
        if (!input_ok) {  // the input is readable once the predecessor of the up kernel completed
          if (P.L > 0) {
            if (btid == 0) wait_flag(&P.flags[5]);
          } else {
            griddep_wait();
          }
          consumer_sync(kBandThreads);
          input_ok = true;
        }
        const int nleaf = 1 << kb;
        const int seglen = 2 * s;
        const int64_t U0 = int64_t(lr) << kb;
        const int64_t i0 = U0 * seglen;
        const int rows = nleaf * seglen;
        const int tcols = (nleaf + 2) * seglen;
        const int tbl = int((P.N - i0) < tcols ? (P.N - i0) : tcols);  // valid band-table entries
        for (int x = btid; x < tcols + 2 * kBandR; x += kBandThreads) {
          const bool ok = x < tbl;
          cp_async8(tb + x + (x >> 4), ok ? P.tabB + i0 + x : P.tabB, ok ? 8u : 0u);
        }
#pragma unroll 1
        for (int v = 0; v < VT; ++v) {
          const int64_t gv = int64_t(tile) * VT + v;
          int lim = 0;  // valid input elements of this vector in the tile
          if (gv < P.batch) lim = int((P.n - i0) < tcols ? (P.n - i0) : tcols);
          if (lim < 0) lim = 0;
          if (P.layout == LC_VEC_CONTIGUOUS) {
            const double* src = P.in + gv * P.ld_in + i0;
            for (int x = btid; x < tcols + 2 * kBandR; x += kBandThreads) {
              const bool ok = x < lim;
              cp_async8(gt + v * tp + x + (x >> 4), ok ? src + x : P.in, ok ? 8u : 0u);
            }
          } else {
            for (int x = btid; x < tcols + 2 * kBandR; x += kBandThreads) {
              const bool ok = x < lim;
              cp_async8(gt + v * tp + x + (x >> 4), ok ? P.in + (i0 + x) * P.ld_in + gv : P.in, ok ? 8u : 0u);
            }
          }
        }
        cp_async_commit();
        cp_async_wait<0>();
        consumer_sync(kBandThreads);
        // item = (v, segment uu, parity sigma, block of kBandR same-parity rows m = kBandR t + r).
        // Band of row i' = i + 2r (i the block's first row): sum_c a[c-r] b[i+r+c] g[i+2c], c >= r,
        // i + 2c < j_end; a = tabA, b = tabB, g = f (L2C) or j f_j (C2L).  Sliding windows of a and
        // b live in registers (slots rotate with c): each step loads 3 values for kBandR rows.
        const int ntb = (s + kBandR - 1) / kBandR;
        const int items = VT * nleaf * 2 * ntb;
        for (int it = btid; it < items; it += kBandThreads) {
          const int tb_i = it % ntb;
          int r_ = it / ntb;
          const int sg = r_ & 1;
          r_ >>= 1;
          const int uu = r_ & (nleaf - 1);
          const int v = r_ >> kb;
          const int m0 = kBandR * tb_i;
          const int ii = uu * seglen + sg + 2 * m0;  // tile-local first row
          const int64_t i = i0 + ii;
          const int64_t je = (int64_t(seglen) * (U0 + uu + 2)) < P.N ? int64_t(seglen) * (U0 + uu + 2) : P.N;
          const int cmax = int((je - i - 1) >> 1);
          const double* gv_t = gt + v * tp;
          double acc[kBandR], aw[kBandR], bw[kBandR];
#pragma unroll
          for (int r = 0; r < kBandR; ++r) {
            acc[r] = 0.0;
            aw[r] = 0.0;
            bw[r] = tb[(ii + r) + ((ii + r) >> 4)];
          }
          // (re-loading b[ii+R-1] at c = 0 is harmless: it is the value already in that slot)
          const int ngrp = (cmax + 1) / kBandR;
          int c0 = 0;
          for (int gi = 0; gi < ngrp; ++gi, c0 += kBandR) {
#pragma unroll
            for (int q = 0; q < kBandR; ++q) {
              const int c = c0 + q;
              aw[q] = ta[c];
              const int xb = ii + kBandR - 1 + c, xg = ii + 2 * c;
              bw[(q + kBandR - 1) % kBandR] = tb[xb + (xb >> 4)];
              double gval = gv_t[xg + (xg >> 4)];
              if (DIR == 1) gval *= double(i + 2 * c);
#pragma unroll
              for (int r = 0; r < kBandR; ++r)
                acc[r] = fma(aw[(q - r + kBandR) % kBandR] * bw[(r + q) % kBandR], gval, acc[r]);
            }
          }
#pragma unroll
          for (int q = 0; q < kBandR; ++q) {  // remainder: c = c0 + q <= cmax
            const int c = c0 + q;
            if (c <= cmax) {
              aw[q] = ta[c];
              const int xb = ii + kBandR - 1 + c, xg = ii + 2 * c;
              bw[(q + kBandR - 1) % kBandR] = tb[xb + (xb >> 4)];
              double gval = gv_t[xg + (xg >> 4)];
              if (DIR == 1) gval *= double(i + 2 * c);
#pragma unroll
              for (int r = 0; r < kBandR; ++r)
                acc[r] = fma(aw[(q - r + kBandR) % kBandR] * bw[(r + q) % kBandR], gval, acc[r]);
            }
          }
#pragma unroll
          for (int r = 0; r < kBandR; ++r) {
            if (m0 + r < s) {
              const int64_t ir = i + 2 * r;
              double z = acc[r];
              if (DIR == 1) {
                z *= double(2 * ir + 1);
                if (ir == 0) z += gv_t[0];  // entry (0,0) of A^{-1}C is 1 (reading R2)
              }
              zst[v * rows + ii + 2 * r] = z;
            }
          }
        }
        consumer_sync(kBandThreads);
        // coalesced store of the band result (step 5 and step 7 are added by the down kernel)
        const int olim = int((P.n - i0) < rows ? (P.n - i0) : rows);
#pragma unroll 1
        for (int v = 0; v < VT; ++v) {
          const int64_t gv = int64_t(tile) * VT + v;
          if (gv >= P.batch) break;
          if (P.layout == LC_VEC_CONTIGUOUS) {
            double* dst = P.out + gv * P.ld_out + i0;
            for (int x = btid; x < olim; x += kBandThreads) dst[x] = zst[v * rows + x];
          } else {
            for (int x = btid; x < olim; x += kBandThreads) P.out[(i0 + x) * P.ld_out + gv] = zst[v * rows + x];
          }
        }
        consumer_sync(kBandThreads);  // tiles are reused by the next band unit
      }
    }
  }
  __syncthreads();
  LC_TS(1, 1);
  if (tid == 0) {  // the last CTA to finish re-arms the readiness flags for the next execution
    if (atomicAdd(&P.flags[4], 1) == int(gridDim.x) - 1) {
      P.flags[1] = 0;
      P.flags[3] = 0;
      P.flags[5] = 0;
      __threadfence();
      atomicExch(&P.flags[4], 0);
    }
  }
}

// ============================================================== down kernel
// One CTA per (subtree of 2^k leaf row segments, tile of VT vectors):
//   cp.async prefetch of T(sigma)^T, the band result z_band of the rows and the c_m2l of the
//   ancestors and of the subtree nodes; step 4 along the ancestor chain (one thread per
//   (sigma, v)) and down the subtree (one thread per node); step 5 + step 7; store.
template <int VT, int DIR>
__global__ void __launch_bounds__(kThreads, 2) lc_down_kernel(const DownParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int s = P.s, k = P.k, gr = P.gr, L = P.L;
  const int tid = threadIdx.x;
  const DownSmem SL = down_smem_layout(VT, k, s, gr);
  double* Tt = reinterpret_cast<double*>(smem + SL.Tt);
  double* zb = reinterpret_cast<double*>(smem + SL.zb);
  double* cm = reinterpret_cast<double*>(smem + SL.cm);

  const int64_t R = blockIdx.x;
  const int64_t tile = blockIdx.y;
  const int64_t VM = int64_t(VT) * kM;
  const int nleaf = 1 << k;
  const int seglen = 2 * s;
  const int64_t U0 = R << k;
  const int64_t i0 = U0 * seglen;
  const int rows = nleaf * seglen;
  // cm layout: ancestors [g][sigma][v][M] (g < gr), then subtree level j at node offset
  // gr + 2^j - 1: [sigma][node][v][M]
  auto cm_anc = [&](int g) { return cm + int64_t(g) * 2 * VM; };
  auto cm_lvl = [&](int j) { return cm + (int64_t(gr) + (1 << j) - 1) * 2 * VM; };

  LC_TS(2, 0);
  for (int i = tid; i < s * kM; i += blockDim.x) cp_async16(Tt + 2 * i, P.Tt + 2 * i);  // plan data
  cp_async_commit();
  griddep_launch();
  griddep_wait();  // c_m2l and the band result (streaming kernel) are ready past this point
  LC_TS(2, 1);

  const double* ct = P.c + tile * P.w_tile;
  if (L > 0) {
    for (int g = 0; g < gr; ++g) {
      const int64_t a = R >> (gr - g);
      for (int sg = 0; sg < 2; ++sg) {
        const double* src = ct + (w_level_offset_units(g) + sg * nseg(g) + a) * VM;
        double* dst = cm_anc(g) + sg * VM;
        for (int i = tid; i < VM / 2; i += blockDim.x) cp_async16(dst + 2 * i, src + 2 * i);
      }
    }
    for (int j = 0; j <= k; ++j) {
      const int g = gr + j;
      const int cnt2 = int((int64_t(1) << j) * VM / 2);
      for (int sg = 0; sg < 2; ++sg) {
        const double* src = ct + (w_level_offset_units(g) + sg * nseg(g) + (R << j)) * VM;
        double* dst = cm_lvl(j) + sg * (int64_t(1) << j) * VM;
        for (int i = tid; i < cnt2; i += blockDim.x) cp_async16(dst + 2 * i, src + 2 * i);
      }
    }
  }
  const int olim = int((P.n - i0) < rows ? (P.n - i0) : rows);  // rows of this tile inside n
#pragma unroll 1
  for (int v = 0; v < VT; ++v) {
    const int64_t gv = tile * VT + v;
    const int lim = gv < P.batch ? olim : 0;
    if (P.layout == LC_VEC_CONTIGUOUS) {
      const double* src = P.out + gv * P.ld_out + i0;
      for (int x = tid; x < rows; x += blockDim.x) {
        const bool ok = x < lim;
        cp_async8(zb + v * rows + x, ok ? src + x : P.out, ok ? 8u : 0u);
      }
    } else {
      for (int x = tid; x < rows; x += blockDim.x) {
        const bool ok = x < lim;
        cp_async8(zb + v * rows + x, ok ? P.out + (i0 + x) * P.ld_out + gv : P.out, ok ? 8u : 0u);
      }
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  LC_TS(2, 2);

  if (L > 0) {
    const int lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    BCol bc;
    load_bcol(bc, P.B, lane);
    // step 4 along the ancestor chain, one warp per (sigma, v): cm_anc(g) += B(p)^T c(a_{g-1}),
    // p = child index of a_g; then the subtree root
    for (int ch = warp; ch < 2 * VT; ch += nwarps) {
      for (int g = 1; g <= gr; ++g) {
        const int p = int((R >> (gr - g)) & 1);
        double* dst = (g < gr ? cm_anc(g) : cm_lvl(0)) + ch * kM;  // [sigma][node 0][v] == ch at the root
        const double r = l2l_warp(bc, cm_anc(g - 1) + ch * kM, p, lane);
        if (lane < kM) dst[lane] += r;
        __syncwarp();
      }
    }
    __syncthreads();
    LC_TS(2, 3);
    // step 4 down the subtree, one warp per (sigma, node, v): c(j) = B(p)^T c(j-1) + c_m2l(j)
    for (int j = 1; j <= k; ++j) {
      const int nodes = 1 << j;
      const double* par = cm_lvl(j - 1);
      double* cur = cm_lvl(j);
      for (int it = warp; it < 2 * nodes * VT; it += nwarps) {
        const int v = it % VT;
        const int sn = it / VT;
        const int node = sn & (nodes - 1);
        const int sg = sn >> j;
        const double r = l2l_warp(bc, par + ((sg * (nodes >> 1) + (node >> 1)) * VT + v) * kM, node & 1, lane);
        if (lane < kM) cur[it * kM + lane] += r;
      }
      __syncthreads();
    }
  }
  LC_TS(2, 4);
  const double* cfin = cm_lvl(k);

  // step 5: z^sigma += c(L-1) T(sigma)^T (eq:step5), 4 same-parity rows per thread (c kept in
  // registers), accumulated into the band result in shared memory
  if (L > 0) {
    constexpr int R5 = 4;
    const int nb5 = (s + R5 - 1) / R5;
    const int items = VT * nleaf * 2 * nb5;
    for (int it = tid; it < items; it += blockDim.x) {
      const int mb = it % nb5;
      int r_ = it / nb5;
      const int sg = r_ & 1;
      r_ >>= 1;
      const int u = r_ & (nleaf - 1);
      const int v = r_ >> k;
      const int m0 = R5 * mb;
      const double* cp = cfin + ((sg * nleaf + u) * VT + v) * kM;
      const double* tq = Tt + sg * kM * s + m0;
      double t5[R5];
#pragma unroll
      for (int r = 0; r < R5; ++r) t5[r] = 0.0;
#pragma unroll
      for (int kk = 0; kk < kM; ++kk) {
        const double cv = cp[kk];
#pragma unroll
        for (int r = 0; r < R5; ++r) t5[r] = fma(cv, tq[kk * s + r], t5[r]);  // (tq beyond s: padding, unused)
      }
      double* zr = zb + v * rows + u * seglen + sg + 2 * m0;
#pragma unroll
      for (int r = 0; r < R5; ++r)
        if (m0 + r < s) zr[2 * r] += t5[r];
    }
    __syncthreads();
  }
  // step 7: C^{-1} (L2C); coalesced store
  const double inv_pi = 0.318309886183790671537767526745028724;
#pragma unroll 1
  for (int v = 0; v < VT; ++v) {
    const int64_t gv = tile * VT + v;
    if (gv >= P.batch) break;
    for (int ii = tid; ii < olim; ii += blockDim.x) {
      const int64_t i = i0 + ii;
      double z = zb[v * rows + ii];
      if (DIR == 0) z *= (i == 0 ? inv_pi : 2.0 * inv_pi);
      if (P.layout == LC_VEC_CONTIGUOUS)
        P.out[gv * P.ld_out + i] = z;
      else
        P.out[i * P.ld_out + gv] = z;
    }
  }
  __syncthreads();
  LC_TS(2, 5);
}

// ============================================================== host side
template <typename K>
static cudaError_t set_max_dyn_smem(K kernel, int smax) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, kernel);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smax - int(fa.sharedSizeBytes));
  if (e != cudaSuccess) return e;
  // without a preference the driver may pick a small shared-memory carveout and cap occupancy
  return cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
}
template <int VT>
static cudaError_t set_attrs_vt(int smax) {
  cudaError_t e = set_max_dyn_smem(lc_up_kernel<VT>, smax);
  if (e == cudaSuccess) e = set_max_dyn_smem(lc_stream_kernel<VT, 0>, smax);
  if (e == cudaSuccess) e = set_max_dyn_smem(lc_stream_kernel<VT, 1>, smax);
  if (e == cudaSuccess) e = set_max_dyn_smem(lc_down_kernel<VT, 0>, smax);
  if (e == cudaSuccess) e = set_max_dyn_smem(lc_down_kernel<VT, 1>, smax);
  return e;
}

static bool g_device_ready[64] = {false};

template <int VT>
static int stream_occupancy(int dir, size_t smem) {
  int occ = 0;
  if (dir == 0)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lc_stream_kernel<VT, 0>, kStreamThreads, smem);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lc_stream_kernel<VT, 1>, kStreamThreads, smem);
  return occ;
}

lc_status configure_kernels(lc_plan* p) {
  int smax = 0;
  cudaError_t ea = cudaDeviceGetAttribute(&smax, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->device);
  if (ea != cudaSuccess) return record_cuda_error(ea);
  if (p->device < 0 || p->device >= 64) return LC_ERR_INVALID_ARG;
  if (!g_device_ready[p->device]) {
    ea = set_attrs_vt<1>(smax);
    if (ea == cudaSuccess) ea = set_attrs_vt<2>(smax);
    if (ea == cudaSuccess) ea = set_attrs_vt<4>(smax);
    if (ea == cudaSuccess) ea = set_attrs_vt<8>(smax);
    if (ea == cudaSuccess) {
      double B[kMM];
      ea = cudaMemcpy(B, p->d_B, sizeof(B), cudaMemcpyDeviceToHost);
      if (ea == cudaSuccess) ea = cudaMemcpyToSymbol(c_B0, B, sizeof(B));
    }
    if (ea != cudaSuccess) return record_cuda_error(ea);
    g_device_ready[p->device] = true;
  }
  smax -= 256;  // static shared memory of the kernels

  const int64_t budget2 = 113 * 1024;  // two CTAs per SM (228 KB minus 1 KB reserved per CTA)
  const int64_t budget3 = 74 * 1024;   // three CTAs per SM
  int vt = p->vt;
  if (vt <= 0) vt = p->batch >= 2 ? 2 : 1;
  if (vt != 1 && vt != 2 && vt != 4 && vt != 8) return LC_ERR_INVALID_ARG;
  const bool user_k = p->k > 0;
  int k = user_k ? p->k : 4;
  int cb = p->bps > 0 ? p->bps : 3;
  int nst = p->nst > 0 ? p->nst : 3;
  if (nst > 8) return LC_ERR_INVALID_ARG;
  const int64_t nleaf_total = p->L > 0 ? (int64_t(2) << p->L) : 2;  // leaf segments (L = 0: the two halves)
  int lnleaf = 0;
  while ((int64_t(1) << (lnleaf + 1)) <= nleaf_total) ++lnleaf;  // log2(nleaf_total)
  if (p->L == 0) {
    k = 1;
  } else {
    k = int(std::min<int64_t>(k, p->L - 1));
  }
  auto down_bytes = [&](int vt_, int k_) {
    const int gr_ = p->L > 0 ? int(p->L - 1 - k_) : 0;
    return down_smem_layout(vt_, k_, int(p->s), gr_).total;
  };
  if (!user_k) {
    while (down_bytes(vt, k) > budget3 && p->L > 0 && k > 1) --k;
  }
  if (down_bytes(vt, k) > smax) return LC_ERR_INVALID_ARG;
  // streaming kernel: band units of 2^kb leaf segments
  int kb = std::min(4, lnleaf);  // 2^kb segments x 2 parities x ceil(s/R) blocks = one item per band thread
  auto stream_bytes = [&](int cb_, int kb_) { return stream_smem_layout(vt, cb_, nst, kb_, int(p->s)).total; };
  while (stream_bytes(cb, kb) > budget2 && kb > 1) --kb;
  while (stream_bytes(cb, kb) > budget2 && cb > 1) --cb;
  if (stream_bytes(cb, kb) > smax) return LC_ERR_INVALID_ARG;
  // up kernel: deeper subtrees (its shared memory is small); continuation step = its depth
  const bool user_kup = p->kup > 0;
  int kup = p->L > 0 ? int(std::min<int64_t>(user_kup ? p->kup : 5, p->L - 1)) : 0;
  while (!user_kup && kup > 0 && up_smem_bytes(vt, kup, int(p->s)) > budget2) --kup;
  if (up_smem_bytes(vt, kup, int(p->s)) > smax) return LC_ERR_INVALID_ARG;
  p->vt = vt;
  p->k = k;
  p->bps = cb;
  p->nst = nst;
  p->kb = kb;
  p->gr = p->L > 0 ? int(p->L - 1 - k) : 0;
  p->kup = kup;
  p->grup = p->L > 0 ? int(p->L - 1 - kup) : 0;
  p->group = std::max(kup, 1);
  p->ntiles = (p->batch + vt - 1) / vt;
  p->smem_down = size_t(down_bytes(vt, k));
  p->smem_up = size_t(up_smem_bytes(vt, kup, int(p->s)));
  p->smem_stream = size_t(stream_bytes(cb, kb));
  int64_t nchunks = 0;
  for (int g = 0; g < p->L; ++g) nchunks += (((int64_t(2) << g) - 1) + cb - 1) / cb;
  p->m2l_units = nchunks * p->ntiles;
  p->band_units = (nleaf_total >> kb) * p->ntiles;
  if (p->m2l_units + p->band_units > 0x7fffffff) return LC_ERR_INVALID_ARG;
  {
    int occ = 0;
    switch (vt) {
      case 1: occ = stream_occupancy<1>(p->dir, p->smem_stream); break;
      case 2: occ = stream_occupancy<2>(p->dir, p->smem_stream); break;
      case 4: occ = stream_occupancy<4>(p->dir, p->smem_stream); break;
      default: occ = stream_occupancy<8>(p->dir, p->smem_stream); break;
    }
    if (occ < 1) return LC_ERR_INVALID_ARG;
    // persistent grid: every CTA co-resident (the producer may wait on flags raised by other grids)
    const int64_t g = int64_t(occ) * p->sm_count;
    p->stream_grid = int(std::max<int64_t>(1, std::min<int64_t>(g, p->m2l_units + p->band_units)));
  }
  if (p->L > 0) {
    p->w_tile_doubles = int64_t(vt) * kM * 2 * ((int64_t(4) << p->L) - 4);
    p->cnt_tile_ints = int64_t(4) << p->L;
  } else {
    p->w_tile_doubles = 0;
    p->cnt_tile_ints = 0;
  }
  // workspace: w | c_m2l | flags (64 ints) | arrival counters (c_m2l rows without a submatrix stay zero)
  const size_t wb = size_t(align_up(p->ntiles * p->w_tile_doubles * 8, 256));
  p->ws_bytes = 2 * wb + 256 + size_t(p->ntiles * p->cnt_tile_ints) * sizeof(int);
  return LC_OK;
}

template <int VT, int DIR>
static cudaError_t launch_vt(const lc_plan* p, const UpParams& up, const StreamParams& sp, const DownParams& dp,
                             dim3 grid_up, dim3 grid, cudaStream_t st, cudaEvent_t const* ev, int nev) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaSuccess;
  int evi = 0;
  if (ev && nev > 0) cudaEventRecord(ev[evi++], st);
  if (p->L > 0) {
    cfg.gridDim = grid_up;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = p->smem_up;
    e = cudaLaunchKernelEx(&cfg, lc_up_kernel<VT>, up);
    if (e != cudaSuccess) return e;
    if (ev && evi < nev) cudaEventRecord(ev[evi++], st);
  }
  cfg.gridDim = dim3(unsigned(p->stream_grid));
  cfg.blockDim = dim3(kStreamThreads);
  cfg.dynamicSmemBytes = p->smem_stream;
  e = cudaLaunchKernelEx(&cfg, lc_stream_kernel<VT, DIR>, sp);
  if (e != cudaSuccess) return e;
  if (ev && evi < nev) cudaEventRecord(ev[evi++], st);
  cfg.gridDim = p->L > 0 ? grid : dim3(1, grid.y);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = p->smem_down;
  e = cudaLaunchKernelEx(&cfg, lc_down_kernel<VT, DIR>, dp);
  if (e != cudaSuccess) return e;
  if (ev && evi < nev) cudaEventRecord(ev[evi++], st);
  return cudaGetLastError();
}

static int64_t extent(int layout, int64_t ld, int64_t n, int64_t batch) {
  return layout == LC_VEC_CONTIGUOUS ? (batch - 1) * ld + n : (n - 1) * ld + batch;
}

lc_status launch_execute(const lc_plan* p, const double* in, double* out, void* ws, cudaStream_t st,
                         cudaEvent_t const* ev, int nev) {
  if (!p || !in || !out) return LC_ERR_INVALID_ARG;
  {
    const char* a0 = reinterpret_cast<const char*>(in);
    const char* a1 = a0 + 8 * extent(p->layout, p->ld_in, p->n, p->batch);
    const char* b0 = reinterpret_cast<const char*>(out);
    const char* b1 = b0 + 8 * extent(p->layout, p->ld_out, p->n, p->batch);
    if (a0 < b1 && b0 < a1) return LC_ERR_ALIASING;
  }
  if (!ws) ws = p->d_ws;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != p->device) cudaSetDevice(p->device);
  const size_t wb = size_t(align_up(p->ntiles * p->w_tile_doubles * 8, 256));
  double* w = reinterpret_cast<double*>(ws);
  double* c = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + wb);
  int* flags = reinterpret_cast<int*>(reinterpret_cast<char*>(ws) + 2 * wb);
  int* cnt = flags + 64;
  UpParams up{};
  up.in = in; up.ld_in = p->ld_in; up.n = p->n; up.N = p->N; up.batch = p->batch;
  up.layout = p->layout; up.L = int(p->L); up.s = int(p->s); up.k = p->kup; up.gr = p->grup; up.G = p->group;
  up.T = p->d_T; up.B = p->d_B; up.w = w; up.cnt = cnt; up.flags = flags; up.w_tile = p->w_tile_doubles;
  up.cnt_tile = p->cnt_tile_ints;
  StreamParams sp{};
  sp.A = p->d_A; sp.w = w; sp.c = c; sp.in = in; sp.out = out; sp.tabA = p->d_tabA; sp.tabB = p->d_tabB;
  sp.flags = flags; sp.w_tile = p->w_tile_doubles; sp.ld_in = p->ld_in; sp.ld_out = p->ld_out; sp.n = p->n;
  sp.N = p->N; sp.batch = p->batch; sp.ntiles = p->ntiles; sp.nm2l = p->m2l_units; sp.nband = p->band_units;
  sp.layout = p->layout; sp.L = int(p->L); sp.s = int(p->s); sp.cb = p->bps; sp.nst = p->nst; sp.kb = p->kb;
  sp.gr_up = p->grup;
  DownParams dp{};
  dp.out = out; dp.ld_out = p->ld_out; dp.n = p->n; dp.N = p->N; dp.batch = p->batch; dp.layout = p->layout;
  dp.L = int(p->L); dp.s = int(p->s); dp.k = p->k; dp.gr = p->gr; dp.Tt = p->d_Tt; dp.B = p->d_B; dp.c = c;
  dp.w_tile = p->w_tile_doubles;
  const int64_t nsub = p->L > 0 ? (int64_t(4) << p->gr) : 1;
  if (nsub > 0x7fffffff || p->ntiles > 65535) {
    if (prev != p->device) cudaSetDevice(prev);
    return LC_ERR_INVALID_ARG;
  }
  const dim3 grid(unsigned(nsub), unsigned(p->ntiles));
  const dim3 grid_up(unsigned(p->L > 0 ? (int64_t(4) << p->grup) : 1), unsigned(p->ntiles));
  cudaError_t e;
  const int key = p->vt * 2 + p->dir;
  switch (key) {
    case 2: e = launch_vt<1, 0>(p, up, sp, dp, grid_up, grid, st, ev, nev); break;
    case 3: e = launch_vt<1, 1>(p, up, sp, dp, grid_up, grid, st, ev, nev); break;
    case 4: e = launch_vt<2, 0>(p, up, sp, dp, grid_up, grid, st, ev, nev); break;
    case 5: e = launch_vt<2, 1>(p, up, sp, dp, grid_up, grid, st, ev, nev); break;
    case 8: e = launch_vt<4, 0>(p, up, sp, dp, grid_up, grid, st, ev, nev); break;
    case 9: e = launch_vt<4, 1>(p, up, sp, dp, grid_up, grid, st, ev, nev); break;
    case 16: e = launch_vt<8, 0>(p, up, sp, dp, grid_up, grid, st, ev, nev); break;
    case 17: e = launch_vt<8, 1>(p, up, sp, dp, grid_up, grid, st, ev, nev); break;
    default: e = cudaErrorInvalidValue;
  }
  if (prev != p->device) cudaSetDevice(prev);
  return e == cudaSuccess ? LC_OK : record_cuda_error(e);
}

}  // namespace lc

extern "C" lc_status lc_execute(const lc_plan* p, const double* in, double* out, void* ws, void* stream) {
  return lc::launch_execute(p, in, out, ws, (cudaStream_t)stream, nullptr, 0);
}

extern "C" lc_status lc_execute_timed(const lc_plan* p, const double* in, double* out, void* ws, void* stream,
                                      void* const* ev, int32_t nev) {
  if (!p || !ev || nev < (p->L > 0 ? 4 : 3)) return LC_ERR_INVALID_ARG;
  return lc::launch_execute(p, in, out, ws, (cudaStream_t)stream, reinterpret_cast<cudaEvent_t const*>(ev), nev);
}

extern "C" lc_status lc_execute_host(const lc_plan* p_, const double* h_in, double* h_out, void* stream) {
  lc_plan* p = const_cast<lc_plan*>(p_);
  if (!p || !h_in || !h_out) return LC_ERR_INVALID_ARG;
  const int64_t ein = lc::extent(p->layout, p->ld_in, p->n, p->batch);
  const int64_t eout = lc::extent(p->layout, p->ld_out, p->n, p->batch);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  const size_t need = size_t(std::max(ein, eout)) * 8;
  if (p->stage_bytes < need) {
    cudaFree(p->d_stage_in);
    cudaFree(p->d_stage_out);
    p->d_stage_in = p->d_stage_out = nullptr;
    p->stage_bytes = 0;
    if (cudaMalloc(&p->d_stage_in, need) != cudaSuccess || cudaMalloc(&p->d_stage_out, need) != cudaSuccess) {
      cudaSetDevice(prev);
      return LC_ERR_OUT_OF_MEMORY;
    }
    p->stage_bytes = need;
  }
  cudaStream_t st = (cudaStream_t)stream;
  lc_status rc = LC_OK;
  cudaError_t e = cudaMemcpyAsync(p->d_stage_in, h_in, size_t(ein) * 8, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) rc = lc::record_cuda_error(e);
  if (rc == LC_OK) rc = lc::launch_execute(p, p->d_stage_in, p->d_stage_out, nullptr, st, nullptr, 0);
  if (rc == LC_OK) {
    e = cudaMemcpyAsync(h_out, p->d_stage_out, size_t(eout) * 8, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) rc = lc::record_cuda_error(e);
  }
  cudaSetDevice(prev);
  return rc;
}

#ifdef LC_PHASE_TIMING
extern "C" int lc_debug_clear() {
  static unsigned long long zero[1 << 16];
  for (int k = 0; k < 3 * 16; ++k)
    if (cudaMemcpyToSymbol(lc::g_lc_ts, zero, sizeof(zero), sizeof(zero) * size_t(k)) != cudaSuccess) return 1;
  return 0;
}
extern "C" int lc_debug_timestamps(int kern, unsigned long long* host_out, long long count) {
  if (kern < 0 || kern > 2 || count > (1 << 20)) return 1;
  return cudaMemcpyFromSymbol(host_out, lc::g_lc_ts, sizeof(unsigned long long) * count,
                              sizeof(unsigned long long) * (size_t(kern) << 20)) == cudaSuccess ? 0 : 1;
}
#endif
