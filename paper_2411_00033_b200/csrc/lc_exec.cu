// lc_exec.cu -- execution stage (Alg. 4, alg:fastercomplete) on sm_100a.
// Both parities are processed together (the same A_hat serves sigma = 0 and 1).
// Three engines (the plan picks one):
//
// Engine 1 (single vectors, small batches), three kernels chained with programmatic dependent
// launch and release/acquire flags in the workspace:
//   lc_up_kernel     one CTA per subtree of 2^kup leaf segments x VT vectors (about one wave):
//                    step 1 (eq:wMM) on the fp64 tensor cores (DMMA, 8 leaves per warp item) and
//                    step 2 (Alg. a.1) inside the subtree; the last CTA of each
//                    group of sibling subtrees continues to level 0.  Writes w of every level.
//   lc_stream_kernel persistent, warp-specialised: a producer lane streams the level-major A_hat
//                    arena and the w windows with TMA bulk copies into an mbarrier ring (finest
//                    level first); 3 M2L warps apply step 3; 4 band warps run
//                    the direct band of step 6 (Alg. 1 restricted to j < j_end(i)) on dynamically
//                    scheduled units.  Both take units from global counters.
//   lc_down_kernel   one CTA per subtree: step 4 ("faster downward spreading")
//                    along the ancestor chain and down the subtree (DMMA), step 5 (eq:step5, DMMA),
//                    step 7 (C^{-1}) added to the band result and stored.
// Engine 2 (batches of short vectors): lc_tile_kernel, one CTA per 8-vector tile, the whole
//   algorithm in one right-to-left pass over the leaf segments with every intermediate on chip.
// Engine 3 (batches of long vectors): lc_up3_kernel (persistent, double-buffered steps 1-2 over chunks
//   of 8-vector subtrees; writes w of every level), then lc_range_kernel, the same pass as engine 2
//   over ranges of leaves of each tile with w read from the workspace.
#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <mutex>
#include <cstdio>
#include <cstring>

#include "lc_internal.h"

namespace lc {


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
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {  // no arrival
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
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
// 1-D TMA bulk copy shared -> global (SASS: UBLKCP), bulk-group completion
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_and_wait_read() {
  asm volatile("cp.async.bulk.commit_group;\n\tcp.async.bulk.wait_group.read 0;" ::: "memory");
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
// padding beyond n).  .cg (L2 only) for data produced by other SMs.
__device__ __forceinline__ void cp_async8(void* dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16z(void* dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
// named barriers of the streaming kernel: 1 = band warps, 2 = M2L warps (the producer joins neither)
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// release/acquire helpers for the readiness flags (gpu scope)
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// gpu-scope acquire-release RMW: releases the CTA's prior stores (ordered before it by a barrier)
// and acquires those released by earlier arrivers (threadfence-reduction without full fences)
__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_flag(const int* p) {
  while (ld_acquire(p) == 0) __nanosleep(64);
}

// fp64 tensor-core MMA (DMMA m8n8k4, row.col): lane l holds A[l>>2][l&3], B[l&3][l>>2] and
// C[l>>2][2(l&3)], C[l>>2][2(l&3)+1]; d += A B.
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// Phase timestamps for the debug build (-DLC_PHASE_TIMING): %globaltimer (ns) per CTA and phase.
#ifdef LC_PHASE_TIMING
__device__ unsigned long long g_lc_ts[3][1 << 20];
__device__ __forceinline__ void lc_ts_any(int kern, int slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  const unsigned cta = blockIdx.y * gridDim.x + blockIdx.x;
  if (cta * 8 + slot < (1u << 20)) g_lc_ts[kern][cta * 8 + slot] = t;
}
#define LC_TS(k, s) \
  do {                                   \
    if (threadIdx.x == 0) lc_ts_any(k, s); \
  } while (0)
#define LC_TS_T(k, s) lc_ts_any(k, s)
#else
#define LC_TS(k, s) ((void)0)
#define LC_TS_T(k, s) ((void)0)
#endif

// ---------------------------------------------------------------- parameters
// flags (workspace ints): [0] up main-phase arrivals, [1] fine levels of w ready,
// [2] finished level-0 continuations, [3] coarse levels of w ready, [4] finished
// streaming CTAs, [5] predecessor complete (input readable), [10] next M2L unit,
// [11] next band unit (dynamic schedule of the streaming kernel), [12] streaming kernel
// complete (for the down kernel), [13] down CTAs past that flag.
struct UpParams {
  const double* in;
  const double* Tpad;  // [2][SMAX][M], zero rows m >= s
  const double* B;     // B(0) [M][M]
  int64_t ld_in, n, N, batch;
  int layout, L, s, k, gr, G, fstride, vec16;
  int noflags;  // engine 3: the range kernel waits for the whole grid (griddepcontrol), no flags
  int ksub;     // M2M levels done inside the CTA's subtree (<= k); the rest by the continuation
  int64_t R0;   // first subtree (partitioned up pass, NEXT-2), else 0
  int nocont;   // partitioned up pass: no continuation (the coarse levels follow the root exchange)
  int phase;    // host side: -1 whole execution; partitioned up pass: 0 the up kernel, 1 coarse levels + rest
  int contonly; // partitioned up pass, phase 1: only the continuation, from groups of the (exchanged) roots
  int kc;       // engine 3 (lc_up3_kernel): subtrees per chunk = 2^kc
  int nbuf;     // engine 3: f buffers of the up pass (1 or 2)
  int tpr;      // rows per parity of Tpad (32 or 64)
  int64_t ntiles;
  double* w;
  int* cnt;
  int* flags;
  int64_t w_tile, cnt_tile;
};
template <int SMAX>
struct UpArgs {
  UpParams p;
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
  int band_lo;      // first band unit (leaf range) of a partitioned plan (NEXT-2), else 0
  int blo[32];      // first M2L block per level (partitioned plan: the rows of its leaf range), else 0
  int nblk[32];     // M2L blocks per level (else 2^(g+1) - 1)
  int layout, L, s, cb, nst, kb, gr_up;
  int lvorder[32];  // M2L level order: position o -> level
  int nup;          // CTAs of the up kernel's main phase (their arrivals on flags[0]: fine levels ready)
};
using StreamArgs = StreamParams;

struct DownParams {
  double* out;
  int* flags;
  const double* c;     // c_m2l
  const double* Tpad;  // [2][SMAX][M], zero rows m >= s
  const double* B;     // B(0) [M][M]
  int64_t ld_out, n, N, batch, w_tile;
  int layout, L, s, k;
  int bulk;  // TMA bulk loads allowed (out 16-byte aligned, ld_out even, full tiles only)
  int nstream;     // CTAs of the streaming kernel (their arrivals on flags[4] release the down kernel)
  int64_t sub_lo;  // first subtree of a partitioned plan (NEXT-2), else 0
};

#ifndef LC_UP3_SKIP
#define LC_UP3_SKIP 0  // experiment builds only: skip parts of the engine-3 up pass (1 w stores, 2 subtree M2M, 4 step 1)
#endif
// ============================================================== up kernel
// Alg. a.1, rows [R0, R1) of one parent:
// parent[n] = sum_{k<=n} b_nk (x0_k + (-1)^(n-k) x1_k)   (B(1) = B(0) with the odd diagonals
// negated, App. A3).  The children are loaded into registers first (sum/difference formed
// once), B(0) is a uniform constant-bank operand (the row group is warp-uniform), and every row
// keeps two partial sums (even / odd k) to halve its dependent DFMA chain.
template <int R0, int R1>
__device__ __forceinline__ void m2m_rows_core(const double* __restrict__ Bs, const double (&zp)[R1],
                                              const double (&zm)[R1], double* __restrict__ out) {
  constexpr int NR = R1 - R0;
  double acc[NR];
#pragma unroll
  for (int n = R0; n < R1; ++n) {
    double ae = 0.0, ao = 0.0;
#pragma unroll
    for (int k = 0; k <= n; k += 2) {
      if (k + 1 <= n) {  // b_{n k}, b_{n k+1}: one broadcast 16-byte load
        const double2 b = *reinterpret_cast<const double2*>(Bs + n * kM + k);
        ae = fma(b.x, ((n - k) & 1) ? zm[k] : zp[k], ae);
        ao = fma(b.y, ((n - k - 1) & 1) ? zm[k + 1] : zp[k + 1], ao);
      } else {
        ae = fma(Bs[n * kM + k], zp[k], ae);
      }
    }
    acc[n - R0] = ae + ao;
  }
#pragma unroll
  for (int i = 0; i < NR; ++i) out[R0 + i] = acc[i];
}

template <int R0, int R1>
__device__ __forceinline__ void m2m_rows(const double* __restrict__ Bs, const double* __restrict__ x0,
                                         const double* __restrict__ x1, double* __restrict__ out) {
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
  m2m_rows_core<R0, R1>(Bs, zp, zm, out);
}

// m2m_rows for one vector per item (VT = 1): a warp's items lie 36 doubles apart, so the 16-byte chunk
// c of every lane's x falls into the bank groups 2P + c (mod 8), half of them; lanes of odd quads load
// the chunks of each pair (c, c ^ 1) in swapped order, so that each load of a warp covers all eight
// groups (no 2-way conflicts), and the pair is swapped back in registers (same arithmetic)
#ifndef LC_M2M_ROT
#define LC_M2M_ROT 1
#endif
template <int R0, int R1>
__device__ __forceinline__ void m2m_rows_rot(const double* __restrict__ Bs, const double* __restrict__ x0,
                                             const double* __restrict__ x1, double* __restrict__ out, bool odd) {
  constexpr int NC = (R1 + 1) / 2;
  double2 ta[NC], tb[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int cp = (c ^ 1) < NC ? (c ^ 1) : c;
    const int cl = odd ? cp : c;
    ta[c] = *reinterpret_cast<const double2*>(x0 + 2 * cl);
    tb[c] = *reinterpret_cast<const double2*>(x1 + 2 * cl);
  }
  double zp[R1], zm[R1];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int cp = (c ^ 1) < NC ? (c ^ 1) : c;
    const double2 a2 = odd ? ta[cp] : ta[c];
    const double2 b2 = odd ? tb[cp] : tb[c];
    zp[2 * c] = a2.x + b2.x;
    zm[2 * c] = a2.x - b2.x;
    if (2 * c + 1 < R1) {
      zp[2 * c + 1] = a2.y + b2.y;
      zm[2 * c + 1] = a2.y - b2.y;
    }
  }
  m2m_rows_core<R0, R1>(Bs, zp, zm, out);
}

// one tree level in shared memory ([sigma][node][v][M]); one thread per (row group, sigma,
// parent, v), each warp on a single row group: [0,10), [10,15), [15,18) carry 55, 65 and 51
// DFMA.  Six of the eight warps work; a level is one round for up to 64 (sigma, parent, v).
template <int VT>
__device__ __forceinline__ void m2m_level(const double* __restrict__ Bs, const double* __restrict__ ch,
                                          double* __restrict__ pa, int lp) {
  const int np = 1 << lp;
  const int per = 2 * np * VT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpr = (blockDim.x >> 5) / 3;  // warps per row group
  if (warp >= 3 * wpr) return;
  const int rg = warp % 3;
  for (int r = (warp / 3) * 32 + lane; r < per; r += wpr * 32) {
    const int v = r % VT;
    const int sp = r / VT;
    const int P = sp & (np - 1);
    const int sg = sp >> lp;
    const double* x0 = ch + ((sg * 2 * np + 2 * P) * VT + v) * kM;
    double* o = pa + r * kM;
    if (VT == 1 && LC_M2M_ROT && per >= 32) {  // whole warps of items (narrow levels: no conflicts to remove)
      const bool odd = (lane >> 2) & 1;
      if (rg == 0)
        m2m_rows_rot<0, 10>(Bs, x0, x0 + VT * kM, o, odd);
      else if (rg == 1)
        m2m_rows_rot<10, 15>(Bs, x0, x0 + VT * kM, o, odd);
      else
        m2m_rows_rot<15, 18>(Bs, x0, x0 + VT * kM, o, odd);
    } else if (rg == 0)
      m2m_rows<0, 10>(Bs, x0, x0 + VT * kM, o);
    else if (rg == 1)
      m2m_rows<10, 15>(Bs, x0, x0 + VT * kM, o);
    else
      m2m_rows<15, 18>(Bs, x0, x0 + VT * kM, o);
  }
}

// stage the leaf range [R 2^k, (R+1) 2^k) of segments of vector tile `tile` into fs ([v][leaf][fst],
// cp.async, not committed), zero padding beyond n
template <int VT>
__device__ __forceinline__ void up_stage(const UpParams& P, double* fs, int64_t R, int64_t tile, int nleaf, int fst) {
  const int tid = threadIdx.x;
  const int seglen = 2 * P.s, tlen = nleaf * seglen;
  const int64_t j0 = R * tlen;
  if (P.layout == LC_VEC_CONTIGUOUS) {
#pragma unroll 1
    for (int v = 0; v < VT; ++v) {
      const int64_t gv = tile * VT + v;
      const double* src = P.in + gv * P.ld_in + j0;
      const int64_t lim = gv < P.batch ? P.n - j0 : 0;  // valid elements of this vector in the tile
      if (P.vec16) {
        const int npair = tlen / 2;
        for (int q = tid; q < npair; q += blockDim.x) {
          const int jj = 2 * q;
          const int lf = jj / seglen, x = jj - lf * seglen;
          const int64_t rem = lim - jj;
          const uint32_t bytes = rem >= 2 ? 16u : (rem == 1 ? 8u : 0u);
          cp_async16z(fs + (v * nleaf + lf) * fst + x, bytes ? src + jj : P.in, bytes);
        }
      } else {
        for (int jj = tid; jj < tlen; jj += blockDim.x) {
          const int lf = jj / seglen, x = jj - lf * seglen;
          const bool ok = jj < lim;
          cp_async8(fs + (v * nleaf + lf) * fst + x, ok ? src + jj : P.in, ok ? 8u : 0u);
        }
      }
    }
  } else {
    for (int idx = tid; idx < VT * tlen; idx += blockDim.x) {
      const int jj = idx / VT, v = idx - jj * VT;  // v fastest: coalesced in the batch layout
      const int64_t gv = tile * VT + v, j = j0 + jj;
      const bool ok = gv < P.batch && j < P.n;
      const int lf = jj / seglen, x = jj - lf * seglen;
      cp_async8(fs + (v * nleaf + lf) * fst + x, ok ? P.in + j * P.ld_in + gv : P.in, ok ? 8u : 0u);
    }
  }
}

template <int VT, int SMAX>
__device__ __forceinline__ void up_step1(const double* __restrict__ Ts, const double* __restrict__ fs, int fst,
                                         int nleaf, int s, double* __restrict__ leaf) {
  // step 1: w(L-1)[t][k] = sum_m f[2s t + 2m + sigma] T(sigma)[m][k]   (eq:wMM), on the fp64
  // tensor cores: one warp item = (vector v, 8 leaves); A = T(sigma)^T (modes padded to 24 = 3
  // row tiles), B[m][leaf] = f[2s leaf + 2m + sigma] (one 16-byte load feeds both parities),
  // K = 4 ceil(s/4) rows of T (rows m >= s are zero, so reads past a segment contribute nothing).
  {
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
    const int lr = lane >> 2, lc = lane & 3;
    // a warp item fills the 8 MMA columns with lpi leaves x vpi vectors (subtrees of < 8 leaves pack
    // several vectors per item); column col = (vector vg vpi + col / lpi, leaf lf0 + col % lpi)
    const int llpi = nleaf >= 8 ? 3 : (nleaf >= 4 ? 2 : (nleaf >= 2 ? 1 : 0));  // log2 lpi (nleaf = 2^k)
    const int lpi = 1 << llpi;
    const int vpi = (8 >> llpi) < VT ? (8 >> llpi) : VT;
    const int ngrp = (nleaf + 7) >> 3;
    const int nitems = (VT / vpi) * ngrp;
    for (int item = warp; item < nitems; item += nw) {
      const int vg = item / ngrp, lf0 = (item - vg * ngrp) * 8;
      const int bv = vg * vpi + (lr >> llpi), blf = lf0 + (lr & (lpi - 1));
      const bool okb = lr < lpi * vpi && blf < nleaf;  // this lane's B column
      const double* fp = fs + (okb ? bv * nleaf + blf : 0) * fst + 2 * lc;
      const double* tq = Ts + lc * kM + lr;
      double acc[2][3][2];
#pragma unroll
      for (int mt = 0; mt < 3; ++mt) acc[0][mt][0] = acc[0][mt][1] = acc[1][mt][0] = acc[1][mt][1] = 0.0;
      auto kstep = [&](int kk) {
        double2 f2 = *reinterpret_cast<const double2*>(fp + 8 * kk);  // f[2m], f[2m+1], m = 4kk + lc
        if (!okb) f2 = make_double2(0.0, 0.0);
        const double* t0 = tq + 4 * kk * kM;  // T(0)[m][8 mt + lr]
#pragma unroll
        for (int mt = 0; mt < 3; ++mt) {
          const bool okm = 8 * mt + lr < kM;
          const double a0 = okm ? t0[8 * mt] : 0.0;
          const double a1 = okm ? t0[SMAX * kM + 8 * mt] : 0.0;
          dmma(acc[0][mt], a0, f2.x);
          dmma(acc[1][mt], a1, f2.y);
        }
      };
      // K = 4 ceil(s/4) rows of T: the rows m >= s are zero, so short segments (s = 20 for
      // n = 10^7) skip the all-zero K steps
      const int nks = (s + 3) >> 2;
      if (nks == SMAX / 4) {
#pragma unroll
        for (int kk = 0; kk < SMAX / 4; ++kk) kstep(kk);
      } else {
#pragma unroll 1
        for (int kk = 0; kk < nks; ++kk) kstep(kk);
      }
#pragma unroll
      for (int sg = 0; sg < 2; ++sg)
#pragma unroll
        for (int mt = 0; mt < 3; ++mt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int col = 2 * lc + h, mode = 8 * mt + lr;
            const int v = vg * vpi + (col >> llpi), lf = lf0 + (col & (lpi - 1));
            if (col < lpi * vpi && lf < nleaf && mode < kM) leaf[((sg * nleaf + lf) * VT + v) * kM + mode] = acc[sg][mt][h];
          }
    }
  }
}

#ifndef LC_UP8_MINB
#define LC_UP8_MINB 2  // resident CTAs per SM of the 8-vector up kernel (engine 3's first pass)
#endif
template <int VT, int SMAX>
__global__ void __launch_bounds__(kThreads, (VT == 8 && SMAX == 32) ? LC_UP8_MINB : 2) lc_up_kernel(const __grid_constant__ UpArgs<SMAX> A) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ int s_last;
  const UpParams& P = A.p;
  const int s = P.s, k = P.k, fst = P.fstride;
  const int tid = threadIdx.x;
  const int nleaf = 1 << k;
  const int seglen = 2 * s;
  double* Ts = reinterpret_cast<double*>(smem);          // [2][SMAX][M], zero rows m >= s
  double* Bs = Ts + 2 * SMAX * kM;                       // B(0) [M][M]
  double* fs = reinterpret_cast<double*>(smem + up_const_bytes(SMAX));  // [v][leaf][fstride]
  double* tree = reinterpret_cast<double*>(smem + up_const_bytes(SMAX) + align_up((int64_t(VT) * nleaf * fst + 2 * SMAX) * 8, 128));
  auto tree_off = [&](int j) { return ((1 << j) - 1) * 2 * VT * kM; };

  const int64_t R = blockIdx.x + P.R0;
  const int64_t tile = blockIdx.y;
  LC_TS(0, 0);
  // plan constants into shared memory (broadcast operands of steps 1 and 2)
  for (int i = tid; i < SMAX * kM; i += blockDim.x) cp_async16(Ts + 2 * i, P.Tpad + 2 * i);
  for (int i = tid; i < kMM / 2; i += blockDim.x) cp_async16(Bs + 2 * i, P.B + 2 * i);
  cp_async_commit();
  griddep_wait();  // the input may be produced by the preceding kernel; w/c of the previous execution are free
  // Trigger the dependent (streaming) launch only now: every streaming CTA then starts after the
  // whole previous execution completed, so it can never observe flags of that execution.
  griddep_launch();
  if (tid == 0 && blockIdx.x == 0 && tile == 0 && !P.contonly)
    st_release(&P.flags[5], 1);  // the streaming kernel may read the input
  double* wt = P.w + tile * P.w_tile;
  const int64_t VM = int64_t(VT) * kM;
  const int ksub = P.ksub;        // subtree levels merged here; the CTA leaves 2^(k-ksub) roots
  const int dsub = k - ksub;
  int g;           // the continuation starts at level g with this CTA's 2^contrib nodes from `node` on
  int64_t node;
  int contrib;
  if (P.contonly) {
    // phase 1 of a partitioned up pass: every subtree root of the vector is in w (exchanged); each
    // CTA takes a group of them and runs the continuation
    g = P.gr;
    contrib = min(P.G, g);
    node = int64_t(blockIdx.x) << contrib;
    cp_async_wait<0>();
    __syncthreads();
  } else {
  up_stage<VT>(P, fs, R, tile, nleaf, fst);
  // zero tail read by the branch-free step 1 of the last leaf (m up to SMAX-1)
  for (int x = tid; x < 2 * SMAX; x += blockDim.x) fs[VT * nleaf * fst + x] = 0.0;
  if (fst > seglen)  // and the segment padding (fstride = 2s + 2 for even s)
    for (int x = tid; x < VT * nleaf; x += blockDim.x) *reinterpret_cast<double2*>(fs + x * fst + seglen) = make_double2(0.0, 0.0);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  LC_TS(0, 1);

  up_step1<VT, SMAX>(Ts, fs, fst, nleaf, s, tree + tree_off(k));
  __syncthreads();
  LC_TS(0, 2);
  // each subtree level goes to the workspace as soon as it exists, so the stores drain while the
  // next M2M levels compute (the release below then waits for little more than the last level)
  auto write_level = [&](int j) {
    const int g = P.gr + j;
    const int cnt2 = int((int64_t(1) << j) * VM / 2);
    for (int sg = 0; sg < 2; ++sg) {
      double2* dst = reinterpret_cast<double2*>(wt + (w_level_offset_units(g) + sg * nseg(g) + (R << j)) * VM);
      const double2* src = reinterpret_cast<const double2*>(tree + tree_off(j) + sg * (int64_t(1) << j) * VM);
      for (int i = tid; i < cnt2; i += blockDim.x) dst[i] = src[i];
    }
  };
  write_level(k);
  // step 2 inside the subtree (ksub levels: an early exit frees the SM for the streaming kernel; the
  // remaining levels are merged by the continuation below, beside the stream)
  for (int j = k; j >= 1 + dsub; --j) {
    m2m_level<VT>(Bs, tree + tree_off(j), tree + tree_off(j - 1), j - 1);
    __syncthreads();
    write_level(j - 1);
  }
  LC_TS(0, 3);
  // the fine levels (gr..L-1) of the whole batch are ready once every CTA got here
  __syncthreads();
  LC_TS(0, 4);
  // release arrival on flags[0]: the streaming kernel acquire-loads the full count (the fine levels of
  // every CTA), so no last arriver needs a second release; the down kernel re-arms the counter
  if (tid == 0 && !P.noflags) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(&P.flags[0]) : "memory");

  if (P.nocont) return;  // partitioned up pass: the coarse levels come after the exchange of the roots
  g = P.gr + dsub;
  node = R << dsub;
  contrib = dsub;
  }
  // upward continuation above the subtree roots: the last arriver of each
  // group of 2^G nodes merges them G levels up (threadfence-reduction pattern).  A CTA that
  // stopped dsub levels early arrives once for its 2^dsub roots (contrib: log2 of the nodes an
  // arrival stands for).
  while (g > 0) {
    const int ge = min(P.G, g);
    const int64_t grp = node >> ge;
    __syncthreads();
    if (tid == 0) {
      int* c = P.cnt + tile * P.cnt_tile + (nseg(g) - 4) + grp;
      const int old = atom_add_acq_rel(c, 1);
      const int last = (old == (1 << (ge - contrib)) - 1);
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
      m2m_level<VT>(Bs, tree + tree_off(j), tree + tree_off(j - 1), j - 1);
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
    g -= ge;  // the next arrival (after a barrier, acquire-release) publishes these stores
    node = grp;
    contrib = 0;
    LC_TS(0, 6);
  }
  if ((P.contonly || P.gr + dsub > 0) && !P.noflags) {  // this CTA produced one of the 4 level-0 nodes of its tile
    __syncthreads();
    if (tid == 0) {
      const int total = 4 * int(gridDim.y);
      if (atom_add_acq_rel(&P.flags[2], 1) == total - 1) {
        atomicExch(&P.flags[2], 0);
        st_release(&P.flags[3], 1);
      }
    }
  }
  LC_TS(0, 7);
}


// one M2M of a pair of siblings held apart: out[sigma][v] = B(0) left[sigma][v] + B(1) right[sigma][v]
// (rows r = (sigma, v) of [2][VT][M], the same row-group split as m2m_level)
template <int VT>
__device__ __forceinline__ void m2m_pair(const double* __restrict__ Bs, const double* __restrict__ left,
                                         const double* __restrict__ right, double* __restrict__ out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpr = (blockDim.x >> 5) / 3;
  if (warp >= 3 * wpr) return;
  const int rg = warp % 3;
  for (int r = (warp / 3) * 32 + lane; r < 2 * VT; r += wpr * 32) {
    const double* x0 = left + r * kM;
    const double* x1 = right + r * kM;
    double* o = out + r * kM;
    if (rg == 0)
      m2m_rows<0, 10>(Bs, x0, x1, o);
    else if (rg == 1)
      m2m_rows<10, 15>(Bs, x0, x1, o);
    else
      m2m_rows<15, 18>(Bs, x0, x1, o);
  }
}

// Engine 3's upward pass (steps 1-2 of Alg. 4 for batches of long vectors), persistent: CTA b takes
// chunks b, b + grid, ... of 2^kc consecutive subtrees (2^k leaf segments x 8 vectors each) and walks
// their subtrees left to right with the f of the next subtree staged (cp.async, double buffer) while
// the current one computes.  A subtree root that is a left child waits in shared memory for its
// sibling; each merge (step 2) stores the parent's w at once, so the chunk root (level gr - kc) is
// reached inside the CTA.  Above it the arrival counters of lc_up_kernel merge groups of 2^G chunk
// roots (the last arriver continues).  No flags: the range kernel waits for the whole grid.
template <int SMAX>
__global__ void __launch_bounds__(kThreads, 2) lc_up3_kernel(const __grid_constant__ UpArgs<SMAX> A) {
  constexpr int VT = 8;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ int s_last;
  const UpParams& P = A.p;
  const int s = P.s, k = P.k, fst = P.fstride, tid = threadIdx.x;
  const int nleaf = 1 << k, seglen = 2 * s;
  const int64_t VM = int64_t(VT) * kM;
  const int64_t fbuf = align_up((int64_t(VT) * nleaf * fst + 2 * SMAX) * 8, 128) / 8;  // doubles per f buffer
  const int nbuf = P.nbuf;                         // 2: double-buffered f; 1: the next f lands during M2M
  double* Ts = reinterpret_cast<double*>(smem);  // [2][SMAX][M], zero rows m >= s
  double* Bs = Ts + 2 * SMAX * kM;               // B(0) [M][M]
  double* fs0 = reinterpret_cast<double*>(smem + up_const_bytes(SMAX));  // nbuf x [v][leaf][fst] + zero tail
  double* tree = fs0 + nbuf * fbuf;
  auto tree_off = [&](int j) { return ((1 << j) - 1) * 2 * VT * kM; };
  double* pend = tree + tree_off(k + 1);  // [kc][2][VT][M]: left siblings waiting, by level
  double* cur = pend + P.kc * 2 * VM;     // [2][2][VT][M]: merged parents (ping-pong)

  for (int i = tid; i < SMAX * kM; i += blockDim.x) {  // [2][SMAX][M] from [2][tpr][M]: SMAX M / 2 pairs per parity
    const int sg = i >= SMAX * kM / 2 ? 1 : 0, jj = i - sg * (SMAX * kM / 2);
    cp_async16(Ts + sg * SMAX * kM + 2 * jj, P.Tpad + int64_t(sg) * P.tpr * kM + 2 * jj);
  }
  for (int i = tid; i < kMM / 2; i += blockDim.x) cp_async16(Bs + 2 * i, P.B + 2 * i);
  for (int b = 0; b < nbuf; ++b) {  // zero tail and segment padding of the buffers (never written by cp.async)
    double* fs = fs0 + b * fbuf;
    for (int x = tid; x < 2 * SMAX; x += blockDim.x) fs[VT * nleaf * fst + x] = 0.0;
    if (fst > seglen)
      for (int x = tid; x < VT * nleaf; x += blockDim.x) *reinterpret_cast<double2*>(fs + x * fst + seglen) = make_double2(0.0, 0.0);
  }
  cp_async_commit();
  griddep_wait();  // the input may be produced by the preceding kernel; w of the previous execution is free
  griddep_launch();

  const int nb = 1 << P.kc;
  const int groot = P.gr - P.kc;                   // level of the chunk roots
  const int64_t cpt = int64_t(4) << groot;         // chunks per tile
  const int64_t nchunks = cpt * P.ntiles;
  const int64_t mych = blockIdx.x < nchunks ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t J = mych * nb;
  auto locate = [&](int64_t j, int64_t& tile, int64_t& R) {
    const int64_t it = blockIdx.x + (j >> P.kc) * int64_t(gridDim.x);
    tile = it / cpt;
    R = (it - tile * cpt) * nb + (j & (nb - 1));
  };
  // VEC layout, 16-byte aligned rows: thread t stages the pairs (leaf q / s, x = 2 (q % s)), q = t and
  // t + 256, of every vector (nleaf s <= 2 x 256 pairs), so the addressing is computed once
  const bool fast = P.layout == LC_VEC_CONTIGUOUS && P.vec16 && nleaf * s <= 2 * int(blockDim.x);
  int my_so[2], my_jj[2];
  bool my_on[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int q = tid + h * int(blockDim.x);
    const int lf = q / s, x = 2 * (q - lf * s);
    my_on[h] = q < nleaf * s;
    my_so[h] = lf * fst + x;
    my_jj[h] = lf * seglen + x;
  }
  auto stage = [&](double* fs, int64_t R, int64_t tile) {
    if (!fast) {
      up_stage<VT>(P, fs, R, tile, nleaf, fst);
      return;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!my_on[h]) continue;
      const int64_t j0 = R * int64_t(nleaf * seglen) + my_jj[h];
      const double* src = P.in + tile * VT * P.ld_in + j0;
#pragma unroll
      for (int v = 0; v < VT; ++v) {
        const int64_t rem = (tile * VT + v < P.batch) ? P.n - j0 : 0;
        const uint32_t bytes = rem >= 2 ? 16u : (rem == 1 ? 8u : 0u);
        cp_async16z(fs + v * nleaf * fst + my_so[h], bytes ? src + v * P.ld_in : P.in, bytes);
      }
    }
  };
  if (J > 0) {
    int64_t t0, r0;
    locate(0, t0, r0);
    stage(fs0, r0, t0);
  }
  cp_async_commit();
  for (int64_t j = 0; j < J; ++j) {
    int64_t tile, R;
    locate(j, tile, R);
    if (nbuf == 2 && j + 1 < J) {
      int64_t t1, r1;
      locate(j + 1, t1, r1);
      stage(fs0 + ((j + 1) & 1) * fbuf, r1, t1);
    }
    cp_async_commit();
    if (nbuf == 2) cp_async_wait<1>(); else cp_async_wait<0>();  // the f of subtree j landed
    __syncthreads();
    if (!(LC_UP3_SKIP & 4)) up_step1<VT, SMAX>(Ts, fs0 + (nbuf == 2 ? (j & 1) * fbuf : 0), fst, nleaf, s, tree + tree_off(k));
    __syncthreads();
    if (nbuf == 1 && j + 1 < J) {  // one buffer: the next subtree's f lands during this one's M2M and stores
      int64_t t1, r1;
      locate(j + 1, t1, r1);
      stage(fs0, r1, t1);
      cp_async_commit();
    }
    double* wt = P.w + tile * P.w_tile;
    auto store_w = [&](int g, int64_t node, int cnt, const double* src) {  // cnt nodes of level g, [sigma][cnt][v][M]
      if (LC_UP3_SKIP & 1) return;
      const int c2 = int(cnt * VM / 2);
      const double2* sp = reinterpret_cast<const double2*>(src);
      double2* d0 = reinterpret_cast<double2*>(wt + (w_level_offset_units(g) + node) * VM);
      double2* d1 = reinterpret_cast<double2*>(wt + (w_level_offset_units(g) + nseg(g) + node) * VM) - c2;
#pragma unroll 4
      for (int i = tid; i < 2 * c2; i += blockDim.x) {
        const double2 x2 = sp[i];
        (i < c2 ? d0 : d1)[i] = x2;
      }
    };
    store_w(P.gr + k, R << k, nleaf, tree + tree_off(k));
    for (int lv = k; lv >= 1; --lv) {
      if (!(LC_UP3_SKIP & 2)) m2m_level<VT>(Bs, tree + tree_off(lv), tree + tree_off(lv - 1), lv - 1);
      __syncthreads();
      store_w(P.gr + lv - 1, R << (lv - 1), 1 << (lv - 1), tree + tree_off(lv - 1));
    }
    // merge with the waiting left siblings while this node is a right child inside the chunk
    int g = P.gr;
    int64_t u = R;
    const double* x = tree;  // [2][VT][M]
    int pp = 0;
    while (g > groot && (u & 1)) {
      double* o = cur + pp * 2 * VM;
      m2m_pair<VT>(Bs, pend + (g - groot - 1) * 2 * VM, x, o);
      __syncthreads();
      --g;
      u >>= 1;
      store_w(g, u, 1, o);
      x = o;
      pp ^= 1;
    }
    if (g > groot) {  // a left child: wait for the sibling
      double* d = pend + (g - groot - 1) * 2 * VM;
      for (int i = tid; i < 2 * VM; i += blockDim.x) d[i] = x[i];
      continue;  // (the barrier at the top of the next subtree orders these copies before any reuse)
    }
    // chunk root (level groot, node u) written: upward continuation across chunks, as lc_up_kernel
    int64_t node = u;
    while (g > 0) {
      const int ge = min(P.G, g);
      const int64_t grp = node >> ge;
      __syncthreads();
      if (tid == 0) {
        int* c = P.cnt + tile * P.cnt_tile + (nseg(g) - 4) + grp;
        const int old = atom_add_acq_rel(c, 1);
        const int last = (old == (1 << ge) - 1);
        if (last) atomicExch(c, 0);  // self-reset for the next launch
        s_last = last;
      }
      __syncthreads();
      if (!s_last) break;
      __threadfence();
      const int cnt2 = int((int64_t(1) << ge) * VM / 2);
      for (int sg = 0; sg < 2; ++sg) {
        const double2* src =
            reinterpret_cast<const double2*>(wt + (w_level_offset_units(g) + sg * nseg(g) + (grp << ge)) * VM);
        double2* dst = reinterpret_cast<double2*>(tree + tree_off(ge) + sg * 2 * cnt2);
        for (int i = tid; i < cnt2; i += blockDim.x) dst[i] = __ldcg(src + i);
      }
      __syncthreads();
      for (int lv = ge; lv >= 1; --lv) {
        m2m_level<VT>(Bs, tree + tree_off(lv), tree + tree_off(lv - 1), lv - 1);
        __syncthreads();
      }
      for (int lv = 0; lv < ge; ++lv) store_w(g - ge + lv, grp << lv, 1 << lv, tree + tree_off(lv));
      g -= ge;
      node = grp;
    }
  }
  cp_async_wait<0>();
}

// ============================================================== streaming kernel
constexpr int kM2lWarps = 3;   // consumer warps applying M2L to the A_hat ring
constexpr int kBandWarps = 4;  // band + down warps (independent pipeline)
constexpr int kStreamThreads = 32 * (1 + kM2lWarps + kBandWarps);
constexpr int kBandThreads = 32 * kBandWarps;
constexpr int kM2lThreads = 32 * kM2lWarps;

__device__ __forceinline__ void band_sync() { named_sync(1, kBandThreads); }

// M2L unit q (< nm2l) = (chunk, tile): chunk = (level g, blocks [b0, b0+nb)), nb <= cb, levels in
// the order lvorder[]; tiles innermost so concurrent CTAs share A_hat in L2.
// cstart[o] = first chunk of the o-th level of the order (shared-memory table).
__device__ __forceinline__ void m2l_unit(int q, int ntiles, int L, int cb, const int* cstart, const int* lvord,
                                         const int* blo, const int* nblk, int& g, int& b0, int& nb, int& tile) {
  int ch = q;
  tile = 0;
  if (ntiles > 1) {
    ch = q / ntiles;
    tile = q - ch * ntiles;
  }
  int o = 0;
  while (o + 1 < L && cstart[o + 1] <= ch) ++o;
  g = lvord[o];
  b0 = blo[g] + (ch - cstart[o]) * cb;
  const int bg = blo[g] + nblk[g];
  nb = (bg - b0) < cb ? (bg - b0) : cb;
}

// ---------------------------------------------------------------- band unit (step 6)
// rows of 2^kb leaf segments x one vector tile; result (without C^{-1}) stored to out,
// where the down unit of the same rows (same CTA, later) picks it up.
template <int VT, int DIR>
__device__ __forceinline__ void band_unit(const StreamParams& P, int tile, int lr, double* ta, double* tb, double* gt,
                                          double* zst, int tp, int btid) {
  // padding of the band tiles: one double every 2^kPadSh.  Several vectors: the lanes of a warp
  // take rows 2 kBandR apart (one pad per 16 separates their banks); one vector: the lanes take
  // consecutive leaf segments 2s apart (one pad per 64 keeps the segment stride odd for s = 32)
  constexpr int kPadSh = VT == 1 ? 6 : 4;
  const int s = P.s, kb = P.kb;
  const int nleaf = 1 << kb;
  const int seglen = 2 * s;
  const int64_t U0 = int64_t(lr) << kb;
  const int64_t i0 = U0 * seglen;
  const int rows = nleaf * seglen;
  const int tcols = (nleaf + 2) * seglen;
  const int tbl = int((P.N - i0) < tcols ? (P.N - i0) : tcols);  // valid band-table entries
  const bool mma8 = VT == 8 && s <= 32;
  const int tp8 = tcols + 2 * kBandR + 2;  // unpadded row stride of the tensor-core path (<= tp)
  if (mma8) {
    // tensor-core path: unpadded tiles, 16-byte cp.async (zero fill beyond N / n)
    for (int x = 2 * btid; x < tcols + 2 * kBandR; x += 2 * kBandThreads) {
      const int valid = tbl - x;
      const uint32_t bytes = valid >= 2 ? 16u : (valid == 1 ? 8u : 0u);
      cp_async16z(tb + x, bytes ? P.tabB + i0 + x : P.tabB, bytes);
    }
#pragma unroll 1
    for (int v = 0; v < VT; ++v) {
      const int64_t gv = int64_t(tile) * VT + v;
      int lim = 0;
      if (gv < P.batch) lim = int((P.n - i0) < tcols ? (P.n - i0) : tcols);
      if (lim < 0) lim = 0;
      if (P.layout == LC_VEC_CONTIGUOUS && (reinterpret_cast<uintptr_t>(P.in) % 16 == 0) && (P.ld_in % 2 == 0)) {
        const double* src = P.in + gv * P.ld_in + i0;
        for (int x = 2 * btid; x < tcols + 2 * kBandR; x += 2 * kBandThreads) {
          const int valid = lim - x;
          const uint32_t bytes = valid >= 2 ? 16u : (valid == 1 ? 8u : 0u);
          cp_async16z(gt + v * tp8 + x, bytes ? src + x : P.in, bytes);
        }
      } else {
        for (int x = btid; x < tcols + 2 * kBandR; x += kBandThreads) {
          const bool ok = x < lim;
          const double* src = P.layout == LC_VEC_CONTIGUOUS ? P.in + gv * P.ld_in + i0 + x : P.in + (i0 + x) * P.ld_in + gv;
          cp_async8(gt + v * tp8 + x, ok ? src : P.in, ok ? 8u : 0u);
        }
      }
    }
  } else {
  for (int x = btid; x < tcols + 2 * kBandR; x += kBandThreads) {
    const bool ok = x < tbl;
    cp_async8(tb + x + (x >> kPadSh), ok ? P.tabB + i0 + x : P.tabB, ok ? 8u : 0u);
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
        cp_async8(gt + v * tp + x + (x >> kPadSh), ok ? src + x : P.in, ok ? 8u : 0u);
      }
    } else {
      for (int x = btid; x < tcols + 2 * kBandR; x += kBandThreads) {
        const bool ok = x < lim;
        cp_async8(gt + v * tp + x + (x >> kPadSh), ok ? P.in + (i0 + x) * P.ld_in + gv : P.in, ok ? 8u : 0u);
      }
    }
  }
  }
  cp_async_commit();
#ifdef LC_PHASE_TIMING
  unsigned long long tb0, tb1, tb2, tb3;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tb0));
#endif
  cp_async_wait<0>();
  band_sync();
#ifdef LC_PHASE_TIMING
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tb1));
#endif
  if (mma8) {
    // fp64 tensor cores (DMMA m8n8k4): per (segment uu, parity sigma) the band is
    // Z[r][v] = sum_{c=r}^{2s-1} K[r][c] G[c][v], rows i = i0 + 2s uu + 2r + sigma, columns
    // j = i0 + 2s uu + 2c + sigma, K[r][c] = a[c-r] b[2s uu + r + c + sigma] (Toeplitz x Hankel,
    // each lane forms its A-fragment element with one DMUL), G[c][v] = g_v[j] (8 vectors = the
    // MMA n dimension).  Blocks with c < r everywhere are skipped; f and b are zero beyond n, N.
    const int warp = btid >> 5, lane = btid & 31;
    const int nrb = (s + 7) / 8, nkc = (2 * s + 3) / 4;
    const int lr_ = lane >> 2, lc_ = lane & 3;
    for (int job = warp; job < nleaf * 2; job += kBandThreads / 32) {
      const int uu = job >> 1, sg = job & 1;
      const int base = uu * seglen + sg;  // tile-local index of row r = 0 / column c = 0
      double acc[4][2];
#pragma unroll
      for (int rb = 0; rb < 4; ++rb) acc[rb][0] = acc[rb][1] = 0.0;
      for (int kc = 0; kc < nkc; ++kc) {
        const int c = 4 * kc + lc_;  // this lane's A column / B row
        const int xg = base + 2 * c;
        double bfr = c < 2 * s ? gt[lr_ * tp8 + xg] : 0.0;  // G[c][v = lane >> 2]
        if (DIR == 1) bfr *= double(i0 + xg);
#pragma unroll
        for (int rb = 0; rb < 4; ++rb) {
          if (rb < nrb && 4 * kc + 3 >= 8 * rb) {  // warp-uniform: the block has entries with c >= r
            const int r = 8 * rb + lr_;
            const int xb = base + r + c;
            const double a = (c >= r && c < 2 * s && r < s) ? ta[c - r] * tb[xb] : 0.0;
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[rb][0]), "+d"(acc[rb][1])
                         : "d"(a), "d"(bfr));
          }
        }
      }
#pragma unroll
      for (int rb = 0; rb < 4; ++rb) {
        const int r = 8 * rb + lr_;
        if (rb < nrb && r < s) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int v = 2 * lc_ + h;
            const int ii = base + 2 * r;
            const int64_t ir = i0 + ii;
            double z = acc[rb][h];
            if (DIR == 1) {
              z *= double(2 * ir + 1);
              if (ir == 0) z += gt[v * tp8];  // entry (0,0) of A^{-1}C is 1 (reading R2)
            }
            zst[(v * rows + ii) + ((v * rows + ii) >> kPadSh)] = z;
          }
        }
      }
    }
  } else {
  // item = (v, segment uu, parity sigma, block of kBandR same-parity rows m = kBandR t + r).
  // Band of row i' = i + 2r (i the block's first row): sum_c a[c-r] b[i+r+c] g[i+2c], c >= r,
  // i + 2c < j_end; a = tabA, b = tabB, g = f (L2C) or j f_j (C2L).  Sliding windows of a and
  // b live in registers (slots rotate with c): each step loads 3 values for kBandR rows.
  const int ntb = (s + kBandR - 1) / kBandR;
  const int items = VT * nleaf * 2 * ntb;
  for (int it = btid; it < items; it += kBandThreads) {
    // single vector: segment fastest, so the lanes of a warp share the row block and with it the
    // trip count of the column loop (no divergence; 1.7x in tools/ubench_band.cu)
    int uu, v, sg, tb_i;
    if (VT == 1) {
      uu = it & (nleaf - 1);
      const int r_ = it >> kb;
      v = 0;
      sg = r_ & 1;
      tb_i = r_ >> 1;
    } else {  // (row block fastest; measured faster with several vectors per tile)
      tb_i = it % ntb;
      int r_ = it / ntb;
      sg = r_ & 1;
      r_ >>= 1;
      uu = r_ & (nleaf - 1);
      v = r_ >> kb;
    }
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
      bw[r] = tb[(ii + r) + ((ii + r) >> kPadSh)];
    }
    const int ngrp = (cmax + 1) / kBandR;
    int c0 = 0;
    for (int gi = 0; gi < ngrp; ++gi, c0 += kBandR) {
#pragma unroll
      for (int q = 0; q < kBandR; ++q) {
        const int c = c0 + q;
        aw[q] = ta[c];
        const int xb = ii + kBandR - 1 + c, xg = ii + 2 * c;
        bw[(q + kBandR - 1) % kBandR] = tb[xb + (xb >> kPadSh)];
        double gval = gv_t[xg + (xg >> kPadSh)];
        if (DIR == 1) gval *= double(i + 2 * c);
#pragma unroll
        for (int r = 0; r < kBandR; ++r) acc[r] = fma(aw[(q - r + kBandR) % kBandR] * bw[(r + q) % kBandR], gval, acc[r]);
      }
    }
#pragma unroll
    for (int q = 0; q < kBandR; ++q) {  // remainder: c = c0 + q <= cmax
      const int c = c0 + q;
      if (c <= cmax) {
        aw[q] = ta[c];
        const int xb = ii + kBandR - 1 + c, xg = ii + 2 * c;
        bw[(q + kBandR - 1) % kBandR] = tb[xb + (xb >> kPadSh)];
        double gval = gv_t[xg + (xg >> kPadSh)];
        if (DIR == 1) gval *= double(i + 2 * c);
#pragma unroll
        for (int r = 0; r < kBandR; ++r) acc[r] = fma(aw[(q - r + kBandR) % kBandR] * bw[(r + q) % kBandR], gval, acc[r]);
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
        zst[(v * rows + ii + 2 * r) + ((v * rows + ii + 2 * r) >> kPadSh)] = z;
      }
    }
  }
  }
  band_sync();
#ifdef LC_PHASE_TIMING
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tb2));
#endif
  // coalesced store of the band result (steps 4, 5 and 7 are added by the down unit)
  const int olim = int((P.n - i0) < rows ? (P.n - i0) : rows);
#pragma unroll 1
  for (int v = 0; v < VT; ++v) {
    const int64_t gv = int64_t(tile) * VT + v;
    if (gv >= P.batch) break;
    if (P.layout == LC_VEC_CONTIGUOUS) {
      double* dst = P.out + gv * P.ld_out + i0;
      for (int x = btid; x < olim; x += kBandThreads) dst[x] = zst[(v * rows + x) + ((v * rows + x) >> kPadSh)];
    } else {
      for (int x = btid; x < olim; x += kBandThreads)
        P.out[(i0 + x) * P.ld_out + gv] = zst[(v * rows + x) + ((v * rows + x) >> kPadSh)];
    }
  }
  band_sync();  // tiles are reused by the next unit
#ifdef LC_PHASE_TIMING
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tb3));
  if (btid == 0) {  // accumulated ns per CTA: [3] load wait, [4] compute, [5] store, [6] units
    const unsigned cta = blockIdx.x;
    g_lc_ts[1][cta * 8 + 3] += tb1 - tb0;
    g_lc_ts[1][cta * 8 + 4] += tb2 - tb1;
    g_lc_ts[1][cta * 8 + 5] += tb3 - tb2;
    g_lc_ts[1][cta * 8 + 6] += 1;
  }
#endif
}

template <int VT, int DIR>
__global__ void __launch_bounds__(kStreamThreads, 2) lc_stream_kernel(const __grid_constant__ StreamArgs A) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ int cstart[32];
  __shared__ int slotq[8];  // M2L unit of each ring slot (-1: end of work)
  __shared__ int s_band;
  const StreamParams& P = A;
  const int tid = threadIdx.x;
  const int s = P.s, cb = P.cb, nst = P.nst, kb = P.kb;
  const int64_t VM = int64_t(VT) * kM;
  const StreamSmem SL = stream_smem_layout(VT, cb, nst, kb, s);
  const int64_t a_bytes = align_up(int64_t(cb) * 3 * kMM * 8, 128);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SL.bars);
  uint64_t* empty = full + nst;
  const int tp = int(SL.tp);

  const int nband = int(P.nband), nm2l = int(P.nm2l);
  if (tid == 0) {
    int acc = 0;
    for (int o = 0; o < P.L && o < 32; ++o) {
      cstart[o] = acc;
      const int g = P.lvorder[o];
      acc += (P.nblk[g] + cb - 1) / cb;
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
        m2l_unit(q, ntiles, P.L, cb, cstart, P.lvorder, P.blo, P.nblk, g, b0, nb, tile);
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
            if (g >= P.gr_up)
              while (ld_acquire(&P.flags[0]) < P.nup) __nanosleep(64);  // every up CTA's fine levels
            else
              wait_flag(&P.flags[3]);
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
      // dynamic schedule: units are taken from a global counter (flags[10]) in the level order,
      // so CTAs that start late (SMs still busy with the up kernel) simply take fewer.  The unit
      // of each ring slot is published to the consumers in slotq[] before the slot's arrive.
      // The A_hat of the first nst units is plan data: issued before any dependency.
      int qs[8];
      int npre = 0;
      for (; npre < nst; ++npre) {
        const int q = atomicAdd(&P.flags[10], 1);
        if (q >= nm2l) break;
        qs[npre] = q;
        slotq[npre] = q;
        issue(q, npre, true, false);
      }
      for (int jj = 0; jj < npre; ++jj) issue(qs[jj], jj, false, true);
      int j = npre;
      if (npre == nst) {
        int qn = atomicAdd(&P.flags[10], 1);
        for (;; ++j) {
          mbar_wait(&empty[j % nst], uint32_t(((j / nst) - 1) & 1));
          if (qn >= nm2l) break;
          const int q = qn;
          qn = atomicAdd(&P.flags[10], 1);  // next unit, resolved while this one streams
          slotq[j % nst] = q;
          issue(q, j, true, true);
        }
      }
      slotq[j % nst] = -1;  // end of work: an arrive without transaction bytes
      mbar_arrive(&full[j % nst]);
    }
  } else if (tid < 32 * (1 + kM2lWarps)) {
    // ------------------------------------------------ M2L consumer warps
    const int ctid = tid - 32;
    for (int j = 0;; ++j) {  // j: M2L ring use counter
      const int slot = j % nst;
      mbar_wait(&full[slot], uint32_t((j / nst) & 1));
      const int q = slotq[slot];
      if (q < 0) break;
      int g, nb, b0, tile;
      m2l_unit(q, ntiles, P.L, cb, cstart, P.lvorder, P.blo, P.nblk, g, b0, nb, tile);
      const double* As = reinterpret_cast<const double*>(smem + SL.ring + slot * SL.slot);
      const double* wwin = reinterpret_cast<const double*>(smem + SL.ring + slot * SL.slot + a_bytes);
      double* ct = P.c + int64_t(tile) * P.w_tile + (w_level_offset_units(g) + 2 * int64_t(b0)) * VM;
      const int64_t sgstride = nseg(g) * VM;
      // item = (block b, mode kk): the even row u = 2b (r = 0 with column t = u+2, r = 1 with
      // t = u+3) and the odd row u+1 (r = 2 with t = u+3), both parities, all VT vectors:
      // 3 A_hat rows x 2 x VT dot products of length 18, each as two partial sums.
      if (VT <= 2) {
      for (int it = ctid; it < nb * kM; it += kM2lThreads) {
        const int bl = it / kM, kk = it - bl * kM;
        double e0[2][VT], e1[2][VT], o0[2][VT], o1[2][VT];  // even row / odd row partial sums
#pragma unroll
        for (int sg = 0; sg < 2; ++sg)
#pragma unroll
          for (int v = 0; v < VT; ++v) e0[sg][v] = e1[sg][v] = o0[sg][v] = o1[sg][v] = 0.0;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const int tloc = 2 * bl + (r == 0 ? 0 : 1);  // t - (2 b0 + 2)
          const double* arow = As + (3 * bl + r) * kMM + kk * kM;
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
              double p0 = 0.0, p1 = 0.0;
#pragma unroll
              for (int l = 0; l < kM; l += 2) {
                const double2 w2 = *reinterpret_cast<const double2*>(wp + l);
                p0 = fma(ar[l], w2.x, p0);
                p1 = fma(ar[l + 1], w2.y, p1);
              }
              if (r < 2) {
                e0[sg][v] += p0;
                e1[sg][v] += p1;
              } else {
                o0[sg][v] = p0;
                o1[sg][v] = p1;
              }
            }
        }
#pragma unroll
        for (int sg = 0; sg < 2; ++sg)
#pragma unroll
          for (int v = 0; v < VT; ++v) {
            ct[sg * sgstride + (2 * bl) * VM + v * kM + kk] = e0[sg][v] + e1[sg][v];
            ct[sg * sgstride + (2 * bl + 1) * VM + v * kM + kk] = o0[sg][v] + o1[sg][v];
          }
      }
      } else if (VT == 8) {
        // fp64 tensor cores (DMMA m8n8k4): output tile = (row segment u, 8 modes, parity sigma) x
        // 8 vectors; c(u) = sum_r A_hat_r w(t_r) with K = 18 modes in steps of 4 (padded to 20)
        const int lane = ctid & 31, warp = ctid >> 5;
        const int lr_ = lane >> 2, lc_ = lane & 3;
        const int ntl = 2 * nb * 3 * 2;  // (row ri, m-tile, sigma)
        for (int t = warp; t < ntl; t += kM2lWarps) {
          const int sg = t & 1, mt = (t >> 1) % 3, ri = (t >> 1) / 3;
          const int bl = ri >> 1;
          double c0 = 0.0, c1 = 0.0;
          const int nmat = (ri & 1) ? 1 : 2;
          for (int mi = 0; mi < nmat; ++mi) {
            const int r = (ri & 1) ? 2 : mi;
            const int tloc = (ri & 1) ? ri : ri + mi;  // t - (2 b0 + 2)
            const double* Am = As + (3 * bl + r) * kMM;
            const double* Wc = wwin + (sg * 2 * cb + tloc) * VM;
            const int row = 8 * mt + lr_;
#pragma unroll
            for (int kk = 0; kk < 5; ++kk) {
              const int kcol = 4 * kk + lc_;
              const double a = (row < kM && kcol < kM) ? Am[row * kM + kcol] : 0.0;
              const double b = kcol < kM ? Wc[lr_ * kM + kcol] : 0.0;  // W[k][vector lane >> 2]
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                           : "+d"(c0), "+d"(c1)
                           : "d"(a), "d"(b));
            }
          }
          const int row = 8 * mt + lr_;
          if (row < kM) {
            ct[sg * sgstride + ri * VM + (2 * lc_) * kM + row] = c0;
            ct[sg * sgstride + ri * VM + (2 * lc_ + 1) * kM + row] = c1;
          }
        }
      } else {  // wide vector tiles: one (row, mode) per thread, one A_hat row at a time
        const int nrows = 2 * nb;
        for (int it = ctid; it < nrows * kM; it += kM2lThreads) {
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
      }
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&empty[slot]);  // this warp is done with the slot
    }
    if (tid == 32) LC_TS_T(1, 7);
  } else {
    // ------------------------------------------------ band + down warps
    const int btid = tid - 32 * (1 + kM2lWarps);
    double* ta = reinterpret_cast<double*>(smem + SL.ta);
    double* tb = reinterpret_cast<double*>(smem + SL.tb);
    double* gt = reinterpret_cast<double*>(smem + SL.gt);
    double* zst = reinterpret_cast<double*>(smem + SL.zst);
    for (int x = btid; x < 2 * s + 2 * kBandR; x += kBandThreads) ta[x] = x < 2 * s ? P.tabA[x] : 0.0;
    {  // the input is readable once the predecessor of the up kernel completed
      if (P.L > 0) {
        if (btid == 0) wait_flag(&P.flags[5]);
      } else {
        griddep_wait();
      }
    }
    band_sync();
    for (;;) {  // dynamic schedule of the band units (flags[11])
      if (btid == 0) s_band = atomicAdd(&P.flags[11], 1);
      band_sync();
      const int u = s_band;
      band_sync();
      if (u >= nband) break;
      const int tile = ntiles > 1 ? u % ntiles : 0;
      const int lr = (ntiles > 1 ? u / ntiles : u) + P.band_lo;
      band_unit<VT, DIR>(P, tile, lr, ta, tb, gt, zst, tp, btid);
    }
    // this CTA's band rows are stored: an acquire-release arrival (the band warps' stores are ordered
    // before it by the band barrier); the last CTA releases flags[14] so the down kernel can fetch the
    // band rows while the M2L tail and the arrivals on flags[4] are still in flight
    band_sync();
    if (btid == 0 && atom_add_acq_rel(&P.flags[15], 1) == int(gridDim.x) - 1) {
      atomicExch(&P.flags[15], 0);
      st_release(&P.flags[14], 1);
    }
    LC_TS_T(1, 2);
  }
  __syncthreads();
  LC_TS(1, 1);
  if (tid == 0) {
    // release arrival: this CTA's c_m2l and band stores (ordered before it by the barrier) are
    // released; the down kernel's acquire load of the complete count synchronises with every arrival
    // (no last-arriver release: one fence per CTA on the critical path instead of two), and the down
    // kernel re-arms the counters
    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(&P.flags[4]) : "memory");
  }
}

// ============================================================== down kernel
// One CTA (8 warps) per (subtree of 2^kd leaf row segments, tile of VT vectors), about one
// wave.  Every dependent step is a warp-level operator with lane = Chebyshev mode:
//   * one cp.async round trip brings the c_m2l of the ancestors and of the whole subtree and
//     the band result of the rows into shared memory;
//   * step 4 along the ancestor chain (Horner: c(g) = B(p_g)^T c(g-1) + c_m2l(g); one warp per
//     (sigma, v)), then down the subtree level by level;
//   * step 5 with lane = row m: z_m = sum_k T(sigma)[m][k] c_k, the T row in registers;
//   * step 7 and a coalesced store.
// Operator inputs are loaded into registers before the arithmetic and every dot product runs
// as four partial sums, so a level costs one shared-memory round trip plus a 5-deep DFMA chain.
constexpr int kDownThreads = 256;
#ifndef LC_DOWN_NARROW_SPLIT
#define LC_DOWN_NARROW_SPLIT 1  // narrow subtree levels split over (sigma, v, parent) warps when 2 VT < warps
#endif
#ifndef LC_DOWN_PAR_ISSUE
#define LC_DOWN_PAR_ISSUE 1  // bulk path: the c_m2l copies issued by the lanes of warp 0 (one copy each)
#endif
#ifndef LC_DOWN_NARROW_JS
#define LC_DOWN_NARROW_JS 4  // subtree levels run as lane operators when split (the rest on DMMA; 3: +0.25 us, 5: +2 us at 10^6)
#endif

// (B(p)^T c)_l = (-1)^{pl} sum_n b_nl (-1)^{pn} c_n   (lane l), with column l of
// B(0) in registers (the ancestor chain and the narrow subtree levels reuse it), c broadcast from
// shared memory, four partial sums
__device__ __forceinline__ double l2l_lane_reg(const double (&b)[kM], const double* __restrict__ c, int p, int l) {
  double x[kM];
#pragma unroll
  for (int n = 0; n < kM; n += 2) {
    const double2 t = *reinterpret_cast<const double2*>(c + n);
    x[n] = t.x;
    x[n + 1] = t.y;
  }
  double e0 = 0.0, e1 = 0.0, o0 = 0.0, o1 = 0.0;
#pragma unroll
  for (int n = 0; n < kM; n += 4) {
    e0 = fma(b[n], x[n], e0);
    o0 = fma(b[n + 1], x[n + 1], o0);
    if (n + 2 < kM) e1 = fma(b[n + 2], x[n + 2], e1);
    if (n + 3 < kM) o1 = fma(b[n + 3], x[n + 3], o1);
  }
  const double e = e0 + e1, o = o0 + o1;
  const double r = p ? e - o : e + o;
  return (p && (l & 1)) ? -r : r;
}

// both children of one parent in one pass: with e = sum_{n even} b_nl c_n and o = sum_{n odd} b_nl c_n,
// (B(0)^T c)_l = e + o and (B(1)^T c)_l = (-1)^l (e - o)   (B(1) = B(0) with odd diagonals negated, App. A3)
__device__ __forceinline__ void l2l_lane_pair(const double (&b)[kM], const double* __restrict__ c, int l,
                                              double& r0, double& r1) {
  double x[kM];
#pragma unroll
  for (int n = 0; n < kM; n += 2) {
    const double2 t = *reinterpret_cast<const double2*>(c + n);
    x[n] = t.x;
    x[n + 1] = t.y;
  }
  double e0 = 0.0, e1 = 0.0, o0 = 0.0, o1 = 0.0;
#pragma unroll
  for (int n = 0; n < kM; n += 4) {
    e0 = fma(b[n], x[n], e0);
    o0 = fma(b[n + 1], x[n + 1], o0);
    if (n + 2 < kM) e1 = fma(b[n + 2], x[n + 2], e1);
    if (n + 3 < kM) o1 = fma(b[n + 3], x[n + 3], o1);
  }
  const double e = e0 + e1, o = o0 + o1;
  r0 = e + o;
  r1 = (l & 1) ? o - e : e - o;
}

template <int VT, int DIR, int SMAX, int NT>
__global__ void __launch_bounds__(NT, 512 / NT) lc_down_kernel(const DownParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int s = P.s, kd = P.k, L = P.L;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nthr = NT, nwarps = NT / 32;  // 256, or 128 for many small vector tiles
  const int gd = L > 0 ? L - 1 - kd : 0;  // level of the subtree root
  const int VM = VT * kM;
  const int nleaf = 1 << kd;
  const int seglen = 2 * s;
  const int64_t R = blockIdx.x + P.sub_lo;
  const int64_t tile = blockIdx.y;
  const int64_t U0 = R << kd;
  const int64_t i0 = U0 * seglen;
  const int rows = nleaf * seglen;
  // shared memory: B(0), T(sigma), cm = ancestors [g][sigma][v][M] (g < gd), subtree level j
  // at node offset gd + 2^j - 1 ([sigma][node][v][M]); zb = [v][rows]
  double* Bsh = reinterpret_cast<double*>(smem);  // B(0) [M][M]
  double* Tsh = Bsh + 2 * (kMM + 4);               // T(sigma) [2][SMAX][M] (after a spare [M][M] slot)
  double* cm = Tsh + 2 * SMAX * kM;
  double* zb = cm + (L > 0 ? (int64_t(gd) + (int64_t(2) << kd) - 1) * 2 * VM : 0);
  auto cm_anc = [&](int g) { return cm + g * 2 * VM; };
  auto cm_lvl = [&](int j) { return cm + (gd + (1 << j) - 1) * 2 * VM; };
  LC_TS(2, 0);
  // plan data first: B(0) and T(sigma) (padded to SMAX rows) into shared memory
  for (int i = tid; i < kMM / 2; i += nthr) cp_async16(Bsh + 2 * i, P.B + 2 * i);
  for (int i = tid; i < SMAX * kM; i += nthr) cp_async16(Tsh + 2 * i, P.Tpad + 2 * i);
  griddep_launch();
  const double* ct = P.c + tile * P.w_tile;
  const int olim = int((P.n - i0) < rows ? (P.n - i0) : rows);  // rows of this tile inside n
  // one TMA bulk-copy round trip when every piece is 16-byte aligned and whole (the c_m2l rows and,
  // in the vector layout, each vector's band rows of a full tile); otherwise per-element cp.async
  // with zero fill beyond n
  const bool bulk = P.bulk && P.layout == LC_VEC_CONTIGUOUS && olim == rows && (tile + 1) * VT <= P.batch;
  __shared__ __align__(8) uint64_t dbar;
  if (bulk && tid == 0) {
    // the band rows are complete once every streaming CTA's band warps arrived (flags[14]): fetch them
    // now, while the last M2L units and the arrivals on flags[4] are still in flight
    mbar_init(&dbar, 1);
    fence_mbar_init();
    wait_flag(&P.flags[14]);
    mbar_expect_tx(&dbar, uint32_t(VT) * uint32_t(rows) * 8u);
    const uint64_t pol = policy_evict_first();
    for (int v = 0; v < VT; ++v)
      bulk_g2s(zb + v * rows, P.out + (tile * VT + v) * P.ld_out + i0, uint32_t(rows) * 8u, &dbar, pol);
  }
  // c_m2l (and every band row) is complete once every streaming CTA arrived on flags[4] with release
  // semantics (cheaper than waiting for the grid to retire); the last down CTA to pass re-arms the
  // counters and readiness flags of this execution for the next one
  if (tid == 0) {
    while (ld_acquire(&P.flags[4]) < P.nstream) __nanosleep(64);
    if (atomicAdd(&P.flags[13], 1) == int(gridDim.x * gridDim.y) - 1) {
      P.flags[13] = 0;
      P.flags[14] = 0;
      P.flags[4] = 0;
      P.flags[0] = 0;
      P.flags[3] = 0;
      P.flags[5] = 0;
      P.flags[10] = 0;
      P.flags[11] = 0;
    }
  }
  __syncthreads();
  LC_TS(2, 1);
  if (bulk) {
    if (LC_DOWN_PAR_ISSUE && warp == 0) {
      // the arrival with the byte count first, then one bulk copy per lane (c_m2l of the gd ancestors and
      // of the kd + 1 subtree levels, both parities): issued in parallel instead of by one thread
      const uint32_t total = L > 0 ? uint32_t(gd + (2 << kd) - 1) * 2u * uint32_t(VM) * 8u : 0u;
      if (lane == 0) mbar_arrive_expect_tx(&dbar, total);  // the phase completes with every copy
      __syncwarp();
      if (L > 0) {
        const uint64_t pol = policy_evict_first();
        for (int c = lane; c < 2 * (gd + kd + 1); c += 32) {
          const int sg = c & 1;
          if (c < 2 * gd) {
            const int g = c >> 1;
            bulk_g2s(cm_anc(g) + sg * VM, ct + (w_level_offset_units(g) + sg * nseg(g) + (R >> (gd - g))) * VM,
                     uint32_t(VM) * 8u, &dbar, pol);
          } else {
            const int j = (c >> 1) - gd;
            bulk_g2s(cm_lvl(j) + sg * (1 << j) * VM, ct + (w_level_offset_units(gd + j) + sg * nseg(gd + j) + (R << j)) * VM,
                     uint32_t((1 << j) * VM) * 8u, &dbar, pol);
          }
        }
      }
    } else if (!LC_DOWN_PAR_ISSUE && tid == 0) {
      const uint32_t total = L > 0 ? uint32_t(gd + (2 << kd) - 1) * 2u * uint32_t(VM) * 8u : 0u;
      mbar_arrive_expect_tx(&dbar, total);  // the arrival: the phase completes with every copy
      const uint64_t pol = policy_evict_first();
      if (L > 0) {
        for (int g = 0; g < gd; ++g)
          for (int sg = 0; sg < 2; ++sg)
            bulk_g2s(cm_anc(g) + sg * VM, ct + (w_level_offset_units(g) + sg * nseg(g) + (R >> (gd - g))) * VM,
                     uint32_t(VM) * 8u, &dbar, pol);
        for (int j = 0; j <= kd; ++j)
          for (int sg = 0; sg < 2; ++sg)
            bulk_g2s(cm_lvl(j) + sg * (1 << j) * VM, ct + (w_level_offset_units(gd + j) + sg * nseg(gd + j) + (R << j)) * VM,
                     uint32_t((1 << j) * VM) * 8u, &dbar, pol);
      }
    }
    __syncthreads();
    mbar_wait(&dbar, 0);
  } else {
  if (L > 0) {
    for (int g = 0; g < gd; ++g) {
      const int64_t a = R >> (gd - g);
      for (int sg = 0; sg < 2; ++sg) {
        const double* src = ct + (w_level_offset_units(g) + sg * nseg(g) + a) * VM;
        double* dst = cm_anc(g) + sg * VM;
        for (int i = tid; i < VM / 2; i += nthr) cp_async16(dst + 2 * i, src + 2 * i);
      }
    }
    for (int j = 0; j <= kd; ++j) {
      const int g = gd + j;
      const int cnt2 = (1 << j) * VM / 2;
      for (int sg = 0; sg < 2; ++sg) {
        const double* src = ct + (w_level_offset_units(g) + sg * nseg(g) + (R << j)) * VM;
        double* dst = cm_lvl(j) + sg * (1 << j) * VM;
        for (int i = tid; i < cnt2; i += nthr) cp_async16(dst + 2 * i, src + 2 * i);
      }
    }
  }
#pragma unroll 1
  for (int v = 0; v < VT; ++v) {
    const int64_t gv = tile * VT + v;
    const int lim = gv < P.batch ? olim : 0;
    for (int x = tid; x < rows; x += nthr) {
      const bool ok = x < lim;
      const double* src = P.layout == LC_VEC_CONTIGUOUS ? P.out + gv * P.ld_out + i0 + x : P.out + (i0 + x) * P.ld_out + gv;
      cp_async8(zb + v * rows + x, ok ? src : P.out, ok ? 8u : 0u);
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  }
  LC_TS(2, 2);

  if (L > 0) {
    // step 4 along the ancestor chain (Horner), one warp per (sigma, v), then the subtree root
    // column `lane` of B(0) in registers for the chain and the narrow subtree levels (b_{n l})
    double bcol[kM];
#pragma unroll
    for (int n = 0; n < kM; ++n) bcol[n] = Bsh[n * kM + (lane < kM ? lane : 0)];
    if (gd > 0) {
      for (int ch = warp; ch < 2 * VT; ch += nwarps) {
        double acc = lane < kM ? cm_anc(0)[ch * kM + lane] : 0.0;
        double* scr = cm_anc(0) + ch * kM;  // the running vector is kept in place of c_m2l(0)
        for (int g = 1; g <= gd; ++g) {
          const double own = lane < kM ? (g < gd ? cm_anc(g) : cm_lvl(0))[ch * kM + lane] : 0.0;
          const int p = int((R >> (gd - g)) & 1);
          const double r = l2l_lane_reg(bcol, scr, p, lane);
          acc = r + own;
          __syncwarp();
          scr = (g < gd ? cm_anc(g) : cm_lvl(0)) + ch * kM;
          if (lane < kM) scr[lane] = acc;
          __syncwarp();
        }
      }
      __syncthreads();
    }
    LC_TS(2, 3);
    // step 4 down the subtree, level by level, every L2L as the lane
    // operator above (lane = child mode, the column of B(0) in registers, both children per parent).
    {
      // narrow levels (j <= 3, at most 4 parents per sigma): one warp per (sigma, v) runs them one after
      // another, lane = mode, both children of a parent in one pass -- no CTA barrier between them
      const bool split = LC_DOWN_NARROW_SPLIT && 2 * VT < nwarps;
      const int jn = min(kd, split ? LC_DOWN_NARROW_JS : 3);
      if (split) {
        // few vectors (2 VT chains < warps): one warp per (sigma, v, parent) and a CTA barrier per level,
        // so the 1 + 2 + 4 parents of a chain are not walked by one warp while the others wait (same
        // arithmetic per element)
        for (int j = 1; j <= jn; ++j) {
          const int nodes = 1 << j, half = nodes >> 1;
          const double* par = cm_lvl(j - 1);
          double* cur = cm_lvl(j);
          for (int it = warp; it < 2 * VT * half; it += nwarps) {
            const int ch = it / half, Pn = it - ch * half;
            const int sg = ch / VT, v = ch - sg * VT;
            double r0, r1;
            l2l_lane_pair(bcol, par + ((sg * half + Pn) * VT + v) * kM, lane, r0, r1);
            if (lane < kM) {
              cur[((sg * nodes + 2 * Pn) * VT + v) * kM + lane] += r0;
              cur[((sg * nodes + 2 * Pn + 1) * VT + v) * kM + lane] += r1;
            }
          }
          __syncthreads();
        }
      } else
      for (int ch = warp; ch < 2 * VT; ch += nwarps) {
        const int sg = ch / VT, v = ch - sg * VT;
        for (int j = 1; j <= jn; ++j) {
          const int nodes = 1 << j;
          const double* par = cm_lvl(j - 1);
          double* cur = cm_lvl(j);
          for (int Pn = 0; Pn < (nodes >> 1); ++Pn) {
            double r0, r1;
            l2l_lane_pair(bcol, par + ((sg * (nodes >> 1) + Pn) * VT + v) * kM, lane, r0, r1);
            if (lane < kM) {
              cur[((sg * nodes + 2 * Pn) * VT + v) * kM + lane] += r0;
              cur[((sg * nodes + 2 * Pn + 1) * VT + v) * kM + lane] += r1;
            }
          }
          __syncwarp();
        }
      }
      __syncthreads();
      if (jn == 3) LC_TS(2, 6);
      // wide levels on the fp64 tensor cores: warp item = 8 parent columns (sigma, P, v); for child
      // parity p, A_p[k][n] = (-1)^(p(k+n)) b_nk (rows k padded to 24, K = n padded to 20; blocks with
      // n < k everywhere skipped), and the children 2P+p accumulate A_p c_parent.  The operator
      // fragments are the same for every level and item: held in registers.
      const int lr = lane >> 2, lc = lane & 3;
      double af[5][3];
#pragma unroll
      for (int kk = 0; kk < 5; ++kk)
#pragma unroll
        for (int mt = 0; mt < 3; ++mt) {
          const int n = 4 * kk + lc, k = 8 * mt + lr;
          af[kk][mt] = (k < kM && n < kM) ? Bsh[n * kM + k] : 0.0;  // b_nk (zero for n < k)
        }
      for (int j = jn + 1; j <= kd; ++j) {
        const int nodes = 1 << j, half = nodes >> 1;
        const double* par = cm_lvl(j - 1);
        double* cur = cm_lvl(j);
        const int ncol = nodes * VT;  // parent columns, both parities
        for (int c0 = warp * 8; c0 < ncol; c0 += nwarps * 8) {
          const int col = c0 + lr;
          const bool okc = col < ncol;
          const double* xp = par + (okc ? col : 0) * kM;
          double bv[5];
#pragma unroll
          for (int kk = 0; kk < 5; ++kk) {
            const int n = 4 * kk + lc;
            bv[kk] = (okc && n < kM) ? xp[n] : 0.0;
          }
          double acc[2][3][2];
#pragma unroll
          for (int mt = 0; mt < 3; ++mt)
            acc[0][mt][0] = acc[0][mt][1] = acc[1][mt][0] = acc[1][mt][1] = 0.0;
#pragma unroll
          for (int kk = 0; kk < 5; ++kk) {
#pragma unroll
            for (int mt = 0; mt < 3; ++mt) {
              if (4 * kk + 3 < 8 * mt) continue;  // n < k for the whole block
              const int k = 8 * mt + lr, n = 4 * kk + lc;
              const double a0 = af[kk][mt];
              const double a1 = ((k + n) & 1) ? -a0 : a0;
              dmma(acc[0][mt], a0, bv[kk]);
              dmma(acc[1][mt], a1, bv[kk]);
            }
          }
#pragma unroll
          for (int mt = 0; mt < 3; ++mt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int k = 8 * mt + lr, co = c0 + 2 * lc + h;
              if (k < kM && co < ncol) {
                const int v = co % VT, sp = co / VT;
                const int Pn = sp & (half - 1), sg = sp >> (j - 1);
                double* d0 = cur + ((sg * nodes + 2 * Pn) * VT + v) * kM + k;
                d0[0] += acc[0][mt][h];
                d0[VT * kM] += acc[1][mt][h];
              }
            }
        }
        __syncthreads();
      }
    }
    LC_TS(2, 7);
    LC_TS(2, 4);
    // step 5: z^sigma += c(L-1) T(sigma)^T (eq:step5) on the fp64 tensor cores: warp item =
    // (sigma, v, 8 leaves); A = T(sigma) (SMAX/8 row tiles of m, K = 18 modes padded to 20),
    // B[k][leaf] = c(L-1)[leaf][k]; the result is added to the band result in zb.
    {
      const int lr = lane >> 2, lc = lane & 3;
      const double* cl = cm_lvl(kd);
      const int ngrp = (nleaf + 7) >> 3;
      for (int item = warp; item < 2 * VT * ngrp; item += nwarps) {
        const int sg = item & 1, r_ = item >> 1;
        const int v = r_ / ngrp, lf0 = (r_ - v * ngrp) * 8;
        const bool okb = lf0 + lr < nleaf;
        const double* cp = cl + ((sg * nleaf + (okb ? lf0 + lr : 0)) * VT + v) * kM;
        const double* tq = Tsh + (sg * SMAX + lr) * kM;
        double acc[SMAX / 8][2];
#pragma unroll
        for (int mt = 0; mt < SMAX / 8; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < (kM + 3) / 4; ++kk) {
          const int kx = 4 * kk + lc;
          const bool okk = kx < kM;
          const double b = (okb && okk) ? cp[kx] : 0.0;
#pragma unroll
          for (int mt = 0; mt < SMAX / 8; ++mt) {
            const double a = okk ? tq[8 * mt * kM + kx] : 0.0;
            dmma(acc[mt], a, b);
          }
        }
#pragma unroll
        for (int mt = 0; mt < SMAX / 8; ++mt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int m = 8 * mt + lr, lf = lf0 + 2 * lc + h;
            if (m < s && lf < nleaf) zb[v * rows + lf * seglen + 2 * m + sg] += acc[mt][h];
          }
      }
    }
    __syncthreads();
  }
  LC_TS(2, 5);
  // step 7: C^{-1} (L2C); coalesced store (whole aligned tiles: scaled in place, one TMA bulk store
  // per vector)
  const double inv_pi = 0.318309886183790671537767526745028724;
  if (bulk) {
    for (int v = 0; v < VT; ++v)
      for (int ii = tid; ii < rows; ii += nthr) {
        const int64_t i = i0 + ii;
        if (DIR == 0) zb[v * rows + ii] *= (i == 0 ? inv_pi : 2.0 * inv_pi);
      }
    fence_proxy_async();  // the scaled rows are visible to the bulk copy (async proxy)
    __syncthreads();
    if (tid == 0) {
      for (int v = 0; v < VT; ++v)
        bulk_s2g(P.out + (tile * VT + v) * P.ld_out + i0, zb + v * rows, uint32_t(rows) * 8u);
      bulk_commit_and_wait_read();  // shared memory stays valid until the copies have read it
    }
    return;
  }
#pragma unroll 1
  for (int v = 0; v < VT; ++v) {
    const int64_t gv = tile * VT + v;
    if (gv >= P.batch) break;
    for (int ii = tid; ii < olim; ii += nthr) {
      const int64_t i = i0 + ii;
      double z = zb[v * rows + ii];
      if (DIR == 0) z *= (i == 0 ? inv_pi : 2.0 * inv_pi);
      if (P.layout == LC_VEC_CONTIGUOUS)
        P.out[gv * P.ld_out + i] = z;
      else
        P.out[i * P.ld_out + gv] = z;
    }
  }
}

// ============================================================== per-tile streaming kernel
// Batched transforms of short vectors (many vector tiles): one CTA runs the whole of Alg. 4 for a
// tile of 8 vectors in ONE right-to-left pass over the leaf segments U = 2^(L+1)-1 .. 0, keeping
// every intermediate on chip (no w / c_m2l round trip through HBM, no inter-CTA flags).
// The pass order works because A is upper triangular and every interaction is local:
//   * row segment u of level g takes the M2L of column segments t = u+2 (and u+3 for even u)
//     (eq:globalij: block b has rows 2b, 2b+1 and columns 2b+2, 2b+3), which lie to its right;
//   * the band of leaf row segment U reaches the end of segment U+1 (j_end, R4);
//   * c of a segment is its M2L plus the L2L of its parent's c (step 4), and a parent is
//     entered (at its rightmost leaf) no later than its children.
// Leaf step U (one CTA barrier per step; a three-stage software pipeline over the leaves):
//   [band]   z(U) = direct band of rows U (step 6)                        warps 0-3
//   [eval]   z(U+1) += T(sigma) c(L-1, U+1) (step 5), C^{-1} (step 7), store      warps 0-3
//   [step 1] w(L-1, U) = f_U^sigma T(sigma)                                warps 4-5
//   [M2M]    w(g-1, u/2) = B(0) w(g, u) + B(1) w(g, u+1) while the segment u completed at leaf
//            U+1 is a left child (step 2)                                  warps 4-5
//   [chain]  c(g, u_g) += B(p)^T c(g-1, u_g/2) for the levels entered at U (step 4)  warps 6-7
//   [M2L]    c_m2l(g, u') for the levels the next leaf U-1 enters (step 3)           warps 4-7
// and the cp.async prefetch of leaf U-2.  Slots are chosen so that nothing a step writes is read
// in the same step: w ring of 3 per level, c by segment parity (mod 3 on the leaf level), z by
// leaf parity, f / lambda ring of 4 leaves.  All contractions run on the fp64 tensor cores (DMMA
// m8n8k4) with the 8 vectors of the tile as the n dimension, 2-3 accumulator chains per warp.
constexpr int kTileThreads = 256;
constexpr int kTileV = 8;                  // vectors per tile (= DMMA n)
constexpr int kTS = kTileV * kM;           // doubles per (segment, sigma) state
// f row stride: >= s and 4 (mod 8) doubles, so the 8-byte reads [lr * fst + lc + 4 kc] of a half warp
// (lr < 4, lc < 4) hit 16 distinct bank pairs; >= 4 ceil(s/4), the K extent of step 1
__host__ __device__ inline int tile_fst(int s) { int f = 4; while (f < s) f += 8; return f; }
// engines 2 and 3 take s <= kTileSMax (5 row tiles of 8); T(sigma) is staged as [2][tile_trows(s)][M]
// with rows >= s zero (step 1 reads 4 ceil(s/4) of them)
constexpr int kTileSMax = 40;
__host__ __device__ inline int tile_trows(int s) { return s <= 32 ? 32 : kTileSMax; }
// the per-tile kernel stages T(sigma) transposed, [2][M][tile_tstride(s)] (row stride 4 or 12 mod 16
// doubles): the A fragments of step 1 (T^T, rows = modes) and of step 5 (T, rows = positions) then hit 16
// distinct bank pairs per half warp (the [m][M] layout's stride 18 gives 2-way conflicts on both)
__host__ __device__ inline int tile_tstride(int s) { return s <= 32 ? 36 : 44; }
// lambda window of a leaf step: the band of rows U reads lambda[(i+j)/2] at offsets r + c + sigma from
// 2sU, at most (s + 6) + (2s + 2) + 1 for the rows and columns the band kernels touch (band_rows: the
// highest started row tile has 8 rb < s, columns c < 4 ceil(s/2)); 3s + 10 instead of 4s leaves room
// for four engine-3 CTAs per SM at s = 39
__host__ __device__ inline int tile_lw(int s) { return (3 * s + 11) & ~1; }  // even: 16-byte aligned regions follow
#ifndef LC_SKIP
#define LC_SKIP 0  // experiment builds only (tools): skip roles of the tile / range kernels (1 band, 2 step 5,
                   // 4 step-4 chain / step 1 + M2M, 8 M2L, 16 staging) to find the one that bounds a leaf step
#endif
#ifndef LC_FRING
#define LC_FRING 3  // leaf slots of the f / lambda ring (3: prefetch one leaf ahead; 4: two)
#endif
// T [2][32][M] | B(0) [M][M]+4 | tabA [80] | f ring [4][2][8][fst] | lambda ring [4][4s] |
// w ring [L][3][2][8][M] | c: levels < L-1 [2][2][8][M], level L-1 [3][2][8][M] | z [2][8][2s+4]
#ifndef LC_TILE_SL
#define LC_TILE_SL 0  // levels whose w / c stay in shared memory (0: all); the rest in a per-CTA scratch
#endif
#ifndef LC_TILE_MINB
#define LC_TILE_MINB 2
#endif
__host__ __device__ inline int tile_gs(int L) { return (LC_TILE_SL == 0 || L <= LC_TILE_SL) ? 0 : L - LC_TILE_SL; }
#ifndef LC_M2L_K36
#define LC_M2L_K36 1  // the two A_hat blocks of an even M2L row as one K = 36 contraction
#endif
__host__ __device__ inline int64_t tile_smem_doubles(int L, int s) {
  const int fst = tile_fst(s);
  const int ns = L - tile_gs(L);  // levels in shared memory
  return 2 * kM * tile_tstride(s) + (kMM + 4) + 80 + LC_FRING * 2 * kTileV * fst + LC_FRING * tile_lw(s) + int64_t(ns) * 3 * 2 * kTS +
         int64_t(2 * ns + 1) * 2 * kTS + 2 * kTileV * (2 * s + 4) + kMM;
}
__host__ __device__ inline int64_t tile_scratch_doubles(int L) { return int64_t(tile_gs(L)) * 5 * 2 * kTS; }

// STAGE = 1: the M2L operands of each job are staged per warp by cp.async (+30 KB; registers bounded
// for 3 CTAs per SM), used when 3 such CTAs fit an SM (s <= 24); otherwise the direct-load variant at
// 4 CTAs per SM (measured at cfg4, s = 20: 17.2 -> 16.7 ms; at n = 2e6, s = 31, staging would drop to
// 2 CTAs per SM and lose 10%)
__host__ __device__ inline int64_t range_smem_doubles(int s, int stage) {
  const int fst = tile_fst(s);
  return 2 * tile_trows(s) * kM + (kMM + 4) + 80 + LC_FRING * 2 * kTileV * fst + LC_FRING * tile_lw(s) + int64_t(5) * 2 * kTS +
         2 * kTileV * (2 * s + 4) + (stage ? 4 * (2 * kMM + 2 * kTS) : 0);
}
#ifndef LC_RANGE_MINB
// CTAs per SM the direct-load range kernel's registers are bounded for (cfg4: 4 -> 17.2 ms, 2 -> 19.8 ms)
#define LC_RANGE_MINB 4
#endif
__host__ __device__ inline int64_t range_scratch_doubles(int L) { return int64_t(L >= 2 ? L - 2 : 0) * 2 * 2 * kTS; }

struct TileParams {
  const double* in;
  double* out;
  const double* A;     // A_hat arena
  const double* tabA;  // 2s
  const double* tabB;  // N
  const double* Tpad;  // [2][tpr][M], rows >= s zero
  int tpr;             // rows per parity of Tpad (32, or 64 for s > 32)
  const double* B;     // B(0)
  const double* wg;    // engine 3: w of every level (up kernel output), tile stride w_tile
  double* scratch;     // engine 3: per-CTA c slots of the levels below L-2
  int64_t w_tile;
  int64_t ld_in, ld_out, n, N, batch, ntiles;
  int layout, L, s;
  int nranges, rlen;   // engine 3: leaf ranges per tile and their length
  int nle;             // engine 3: leaf segments holding outputs (the ranges stop there: past n is padding)
  int64_t oblk;        // > 0: column-blocked output (out[(i / oblk) batch oblk + v oblk + i % oblk])
};

// debug build: per (CTA, warp) cycle accounting of the tile kernel in g_lc_ts[0]:
// [0] band / step 1 / chain, [1] eval / cascade, [2] M2L jobs, [3] end of step, [4] steps
#ifdef LC_PHASE_TIMING
#define TP_DECL                                  \
  long long tp_t0 = clock64();                   \
  unsigned long long tp_acc[6] = {0, 0, 0, 0, 0, 0};
#define TP_MARK(slot)                            \
  do {                                           \
    const long long tp_t1 = clock64();           \
    tp_acc[slot] += (unsigned long long)(tp_t1 - tp_t0); \
    tp_t0 = tp_t1;                               \
  } while (0)
#define TP_COUNT(slot, v) (tp_acc[slot] += (v))
#define TP_FLUSH                                                                          \
  do {                                                                                    \
    if (lane == 0 && blockIdx.x < 4096)                                                   \
      for (int q = 0; q < 6; ++q) g_lc_ts[0][(blockIdx.x * 8 + warp) * 8 + q] += tp_acc[q]; \
  } while (0)
#else
#define TP_DECL
#define TP_MARK(slot) ((void)0)
#define TP_COUNT(slot, v) ((void)0)
#define TP_FLUSH ((void)0)
#endif

// Step 6 of one leaf for s != 32, row tiles R0, R1 (and R2 >= 0) of this warp: rows r = 8 rb + lr,
// columns c = 4 kc + lc in [8 rb, 2s) of the segment pair (U, U+1); K[r][c] = a[c-r] lambda[(i+j)/2]
// per lane, G[c][v] = f_v[j] (C2L: j f_j).  The k-steps are unrolled at compile time (immediate shared-
// memory offsets; the loop ends at nkc = ceil(s/2)); only the diagonal chunks mask c < r.  Rows r >= s of
// a partly used tile compute values that are never stored (the caller writes r < s; tiles with 8 rb >= s
// are skipped), and columns c >= 2s have b = 0 (their a stays inside the 4s lambda window: finite).
// fU / fU1 -> f[sigma][v = lr][0] of U / U+1, lamw -> lambda window + sigma + lr + lc, tap -> tabA + lc - lr.
// Per warp group at s = 40: {0, 1} 38 and {2, 3, 4} 42 k-steps; at s = 31: {0, 3} 26 and {1, 2} 26.
template <int DIR, int R0, int R1, int R2, bool ALIGNED>
__device__ __forceinline__ void band_rows(const double* __restrict__ fU, const double* __restrict__ fU1,
                                          const double* __restrict__ lamw, const double* __restrict__ tap,
                                          int64_t i0, int s, int sg, int lr, int lc, double (&acc)[3][2]) {
  constexpr int RMIN = R0 < R1 ? R0 : R1;
  const int nkc = (2 * s + 3) >> 2;
  const double jb = double(i0 + 2 * lc + sg);  // C2L column weight j = jb + 8 kc (exact integers)
  // (s > 32: every listed tile holds rows, no run-time check)
  const bool on1 = R2 >= 0 || R1 < 2 || 8 * R1 < s, on2 = R2 >= 0;
#pragma unroll
  for (int kc = 2 * RMIN; kc < kTileSMax / 2; ++kc) {
    if (kc >= nkc) break;
    const int c = 4 * kc + lc;
    double b;
    if (ALIGNED) {  // s = 0 (mod 4): the chunk boundary is the segment boundary, nkc = s/2 (no c >= 2s)
      b = (4 * kc < s ? fU : fU1 - s)[c];
    } else {
      const double* pb = c < s ? fU + c : fU1 + (c - s);
      b = c < 2 * s ? *pb : 0.0;
    }
    if (DIR == 1) b *= jb + double(8 * kc);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int rb = q == 0 ? R0 : (q == 1 ? R1 : R2);
      if (rb >= 0 && kc >= 2 * rb && (q == 0 || (q == 1 ? on1 : on2))) {
        const int d = 4 * kc - 8 * rb;
        double a = tap[d] * lamw[8 * rb + 4 * kc];
        if (d < 8 && lc + d < lr) a = 0.0;
        dmma(acc[q], a, b);
      }
    }
  }
}

// Step 6 of one leaf for s = 32, row tiles RLO < RHI, everything unrolled at compile time:
// K[r][c] = a[c-r] lambda[(i+j)/2] (per lane, one DMUL), G[c][v] = f_v[j] (C2L: j f_j).  Pointers are
// pre-offset by the lane: fU/fU1 -> f[sigma][v = lr][lc], lamw -> lambda window + sigma + lr + lc,
// tap -> a + lc - lr; the c >= r mask only exists in the two diagonal chunks of each row tile.
template <int DIR, int RLO, int RHI>
__device__ __forceinline__ void band32(const double* __restrict__ fU, const double* __restrict__ fU1,
                                       const double* __restrict__ lamw, const double* __restrict__ tap,
                                       int64_t i0, int sg, int lc, int lr, double (&acc)[3][2]) {
  const double jb = double(i0 + 2 * lc + sg);  // C2L column weight j = jb + 8 kc (exact integers)
#pragma unroll
  for (int kc = 2 * RLO; kc < 16; ++kc) {
    double b = kc < 8 ? fU[4 * kc] : fU1[4 * kc - 32];
    if (DIR == 1) b *= jb + double(8 * kc);
    {
      constexpr int dummy = 0;
      (void)dummy;
      double a = tap[4 * kc - 8 * RLO] * lamw[8 * RLO + 4 * kc];
      if (kc < 2 * RLO + 2 && lc + 4 * (kc - 2 * RLO) < lr) a = 0.0;
      dmma(acc[0], a, b);
    }
    if (kc >= 2 * RHI) {
      double a = tap[4 * kc - 8 * RHI] * lamw[8 * RHI + 4 * kc];
      if (kc < 2 * RHI + 2 && lc + 4 * (kc - 2 * RHI) < lr) a = 0.0;
      dmma(acc[1], a, b);
    }
  }
}

// Step 5 of leaf V1 for row tile mt (m = 8 mt + lr) of both parities: z[v][2m + sigma] += sum_k
// T(sigma)[m][k] c(L-1, V1)[sigma][v][k] (cc = c(L-1, V1), [sigma][v][k]), then C^{-1} (step 7) and the
// store: a lane holds rows i0 + 2m and i0 + 2m + 1 of vectors 2 lc and 2 lc + 1, written as one 16-byte
// store where the output layout allows it (v2ok)
template <int DIR, bool TT>
__device__ __forceinline__ void step5_store(const TileParams& P, const double* __restrict__ Tq, int tr,
                                            const double* __restrict__ cc, const double* __restrict__ zb, int zst,
                                            int64_t tile, int64_t i0, int mt, int s, int lr, int lc, bool v2ok,
                                            double* ob0 = nullptr, double* ob1 = nullptr) {
  const int m = 8 * mt + lr;
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int kk = 0; kk < 5; ++kk) {
    const int k = 4 * kk + lc;
#pragma unroll
    for (int sg = 0; sg < 2; ++sg) {
      const double bb = k < kM ? cc[sg * kTS + lr * kM + k] : 0.0;
      // T(sigma)[m][k]: [2][tr][M] (TT = false) or transposed [2][M][tr] (TT = true)
      const double a = k < kM ? (TT ? Tq[(sg * kM + k) * tr + m] : Tq[(sg * tr + m) * kM + k]) : 0.0;
      dmma(acc[sg], a, bb);
    }
  }
  if (m >= s) return;
  const double inv_pi = 0.318309886183790671537767526745028724;
  const int64_t i = i0 + 2 * m;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int v = 2 * lc + h;
    const int64_t gv = tile * kTileV + v;
    const double2 zz = *reinterpret_cast<const double2*>(zb + v * zst + 2 * m);
    double z0 = zz.x + acc[0][h], z1 = zz.y + acc[1][h];
    if (DIR == 0) {
      z0 *= (i == 0 ? inv_pi : 2.0 * inv_pi);
      z1 *= 2.0 * inv_pi;
    }
    if (gv >= P.batch) continue;
    if (ob0 && i + 1 < P.n) {  // hoisted row pointers of the lane's two vectors (vector layout, 16-byte stores)
      *reinterpret_cast<double2*>((h ? ob1 : ob0) + i) = make_double2(z0, z1);
    } else if (v2ok && i + 1 < P.n) {
      double* o = P.oblk ? P.out + (i / P.oblk) * P.batch * P.oblk + gv * P.oblk + i % P.oblk : P.out + gv * P.ld_out + i;
      *reinterpret_cast<double2*>(o) = make_double2(z0, z1);
    } else {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t ie = i + e;
        const double z = e ? z1 : z0;
        if (ie < P.n) {
          if (P.oblk) P.out[(ie / P.oblk) * P.batch * P.oblk + gv * P.oblk + ie % P.oblk] = z;
          else if (P.layout == LC_VEC_CONTIGUOUS) P.out[gv * P.ld_out + ie] = z;
          else P.out[ie * P.ld_out + gv] = z;
        }
      }
    }
  }
}
__device__ __forceinline__ bool step5_v2ok(const TileParams& P) {
  const bool lay = P.oblk ? (P.oblk & 1) == 0 : (P.layout == LC_VEC_CONTIGUOUS && (P.ld_out & 1) == 0);
  return lay && (reinterpret_cast<uintptr_t>(P.out) & 15) == 0;
}

template <int DIR>
__global__ void __launch_bounds__(kTileThreads, LC_TILE_MINB) lc_tile_kernel(const __grid_constant__ TileParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  const int s = P.s, L = P.L, seglen = 2 * s;
  const int fst = tile_fst(s), zst_ = 2 * s + 4;
  const int nls = 2 << L;  // leaf segments
  const int TS = tile_tstride(s);
  double* Tq = reinterpret_cast<double*>(smem);  // T(sigma) transposed: [2][M][TS]
  double* Bq = Tq + 2 * kM * TS;                  // B(0) [M][M]
  double* taq = Bq + kMM + 4;                     // tabA [80]
  double* fr = taq + 80;                          // [LC_FRING][2][8][fst]
  double* lmr = fr + LC_FRING * 2 * kTileV * fst; // [LC_FRING][4s]
  const int gs = tile_gs(L);                      // levels >= gs in shared memory, below in scratch
  const int ns = L - gs;
  double* wr = lmr + LC_FRING * tile_lw(s);       // [ns][3][2][8][M]
  double* cs = wr + ns * 3 * 2 * kTS;             // levels gs..L-2: [2][2][8][M], then leaf [3][2][8][M]
  double* zs = cs + (2 * ns + 1) * 2 * kTS;       // [2][8][2s+4]
  double* Bqs = zs + 2 * kTileV * zst_;           // sign-folded B(0): (-1)^(n-k) b_nk (child 1 / parity 1)
  double* gw = P.scratch + int64_t(blockIdx.x) * tile_scratch_doubles(L);  // [gs][3][2][8][M]
  double* gc = gw + gs * 3 * 2 * kTS;                                       // [gs][2][2][8][M]
  auto fslot = [&](int U) { return fr + ((U + LC_FRING) % LC_FRING) * 2 * kTileV * fst; };  // U >= -1
  auto lslot = [&](int U) { return lmr + ((U + LC_FRING) % LC_FRING) * tile_lw(s); };
  auto wslot = [&](int g, int t) {
    return g >= gs ? wr + ((g - gs) * 3 + t % 3) * 2 * kTS : gw + (g * 3 + t % 3) * 2 * kTS;
  };
  auto cslot = [&](int g, int u) {
    return g == L - 1 ? cs + (2 * (ns - 1) + u % 3) * 2 * kTS
                      : (g >= gs ? cs + ((g - gs) * 2 + (u & 1)) * 2 * kTS : gc + (g * 2 + (u & 1)) * 2 * kTS);
  };
  auto zbuf = [&](int U) { return zs + (U & 1) * kTileV * zst_; };

  for (int i = tid; i < 2 * kM * TS; i += kTileThreads) {  // [2][M][TS] from [2][tpr][M] (rows m >= s are zero)
    const int sg = i / (kM * TS), r = i - sg * kM * TS, k = r / TS, m = r - k * TS;
    Tq[i] = m < P.tpr ? __ldg(P.Tpad + (int64_t(sg) * P.tpr + m) * kM + k) : 0.0;
  }
  for (int i = tid; i < kMM / 2; i += kTileThreads) cp_async16(Bq + 2 * i, P.B + 2 * i);
  for (int i = tid; i < 80; i += kTileThreads) taq[i] = i < seglen ? P.tabA[i] : 0.0;
  // rows m in [s, fst) of every f slot stay zero (read by the K = 4 ceil(s/4) steps of step 1)
  for (int i = tid; i < LC_FRING * 2 * kTileV * fst; i += kTileThreads) fr[i] = 0.0;
  for (int i = tid; i < kMM; i += kTileThreads) {
    const double b = __ldg(P.B + i);
    Bqs[i] = ((i / kM - i % kM) & 1) ? -b : b;
  }
  cp_async_commit();
  __syncthreads();  // the zero fill precedes every cp.async into the ring (other threads' elements)
  griddep_wait();  // the input may be produced by the preceding kernel
  griddep_launch();

  // stage leaf segment U of the tile: f de-interleaved by parity ([sigma][v][m]), and the lambda
  // (tabB) window [2sU, 2sU + 3s + 10) that the band of rows U reads (tile_lw); zero beyond N
  auto stage = [&](int64_t tile, int U) {
    double* fd = fslot(U);
    const int64_t j0 = int64_t(U) * seglen;
    if (P.layout == LC_VEC_CONTIGUOUS) {  // warp = vector, lanes along the segment
      const int64_t gv = tile * kTileV + warp;
      const double* src = P.in + gv * P.ld_in + j0;
      const int64_t lim = gv < P.batch ? P.n - j0 : 0;
      for (int x = lane; x < seglen; x += 32) {
        const bool ok = x < lim;
        cp_async8(fd + ((x & 1) * kTileV + warp) * fst + (x >> 1), ok ? src + x : P.in, ok ? 8u : 0u);
      }
    } else {  // vectors fastest
      for (int idx = tid; idx < kTileV * seglen; idx += kTileThreads) {
        const int x = idx >> 3, v = idx & 7;
        const int64_t gv = tile * kTileV + v, j = j0 + x;
        const bool ok = gv < P.batch && j < P.n;
        cp_async8(fd + ((x & 1) * kTileV + v) * fst + (x >> 1), ok ? P.in + j * P.ld_in + gv : P.in, ok ? 8u : 0u);
      }
    }
    double* ld = lslot(U);
    for (int x = tid; x < tile_lw(s); x += kTileThreads) {
      const bool ok = j0 + x < P.N;
      cp_async8(ld + x, ok ? P.tabB + j0 + x : P.tabB, ok ? 8u : 0u);
    }
  };
  // first level entered at leaf U (U is the rightmost leaf of its segments on levels >= gmin)
  auto gmin_of = [&](int U) {
    const int ones = __ffs(~U) - 1;  // trailing one bits
    const int g = L - 1 - ones;
    return g < 0 ? 0 : g;
  };
  const bool v2ok = step5_v2ok(P);  // 16-byte output stores

  for (int64_t tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x) {
    // the lane's two output rows (vectors 2 lc, 2 lc + 1) for step 7's 16-byte stores
    const bool hoist = v2ok && !P.oblk && P.layout == LC_VEC_CONTIGUOUS;
    double* const ob0 = hoist ? P.out + (tile * kTileV + 2 * lc) * P.ld_out : nullptr;
    double* const ob1 = hoist ? P.out + (tile * kTileV + 2 * lc + 1) * P.ld_out : nullptr;
    for (int i = tid; i < (2 * ns + 1) * 2 * kTS; i += kTileThreads) cs[i] = 0.0;  // rows without M2L stay 0
    for (int i = tid; i < gs * 2 * 2 * kTS; i += kTileThreads) gc[i] = 0.0;
    {
      double* fz = fslot(nls);  // the segment past the end reads as zero
      for (int i = tid; i < 2 * kTileV * fst; i += kTileThreads) fz[i] = 0.0;
    }
    stage(tile, nls - 1);
    cp_async_commit();
    if (LC_FRING == 4) stage(tile, nls - 2);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();

    TP_DECL
    for (int U = nls - 1; U >= -1; --U) {
      // prefetch distance: two leaves with a ring of 4, one leaf (a whole step to land) with 3
      if (!(LC_SKIP & 16) && (LC_FRING == 4 ? U >= 2 : U >= 1)) stage(tile, LC_FRING == 4 ? U - 2 : U - 1);
      cp_async_commit();
      TP_MARK(5);
      const int V1 = U + 1;  // the leaf whose step 5 / step 2 run in this step
      if (warp < 4) {
        if (!(LC_SKIP & 1) && U >= 0 && 8 * ((warp >> 1) ? 1 : 0) < s) {
          // ---- step 6: rows i = 2sU + 2r + sigma, columns j = 2sU + 2c + sigma (c >= r, j < j_end),
          // K[r][c] = a[c-r] b[(i+j)/2] formed per lane, G[c][v] = f_v[j] (C2L: j f_j); two or three
          // row tiles per warp (one accumulator chain each)
          const int sg = warp & 1;
          const int grp = warp >> 1;
          const double* fU = fslot(U) + (sg * kTileV + lr) * fst;
          const double* fU1 = fslot(U + 1) + (sg * kTileV + lr) * fst;
          const double* lamw = lslot(U) + sg + lr + lc;  // lambda[(i+j)/2 - 2sU] = lamw[8 rb + 4 kc]
          const double* tap = taq + lc - lr;              // a[c - r] = tap[4 kc - 8 rb]
          const int64_t i0 = int64_t(U) * seglen;
          // row tiles per warp group: s <= 32 {0, 3} / {1, 2}; s in (32, 40] {0, 1} / {2, 3, 4}
          const int rq0 = s > 32 ? (grp ? 2 : 0) : (grp ? 1 : 0);
          const int rq1 = s > 32 ? (grp ? 3 : 1) : (grp ? 2 : 3);
          const int rq2 = (s > 32 && grp) ? 4 : 99;
          double acc[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
          if (s == 32) {
            if (grp == 0)
              band32<DIR, 0, 3>(fU + lc, fU1 + lc, lamw, tap, i0, sg, lc, lr, acc);
            else
              band32<DIR, 1, 2>(fU + lc, fU1 + lc, lamw, tap, i0, sg, lc, lr, acc);
          } else if (s > 32) {
            if (grp == 0)
              band_rows<DIR, 0, 1, -1, false>(fU, fU1, lamw, tap, i0, s, sg, lr, lc, acc);
            else
              band_rows<DIR, 2, 3, 4, false>(fU, fU1, lamw, tap, i0, s, sg, lr, lc, acc);
          } else if ((s & 3) == 0) {
            if (grp == 0)
              band_rows<DIR, 0, 3, -1, true>(fU, fU1, lamw, tap, i0, s, sg, lr, lc, acc);
            else
              band_rows<DIR, 1, 2, -1, true>(fU, fU1, lamw, tap, i0, s, sg, lr, lc, acc);
          } else {
            if (grp == 0)
              band_rows<DIR, 0, 3, -1, false>(fU, fU1, lamw, tap, i0, s, sg, lr, lc, acc);
            else
              band_rows<DIR, 1, 2, -1, false>(fU, fU1, lamw, tap, i0, s, sg, lr, lc, acc);
          }
          double* zb = zbuf(U);
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const int r = 8 * (q == 0 ? rq0 : (q == 1 ? rq1 : rq2)) + lr;
            if (r < s) {
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int v = 2 * lc + h;
                double z = acc[q][h];
                if (DIR == 1) {
                  const int64_t ir = i0 + 2 * r + sg;
                  z *= double(2 * ir + 1);
                  if (ir == 0) z += fslot(U)[v * fst];  // entry (0,0) of A^{-1}C is 1 (R2)
                }
                zb[v * zst_ + 2 * r + sg] = z;
              }
            }
          }
        }
        TP_MARK(0);
        // ---- step 5 + 7 of leaf V1, row tile = warp (and 4 on warp 0 for s > 32), both parities
        if (!(LC_SKIP & 2) && V1 < nls)
          for (int mt = warp; 8 * mt < s; mt += 4)
            step5_store<DIR, true>(P, Tq, TS, cslot(L - 1, V1), zbuf(V1), zst_, tile, int64_t(V1) * seglen, mt, s, lr, lc, v2ok,
                                   ob0, ob1);
      } else {
        const int sg = warp & 1;
        if (warp < 6) {
          if (U >= 0) {
            // ---- step 1: w(L-1, U)[sigma][v][mode] = sum_m T(sigma)[m][mode] f_v[2sU + 2m + sigma]
            const double* fv = fslot(U) + (sg * kTileV + lr) * fst;
            const double* Tm = Tq + sg * kM * TS;  // T(sigma)^T: [mode][TS]
            double acc[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
            if (s == 32) {  // compile-time K: immediate offsets, no loop control
              const double* fq = fv + lc;
              const double* tq = Tm + lr * TS + lc;
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) {
                const double bb = fq[4 * kk];
#pragma unroll
                for (int mt = 0; mt < 3; ++mt)
                  dmma(acc[mt], (mt < 2 || lr < 2) ? tq[8 * mt * TS + 4 * kk] : 0.0, bb);
              }
            } else {
              const int nks = (s + 3) >> 2;
              for (int kk = 0; kk < nks; ++kk) {
                const int m = 4 * kk + lc;
                const double bb = fv[m];
#pragma unroll
                for (int mt = 0; mt < 3; ++mt) {
                  const int mode = 8 * mt + lr;
                  dmma(acc[mt], mode < kM ? Tm[mode * TS + m] : 0.0, bb);
                }
              }
            }
            double* dst = wslot(L - 1, U) + sg * kTS;
#pragma unroll
            for (int mt = 0; mt < 3; ++mt) {
              const int mode = 8 * mt + lr;
              if (mode < kM) {
                dst[(2 * lc) * kM + mode] = acc[mt][0];
                dst[(2 * lc + 1) * kM + mode] = acc[mt][1];
              }
            }
          }
          TP_MARK(0);
          // ---- step 2 cascade from leaf V1 (complete since the last step) while it is a left child
          // (w(g, 0) feeds no M2L: the cascade of leaf 0 is skipped)
          if (V1 >= 2 && V1 < nls && (V1 & 1) == 0) {
            int g = L - 1, u = V1;
            while (g > 0 && (u & 1) == 0) {
              const double* x0 = wslot(g, u) + sg * kTS;
              const double* x1 = wslot(g, u + 1) + sg * kTS;
              double* o = wslot(g - 1, u >> 1) + sg * kTS;
              double acc[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
              for (int kk = 0; kk < 9; ++kk) {
                const int kap = 4 * kk + lc;
                const int child = kap >= kM ? 1 : 0;
                const int kx = kap - child * kM;
                const double bb = (child ? x1 : x0)[lr * kM + kx];
#pragma unroll
                for (int mt = 0; mt < 3; ++mt) {
                  if (mt == 0 && (kk == 2 || kk == 3 || kk == 7 || kk == 8)) continue;  // k >= 8 > n
                  const int nn = 8 * mt + lr;
                  const double a = nn < kM ? (child ? Bqs : Bq)[nn * kM + kx] : 0.0;
                  dmma(acc[mt], a, bb);
                }
              }
#pragma unroll
              for (int mt = 0; mt < 3; ++mt) {
                const int nn = 8 * mt + lr;
                if (nn < kM) {
                  o[(2 * lc) * kM + nn] = acc[mt][0];
                  o[(2 * lc + 1) * kM + nn] = acc[mt][1];
                }
              }
              __syncwarp();
              --g;
              u >>= 1;
            }
          }
        } else if (!(LC_SKIP & 4) && U >= 0) {
          // ---- step 4 chain (sigma) over the levels entered at U, coarse to fine
          const int gA = gmin_of(U);
          for (int g = (gA > 0 ? gA : 1); g < L; ++g) {
            const int u = U >> (L - 1 - g);
            const int p = u & 1;
            const double* par = cslot(g - 1, u >> 1) + sg * kTS;
            double* dst = cslot(g, u) + sg * kTS;
            double acc[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
            for (int kk = 0; kk < 5; ++kk) {
              const int nn = 4 * kk + lc;
              const double bb = nn < kM ? par[lr * kM + nn] : 0.0;
#pragma unroll
              for (int mt = 0; mt < 3; ++mt) {
                if (4 * kk + 3 < 8 * mt) continue;  // n < k everywhere
                const int k = 8 * mt + lr;
                const double a = (k < kM && nn < kM) ? (p ? Bqs : Bq)[nn * kM + k] : 0.0;  // b_{n k}, sign-folded
                dmma(acc[mt], a, bb);
              }
            }
#pragma unroll
            for (int mt = 0; mt < 3; ++mt) {
              const int k = 8 * mt + lr;
              if (k < kM) {
                dst[(2 * lc) * kM + k] += acc[mt][0];
                dst[(2 * lc + 1) * kM + k] += acc[mt][1];
              }
            }
            __syncwarp();
          }
        }
        TP_MARK(1);
      }
      // (all eight warps: the jobs past the first four go to the band warps, not back to the chain warps)
      const int m2l_pos = warp >= 6 ? warp - 6 : (warp >= 4 ? warp - 2 : warp + 4);
      // ---- step 3 for the rows the next leaf enters: job k = (level gN + k/2, sigma k&1) on warp
      // 6, 7, 4, 5, 0, 1, 2, 3, 6, ...: c(u') = sum_r A_hat_r w(t_r)
      if (!(LC_SKIP & 8) && U >= 1) {
        const int gN = gmin_of(U - 1);
        const int nm2l = (L - gN) * 2;
        for (int k = m2l_pos; k < nm2l; k += 8) {
          const int g = gN + (k >> 1), sgk = k & 1;
          const int u = (U - 1) >> (L - 1 - g);
          double acc[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
          if (u < (4 << g) - 2) {
            const int b = u >> 1, p = u & 1;
            if (LC_M2L_K36 && p == 0) {
              // even row: both blocks as one K = 36 contraction [A_hat_0 | A_hat_1] [w(u+2); w(u+3)]
              // (9 K steps instead of 2 x 5 with the padding to 20)
              const double* A0 = P.A + (ahat_level_offset(g) + 3 * int64_t(b)) * kMM;
              const double* W0 = wslot(g, u + 2) + sgk * kTS;
              const double* W1 = wslot(g, u + 3) + sgk * kTS;
#pragma unroll
              for (int kk = 0; kk < 9; ++kk) {
                const int kx = 4 * kk + lc;
                const int blk = kx >= kM ? 1 : 0, kc = kx - blk * kM;
                const double bb = (blk ? W1 : W0)[lr * kM + kc];
#pragma unroll
                for (int mt = 0; mt < 3; ++mt) {
                  const int mode = 8 * mt + lr;
                  dmma(acc[mt], mode < kM ? __ldg(A0 + blk * kMM + mode * kM + kc) : 0.0, bb);
                }
              }
            } else
            for (int mi = 0; mi < (p ? 1 : 2); ++mi) {
              const int r = p ? 2 : mi;
              const int t = u + 2 + (p ? 0 : mi);
              const double* Am = P.A + (ahat_level_offset(g) + 3 * int64_t(b) + r) * kMM;
              const double* W = wslot(g, t) + sgk * kTS;
              double av[3][5];
#pragma unroll
              for (int mt = 0; mt < 3; ++mt)
#pragma unroll
                for (int kk = 0; kk < 5; ++kk) {
                  const int kx = 4 * kk + lc, mode = 8 * mt + lr;
                  av[mt][kk] = (mode < kM && kx < kM) ? __ldg(Am + mode * kM + kx) : 0.0;
                }
#pragma unroll
              for (int kk = 0; kk < 5; ++kk) {
                const int kx = 4 * kk + lc;
                const double bb = kx < kM ? W[lr * kM + kx] : 0.0;
#pragma unroll
                for (int mt = 0; mt < 3; ++mt) dmma(acc[mt], av[mt][kk], bb);
              }
            }
          }
          double* dst = cslot(g, u) + sgk * kTS;
#pragma unroll
          for (int mt = 0; mt < 3; ++mt) {
            const int mode = 8 * mt + lr;
            if (mode < kM) {
              dst[(2 * lc) * kM + mode] = acc[mt][0];
              dst[(2 * lc + 1) * kM + mode] = acc[mt][1];
            }
          }
        }
      }
      TP_MARK(2);
      if (LC_FRING == 4) cp_async_wait<1>(); else cp_async_wait<0>();  // f(U-1) landed
      __syncthreads();
      TP_MARK(3);
      TP_COUNT(4, 1);
    }
    TP_FLUSH;
    cp_async_wait<0>();
    __syncthreads();
  }
}

// Engine 3 (batches of long vectors, few tiles): lc_up3_kernel writes w of every level, then this
// kernel runs the per-tile right-to-left pass over a RANGE of leaves of a tile (ranges x tiles fill
// the GPU): steps 3-7 exactly as in lc_tile_kernel, with w read from the workspace, the step-4 chain
// started at the range's rightmost leaf from the top level down, and the c of the levels below L-2 in
// a per-CTA global scratch (the footprint does not grow with L).
template <int DIR, int STAGE>
__global__ void __launch_bounds__(kTileThreads, STAGE ? 3 : LC_RANGE_MINB) lc_range_kernel(const __grid_constant__ TileParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  const int s = P.s, L = P.L, seglen = 2 * s;
  const int fst = tile_fst(s), zst_ = 2 * s + 4;
  const int TR = tile_trows(s);
  double* Tq = reinterpret_cast<double*>(smem);  // [2][TR][M]
  double* Bq = Tq + 2 * TR * kM;                  // B(0) [M][M]
  double* taq = Bq + kMM + 4;                     // tabA [80]
  double* fr = taq + 80;                          // [LC_FRING][2][8][fst]
  double* lmr = fr + LC_FRING * 2 * kTileV * fst; // [LC_FRING][4s]
  double* cs = lmr + LC_FRING * tile_lw(s);       // leaf level [3], level L-2 [2] x [2][8][M]
  double* zs = cs + 5 * 2 * kTS;                  // [2][8][2s+4]
  double* mbuf = zs + 2 * kTileV * (2 * s + 4);    // STAGE: [4 M2L warps][2 A_hat + 2 w]
  double* gc = P.scratch + int64_t(blockIdx.x) * range_scratch_doubles(L);  // levels < L-2: [L-2][2][2][8][M]
  auto fslot = [&](int U) { return fr + ((U + LC_FRING) % LC_FRING) * 2 * kTileV * fst; };  // U >= -1
  auto lslot = [&](int U) { return lmr + ((U + LC_FRING) % LC_FRING) * tile_lw(s); };
  // w of every level comes from the up kernel (global workspace, read-only here)
  auto wglob = [&](int64_t tile, int g, int t, int sg) {
    return P.wg + tile * P.w_tile + (w_level_offset_units(g) + sg * nseg(g) + t) * kTS;
  };
  auto cslot = [&](int g, int u) {
    return g == L - 1 ? cs + (u % 3) * 2 * kTS
                      : (g == L - 2 ? cs + (3 + (u & 1)) * 2 * kTS : gc + (g * 2 + (u & 1)) * 2 * kTS);
  };
  auto zbuf = [&](int U) { return zs + (U & 1) * kTileV * zst_; };

  for (int i = tid; i < TR * kM; i += kTileThreads) {  // [2][TR][M] from [2][tpr][M]: TR * M / 2 pairs per parity
    const int sg = i >= TR * kM / 2 ? 1 : 0, j = i - sg * (TR * kM / 2);
    cp_async16(Tq + sg * TR * kM + 2 * j, P.Tpad + int64_t(sg) * P.tpr * kM + 2 * j);
  }
  for (int i = tid; i < kMM / 2; i += kTileThreads) cp_async16(Bq + 2 * i, P.B + 2 * i);
  for (int i = tid; i < 80; i += kTileThreads) taq[i] = i < seglen ? P.tabA[i] : 0.0;
  // rows m in [s, fst) of every f slot stay zero (read by the K = 4 ceil(s/4) steps of step 1)
  for (int i = tid; i < LC_FRING * 2 * kTileV * fst; i += kTileThreads) fr[i] = 0.0;
  cp_async_commit();
  __syncthreads();  // the zero fill precedes every cp.async into the ring (other threads' elements)
  griddep_wait();  // the input may be produced by the preceding kernel
  griddep_launch();

  // stage leaf segment U of the tile: f de-interleaved by parity ([sigma][v][m]), and the lambda
  // (tabB) window [2sU, 2sU + 3s + 10) that the band of rows U reads (tile_lw); zero beyond N
  auto stage = [&](int64_t tile, int U) {
    if (STAGE && warp >= 4) return;  // the M2L warps' cp.async groups stay their own
    double* fd = fslot(U);
    const int64_t j0 = int64_t(U) * seglen;
    constexpr int nstw = STAGE ? 4 : 8;  // staging warps
    if (P.layout == LC_VEC_CONTIGUOUS) {  // warp = vector, lanes along the segment
      for (int vv = warp; vv < kTileV; vv += nstw) {
        const int64_t gv = tile * kTileV + vv;
        const double* src = P.in + gv * P.ld_in + j0;
        const int64_t lim = gv < P.batch ? P.n - j0 : 0;
        for (int x = lane; x < seglen; x += 32) {
          const bool ok = x < lim;
          cp_async8(fd + ((x & 1) * kTileV + vv) * fst + (x >> 1), ok ? src + x : P.in, ok ? 8u : 0u);
        }
      }
    } else {  // vectors fastest
      for (int idx = tid; idx < kTileV * seglen; idx += 32 * nstw) {
        const int x = idx >> 3, v = idx & 7;
        const int64_t gv = tile * kTileV + v, j = j0 + x;
        const bool ok = gv < P.batch && j < P.n;
        cp_async8(fd + ((x & 1) * kTileV + v) * fst + (x >> 1), ok ? P.in + j * P.ld_in + gv : P.in, ok ? 8u : 0u);
      }
    }
    double* ld = lslot(U);
    for (int x = tid; x < tile_lw(s); x += 32 * nstw) {
      const bool ok = j0 + x < P.N;
      cp_async8(ld + x, ok ? P.tabB + j0 + x : P.tabB, ok ? 8u : 0u);
    }
  };
  // first level entered at leaf U (U is the rightmost leaf of its segments on levels >= gmin)
  auto gmin_of = [&](int U) {
    const int ones = __ffs(~U) - 1;  // trailing one bits
    const int g = L - 1 - ones;
    return g < 0 ? 0 : g;
  };
  const bool v2ok = step5_v2ok(P);  // 16-byte output stores

  const int64_t nunits = P.ntiles * P.nranges;
  for (int64_t unit = blockIdx.x; unit < nunits; unit += gridDim.x) {
    const int64_t tile = unit / P.nranges;
    const int Ua = int(unit - tile * P.nranges) * P.rlen;
    const int Ub = min(P.nle, Ua + P.rlen) - 1;
    const bool hoist = v2ok && !P.oblk && P.layout == LC_VEC_CONTIGUOUS;  // step 7's row pointers per lane
    double* const ob0 = hoist ? P.out + (tile * kTileV + 2 * lc) * P.ld_out : nullptr;
    double* const ob1 = hoist ? P.out + (tile * kTileV + 2 * lc + 1) * P.ld_out : nullptr;
    // entering the range at its rightmost leaf Ub enters every level; the "step" Ub+1 only computes
    // the M2L of Ub's rows on all levels (and stages f(Ub+1), zero past the end)
    auto gentry = [&](int U) { return U == Ub ? 0 : gmin_of(U); };
    stage(tile, Ub + 1);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();

    TP_DECL
    for (int U = Ub + 1; U >= Ua - 1; --U) {
      if (!(LC_SKIP & 16) && U - 1 >= Ua) stage(tile, U - 1);  // one leaf ahead (a whole step to land)
      cp_async_commit();
      TP_MARK(5);
      const int V1 = U + 1;  // the leaf whose step 5 runs in this step
      const bool inU = U >= Ua && U <= Ub;
      if (warp < 4) {
        if (!(LC_SKIP & 1) && inU && 8 * ((warp >> 1) ? 1 : 0) < s) {
          // ---- step 6: rows i = 2sU + 2r + sigma, columns j = 2sU + 2c + sigma (c >= r, j < j_end),
          // K[r][c] = a[c-r] b[(i+j)/2] formed per lane, G[c][v] = f_v[j] (C2L: j f_j); two or three
          // row tiles per warp (one accumulator chain each)
          const int sg = warp & 1;
          const int grp = warp >> 1;
          const double* fU = fslot(U) + (sg * kTileV + lr) * fst;
          const double* fU1 = fslot(U + 1) + (sg * kTileV + lr) * fst;
          const double* lamw = lslot(U) + sg + lr + lc;  // lambda[(i+j)/2 - 2sU] = lamw[8 rb + 4 kc]
          const double* tap = taq + lc - lr;              // a[c - r] = tap[4 kc - 8 rb]
          const int64_t i0 = int64_t(U) * seglen;
          // row tiles per warp group: s <= 32 {0, 3} / {1, 2}; s in (32, 40] {0, 1} / {2, 3, 4}
          const int rq0 = s > 32 ? (grp ? 2 : 0) : (grp ? 1 : 0);
          const int rq1 = s > 32 ? (grp ? 3 : 1) : (grp ? 2 : 3);
          const int rq2 = (s > 32 && grp) ? 4 : 99;
          double acc[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
          if (s == 32) {
            if (grp == 0)
              band32<DIR, 0, 3>(fU + lc, fU1 + lc, lamw, tap, i0, sg, lc, lr, acc);
            else
              band32<DIR, 1, 2>(fU + lc, fU1 + lc, lamw, tap, i0, sg, lc, lr, acc);
          } else if (s > 32) {
            if (grp == 0)
              band_rows<DIR, 0, 1, -1, false>(fU, fU1, lamw, tap, i0, s, sg, lr, lc, acc);
            else
              band_rows<DIR, 2, 3, 4, false>(fU, fU1, lamw, tap, i0, s, sg, lr, lc, acc);
          } else if ((s & 3) == 0) {
            if (grp == 0)
              band_rows<DIR, 0, 3, -1, true>(fU, fU1, lamw, tap, i0, s, sg, lr, lc, acc);
            else
              band_rows<DIR, 1, 2, -1, true>(fU, fU1, lamw, tap, i0, s, sg, lr, lc, acc);
          } else {
            if (grp == 0)
              band_rows<DIR, 0, 3, -1, false>(fU, fU1, lamw, tap, i0, s, sg, lr, lc, acc);
            else
              band_rows<DIR, 1, 2, -1, false>(fU, fU1, lamw, tap, i0, s, sg, lr, lc, acc);
          }
          double* zb = zbuf(U);
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const int r = 8 * (q == 0 ? rq0 : (q == 1 ? rq1 : rq2)) + lr;
            if (r < s) {
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int v = 2 * lc + h;
                double z = acc[q][h];
                if (DIR == 1) {
                  const int64_t ir = i0 + 2 * r + sg;
                  z *= double(2 * ir + 1);
                  if (ir == 0) z += fslot(U)[v * fst];  // entry (0,0) of A^{-1}C is 1 (R2)
                }
                zb[v * zst_ + 2 * r + sg] = z;
              }
            }
          }
        }
        TP_MARK(0);
        // ---- step 5 + 7 of leaf V1, row tile = warp, both parities (s > 32: on warps 4 and 5, below)
        if (!(LC_SKIP & 2) && s <= 32 && V1 >= Ua && V1 <= Ub && 8 * warp < s)
          step5_store<DIR, false>(P, Tq, TR, cslot(L - 1, V1), zbuf(V1), zst_, tile, int64_t(V1) * seglen, warp, s, lr, lc, v2ok,
                                  ob0, ob1);
      } else {
        const int sg = warp & 1;
        // s in (32, 40]: the band warps carry five row tiles, so step 5 + 7 of leaf V1 (its c and z
        // slots are not written in this step) runs on warps 4 and 5: row tiles {0, 2, 4} and {1, 3}
        if (!(LC_SKIP & 2) && s > 32 && warp < 6 && V1 >= Ua && V1 <= Ub)
          for (int mt = warp - 4; 8 * mt < s; mt += 2)
            step5_store<DIR, false>(P, Tq, TR, cslot(L - 1, V1), zbuf(V1), zst_, tile, int64_t(V1) * seglen, mt, s, lr, lc, v2ok,
                                    ob0, ob1);
        if (!(LC_SKIP & 4) && warp >= 6 && inU) {
          // ---- step 4 chain (sigma) over the levels entered at U, coarse to fine
          const int gA = gentry(U);
          for (int g = (gA > 0 ? gA : 1); g < L; ++g) {
            const int u = U >> (L - 1 - g);
            const int p = u & 1;
            const double* par = cslot(g - 1, u >> 1) + sg * kTS;
            double* dst = cslot(g, u) + sg * kTS;
            double acc[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
            for (int kk = 0; kk < 5; ++kk) {
              const int nn = 4 * kk + lc;
              const double bb = nn < kM ? par[lr * kM + nn] : 0.0;
#pragma unroll
              for (int mt = 0; mt < 3; ++mt) {
                if (4 * kk + 3 < 8 * mt) continue;  // n < k everywhere
                const int k = 8 * mt + lr;
                double a = (k < kM && nn < kM) ? Bq[nn * kM + k] : 0.0;  // b_{n k}
                if (p && ((k + nn) & 1)) a = -a;
                dmma(acc[mt], a, bb);
              }
            }
#pragma unroll
            for (int mt = 0; mt < 3; ++mt) {
              const int k = 8 * mt + lr;
              if (k < kM) {
                dst[(2 * lc) * kM + k] += acc[mt][0];
                dst[(2 * lc + 1) * kM + k] += acc[mt][1];
              }
            }
            __syncwarp();
          }
        }
        TP_MARK(1);
      }
      // ---- step 3 for the rows the next leaf enters: job k = (level gN + k/2, sigma k&1) on warp
      // 4, 5, 6, 7, 4, ...: c(u') = sum_r A_hat_r w(t_r), w from the up kernel's output (handing the
      // jobs past the first four to the band warps, as lc_tile_kernel does, measured 0.6% slower here)
      // s > 32 (all eight warps; per-warp cycle accounting, tools/tile_roles.py): jobs to warps
      // 5, 4 (step 5), 0, 1 (band), 6, 7 (step-4 chain), 2, 3 (the longer band group), then around again
      if (!(LC_SKIP & 8) && (warp >= 4 || s > 32) && U - 1 >= Ua) {
        const int gN = gentry(U - 1);
        const int nm2l = (L - gN) * 2;
        const int kpos = s > 32 ? (warp == 5 ? 0 : warp == 4 ? 1 : warp < 2 ? warp + 2 : warp >= 6 ? warp - 2 : warp + 4)
                                : warp - 4;
        const int kstep = s > 32 ? 8 : 4;
        for (int k = kpos; k < nm2l; k += kstep) {
          const int g = gN + (k >> 1), sgk = k & 1;
          const int u = (U - 1) >> (L - 1 - g);
          double acc[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
          if (STAGE && u < (4 << g) - 2) {
            // the job's A_hat block(s) and w node(s) (contiguous) land in this warp's buffer in one round
            const int b = u >> 1, p = u & 1, nb = p ? 1 : 2;
            double* ab = mbuf + (warp - 4) * (2 * kMM + 2 * kTS);
            double* wb = ab + 2 * kMM;
            const double* As = P.A + (ahat_level_offset(g) + 3 * int64_t(b) + (p ? 2 : 0)) * kMM;
            const double* Wsrc = wglob(tile, g, u + 2, sgk);
            __syncwarp();
            for (int i = lane; i < nb * (kMM / 2); i += 32) cp_async16(ab + 2 * i, As + 2 * i);
            for (int i = lane; i < nb * (kTS / 2); i += 32) cp_async16(wb + 2 * i, Wsrc + 2 * i);
            cp_async_commit();
            cp_async_wait<0>();
            __syncwarp();
            auto kstep = [&](int kk, bool one) {
              const int kx = 4 * kk + lc;
              const int blk = kx >= kM ? 1 : 0, kc = kx - blk * kM;
              const bool okk = !one || kx < kM;
              const double bb = okk ? wb[blk * kTS + lr * kM + kc] : 0.0;
#pragma unroll
              for (int mt = 0; mt < 3; ++mt) {
                const int mode = 8 * mt + lr;
                dmma(acc[mt], (okk && mode < kM) ? ab[blk * kMM + mode * kM + kc] : 0.0, bb);
              }
            };
            if (p) {
#pragma unroll
              for (int kk = 0; kk < 5; ++kk) kstep(kk, true);
            } else {
#pragma unroll
              for (int kk = 0; kk < 9; ++kk) kstep(kk, false);
            }
          } else if (u < (4 << g) - 2) {
            const int b = u >> 1, p = u & 1;
            if (LC_M2L_K36 && p == 0) {
              // even row: both blocks as one K = 36 contraction [A_hat_0 | A_hat_1] [w(u+2); w(u+3)]
              // (9 K steps instead of 2 x 5 with the padding to 20)
              const double* A0 = P.A + (ahat_level_offset(g) + 3 * int64_t(b)) * kMM;
              const double* W0 = wglob(tile, g, u + 2, sgk);
              const double* W1 = wglob(tile, g, u + 3, sgk);
#pragma unroll
              for (int kk = 0; kk < 9; ++kk) {
                const int kx = 4 * kk + lc;
                const int blk = kx >= kM ? 1 : 0, kc = kx - blk * kM;
                const double bb = __ldg((blk ? W1 : W0) + lr * kM + kc);
#pragma unroll
                for (int mt = 0; mt < 3; ++mt) {
                  const int mode = 8 * mt + lr;
                  dmma(acc[mt], mode < kM ? __ldg(A0 + blk * kMM + mode * kM + kc) : 0.0, bb);
                }
              }
            } else
            for (int mi = 0; mi < (p ? 1 : 2); ++mi) {
              const int r = p ? 2 : mi;
              const int t = u + 2 + (p ? 0 : mi);
              const double* Am = P.A + (ahat_level_offset(g) + 3 * int64_t(b) + r) * kMM;
              const double* W = wglob(tile, g, t, sgk);
              double av[3][5];
#pragma unroll
              for (int mt = 0; mt < 3; ++mt)
#pragma unroll
                for (int kk = 0; kk < 5; ++kk) {
                  const int kx = 4 * kk + lc, mode = 8 * mt + lr;
                  av[mt][kk] = (mode < kM && kx < kM) ? __ldg(Am + mode * kM + kx) : 0.0;
                }
#pragma unroll
              for (int kk = 0; kk < 5; ++kk) {
                const int kx = 4 * kk + lc;
                const double bb = kx < kM ? __ldg(W + lr * kM + kx) : 0.0;
#pragma unroll
                for (int mt = 0; mt < 3; ++mt) dmma(acc[mt], av[mt][kk], bb);
              }
            }
          }
          double* dst = cslot(g, u) + sgk * kTS;
#pragma unroll
          for (int mt = 0; mt < 3; ++mt) {
            const int mode = 8 * mt + lr;
            if (mode < kM) {
              dst[(2 * lc) * kM + mode] = acc[mt][0];
              dst[(2 * lc + 1) * kM + mode] = acc[mt][1];
            }
          }
        }
      }
      TP_MARK(2);
      if (LC_FRING == 4) cp_async_wait<1>(); else cp_async_wait<0>();  // f(U-1) landed
      __syncthreads();
      TP_MARK(3);
      TP_COUNT(4, 1);
    }
    TP_FLUSH;
    cp_async_wait<0>();
    __syncthreads();
  }
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
template <int VT, int SMAX>
static cudaError_t set_attrs_vt(int smax) {
  cudaError_t e = set_max_dyn_smem(lc_up_kernel<VT, SMAX>, smax);
  if (e == cudaSuccess) e = set_max_dyn_smem(lc_stream_kernel<VT, 0>, smax);
  if (e == cudaSuccess) e = set_max_dyn_smem(lc_stream_kernel<VT, 1>, smax);
  if (e == cudaSuccess) e = set_max_dyn_smem(lc_down_kernel<VT, 0, SMAX, kDownThreads>, smax);
  if (e == cudaSuccess) e = set_max_dyn_smem(lc_down_kernel<VT, 1, SMAX, kDownThreads>, smax);
  if (e == cudaSuccess) e = set_max_dyn_smem(lc_down_kernel<VT, 0, SMAX, kDownThreads / 2>, smax);
  if (e == cudaSuccess) e = set_max_dyn_smem(lc_down_kernel<VT, 1, SMAX, kDownThreads / 2>, smax);
  return e;
}
template <int SMAX>
static cudaError_t set_attrs_all(int smax) {
  cudaError_t e = set_attrs_vt<1, SMAX>(smax);
  if (e == cudaSuccess) e = set_attrs_vt<2, SMAX>(smax);
  if (e == cudaSuccess) e = set_attrs_vt<4, SMAX>(smax);
  if (e == cudaSuccess) e = set_attrs_vt<8, SMAX>(smax);
  return e;
}

static std::atomic<bool> g_device_ready[64];
static std::mutex g_config_mu;  // cudaFuncSetAttribute of the kernels, once per device

template <int VT>
static int stream_occupancy(int dir, size_t smem) {
  int occ = 0;
  if (dir == 0)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lc_stream_kernel<VT, 0>, kStreamThreads, smem);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lc_stream_kernel<VT, 1>, kStreamThreads, smem);
  return occ;
}
static int stream_occupancy_vt(int vt, int dir, size_t smem) {
  switch (vt) {
    case 1: return stream_occupancy<1>(dir, smem);
    case 2: return stream_occupancy<2>(dir, smem);
    case 4: return stream_occupancy<4>(dir, smem);
    default: return stream_occupancy<8>(dir, smem);
  }
}

lc_status configure_kernels(lc_plan* p) {
  int smax = 0;
  cudaError_t ea = cudaDeviceGetAttribute(&smax, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->device);
  if (ea != cudaSuccess) return record_cuda_error(ea);
  if (p->device < 0 || p->device >= 64) return LC_ERR_INVALID_ARG;
  std::unique_lock<std::mutex> cfg_lock(g_config_mu);
  if (!g_device_ready[p->device].load()) {
    ea = set_attrs_all<32>(smax);
    if (ea == cudaSuccess) ea = set_attrs_all<64>(smax);
    if (ea == cudaSuccess) ea = set_max_dyn_smem(lc_tile_kernel<0>, smax);
    if (ea == cudaSuccess) ea = set_max_dyn_smem(lc_tile_kernel<1>, smax);
    if (ea == cudaSuccess) ea = set_max_dyn_smem(lc_up3_kernel<32>, smax);
    if (ea == cudaSuccess) ea = set_max_dyn_smem(lc_up3_kernel<40>, smax);
    if (ea == cudaSuccess) ea = set_max_dyn_smem(lc_range_kernel<0, 0>, smax);
    if (ea == cudaSuccess) ea = set_max_dyn_smem(lc_range_kernel<1, 0>, smax);
    if (ea == cudaSuccess) ea = set_max_dyn_smem(lc_range_kernel<0, 1>, smax);
    if (ea == cudaSuccess) ea = set_max_dyn_smem(lc_range_kernel<1, 1>, smax);
    if (ea != cudaSuccess) return record_cuda_error(ea);
    g_device_ready[p->device].store(true);
  }
  cfg_lock.unlock();
  smax -= 256;  // static shared memory of the kernels
  const int L = int(p->L);
  if (L > 0 && L - 1 > 62) return LC_ERR_INVALID_ARG;
  p->smax = p->s <= 32 ? 32 : 64;

  const int64_t budget2 = 113 * 1024;  // two CTAs per SM (228 KB minus 1 KB reserved per CTA)
  int vt = p->vt;
  // automatic engine 3 (tools/engine_cross_all.py on the B200, round 2, ranges of >= 8 leaves): batches of
  // 8+ vectors with at least ~1.6e6 coefficients in all (below, the level-pipelined kernels win: 65536 x 16
  // engine 1 55 vs 68 us, 150000 x 8 70 vs 91 us; above, engine 3: 16384 x 128 73 vs 102 us, 10^6 x 8 267
  // vs 374 us, 3e6 x 8 810 vs 1587 us, 64 x 10^7 14.4 vs 36 ms), fewer 8-vector tiles than SMs (else the
  // per-tile kernel)
  if (p->engine == 0 && p->part_count <= 1 && p->vt <= 0 && L >= 7 && p->s <= kTileSMax && p->batch >= 8 &&
      p->n * p->batch >= 1600000 && ((p->batch + kTileV - 1) / kTileV) < int64_t(p->sm_count))
    p->engine = 3;
  if (p->engine == 3) {  // up kernel of 8-vector tiles feeding the per-range pass
    if (L < 1 || p->s > kTileSMax) return LC_ERR_INVALID_ARG;
    vt = 8;
  }
  if (vt <= 0) vt = p->batch >= 2 ? 2 : 1;
  if (vt != 1 && vt != 2 && vt != 4 && vt != 8) return LC_ERR_INVALID_ARG;
  const int64_t nleaf_total = L > 0 ? (int64_t(2) << L) : 2;  // leaf segments (L = 0: the two halves)
  int lnleaf = 0;
  while ((int64_t(1) << (lnleaf + 1)) <= nleaf_total) ++lnleaf;  // log2(nleaf_total)
  const int s = int(p->s);
  // down kernel: subtrees of 2^kd leaf segments (kd <= L-1; L = 0: the whole vector), about
  // one wave of 8-warp CTAs at two per SM when the shared memory allows
  const bool user_k = p->k > 0;
  int kd = 1;
  if (L >= 1) {
    const int64_t ntiles_ = (p->batch + vt - 1) / vt;
    kd = 0;
    while (kd < L - 1 && (nleaf_total >> kd) * ntiles_ > 2 * int64_t(p->sm_count) &&
           down_smem_bytes(vt, kd + 1, s, L) <= budget2)
      ++kd;
    if (user_k) kd = std::min(p->k, L - 1);
    if (p->part_count > 1) kd = std::min(kd, part_align_log2(L));  // down subtrees inside one part
  }
  if (down_smem_bytes(vt, kd, s, L) > smax) return LC_ERR_INVALID_ARG;
  // streaming kernel: band units of 2^kb leaf segments
  int kb = std::min(4, lnleaf);
  int cb = p->bps > 0 ? p->bps : 3;
  int nst = p->nst > 0 ? p->nst : 3;
  if (nst > 8 || cb > 64) return LC_ERR_INVALID_ARG;
  auto stream_bytes = [&](int cb_, int kb_) { return stream_smem_layout(vt, cb_, nst, kb_, s).total; };
  while (stream_bytes(cb, kb) > budget2 && kb > 1) --kb;
  while (p->bps <= 0 && stream_bytes(cb, kb) > budget2 && cb > 1) --cb;
  if (stream_bytes(cb, kb) > smax) return LC_ERR_INVALID_ARG;
  // up kernel: about one wave of subtrees (2 CTAs per SM) if the shared memory allows
  const bool user_kup = p->kup > 0;
  int kup = 0;
  if (L > 0) {
    const int64_t ntiles_ = (p->batch + vt - 1) / vt;
    int kmax = L - 1;
    while (kmax > 0 && up_smem_bytes(vt, kmax, s) > budget2) --kmax;
    if (user_kup) {
      kup = std::min(p->kup, L - 1);
    } else {
      kup = 0;
      while (kup < kmax && (nleaf_total >> kup) * ntiles_ > 2 * int64_t(p->sm_count)) ++kup;
      if (L >= 2) kup = std::max(kup, 1);
    }
  }
  if (p->part_up) kup = std::max(1, std::min(kup, part_align_log2(L)));  // the parts' subtrees are whole
  if (up_smem_bytes(vt, kup, s) > smax) return LC_ERR_INVALID_ARG;
  {
    p->down_bulk = 1;  // TMA bulk loads in the down kernel (LC_DOWN_BULK=0: per-element cp.async, A/B runs)
    // M2M levels merged inside the up kernel's subtree (the rest by the continuation); fewer levels
    // free the SMs for the A_hat stream earlier (LC_UP_KSUB overrides, for A/B runs)
    // measured on cfg2 (tools/r2_job10.sh): 3 levels in the CTA, 3 by the continuation saves ~0.7 us per
    // transform over all 6 in the CTA (the up CTAs leave ~1.7 us earlier); 2 is slower again
    int ksub = (L >= 10 && kup >= 4 && !p->part_up) ? 3 : kup;
    if (const char* e = std::getenv("LC_UP_KSUB")) ksub = std::max(0, std::min(kup, std::atoi(e)));
    if (kup - ksub > std::max(kup, 1)) ksub = kup;  // a continuation group must cover the CTA's roots
    p->up_ksub = ksub;
    if (const char* e = std::getenv("LC_DOWN_BULK")) p->down_bulk = std::atoi(e) != 0;
  }
  p->vt = vt;
  p->k = kd;
  p->kb = kb;
  p->bps = cb;
  p->nst = nst;
  p->kup = kup;
  p->grup = L > 0 ? L - 1 - kup : 0;
  p->gr = L > 0 ? L - 1 - kd : 0;
  p->group = std::max(kup, 1);
  p->ntiles = (p->batch + vt - 1) / vt;
  p->smem_up = size_t(up_smem_bytes(vt, kup, s));
  p->smem_stream = size_t(stream_bytes(cb, kb));
  p->smem_down = size_t(down_smem_bytes(vt, kd, s, L));
  // M2L level order: the finest level first (its w is ready after the up kernel's main phase),
  // down to the subtree roots, then the coarse levels (after the up kernel's continuation)
  {
    int o = 0;
    {
      const int gtop = p->grup + (p->kup - p->up_ksub);
      for (int g = L - 1; g >= gtop; --g) p->lvorder[o++] = g;
      for (int g = 0; g < gtop; ++g) p->lvorder[o++] = g;
    }
    if (o != L) return LC_ERR_INTERNAL;
  }
  // M2L blocks per level: all of them, or (a partitioned plan, NEXT-2) the row blocks of the segments
  // that contain a leaf of the part, i.e. its own rows and their ancestors' (the down kernel's chain)
  // A whole plan likewise stops at the last group of 2^max(kd, kb) leaves holding outputs: the zero
  // padding past n has no rows to return, so its band units, down subtrees and M2L rows
  // are skipped (its w, all zeros, is still projected by the up kernel: columns of the last rows).
  int64_t lo_leaf = 0, hi_leaf = nleaf_total;
  if (p->part_count > 1) {
    lo_leaf = p->part_lo;
    hi_leaf = p->part_hi;
  } else if (L >= 1) {
    const int64_t a = int64_t(1) << std::max(kd, kb);
    hi_leaf = std::min(nleaf_total, ((p->n + 2 * s - 1) / (2 * s) + a - 1) / a * a);
  }
  int64_t nchunks = 0;
  for (int g = 0; g < L; ++g) {
    const int64_t bg = (int64_t(2) << g) - 1;
    int64_t blo = 0, nb = bg;
    {
      const int sh = L - 1 - g;
      if (hi_leaf > lo_leaf) {
        const int64_t ulo = lo_leaf >> sh, uhi = (hi_leaf - 1) >> sh;
        blo = std::min(bg, ulo >> 1);
        nb = std::max<int64_t>(0, std::min(bg, (uhi >> 1) + 1) - blo);
      } else {
        nb = 0;
      }
    }
    p->blo[g] = int(blo);
    p->nblk[g] = int(nb);
    nchunks += (nb + cb - 1) / cb;
  }
  p->m2l_units = nchunks * p->ntiles;
  if (p->part_count > 1) {
    p->band_lo = int(p->part_lo >> kb);
    p->band_units = ((p->part_hi - p->part_lo) >> kb) * p->ntiles;
    p->sub_lo = p->part_lo >> kd;
    p->nsub_down = (p->part_hi - p->part_lo) >> kd;
  } else {
    p->band_lo = 0;
    p->band_units = (hi_leaf >> kb) * p->ntiles;
    p->sub_lo = 0;
    p->nsub_down = L > 0 ? hi_leaf >> kd : 1;
  }
  if (p->m2l_units + p->band_units > 0x7fffffff) return LC_ERR_INVALID_ARG;
  {
    const int occ = stream_occupancy_vt(vt, p->dir, p->smem_stream);
    if (occ < 1) return LC_ERR_INVALID_ARG;
    p->stream_occ = occ;
    // persistent grid: every CTA co-resident (the producer waits on flags raised by the up kernel)
    const int64_t g = int64_t(occ) * p->sm_count;
    p->stream_grid = int(std::max<int64_t>(1, std::min<int64_t>(g, std::max(p->m2l_units, p->band_units))));
  }
  if (L > 0) {
    p->w_tile_doubles = int64_t(vt) * kM * 2 * ((int64_t(4) << L) - 4);
    p->cnt_tile_ints = int64_t(4) << L;
  } else {
    p->w_tile_doubles = 0;
    p->cnt_tile_ints = 0;
  }
  // workspace: w | c_m2l | flags (64 ints) | arrival counters (c_m2l rows without a submatrix stay zero)
  const size_t wb = size_t(align_up(p->ntiles * p->w_tile_doubles * 8, 256));
  p->ws_bytes = 2 * wb + 256 + size_t(p->ntiles * p->cnt_tile_ints) * sizeof(int) + 64 * sizeof(int);
  if (p->part_count > 1) {  // partitioned plans (NEXT-2) run the level-pipelined kernels
    if (p->engine != 0 && p->engine != 1) return LC_ERR_INVALID_ARG;
    p->engine = 1;
    return LC_OK;
  }
  // per-tile streaming kernel (engine 2): many 8-vector tiles of short vectors
  {
    const int64_t ntiles8 = (p->batch + kTileV - 1) / kTileV;
    const int64_t tsm = L >= 1 ? tile_smem_doubles(L, s) * 8 : 0;
    const bool tile_ok = L >= 1 && s <= kTileSMax && tsm <= smax;
    if (p->engine == 2 && !tile_ok) return LC_ERR_INVALID_ARG;
    if (p->engine == 3) {
      // the staged-M2L variant where three of its CTAs fit an SM, else the direct-load one
      int occ = 0;
      size_t rsm = size_t(range_smem_doubles(s, 1) * 8);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, p->dir == 0 ? lc_range_kernel<0, 1> : lc_range_kernel<1, 1>,
                                                    kTileThreads, rsm);
      p->range_stage = occ >= 3 ? 1 : 0;
      if (!p->range_stage) {
        rsm = size_t(range_smem_doubles(s, 0) * 8);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, p->dir == 0 ? lc_range_kernel<0, 0> : lc_range_kernel<1, 0>,
                                                      kTileThreads, rsm);
      }
      if (occ < 1) return LC_ERR_INVALID_ARG;
      const int64_t slots = int64_t(occ) * p->sm_count;
      // the ranges cover the leaf segments that hold outputs: the zero padding past n has
      // w = 0 (written by the up pass) and no rows to return, so no range walks it
      const int64_t nls = std::min<int64_t>(int64_t(2) << L, (p->n + 2 * s - 1) / (2 * s));
      p->range_nle = int(nls);
      int64_t nr = std::max<int64_t>(1, slots / p->ntiles);  // units <= slots: one wave, no straggler round
      // ranges of >= 8 leaves (LC_RANGE_MIN; entering a range costs the whole step-4 chain and the M2L of every
      // level): the kernel time follows the leaf steps of one CTA, so below one wave shorter ranges win
      int rmin = 8;
      if (const char* e = std::getenv("LC_RANGE_MIN")) rmin = std::max(1, std::atoi(e));
      nr = std::max<int64_t>(1, std::min<int64_t>(nr, nls / rmin));
      const int64_t rlen = (nls + nr - 1) / nr;
      nr = (nls + rlen - 1) / rlen;
      p->range_n = int(nr);
      p->range_len = int(rlen);
      p->smem_tile = rsm;
      p->tile_grid = int(std::min<int64_t>(p->ntiles * nr, slots));
      // persistent up pass: subtrees of 2^kup leaves (two CTAs per SM), chunks of 2^kc subtrees; the
      // largest subtree (<= 8 leaves) that fits two CTAs per SM, double-buffered f if that fits too
      // (s = 39: 8 leaves single-buffered, 4.18 -> ... ms at cfg4, instead of 4 leaves double-buffered)
      {
        int ku = std::max(0, std::min(p->kup, 3));
        int nbuf = 2;
        int kc = std::min(6, L - 1 - ku);
        int force_nbuf = 0;
        if (const char* e = std::getenv("LC_UP3_NBUF")) force_nbuf = std::atoi(e);
        for (;;) {
          kc = std::min(6, L - 1 - ku);
          if (force_nbuf != 1 && up3_smem_bytes(ku, s, kc, 2) <= budget2) { nbuf = 2; break; }
          if (force_nbuf != 2 && up3_smem_bytes(ku, s, kc, 1) <= budget2) { nbuf = 1; break; }
          if (ku == 0) { nbuf = 1; break; }
          --ku;
        }
        // chunks of 2^kc subtrees, but at least two chunks per SM where the tree allows (small batches
        // of shorter vectors: 16 x 3e5 had 16 chunks for 148 SMs at kc = 6)
        while (kc > 0 && p->ntiles * (int64_t(4) << (L - 1 - ku - kc)) < 2 * int64_t(p->sm_count)) --kc;
        if (up3_smem_bytes(ku, s, kc, nbuf) > smax) return LC_ERR_INVALID_ARG;
        p->kup = ku;
        p->grup = L - 1 - ku;
        p->group = std::max(ku, 1);
        p->up3_kc = kc;
        p->up3_nbuf = nbuf;
        p->smem_up = size_t(up3_smem_bytes(ku, s, kc, nbuf));
        int uocc = 0;
        if (s <= 32)
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&uocc, lc_up3_kernel<32>, kThreads, p->smem_up);
        else
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&uocc, lc_up3_kernel<40>, kThreads, p->smem_up);
        if (uocc < 1) return LC_ERR_INVALID_ARG;
        const int64_t nch = p->ntiles * ((int64_t(4) << p->grup) >> kc);
        const int64_t uslots = int64_t(uocc) * p->sm_count;
        const int64_t per = (nch + uslots - 1) / uslots;
        p->up3_grid = (nch + per - 1) / per;
      }
      p->ws_range_off = align_up(int64_t(p->ws_bytes), 256);
      p->ws_bytes = size_t(p->ws_range_off + int64_t(p->tile_grid) * range_scratch_doubles(L) * 8 + 256);
      return LC_OK;
    }
    // automatic choice (tools/engine_cross.py on the B200): the per-tile pass wins once there is
    // about one 8-vector tile per SM (e.g. n = 4096: 256 tiles 181 vs 355 us), and earlier for short
    // vectors (n = 1024: 64 tiles 32 vs 58 us); below that the level-pipelined kernels win
    if (p->engine == 0)
      p->engine = (tile_ok && (ntiles8 >= int64_t(p->sm_count) || (p->n <= 2048 && 3 * ntiles8 >= int64_t(p->sm_count))))
                      ? 2 : 1;
    // the column-blocked output (2-D exchange packed by destination) is written by engines 2 and 3
    if (p->out_block > 0 && p->engine == 1) {
      if (!tile_ok) return LC_ERR_INVALID_ARG;
      p->engine = 2;
    }
    if (p->engine == 2) {
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, p->dir == 0 ? lc_tile_kernel<0> : lc_tile_kernel<1>,
                                                    kTileThreads, size_t(tsm));
      if (occ < 1) return LC_ERR_INVALID_ARG;
      p->smem_tile = size_t(tsm);
      p->tile_grid = int(std::min<int64_t>(ntiles8, int64_t(occ) * p->sm_count));
      p->vt = kTileV;
      p->ntiles = ntiles8;
      p->ws_bytes = size_t(std::max<int64_t>(256, int64_t(p->tile_grid) * tile_scratch_doubles(L) * 8));
    }
  }
  return LC_OK;
}

template <int VT, int DIR, int SMAX>
static cudaError_t launch_vt(const lc_plan* p, const UpParams& up, const StreamParams& sp, const DownParams& dp,
                             dim3 grid_up, dim3 grid_down, cudaStream_t st, cudaEvent_t const* ev, int nev) {
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
  if (p->L > 0 && up.phase == 1) {
    // partitioned up pass, after the exchange of the roots: the continuation from groups of them
    // (stream order after the exchange, no programmatic overlap)
    UpArgs<SMAX> ua;
    ua.p = up;
    ua.p.contonly = 1;
    cudaLaunchConfig_t c1 = cfg;
    c1.numAttrs = 0;
    const int cg = std::min(std::max(p->kup, 1), int(p->grup));
    c1.gridDim = dim3(unsigned(nseg(p->grup) >> cg), unsigned(p->ntiles));
    c1.blockDim = dim3(kThreads);
    c1.dynamicSmemBytes = p->smem_up;
    e = cudaLaunchKernelEx(&c1, lc_up_kernel<VT, SMAX>, ua);
    if (e != cudaSuccess) return e;
    if (ev && evi < nev) cudaEventRecord(ev[evi++], st);
  } else if (p->L > 0) {
    UpArgs<SMAX> ua;
    ua.p = up;
    cfg.gridDim = grid_up;
    // many CTAs (small vector tiles or deep trees): 128-thread CTAs (four per SM) overlap their
    // latency-bound phases
    const bool small_up = int64_t(grid_up.x) * grid_up.y > 8 * p->sm_count && p->smem_up <= 56 * 1024;
    cfg.blockDim = dim3(small_up ? kThreads / 2 : kThreads);
    cfg.dynamicSmemBytes = p->smem_up;
    e = cudaLaunchKernelEx(&cfg, lc_up_kernel<VT, SMAX>, ua);
    if (e != cudaSuccess) return e;
    if (ev && evi < nev) cudaEventRecord(ev[evi++], st);
    if (up.phase == 0) return cudaGetLastError();  // partitioned up pass: the roots are exchanged next
  }
  cfg.gridDim = dim3(unsigned(p->stream_grid));
  cfg.blockDim = dim3(kStreamThreads);
  cfg.dynamicSmemBytes = p->smem_stream;
  e = cudaLaunchKernelEx(&cfg, lc_stream_kernel<VT, DIR>, sp);
  if (e != cudaSuccess) return e;
  if (ev && evi < nev) cudaEventRecord(ev[evi++], st);
  cfg.gridDim = grid_down;
  cfg.dynamicSmemBytes = p->smem_down;
  if (int64_t(grid_down.x) * grid_down.y > 8 * p->sm_count && p->smem_down <= 56 * 1024) {
    // many small CTAs: 4-warp CTAs, four per SM
    cfg.blockDim = dim3(kDownThreads / 2);
    e = cudaLaunchKernelEx(&cfg, lc_down_kernel<VT, DIR, SMAX, kDownThreads / 2>, dp);
  } else {
    cfg.blockDim = dim3(kDownThreads);
    e = cudaLaunchKernelEx(&cfg, lc_down_kernel<VT, DIR, SMAX, kDownThreads>, dp);
  }
  if (e != cudaSuccess) return e;
  if (ev && evi < nev) cudaEventRecord(ev[evi++], st);
  return cudaGetLastError();
}

template <int SMAX>
static cudaError_t launch_dispatch(const lc_plan* p, const UpParams& up, const StreamParams& sp, const DownParams& dp,
                                   dim3 gu, dim3 gd, cudaStream_t st, cudaEvent_t const* ev, int nev) {
  switch (p->vt * 2 + p->dir) {
    case 2: return launch_vt<1, 0, SMAX>(p, up, sp, dp, gu, gd, st, ev, nev);
    case 3: return launch_vt<1, 1, SMAX>(p, up, sp, dp, gu, gd, st, ev, nev);
    case 4: return launch_vt<2, 0, SMAX>(p, up, sp, dp, gu, gd, st, ev, nev);
    case 5: return launch_vt<2, 1, SMAX>(p, up, sp, dp, gu, gd, st, ev, nev);
    case 8: return launch_vt<4, 0, SMAX>(p, up, sp, dp, gu, gd, st, ev, nev);
    case 9: return launch_vt<4, 1, SMAX>(p, up, sp, dp, gu, gd, st, ev, nev);
    case 16: return launch_vt<8, 0, SMAX>(p, up, sp, dp, gu, gd, st, ev, nev);
    case 17: return launch_vt<8, 1, SMAX>(p, up, sp, dp, gu, gd, st, ev, nev);
  }
  return cudaErrorInvalidValue;
}

static lc_status launch_execute_impl(const lc_plan* p, const double* in, double* out, void* ws, cudaStream_t st,
                                     cudaEvent_t const* ev, int nev, int phase) {
  if (!p || !in || !out) return LC_ERR_INVALID_ARG;
  // a plan with a partitioned up pass runs in two phases around the exchange of its subtree roots
  if ((phase >= 0) != (p->part_up != 0)) return LC_ERR_INVALID_ARG;
  {
    const char* a0 = reinterpret_cast<const char*>(in);
    const char* a1 = a0 + 8 * in_extent(p);
    const char* b0 = reinterpret_cast<const char*>(out);
    const char* b1 = b0 + 8 * out_extent(p);
    if (a0 < b1 && b0 < a1) return LC_ERR_ALIASING;
  }
  if (!ws) ws = p->d_ws;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != p->device) cudaSetDevice(p->device);
  if (p->engine == 2) {
    TileParams tp{};
    tp.in = in; tp.out = out; tp.A = p->d_A; tp.tabA = p->d_tabA; tp.tabB = p->d_tabB; tp.Tpad = p->d_Tpad; tp.tpr = p->smax;
    tp.B = p->d_B; tp.ld_in = p->ld_in; tp.ld_out = p->ld_out; tp.n = p->n; tp.N = p->N; tp.batch = p->batch;
    tp.ntiles = p->ntiles; tp.layout = p->layout; tp.L = int(p->L); tp.s = int(p->s);
    tp.scratch = reinterpret_cast<double*>(ws);
    tp.oblk = p->out_block;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(unsigned(p->tile_grid));
    cfg.blockDim = dim3(kTileThreads);
    cfg.dynamicSmemBytes = p->smem_tile;
    if (ev && nev > 0) cudaEventRecord(ev[0], st);
    cudaError_t e = p->dir == 0 ? cudaLaunchKernelEx(&cfg, lc_tile_kernel<0>, tp) : cudaLaunchKernelEx(&cfg, lc_tile_kernel<1>, tp);
    if (e == cudaSuccess && ev && nev > 1) cudaEventRecord(ev[1], st);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (prev != p->device) cudaSetDevice(prev);
    return e == cudaSuccess ? LC_OK : record_cuda_error(e);
  }
  const size_t wb = size_t(align_up(p->ntiles * p->w_tile_doubles * 8, 256));
  double* w = reinterpret_cast<double*>(ws);
  double* c = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + wb);
  int* flags = reinterpret_cast<int*>(reinterpret_cast<char*>(ws) + 2 * wb);
  int* cnt = flags + 64;
  UpParams up{};
  up.in = in; up.Tpad = p->d_Tpad; up.B = p->d_B; up.ld_in = p->ld_in; up.n = p->n; up.N = p->N; up.batch = p->batch;
  up.layout = p->layout; up.L = int(p->L); up.s = int(p->s); up.k = p->kup; up.gr = p->grup; up.G = p->group;
  up.fstride = up_fstride(int(p->s));
  up.vec16 = (reinterpret_cast<uintptr_t>(in) % 16 == 0) && (p->ld_in % 2 == 0) ? 1 : 0;
  up.noflags = p->engine == 3 ? 1 : 0;
  up.ksub = p->engine == 1 ? p->up_ksub : p->kup;
  up.R0 = p->part_up ? (p->part_lo >> p->kup) : 0;
  up.nocont = p->part_up;
  up.phase = phase;
  up.contonly = 0;
  up.kc = p->up3_kc;
  up.nbuf = p->up3_nbuf;
  up.tpr = p->smax;
  up.ntiles = p->ntiles;
  up.w = w; up.cnt = cnt; up.flags = flags; up.w_tile = p->w_tile_doubles; up.cnt_tile = p->cnt_tile_ints;
  StreamParams sp{};
  sp.A = p->d_A; sp.w = w; sp.c = c; sp.in = in; sp.out = out; sp.tabA = p->d_tabA; sp.tabB = p->d_tabB;
  sp.flags = flags; sp.w_tile = p->w_tile_doubles;
  sp.ld_in = p->ld_in; sp.ld_out = p->ld_out; sp.n = p->n;
  sp.N = p->N; sp.batch = p->batch; sp.ntiles = p->ntiles; sp.nm2l = p->m2l_units; sp.nband = p->band_units;
  sp.layout = p->layout; sp.L = int(p->L); sp.s = int(p->s); sp.cb = p->bps; sp.nst = p->nst; sp.kb = p->kb;
  sp.gr_up = p->grup + (p->kup - p->up_ksub);  // finest level left to the continuation + 1
  for (int i = 0; i < 32; ++i) {
    sp.lvorder[i] = p->lvorder[i];
    sp.blo[i] = p->blo[i];
    sp.nblk[i] = p->nblk[i];
  }
  sp.band_lo = p->band_lo;
  DownParams dp{};
  dp.out = out; dp.flags = flags; dp.c = c; dp.Tpad = p->d_Tpad; dp.B = p->d_B; dp.ld_out = p->ld_out; dp.n = p->n; dp.N = p->N; dp.batch = p->batch;
  dp.w_tile = p->w_tile_doubles; dp.layout = p->layout; dp.L = int(p->L); dp.s = int(p->s); dp.k = p->k;
  dp.bulk = (p->down_bulk && reinterpret_cast<uintptr_t>(out) % 16 == 0 && p->ld_out % 2 == 0) ? 1 : 0;
  dp.nstream = p->stream_grid;
  dp.sub_lo = p->sub_lo;
  const int64_t ndown = p->nsub_down;
  if (p->part_count > 1 && (ndown == 0 || p->m2l_units + p->band_units == 0)) {
    if (prev != p->device) cudaSetDevice(prev);
    return LC_OK;  // an empty part of a partitioned plan: no rows to compute
  }
  const int64_t nsub = p->L > 0 ? (int64_t(4) << p->grup) : 1;
  if (nsub > 0x7fffffff || ndown > 0x7fffffff || p->ntiles > 65535) {
    if (prev != p->device) cudaSetDevice(prev);
    return LC_ERR_INVALID_ARG;
  }
  const dim3 grid_up(unsigned(p->part_up ? ((p->part_hi - p->part_lo) >> p->kup) : nsub), unsigned(p->ntiles));
  sp.nup = int(grid_up.x * grid_up.y);  // (phase 1 of a part_up plan: the arrivals of its phase 0)
  const dim3 grid_down(unsigned(ndown), unsigned(p->ntiles));
  if (p->engine == 3) {
    TileParams tp{};
    tp.in = in; tp.out = out; tp.A = p->d_A; tp.tabA = p->d_tabA; tp.tabB = p->d_tabB; tp.Tpad = p->d_Tpad; tp.tpr = p->smax;
    tp.B = p->d_B; tp.ld_in = p->ld_in; tp.ld_out = p->ld_out; tp.n = p->n; tp.N = p->N; tp.batch = p->batch;
    tp.ntiles = p->ntiles; tp.layout = p->layout; tp.L = int(p->L); tp.s = int(p->s);
    tp.wg = w; tp.w_tile = p->w_tile_doubles; tp.nranges = p->range_n; tp.rlen = p->range_len;
    tp.nle = p->range_nle;
    tp.oblk = p->out_block;
    tp.scratch = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + p->ws_range_off);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int evi = 0;
    if (ev && nev > 0) cudaEventRecord(ev[evi++], st);
    cfg.gridDim = dim3(unsigned(p->up3_grid));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = p->smem_up;
    cudaError_t e = cudaSuccess;
    if (p->s <= 32) {
      UpArgs<32> ua;
      ua.p = up;
      e = cudaLaunchKernelEx(&cfg, lc_up3_kernel<32>, ua);
    } else {
      UpArgs<40> ua;
      ua.p = up;
      e = cudaLaunchKernelEx(&cfg, lc_up3_kernel<40>, ua);
    }
    if (e == cudaSuccess && ev && evi < nev) cudaEventRecord(ev[evi++], st);
    if (e == cudaSuccess) {
      cfg.gridDim = dim3(unsigned(p->tile_grid));
      cfg.blockDim = dim3(kTileThreads);
      cfg.dynamicSmemBytes = p->smem_tile;
      if (p->range_stage)
        e = p->dir == 0 ? cudaLaunchKernelEx(&cfg, lc_range_kernel<0, 1>, tp) : cudaLaunchKernelEx(&cfg, lc_range_kernel<1, 1>, tp);
      else
        e = p->dir == 0 ? cudaLaunchKernelEx(&cfg, lc_range_kernel<0, 0>, tp) : cudaLaunchKernelEx(&cfg, lc_range_kernel<1, 0>, tp);
    }
    if (e == cudaSuccess && ev && evi < nev) cudaEventRecord(ev[evi++], st);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (prev != p->device) cudaSetDevice(prev);
    return e == cudaSuccess ? LC_OK : record_cuda_error(e);
  }
  const cudaError_t e = p->smax == 32 ? launch_dispatch<32>(p, up, sp, dp, grid_up, grid_down, st, ev, nev)
                                      : launch_dispatch<64>(p, up, sp, dp, grid_up, grid_down, st, ev, nev);
  if (prev != p->device) cudaSetDevice(prev);
  return e == cudaSuccess ? LC_OK : record_cuda_error(e);
}

lc_status launch_execute(const lc_plan* p, const double* in, double* out, void* ws, cudaStream_t st,
                         cudaEvent_t const* ev, int nev, int phase) {
  if (!p) return LC_ERR_INVALID_ARG;
  const lc_status rc = launch_execute_impl(p, in, out, ws, st, ev, nev, phase);
  if (rc == LC_OK) {
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != p->device) cudaSetDevice(p->device);
    note_execute(p, st);
    if (prev != p->device) cudaSetDevice(prev);
  }
  return rc;
}

}  // namespace lc

extern "C" lc_status lc_plan_kernel_info(const lc_plan* p, int64_t* out, int32_t count, int32_t* written) {
  if (!p || !out) return LC_ERR_INVALID_ARG;
  const int64_t up_grid = p->engine == 3 ? p->up3_grid : (p->L > 0 ? (int64_t(4) << p->grup) * p->ntiles : 0);
  const int64_t v[] = {p->stream_grid, int64_t(p->smem_stream), int64_t(p->smem_up), p->kup, p->grup, p->kb,
                       p->bps, p->nst, p->vt, p->stream_occ, p->m2l_units, p->band_units, up_grid, p->k,
                       int64_t(p->smem_down), p->engine, p->tile_grid, int64_t(p->smem_tile), p->range_n, p->range_len,
                       p->up_ksub, p->part_lo, p->part_hi, p->part_up};
  const int32_t nv = int32_t(sizeof(v) / sizeof(v[0]));
  int32_t i = 0;
  for (; i < nv && i < count; ++i) out[i] = v[i];
  if (written) *written = i;
  return LC_OK;
}

extern "C" lc_status lc_execute(const lc_plan* p, const double* in, double* out, void* ws, void* stream) {
  return lc::launch_execute(p, in, out, ws, (cudaStream_t)stream, nullptr, 0, -1);
}

extern "C" lc_status lc_execute_part(const lc_plan* p, int32_t phase, const double* in, double* out, void* ws,
                                     void* stream) {
  if (!p || !p->part_up || (phase != 0 && phase != 1) || !ws) return LC_ERR_INVALID_ARG;
  return lc::launch_execute(p, in, out, ws, (cudaStream_t)stream, nullptr, 0, phase);
}

extern "C" lc_status lc_execute_timed(const lc_plan* p, const double* in, double* out, void* ws, void* stream,
                                      void* const* ev, int32_t nev) {
  if (!p || !ev || nev < lc::kernels_per_execute(p) + 1) return LC_ERR_INVALID_ARG;
  return lc::launch_execute(p, in, out, ws, (cudaStream_t)stream, reinterpret_cast<cudaEvent_t const*>(ev), nev, -1);
}

extern "C" lc_status lc_execute_host(const lc_plan* p, const double* h_in, double* h_out, void* d_stage,
                                     void* ws, void* stream) {
  if (!p || !h_in || !h_out) return LC_ERR_INVALID_ARG;
  const int64_t ein = lc::in_extent(p);
  const int64_t eout = lc::out_extent(p);
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != p->device) cudaSetDevice(p->device);
  double* stage = static_cast<double*>(d_stage);
  if (!stage) stage = lc::plan_stage(p);  // plan-owned, allocated once under the plan's mutex
  if (!stage) {
    if (prev != p->device) cudaSetDevice(prev);
    return LC_ERR_OUT_OF_MEMORY;
  }
  double* d_in = stage;
  double* d_out = reinterpret_cast<double*>(reinterpret_cast<char*>(stage) + lc::align_up(ein * 8, 256));
  cudaStream_t st = (cudaStream_t)stream;
  lc_status rc = LC_OK;
  cudaError_t e = cudaMemcpyAsync(d_in, h_in, size_t(ein) * 8, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) rc = lc::record_cuda_error(e);
  if (rc == LC_OK) rc = lc::launch_execute(p, d_in, d_out, ws, st, nullptr, 0, -1);
  if (rc == LC_OK) {
    e = cudaMemcpyAsync(h_out, d_out, size_t(eout) * 8, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) rc = lc::record_cuda_error(e);
    else lc::note_execute(p, st);  // destroy also waits for the read-back of the staging
  }
  if (prev != p->device) cudaSetDevice(prev);
  return rc;
}

static int64_t chain_half(const lc_plan* const* plans, int nplans) {
  int64_t m = 0;
  for (int k = 0; k < nplans; ++k) m = std::max(m, std::max(lc::in_extent(plans[k]), lc::out_extent(plans[k])));
  return lc::align_up(m * 8, 256);
}

extern "C" size_t lc_host_chain_stage_bytes(const lc_plan* const* plans, int nplans) {
  if (!plans || nplans < 1) return 0;
  for (int k = 0; k < nplans; ++k)
    if (!plans[k]) return 0;
  return size_t(2 * chain_half(plans, nplans));
}

extern "C" lc_status lc_execute_host_chain(const lc_plan* const* plans, int nplans, const double* h_in, double* h_out,
                                           void* d_stage, void* const* workspaces, void* stream) {
  if (!plans || nplans < 1 || !h_in || !h_out || !d_stage) return LC_ERR_INVALID_ARG;
  for (int k = 0; k < nplans; ++k) {
    if (!plans[k] || plans[k]->device != plans[0]->device || plans[k]->part_up) return LC_ERR_INVALID_ARG;
    if (k > 0 && lc::out_extent(plans[k - 1]) < lc::in_extent(plans[k])) return LC_ERR_INVALID_ARG;
  }
  const int dev = plans[0]->device;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != dev) cudaSetDevice(dev);
  // ping-pong staging: plan k reads buf[k & 1] and writes buf[(k + 1) & 1]
  double* buf[2] = {static_cast<double*>(d_stage),
                    reinterpret_cast<double*>(static_cast<char*>(d_stage) + chain_half(plans, nplans))};
  cudaStream_t st = (cudaStream_t)stream;
  lc_status rc = LC_OK;
  cudaError_t e = cudaMemcpyAsync(buf[0], h_in, size_t(lc::in_extent(plans[0])) * 8, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) rc = lc::record_cuda_error(e);
  for (int k = 0; k < nplans && rc == LC_OK; ++k)
    rc = lc::launch_execute(plans[k], buf[k & 1], buf[(k + 1) & 1], workspaces ? workspaces[k] : nullptr, st,
                            nullptr, 0, -1);
  if (rc == LC_OK) {
    e = cudaMemcpyAsync(h_out, buf[nplans & 1], size_t(lc::out_extent(plans[nplans - 1])) * 8,
                        cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) rc = lc::record_cuda_error(e);
    else
      for (int k = 0; k < nplans; ++k) lc::note_execute(plans[k], st);
  }
  if (prev != dev) cudaSetDevice(prev);
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
