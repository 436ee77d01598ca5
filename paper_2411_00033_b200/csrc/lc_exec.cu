// lc_exec.cu -- execution stage (Alg. 4, alg:fastercomplete)
// as two sm_100a kernels per transform, both parities fused (PAPER.md:272:
// the same A_hat serves sigma = 0 and 1, so it is streamed once).
//
//   lc_up_kernel   (one CTA per subtree of 2^k leaf segments x VT vectors):
//       step 1 (eq:wMM, leaf projection w = f^sigma T(sigma)) and step 2
//       (eq:wtk via Alg. a.1) inside the subtree; the last
//       CTA of each group of 2^G sibling subtrees (atomic arrival counter)
//       continues the upward pass G levels, until level 0.  Writes w(g) for
//       every level to the workspace.
//   lc_down_kernel (same grid): the ancestor chain of its subtree root
//       (step 3 M2L of the 1-2 ancestor submatrices per coarser level, all
//       issued in parallel, then the step 4 chain B(p)^T), then level by
//       level inside the subtree: step 4 (B(p)^T push, "faster downward
//       spreading") and step 3 (M2L) with the
//       A_hat arena streamed by TMA bulk copies (cp.async.bulk + mbarrier ring,
//       L2 evict-first); then the epilogue: step 5 (eq:step5), step 6 (direct
//       band, Alg. 1 restricted to j < j_end(i)), step 7 (C^{-1}), store.
//
// The two kernels are chained with programmatic dependent launch: the down
// kernel issues its A_hat prefetch before griddepcontrol.wait.
#include <algorithm>
#include <cstdio>

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
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
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

__device__ __forceinline__ int64_t vaddr(int layout, int64_t ld, int64_t v, int64_t j) {
  return layout == LC_VEC_CONTIGUOUS ? v * ld + j : j * ld + v;
}

// ---------------------------------------------------------------- parameters
struct UpParams {
  const double* in;
  int64_t ld_in, n, N, batch;
  int layout, L, s, k, gr, G;
  const double* T;  // [2][s][M]
  const double* B;  // [M][M]
  double* w;
  int* cnt;
  int64_t w_tile, cnt_tile;
};

struct DownParams {
  const double* in;
  double* out;
  int64_t ld_in, ld_out, n, N, batch;
  int layout, L, s, k, gr, bps, nst;
  const double* A;
  const double* Tt;  // [2][M][s]
  const double* B;
  const double* tabA;
  const double* tabB;
  const double* w;
  int64_t w_tile;
};

// Alg. a.1 for a whole tree level held in shared memory:
// parent P <- B(0) child(2P) + B(1) child(2P+1) = sum_{k<=n} b_nk (x0_k +- x1_k),
// "+" on even diagonals (n-k even), "-" on odd ones (B(1) = B(0) with odd
// diagonals negated, App. A3).  Layout [sigma][node][v][M].
template <int VT>
__device__ __forceinline__ void m2m_level(const double* __restrict__ ch, double* __restrict__ pa, int nparent,
                                          const double* __restrict__ Bs) {
  const int items = 2 * nparent * VT * kM;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int nn = it % kM;
    int r = it / kM;
    const int v = r % VT;
    r /= VT;
    const int P = r % nparent;
    const int sg = r / nparent;
    const double* x0 = ch + ((sg * 2 * nparent + 2 * P) * VT + v) * kM;
    const double* x1 = x0 + VT * kM;
    double acc = 0.0;
    for (int kk = 0; kk <= nn; ++kk) {
      const double b = Bs[nn * kM + kk];
      acc = fma(b, ((nn - kk) & 1) ? (x0[kk] - x1[kk]) : (x0[kk] + x1[kk]), acc);
    }
    pa[((sg * nparent + P) * VT + v) * kM + nn] = acc;
  }
}

// (B(p)^T c)_k = sum_{n>=k} b_nk (-1)^{p(n-k)} c_n   (step 4)
__device__ __forceinline__ double l2l_entry(const double* __restrict__ src, int p, int kk,
                                            const double* __restrict__ Bs) {
  double e = 0.0, o = 0.0;
  for (int nn = kk; nn < kM; nn += 2) e = fma(Bs[nn * kM + kk], src[nn], e);
  for (int nn = kk + 1; nn < kM; nn += 2) o = fma(Bs[nn * kM + kk], src[nn], o);
  return p ? e - o : e + o;
}

// cp.async (LDGSTS): per-element asynchronous global->shared copies, used for
// the small gathers (w windows, band tiles) whose shared-memory destinations
// are padded or scattered; src_bytes = 0 zero-fills (padding beyond n).
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

// ============================================================== up kernel
// Step 1 (eq:wMM) and step 2 (eq:wtk / Alg. a.1) for a subtree of 2^k leaf
// segments, then the group continuation up to level 0.
template <int VT>
__global__ void __launch_bounds__(kThreads) lc_up_kernel(const UpParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ int s_last;
  const int s = P.s, k = P.k;
  const int tid = threadIdx.x;
  double* Ts = reinterpret_cast<double*>(smem);
  double* Bs = reinterpret_cast<double*>(smem + align_up(int64_t(2) * s * kM * 8, 128));
  double* fs = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(Bs) + align_up(int64_t(kMM) * 8, 128));
  const int nleaf = 1 << k;
  const int64_t seglen = 2 * s;
  const int64_t tlen = nleaf * seglen;
  double* tree = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(fs) + align_up(VT * tlen * 8, 128));
  auto tree_off = [&](int j) { return ((1 << j) - 1) * 2 * VT * kM; };

  const int64_t R = blockIdx.x;
  const int64_t tile = blockIdx.y;
  griddep_launch();
  for (int i = tid; i < 2 * s * kM; i += blockDim.x) Ts[i] = __ldg(P.T + i);
  for (int i = tid; i < kMM; i += blockDim.x) Bs[i] = __ldg(P.B + i);
  griddep_wait();  // the input may be produced by the preceding kernel

  // stage the leaf range [R 2^k, (R+1) 2^k) of segments, zero padding beyond n
  const int64_t j0 = R * tlen;
  if (P.layout == LC_VEC_CONTIGUOUS) {
    for (int64_t idx = tid; idx < VT * tlen; idx += blockDim.x) {
      const int64_t v = idx / tlen, jj = idx - v * tlen;
      const int64_t gv = tile * VT + v, j = j0 + jj;
      const bool ok = gv < P.batch && j < P.n;
      cp_async8(fs + idx, ok ? P.in + gv * P.ld_in + j : P.in, ok ? 8u : 0u);
    }
  } else {
    for (int64_t idx = tid; idx < VT * tlen; idx += blockDim.x) {
      const int64_t jj = idx / VT, v = idx - jj * VT;  // v fastest: coalesced in the batch layout
      const int64_t gv = tile * VT + v, j = j0 + jj;
      const bool ok = gv < P.batch && j < P.n;
      cp_async8(fs + v * tlen + jj, ok ? P.in + j * P.ld_in + gv : P.in, ok ? 8u : 0u);
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();

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
      const int seg = r % nleaf;
      const int v = r / nleaf;
      const double* fp = fs + v * tlen + seg * seglen + sg;
      const double* tp = Ts + sg * s * kM + 6 * kg;
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0;
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
      o[0] = a0; o[1] = a1; o[2] = a2; o[3] = a3; o[4] = a4; o[5] = a5;
    }
  }
  __syncthreads();
  // step 2 inside the subtree
  for (int j = k; j >= 1; --j) {
    m2m_level<VT>(tree + tree_off(j), tree + tree_off(j - 1), 1 << (j - 1), Bs);
    __syncthreads();
  }
  double* wt = P.w + tile * P.w_tile;
  const int64_t VM = int64_t(VT) * kM;
  for (int j = 0; j <= k; ++j) {
    const int g = P.gr + j;
    const int64_t cntd = (int64_t(1) << j) * VM;
    for (int sg = 0; sg < 2; ++sg) {
      double2* dst = reinterpret_cast<double2*>(wt + (w_level_offset_units(g) + sg * nseg(g) + (R << j)) * VM);
      const double2* src = reinterpret_cast<const double2*>(tree + tree_off(j) + sg * (int64_t(1) << j) * VM);
      for (int64_t i = tid; i < cntd / 2; i += blockDim.x) dst[i] = src[i];
    }
  }

  // upward continuation above the subtree roots: the last arriver of each
  // group of 2^G nodes merges them G levels up (threadfence-reduction pattern).
  int g = P.gr;
  int64_t node = R;
  while (g > 0) {
    const int ge = min(P.G, g);
    const int64_t grp = node >> ge;
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      int* c = P.cnt + tile * P.cnt_tile + (nseg(g) - 4) + grp;
      const int old = atomicAdd(c, 1);
      const int last = (old == (1 << ge) - 1);
      if (last) atomicExch(c, 0);  // self-reset for the next launch
      s_last = last;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int64_t cntd = (int64_t(1) << ge) * VM;
    for (int sg = 0; sg < 2; ++sg) {
      const double* src = wt + (w_level_offset_units(g) + sg * nseg(g) + (grp << ge)) * VM;
      double* dst = tree + tree_off(ge) + sg * cntd;
      for (int64_t i = tid; i < cntd; i += blockDim.x) dst[i] = __ldcg(src + i);
    }
    __syncthreads();
    for (int j = ge; j >= 1; --j) {
      m2m_level<VT>(tree + tree_off(j), tree + tree_off(j - 1), 1 << (j - 1), Bs);
      __syncthreads();
    }
    for (int j = 0; j < ge; ++j) {
      const int gg = g - ge + j;
      const int64_t cj = (int64_t(1) << j) * VM;
      for (int sg = 0; sg < 2; ++sg) {
        double* dst = wt + (w_level_offset_units(gg) + sg * nseg(gg) + (grp << j)) * VM;
        const double* src = tree + tree_off(j) + sg * cj;
        for (int64_t i = tid; i < cj; i += blockDim.x) dst[i] = src[i];
      }
    }
    g -= ge;
    node = grp;
  }
}

// ============================================================== down kernel
// One CTA per (subtree of 2^k leaf row segments, tile of VT vectors).
template <int VT, int DIR>
__global__ void __launch_bounds__(kThreads, 2) lc_down_kernel(const DownParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ int s_nstages;
  const int s = P.s, k = P.k, gr = P.gr, L = P.L;
  const int tid = threadIdx.x;
  const DownSmem SL = down_smem_layout(VT, k, s, P.bps, P.nst, gr);
  double* Tt = reinterpret_cast<double*>(smem + SL.Tt);
  double* Bs = reinterpret_cast<double*>(smem + SL.Bs);
  double* ta = reinterpret_cast<double*>(smem + SL.ta);
  double* cA = reinterpret_cast<double*>(smem + SL.cA);
  double* cB = reinterpret_cast<double*>(smem + SL.cB);
  double* wall = reinterpret_cast<double*>(smem + SL.wall);
  double* anc = reinterpret_cast<double*>(smem + SL.anc);
  double* chain = reinterpret_cast<double*>(smem + SL.chain);
  double* ring = reinterpret_cast<double*>(smem + SL.ring);
  double* gt = reinterpret_cast<double*>(smem + SL.gt);
  double* tb = reinterpret_cast<double*>(smem + SL.tb);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SL.bars);
  StageDesc* stab = reinterpret_cast<StageDesc*>(smem + SL.stab);
  const int64_t tp = SL.tp;

  const int64_t R = blockIdx.x;
  const int64_t tile = blockIdx.y;
  const int64_t VM = int64_t(VT) * kM;
  const int64_t slot_doubles = int64_t(P.bps) * 3 * kMM;
  const int nleaf = 1 << k;
  const int64_t seglen = 2 * s;
  const int64_t U0 = R << k;
  const int64_t i0 = U0 * seglen;
  const int64_t rows = nleaf * seglen;
  const int64_t tcols = (nleaf + 2) * seglen;

  // ---- stage table of this CTA's A_hat stream (level-major arena, contiguous per level)
  if (tid == 0) {
    int ns = 0;
    if (L > 0) {
      for (int j = 0; j <= k; ++j) {
        const int g = gr + j;
        const int64_t bg = (int64_t(2) << g) - 1;  // b_g (eq:Nb)
        const int64_t abase = ahat_level_offset(g);
        if (j == 0) {
          const int64_t b = R >> 1;
          if (b < bg) {
            StageDesc d;
            d.j = 0; d.b0 = int(b); d.nb = 1; d.r0 = (R & 1) ? 2 : 0; d.nmat = (R & 1) ? 1 : 2; d.pad = 0;
            d.mat0 = abase + 3 * b + d.r0;
            stab[ns++] = d;
          }
        } else {
          const int64_t bb0 = R << (j - 1);
          const int64_t lim = bb0 + (int64_t(1) << (j - 1));
          const int64_t bend = lim < bg ? lim : bg;
          for (int64_t b = bb0; b < bend; b += P.bps) {
            StageDesc d;
            d.j = j; d.b0 = int(b); d.nb = int((bend - b) < P.bps ? (bend - b) : P.bps); d.r0 = 0;
            d.nmat = 3 * d.nb; d.pad = 0;
            d.mat0 = abase + 3 * b;
            stab[ns++] = d;
          }
        }
      }
      for (int i = 0; i < P.nst; ++i) mbar_init(&bars[i], 1);
      fence_mbar_init();
    }
    s_nstages = ns;
  }
  __syncthreads();
  const int nstages = s_nstages;
  uint64_t pol = 0;
  auto issue = [&](int st) {
    const StageDesc d = stab[st];
    const int slot = st % P.nst;
    const uint32_t bytes = uint32_t(d.nmat) * kMM * 8u;
    fence_proxy_async();
    mbar_expect_tx(&bars[slot], bytes);
    bulk_g2s(ring + slot * slot_doubles, P.A + d.mat0 * kMM, bytes, &bars[slot], pol);
  };
  if (tid == 0 && nstages > 0) {
    pol = policy_evict_first();
    for (int st = 0; st < min(P.nst, nstages); ++st) issue(st);
  }
  // ---- plan constants (cp.async group 0): T(sigma)^T, B(0), band tables
  for (int i = tid; i < 2 * s * kM / 2; i += blockDim.x) cp_async16(Tt + 2 * i, P.Tt + 2 * i);
  for (int i = tid; i < kMM / 2; i += blockDim.x) cp_async16(Bs + 2 * i, P.B + 2 * i);
  for (int x = tid; x < 2 * s + 2 * kBandR; x += blockDim.x)
    cp_async8(ta + x, x < 2 * s ? P.tabA + x : P.tabA, x < 2 * s ? 8u : 0u);
  for (int64_t x = tid; x < tcols + 2 * kBandR; x += blockDim.x) {
    const bool ok = x < tcols && i0 + x < P.N;
    cp_async8(tb + pidx(x), ok ? P.tabB + i0 + x : P.tabB, ok ? 8u : 0u);
  }
  cp_async_commit();
  griddep_launch();
  griddep_wait();  // w (up kernel) and the input are ready past this point

  // ---- data of this CTA (cp.async group 1): w windows of every subtree level, input tile
  const double* wt = P.w + tile * P.w_tile;
  if (L > 0) {
    for (int j = 0; j <= k; ++j) {
      const int g = gr + j;
      const int64_t nodes = int64_t(1) << j;
      const int64_t tw0 = (R << j) + 2;
      const int64_t nw = nodes > 2 ? nodes : 2;
      const int64_t twe = (tw0 + nw) < nseg(g) ? (tw0 + nw) : nseg(g);
      if (twe <= tw0) continue;
      const int64_t cnt2 = (twe - tw0) * VM / 2;
      for (int sg = 0; sg < 2; ++sg) {
        const double* src = wt + (w_level_offset_units(g) + sg * nseg(g) + tw0) * VM;
        double* dst = wall + (wall_nodes_before(j) * 2 + sg * nw) * VM;
        for (int64_t i = tid; i < cnt2; i += blockDim.x) cp_async16(dst + 2 * i, src + 2 * i);
      }
    }
  }
  for (int64_t idx = tid; idx < VT * (tcols + 2 * kBandR); idx += blockDim.x) {
    const int64_t v = idx / (tcols + 2 * kBandR), x = idx - v * (tcols + 2 * kBandR);
    const int64_t gv = tile * VT + v, j = i0 + x;
    const bool ok = x < tcols && gv < P.batch && j < P.n;
    const double* src = ok ? P.in + vaddr(P.layout, P.ld_in, gv, j) : P.in;
    cp_async8(gt + v * tp + pidx(x), src, ok ? 8u : 0u);
  }
  cp_async_commit();

  const double* cfin = cA;
  if (L > 0) {
    // ---- ancestor chain: M2L of every ancestor of the subtree root, all in parallel (L2-resident A_hat)
    const double* chain_final = chain;
    if (gr > 0) {
      for (int it = tid; it < gr * kM; it += blockDim.x) {
        const int g = it / kM, kk = it % kM;
        const int64_t a = R >> (gr - g);
        double acc[2][VT];
#pragma unroll
        for (int sg = 0; sg < 2; ++sg)
#pragma unroll
          for (int v = 0; v < VT; ++v) acc[sg][v] = 0.0;
        if (a <= nseg(g) - 3) {
          const int64_t b = a >> 1;
          const int64_t abase = ahat_level_offset(g);
          const int nmat = (a & 1) ? 1 : 2;
          for (int mi = 0; mi < nmat; ++mi) {
            const int r = (a & 1) ? 2 : mi;
            const int64_t t = (a & 1) ? a + 2 : a + 2 + mi;  // r=0: t=a+2, r=1: t=a+3; r=2 (odd a): t=a+2
            const double2* arow = reinterpret_cast<const double2*>(P.A + (abase + 3 * b + r) * kMM + kk * kM);
            double ar[kM];
#pragma unroll
            for (int l = 0; l < kM / 2; ++l) {
              const double2 a2 = __ldg(arow + l);
              ar[2 * l] = a2.x;
              ar[2 * l + 1] = a2.y;
            }
#pragma unroll
            for (int sg = 0; sg < 2; ++sg)
#pragma unroll
              for (int v = 0; v < VT; ++v) {
                const double2* wp =
                    reinterpret_cast<const double2*>(wt + (w_level_offset_units(g) + sg * nseg(g) + t) * VM + v * kM);
                double sacc = 0.0;
#pragma unroll
                for (int l = 0; l < kM / 2; ++l) {
                  const double2 w2 = __ldcg(wp + l);
                  sacc = fma(ar[2 * l], w2.x, sacc);
                  sacc = fma(ar[2 * l + 1], w2.y, sacc);
                }
                acc[sg][v] += sacc;
              }
          }
        }
#pragma unroll
        for (int sg = 0; sg < 2; ++sg)
#pragma unroll
          for (int v = 0; v < VT; ++v) anc[((g * 2 + sg) * VT + v) * kM + kk] = acc[sg][v];
      }
    }
    cp_async_wait<1>();  // constants (B) have landed
    __syncthreads();
    if (gr > 0) {
      // Horner chain of step 4 down to level gr-1
      double* cb0 = chain;
      double* cb1 = chain + 2 * VM;
      for (int i = tid; i < 2 * VM; i += blockDim.x) cb0[i] = anc[i];
      __syncthreads();
      for (int g = 1; g < gr; ++g) {
        const int p = int((R >> (gr - g)) & 1);
        for (int it = tid; it < 2 * VM; it += blockDim.x) {
          const int kk = it % kM;
          const int sv = it / kM;  // sigma*VT + v
          cb1[it] = anc[g * 2 * VM + it] + l2l_entry(cb0 + sv * kM, p, kk, Bs);
        }
        __syncthreads();
        double* t = cb0; cb0 = cb1; cb1 = t;
      }
      chain_final = cb0;
    }
    cp_async_wait<0>();  // w windows and the input tile
    __syncthreads();

    // ---- the subtree, level by level: step 4 push then step 3 M2L (streamed A_hat)
    int st = 0;
    for (int j = 0; j <= k; ++j) {
      const int nodes = 1 << j;
      const int64_t u0 = R << j;
      const int64_t tw0 = u0 + 2;
      const int nw = nodes > 2 ? nodes : 2;
      const double* wwin = wall + wall_nodes_before(j) * 2 * VM;
      double* cur = (j & 1) ? cB : cA;
      const double* par = (j & 1) ? cA : cB;
      {
        const int items = nodes * 2 * VT * kM;
        for (int it = tid; it < items; it += blockDim.x) {
          const int kk = it % kM;
          int r = it / kM;
          const int v = r % VT;
          r /= VT;
          const int node = r % nodes;
          const int sg = r / nodes;
          double val = 0.0;
          if (j == 0) {
            if (gr > 0) val = l2l_entry(chain_final + (sg * VT + v) * kM, int(R & 1), kk, Bs);
          } else {
            const double* src = par + ((sg * (nodes >> 1) + (node >> 1)) * VT + v) * kM;
            val = l2l_entry(src, node & 1, kk, Bs);
          }
          cur[((sg * nodes + node) * VT + v) * kM + kk] = val;
        }
      }
      __syncthreads();
      while (st < nstages && stab[st].j == j) {
        const StageDesc d = stab[st];
        const int slot = st % P.nst;
        mbar_wait(&bars[slot], uint32_t((st / P.nst) & 1));
        const double* As = ring + slot * slot_doubles;
        const int nrows = (j == 0) ? 1 : 2 * d.nb;
        for (int it = tid; it < nrows * kM; it += blockDim.x) {
          const int ri = it / kM, kk = it % kM;
          const int64_t u = (j == 0) ? R : (2 * int64_t(d.b0) + ri);
          const int64_t b = u >> 1;
          double acc[2][VT];
#pragma unroll
          for (int sg = 0; sg < 2; ++sg)
#pragma unroll
            for (int v = 0; v < VT; ++v) acc[sg][v] = 0.0;
          const int nmat = (u & 1) ? 1 : 2;
          for (int mi = 0; mi < nmat; ++mi) {
            const int r = (u & 1) ? 2 : mi;
            const int64_t t = (u & 1) ? u + 2 : u + 2 + mi;
            const double* arow = As + (3 * (b - d.b0) + r - d.r0) * kMM + kk * kM;
            double ar[kM];
#pragma unroll
            for (int l = 0; l < kM; l += 2) {
              const double2 a2 = *reinterpret_cast<const double2*>(arow + l);
              ar[l] = a2.x;
              ar[l + 1] = a2.y;
            }
#pragma unroll
            for (int sg = 0; sg < 2; ++sg)
#pragma unroll
              for (int v = 0; v < VT; ++v) {
                const double* wp = wwin + (sg * nw + (t - tw0)) * VM + v * kM;
                double sacc = 0.0;
#pragma unroll
                for (int l = 0; l < kM; ++l) sacc = fma(ar[l], wp[l], sacc);
                acc[sg][v] += sacc;
              }
          }
#pragma unroll
          for (int sg = 0; sg < 2; ++sg)
#pragma unroll
            for (int v = 0; v < VT; ++v) cur[((sg * nodes + (u - u0)) * VT + v) * kM + kk] += acc[sg][v];
        }
        __syncthreads();
        if (tid == 0 && st + P.nst < nstages) issue(st + P.nst);
        ++st;
      }
    }
    cfin = (k & 1) ? cB : cA;
  } else {
    cp_async_wait<0>();
    __syncthreads();
  }

  // ---- epilogue: step 5 (eq:step5), step 6 (direct band, register-blocked), step 7 (C^{-1})
  // item = (v, segment u, parity sigma, block t of kBandR same-parity rows m = kBandR t + r).
  // Band for row i' = i + 2r (i the block's first row): sum_c a[c-r] b[i+r+c] g[i+2c], c >= r,
  // i + 2c < j_end; a[.] = tabA, b[.] = tabB, g = f (L2C) or j f_j (C2L).  Sliding windows of a
  // and b are kept in registers (slots rotate with c), so each step loads 3 values for kBandR rows.
  double* zst = ring;  // [VT][rows] staging for a coalesced store
  const double inv_pi = 0.318309886183790671537767526745028724;
  const int ntb = (s + kBandR - 1) / kBandR;
  const int items = VT * nleaf * 2 * ntb;
  for (int it = tid; it < items; it += blockDim.x) {
    const int tb_i = it % ntb;
    int r_ = it / ntb;
    const int sg = r_ & 1;
    r_ >>= 1;
    const int u = r_ % nleaf;
    const int v = r_ / nleaf;
    const int m0 = kBandR * tb_i;
    const int64_t ii = int64_t(u) * seglen + sg + 2 * m0;  // tile-local first row
    const int64_t i = i0 + ii;
    const int64_t je = (seglen * (U0 + u + 2)) < P.N ? seglen * (U0 + u + 2) : P.N;
    const int cmax = int((je - i - 1) >> 1);
    const double* gv_t = gt + v * tp;
    double acc[kBandR], aw[kBandR], bw[kBandR];
#pragma unroll
    for (int r = 0; r < kBandR; ++r) {
      acc[r] = 0.0;
      aw[r] = 0.0;
      bw[r] = tb[pidx(ii + r)];
    }
    for (int c0 = 0; c0 <= cmax; c0 += kBandR) {
#pragma unroll
      for (int uu = 0; uu < kBandR; ++uu) {
        const int c = c0 + uu;
        if (c <= cmax) {
          aw[uu] = ta[c];
          if (c >= 1) bw[(uu + kBandR - 1) % kBandR] = tb[pidx(ii + kBandR - 1 + c)];
          double gval = gv_t[pidx(ii + 2 * c)];
          if (DIR == 1) gval *= double(i + 2 * c);
#pragma unroll
          for (int r = 0; r < kBandR; ++r)
            acc[r] = fma(aw[(uu - r + kBandR) % kBandR] * bw[(r + uu) % kBandR], gval, acc[r]);
        }
      }
    }
    // step 5: z^sigma = c(L-1) T(sigma)^T
    double t5[kBandR];
#pragma unroll
    for (int r = 0; r < kBandR; ++r) t5[r] = 0.0;
    if (L > 0) {
      const double* cp = cfin + ((sg * nleaf + u) * VT + v) * kM;
      const double* tq = Tt + sg * kM * s + m0;
#pragma unroll
      for (int kk = 0; kk < kM; ++kk) {
        const double cv = cp[kk];
#pragma unroll
        for (int r = 0; r < kBandR; ++r) t5[r] = fma(cv, tq[kk * s + r], t5[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < kBandR; ++r) {
      if (m0 + r < s) {
        const int64_t ir = i + 2 * r;
        double z;
        if (DIR == 0) {
          z = (t5[r] + acc[r]) * (ir == 0 ? inv_pi : 2.0 * inv_pi);  // step 7: C^{-1}
        } else {
          z = t5[r] + double(2 * ir + 1) * acc[r];
          if (ir == 0) z += gv_t[pidx(0)];  // entry (0,0) of A^{-1}C is 1 (reading R2)
        }
        zst[v * rows + ii + 2 * r] = z;
      }
    }
  }
  __syncthreads();
  if (P.layout == LC_VEC_CONTIGUOUS) {
    for (int64_t idx = tid; idx < VT * rows; idx += blockDim.x) {
      const int64_t v = idx / rows, ii = idx - v * rows;
      const int64_t gv = tile * VT + v, i = i0 + ii;
      if (gv < P.batch && i < P.n) P.out[gv * P.ld_out + i] = zst[idx];
    }
  } else {
    for (int64_t idx = tid; idx < VT * rows; idx += blockDim.x) {
      const int64_t ii = idx / VT, v = idx - ii * VT;
      const int64_t gv = tile * VT + v, i = i0 + ii;
      if (gv < P.batch && i < P.n) P.out[i * P.ld_out + gv] = zst[v * rows + ii];
    }
  }
}

// ============================================================== host side
template <typename K>
static cudaError_t set_max_dyn_smem(K kernel, int smax) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, kernel);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smax - int(fa.sharedSizeBytes));
}
template <int VT>
static cudaError_t set_attrs_vt(int smax) {
  cudaError_t e = set_max_dyn_smem(lc_up_kernel<VT>, smax);
  if (e == cudaSuccess) e = set_max_dyn_smem(lc_down_kernel<VT, 0>, smax);
  if (e == cudaSuccess) e = set_max_dyn_smem(lc_down_kernel<VT, 1>, smax);
  return e;
}

lc_status configure_kernels(lc_plan* p) {
  int smax = 0;
  if (cudaDeviceGetAttribute(&smax, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->device) != cudaSuccess)
    return LC_ERR_CUDA;
  cudaError_t ea = set_attrs_vt<1>(smax);
  if (ea == cudaSuccess) ea = set_attrs_vt<2>(smax);
  if (ea == cudaSuccess) ea = set_attrs_vt<4>(smax);
  if (ea == cudaSuccess) ea = set_attrs_vt<8>(smax);
  if (ea != cudaSuccess) return record_cuda_error(ea);
  smax -= 256;  // static shared memory of the kernels

  const int64_t budget = 113 * 1024;  // two CTAs per SM (228 KB minus 1 KB reserved per CTA)
  int vt = p->vt;
  if (vt <= 0) vt = p->batch >= 2 ? 2 : 1;
  if (vt != 1 && vt != 2 && vt != 4 && vt != 8) return LC_ERR_INVALID_ARG;
  const bool user_k = p->k > 0;
  int k = user_k ? p->k : 4;
  int bps = p->bps > 0 ? p->bps : 2;
  int nst = p->nst > 0 ? p->nst : 3;
  if (p->L == 0) {
    k = 1;
  } else {
    k = int(std::min<int64_t>(k, p->L - 1));
  }
  auto down_bytes = [&](int vt_, int k_) {
    const int gr_ = p->L > 0 ? int(p->L - 1 - k_) : 0;
    return down_smem_layout(vt_, k_, int(p->s), bps, nst, gr_).total;
  };
  if (!user_k) {
    while (down_bytes(vt, k) > budget && p->L > 0 && k > 1) --k;
  }
  if (down_bytes(vt, k) > smax) return LC_ERR_INVALID_ARG;
  // up kernel: deeper subtrees (its shared memory is small); continuation step = its depth
  int kup = p->L > 0 ? int(std::min<int64_t>(5, p->L - 1)) : 0;
  while (kup > 0 && up_smem_bytes(vt, kup, int(p->s)) > budget) --kup;
  p->vt = vt;
  p->k = k;
  p->bps = bps;
  p->nst = nst;
  p->gr = p->L > 0 ? int(p->L - 1 - k) : 0;
  p->kup = kup;
  p->grup = p->L > 0 ? int(p->L - 1 - kup) : 0;
  p->group = std::max(kup, 1);
  p->ntiles = (p->batch + vt - 1) / vt;
  // stage-table capacity
  if (p->L > 0) {
    int64_t ns = 1;
    for (int j = 1; j <= k; ++j) ns += ((int64_t(1) << (j - 1)) + bps - 1) / bps;
    if (ns > kMaxStages) return LC_ERR_INVALID_ARG;
  }
  p->smem_down = size_t(down_bytes(vt, k));
  p->smem_up = size_t(up_smem_bytes(vt, kup, int(p->s)));
  if (p->L > 0) {
    p->w_tile_doubles = int64_t(vt) * kM * 2 * ((int64_t(4) << p->L) - 4);
    p->cnt_tile_ints = int64_t(4) << p->L;
  } else {
    p->w_tile_doubles = 0;
    p->cnt_tile_ints = 0;
  }
  const size_t wb = size_t(align_up(p->ntiles * p->w_tile_doubles * 8, 256));
  p->ws_bytes = wb + size_t(p->ntiles * p->cnt_tile_ints) * sizeof(int);
  return LC_OK;
}

template <int VT>
static cudaError_t launch_vt(const lc_plan* p, const UpParams& up, const DownParams& dp, dim3 grid_up, dim3 grid,
                             cudaStream_t st, cudaEvent_t const* ev, int nev) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kThreads);
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaSuccess;
  int evi = 0;
  if (ev && nev > 0) cudaEventRecord(ev[evi++], st);
  if (p->L > 0) {
    cfg.gridDim = grid_up;
    cfg.dynamicSmemBytes = p->smem_up;
    e = cudaLaunchKernelEx(&cfg, lc_up_kernel<VT>, up);
    if (e != cudaSuccess) return e;
    if (ev && evi < nev) cudaEventRecord(ev[evi++], st);
  }
  cfg.gridDim = p->L > 0 ? grid : dim3(1, grid.y);
  cfg.dynamicSmemBytes = p->smem_down;
  if (p->dir == 0)
    e = cudaLaunchKernelEx(&cfg, lc_down_kernel<VT, 0>, dp);
  else
    e = cudaLaunchKernelEx(&cfg, lc_down_kernel<VT, 1>, dp);
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
  double* w = reinterpret_cast<double*>(ws);
  int* cnt = reinterpret_cast<int*>(reinterpret_cast<char*>(ws) +
                                    align_up(p->ntiles * p->w_tile_doubles * 8, 256));
  UpParams up{};
  up.in = in; up.ld_in = p->ld_in; up.n = p->n; up.N = p->N; up.batch = p->batch;
  up.layout = p->layout; up.L = int(p->L); up.s = int(p->s); up.k = p->kup; up.gr = p->grup; up.G = p->group;
  up.T = p->d_T; up.B = p->d_B; up.w = w; up.cnt = cnt; up.w_tile = p->w_tile_doubles; up.cnt_tile = p->cnt_tile_ints;
  DownParams dp{};
  dp.in = in; dp.out = out; dp.ld_in = p->ld_in; dp.ld_out = p->ld_out; dp.n = p->n; dp.N = p->N;
  dp.batch = p->batch; dp.layout = p->layout; dp.L = int(p->L); dp.s = int(p->s); dp.k = p->k; dp.gr = p->gr;
  dp.bps = p->bps; dp.nst = p->nst; dp.A = p->d_A; dp.Tt = p->d_Tt; dp.B = p->d_B; dp.tabA = p->d_tabA;
  dp.tabB = p->d_tabB; dp.w = w; dp.w_tile = p->w_tile_doubles;
  const int64_t nsub = p->L > 0 ? (int64_t(4) << p->gr) : 1;
  if (nsub > 0x7fffffff || p->ntiles > 65535) {
    if (prev != p->device) cudaSetDevice(prev);
    return LC_ERR_INVALID_ARG;
  }
  const dim3 grid(unsigned(nsub), unsigned(p->ntiles));
  const dim3 grid_up(unsigned(p->L > 0 ? (int64_t(4) << p->grup) : 1), unsigned(p->ntiles));
  cudaError_t e;
  switch (p->vt) {
    case 1: e = launch_vt<1>(p, up, dp, grid_up, grid, st, ev, nev); break;
    case 2: e = launch_vt<2>(p, up, dp, grid_up, grid, st, ev, nev); break;
    case 4: e = launch_vt<4>(p, up, dp, grid_up, grid, st, ev, nev); break;
    case 8: e = launch_vt<8>(p, up, dp, grid_up, grid, st, ev, nev); break;
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
  if (!ev || nev < (p && p->L > 0 ? 3 : 2)) return LC_ERR_INVALID_ARG;
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
  if (cudaMemcpyAsync(p->d_stage_in, h_in, size_t(ein) * 8, cudaMemcpyHostToDevice, st) != cudaSuccess) rc = LC_ERR_CUDA;
  if (rc == LC_OK) rc = lc::launch_execute(p, p->d_stage_in, p->d_stage_out, nullptr, st, nullptr, 0);
  if (rc == LC_OK &&
      cudaMemcpyAsync(h_out, p->d_stage_out, size_t(eout) * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    rc = LC_ERR_CUDA;
  cudaSetDevice(prev);
  return rc;
}
