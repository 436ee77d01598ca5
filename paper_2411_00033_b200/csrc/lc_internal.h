// lc_internal.h -- internal definitions shared by the planner and the
// execution kernels of the B200 Legendre<->Chebyshev library.
//
// Notation follows arXiv 2411.00033: levels g = 0..L-1, h_g =
// s 2^(L-g-1), b_g = 2^(g+1)-1 blocks, three submatrices r = 0,1,2 per block
// (eq:cfrompq), M = 18 Chebyshev modes.  DESIGN.md "Data layout" defines the
// segment indexing used here: level g cuts the padded vector into 2^(g+2)
// segments of length 2h_g; column block (g,b,q) is segment t = 2b+q+2
// (eq:globalij), row block (g,b,p) is segment u = 2b+p; segment t of level g
// is segments 2t, 2t+1 of level g+1 (eq:flevels, eq:zlevels).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/legcheb.h"

namespace lc {

constexpr int kM = 18;               // Chebyshev modes
constexpr int kMM = kM * kM;
constexpr int kThreads = 256;        // threads per CTA of the execution kernels

// First A_hat index of level g in the level-major (g, b, r) arena:
// 3 * sum_{g'<g} b_g' = 3 (2^(g+1) - 2 - g).
__host__ __device__ inline int64_t ahat_level_offset(int g) {
  return 3 * ((int64_t(2) << g) - 2 - g);
}
// Segments on level g (all of them; rows u < 2^(g+2)-2 carry M2L, columns t >= 2 carry w).
__host__ __device__ inline int64_t nseg(int g) { return int64_t(4) << g; }
// Offset (in units of VT*M doubles) of level g inside one vector tile of w:
// sum_{g'<g} 2 * 2^(g'+2) = 2 (2^(g+2) - 4).
__host__ __device__ inline int64_t w_level_offset_units(int g) { return 2 * ((int64_t(4) << g) - 4); }

struct Geometry {
  int64_t n, N, L, s, nc;
};

// log2 of the leaf-segment alignment of a part (NEXT-2): 64 leaves (or all of them for short trees)
inline int part_align_log2(int64_t L) { return int(L + 1 < 6 ? L + 1 : 6); }

// Default s_hat (reading R17): s = ceil(n / 2^(L+2)) then lies in [s_hat/2, s_hat] = [20, 40],
// within a factor sqrt(2) of the flop-optimal s = 29 of eq:totalnumflopsnew for every n
// (s_hat = 32 keeps power-of-two n at s = 32, but lets s fall to 16: n = 10^7 gets s = 20, whose M2L work
// and A_hat bytes per coefficient are twice those of s = 39).
constexpr int64_t kSHatDefault = 40;

// eq:numlevels; L clamped at 0 (band only) for n <= 4 s_hat.
inline Geometry geometry(int64_t n, int64_t s_hat) {
  Geometry G{};
  int64_t lp = 0;
  while ((s_hat << lp) < n) ++lp;
  G.L = lp >= 2 ? lp - 2 : 0;
  G.n = n;
  G.s = (n + (int64_t(1) << (G.L + 2)) - 1) >> (G.L + 2);
  G.N = G.s << (G.L + 2);
  G.nc = G.L > 0 ? 3 * ((G.N / (2 * G.s)) - G.L - 2) : 0;  // eq:total_blocks_and_mats
  return G;
}

constexpr int kBandR = 8;            // rows per thread in the register-blocked band (step 6)

// Padded index of the band tiles: one pad double every 16, so that threads
// whose rows are 2*kBandR apart hit distinct shared-memory banks.
__host__ __device__ inline int64_t pidx(int64_t x) { return x + (x >> 4); }

__host__ __device__ inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Streaming kernel: a ring of nst slots, each with the A_hat of `cb` blocks plus the w window
// (2 cb column segments, both parities, VT vectors); and the band region for a band unit of
// 2^kb leaf segments: tabA, padded tabB and input tiles, and the z staging tile.
struct StreamSmem {
  int64_t slot, ring, ta, tb, gt, zst, bars, total;
  int64_t tp;  // padded band-tile length (doubles)
};
__host__ __device__ inline StreamSmem stream_smem_layout(int VT, int cb, int nst, int kb, int s) {
  StreamSmem S{};
  S.slot = align_up(int64_t(cb) * 3 * kMM * 8, 128) + align_up(int64_t(2) * (2 * cb) * VT * kM * 8, 128);
  int64_t o = 0;
  S.ring = o;  o += int64_t(nst) * S.slot;
  const int64_t nleaf = int64_t(1) << kb;
  const int64_t tcols = (nleaf + 2) * 2 * s;
  S.tp = pidx(tcols + 2 * kBandR) + 2;
  S.ta = o;   o = align_up(o + (int64_t(2) * s + 2 * kBandR) * 8, 128);
  S.tb = o;   o = align_up(o + S.tp * 8, 128);
  S.gt = o;   o = align_up(o + int64_t(VT) * S.tp * 8, 128);
  S.zst = o;  o = align_up(o + (pidx(int64_t(VT) * nleaf * 2 * s) + 2) * 8, 128);  // padded like the band tiles
  S.bars = o; o = align_up(o + int64_t(2) * nst * 8, 128);
  S.total = o;
  return S;
}

// Down kernel: c_m2l of the gd ancestors and of the 2^(kd+1)-1 subtree nodes (both parities,
// VT vectors), then the band result of the 2^kd leaf segments.
__host__ __device__ inline int64_t down_smem_bytes(int VT, int kd, int s, int L) {
  const int gd = L > 0 ? L - 1 - kd : 0;
  const int64_t nodes = L > 0 ? int64_t(gd) + ((int64_t(2) << kd) - 1) : 0;
  const int64_t smax = s <= 32 ? 32 : 64;
  return align_up((2 * (kMM + 4) + 2 * smax * kM) * 8 + nodes * 2 * VT * kM * 8 + int64_t(VT) * (int64_t(1) << kd) * 2 * s * 8,
                  128);
}

// segment stride of the up kernel's f tile: 2s rounded up to 2 (mod 4) doubles, so that the
// 16-byte reads of 32 consecutive leaves hit distinct bank quads
__host__ __device__ inline int up_fstride(int s) { return (2 * s) % 4 == 2 ? 2 * s : 2 * s + 2; }

// T(sigma) [2][SMAX][M] and B(0) in shared memory, 128-byte aligned (SMAX = 32 for s <= 32, else 64)
__host__ __device__ constexpr int64_t up_const_bytes(int smax) { return ((2 * smax * kM + kMM) * 8 + 127) / 128 * 128; }

__host__ __device__ inline int64_t up_smem_bytes(int VT, int k, int s) {
  int64_t o = up_const_bytes(s <= 32 ? 32 : 64);
  o = align_up(o + (int64_t(VT) * (int64_t(1) << k) * up_fstride(s) + 2 * 64) * 8, 128);  // f tile + zero tail
  o = align_up(o + ((int64_t(2) << k) - 1) * 2 * VT * kM * 8, 128);          // w tree
  o += 16;
  return o;
}

}  // namespace lc

struct lc_plan {
  int64_t n, N, L, s, M, batch, nc;
  int dir;
  int layout;
  int64_t ld_in, ld_out;
  int device;
  int sm_count;
  // kernel configuration
  int vt, k, gr, bps, nst, group, kup, grup, kb;
  int smax;            // 32 or 64: rows of the padded copy of T(sigma)
  int up3_nbuf;        // engine 3: f buffers of the up pass
  int lvorder[32];     // M2L level order of the streaming kernel
  double* h_Tpad;      // host [2][smax][M] copy of T(sigma), zero rows m >= s (kernel parameter)
  double* d_Tpad;      // device copy of h_Tpad
  int64_t m2l_units;   // (chunk, tile) M2L work units of the streaming kernel
  int64_t band_units;  // (leaf range, tile) band work units of the streaming kernel
  int stream_grid, stream_occ;
  int engine;          // 1 = up / stream / down kernels, 2 = per-tile streaming kernel
  int down_bulk;       // engine 1 down kernel: TMA bulk loads of c_m2l and the band rows
  int up_ksub;         // engine 1: M2M levels merged inside the up kernel's subtree (<= kup)
  // partitioned single-vector plan (NEXT-2): part part_index of part_count computes the output rows
  // [row_lo, row_hi) = leaf segments [part_lo, part_hi); the up pass stays whole (replicated)
  int part_index, part_count;
  int part_up;            // the up pass partitioned too (two-phase execution around a root/halo exchange)
  int64_t part_lo, part_hi, row_lo, row_hi;
  int blo[32], nblk[32];  // M2L row blocks per level
  int band_lo;            // first band unit
  int64_t sub_lo, nsub_down;  // down-kernel subtrees
  int tile_grid;       // CTAs of the per-tile kernel (engine 2)
  size_t smem_tile;
  int range_n, range_len;   // engine 3: leaf ranges per tile and their length
  int range_nle;            // engine 3: leaf segments holding outputs (ranges stop there)
  int64_t out_block;        // > 0: column-blocked output of width out_block (engines 2 and 3)
  int range_stage;          // engine 3: range kernel with per-warp staged M2L operands (3 CTAs per SM)
  int64_t ws_range_off;     // engine 3: byte offset of the per-CTA scratch in the workspace
  int up3_kc;               // engine 3: subtrees per chunk of the persistent up pass = 2^up3_kc
  int64_t up3_grid;         // engine 3: CTAs of the persistent up pass
  size_t smem_stream;
  int64_t ntiles;
  int64_t w_tile_doubles, cnt_tile_ints;
  size_t ws_bytes;
  size_t smem_up, smem_down;
  // device data (plan-owned)
  double* d_A;      // nc * M * M
  double* d_tabB;   // N    (L2C: lambda_m; C2L: rho_m = 1/(2m(2m+1) lambda_m), rho_0 = 0)
  double* d_tabA;   // 2s   (L2C: lambda_k; C2L: kappa_k = lambda_k/(1-2k))
  double* d_T;      // [2][s][M]
  double* d_Tt;     // [2][M][s]
  double* d_B;      // [M][M]
  void* d_ws;       // plan-owned workspace
  double* d_stage;      // plan-owned lc_execute_host staging (allocated once, on first use, under sync->mu)
  size_t stage_bytes;   // lc_host_stage_bytes(): input staging + output staging, 256-byte aligned halves
  cudaStream_t own;     // plan-internal non-blocking stream: planning kernels, allocations, frees
  struct lc_plan_sync* sync;  // host-only: mutex + last-execute event per stream (lc_plan.cu)
  double plan_ms;       // device time of the planning kernels (CUDA events on `own`)
  int64_t band_nnz;
  double flops_alg, bytes_alg;
  size_t plan_bytes;
};

namespace lc {
// elements spanned by the input / the output array of one execute (layout, leading dimensions and,
// for the output, the column blocking of out_block plans)
inline int64_t in_extent(const lc_plan* p) {
  return p->layout == LC_VEC_CONTIGUOUS ? (p->batch - 1) * p->ld_in + p->n : (p->n - 1) * p->ld_in + p->batch;
}
inline int64_t out_extent(const lc_plan* p) {
  if (p->out_block > 0) return (p->n + p->out_block - 1) / p->out_block * p->batch * p->out_block;
  return p->layout == LC_VEC_CONTIGUOUS ? (p->batch - 1) * p->ld_out + p->n : (p->n - 1) * p->ld_out + p->batch;
}
// remembers the last CUDA error (thread-local) for lc_last_error(); returns LC_ERR_CUDA or OUT_OF_MEMORY
lc_status record_cuda_error(cudaError_t e);
lc_status launch_execute(const lc_plan* p, const double* in, double* out, void* ws, cudaStream_t st,
                         cudaEvent_t const* ev, int nev, int phase);
// records that p was used on stream st (after the enqueued work) so lc_plan_destroy can wait for it;
// a no-op on a capturing stream (graph launches are the caller's to finish before destroy)
void note_execute(const lc_plan* p, cudaStream_t st);
// kernel launches of one lc_execute
inline int kernels_per_execute(const lc_plan* p) {
  if (p->engine == 2) return 1;
  if (p->engine == 3) return 2;
  return p->L > 0 ? 3 : 2;
}
// the plan-owned lc_execute_host staging (allocated once, thread-safe), or nullptr on failure
double* plan_stage(const lc_plan* p);
int64_t band_nnz(int64_t N, int64_t s);
// engine 3's persistent up pass (lc_up3_kernel, 8 vectors, s <= 32): constants, two f buffers,
// the subtree tree, kc waiting left siblings and two merged parents
// (T(sigma) staged with 32 rows for s <= 32, else 40: engines 2 / 3 take s <= 40)
__host__ __device__ inline int64_t up3_smem_bytes(int k, int s, int kc, int nbuf) {
  const int smax = s <= 32 ? 32 : 40;
  int64_t o = up_const_bytes(smax);
  o += nbuf * align_up((int64_t(8) * (int64_t(1) << k) * up_fstride(s) + 2 * smax) * 8, 128);
  o += ((int64_t(2) << k) - 1) * 2 * 8 * kM * 8;
  o += int64_t(kc + 2) * 2 * 8 * kM * 8;
  return o + 16;
}

}  // namespace lc
