/*
 * legcheb.h -- C ABI of the B200 (sm_100a) execution stage of the modal FMM
 * Legendre<->Chebyshev coefficient transform of arXiv 2411.00033.
 *
 * Citations "PAPER.md:L" are lines of the paper's LaTeX source; equation and
 * algorithm names are its LaTeX labels.
 *
 *   leg2cheb (L2C):  f_cheb = C^{-1} A f_leg                         PAPER.md:29-32 (eq:directmv)
 *   cheb2leg (C2L):  f_leg  = A^{-1} C f_cheb                        PAPER.md:29-32 (eq:directmv)
 *   a_{i,i+2k} = Lambda(k) Lambda(i+k),  Lambda(x) = Gamma(x+1/2)/Gamma(x+1)
 *   C = diag(c_i pi/2), c_0 = 2, c_i = 1
 *
 * The transform is evaluated with the paper's O(N) algorithm (Alg. 4,
 * alg:fastercomplete): leaf projection (step 1), upward
 * modal transfer with the exact triangular B(l) (step 2, eq:wtk, Alg. a.1),
 * low-rank M2L with the precomputed M x M Chebyshev coefficient matrices
 * A_hat (step 3, eq:aklmore), the "faster downward spreading" B(p)^T
 * (step 4), leaf evaluation (step 5), the direct near-diagonal band
 * (step 6, Alg. 1 restricted to j < j_end(i) = min(N, 2s(floor(i/2s)+2))) and
 * C^{-1} (step 7).  C2L uses the kernel L(x,y) of eq:Lxymod
 * in the band and in A_hat.  Both parities share one A_hat.
 *
 * Conventions common to all entry points
 * --------------------------------------
 *  - All floating point data are IEEE fp64 (double).
 *  - Device pointers are CUDA device addresses on the plan's device; host
 *    pointers are ordinary (preferably page-locked) host addresses.
 *  - Nothing here throws; every function returns an lc_status.  A CUDA
 *    error detected during a call is returned as LC_ERR_CUDA; asynchronous
 *    kernel faults surface at the caller's next synchronisation.
 *  - Thread safety: a plan is immutable after lc_plan_create (its only
 *    mutable state -- the lazily allocated lc_execute_host staging and the
 *    per-stream record of executions used by lc_plan_destroy -- is guarded by
 *    a per-plan mutex) and may be shared by threads.  Concurrent lc_execute /
 *    lc_execute_host calls on one plan need distinct workspaces (and, for
 *    lc_execute_host, distinct staging buffers); a NULL workspace or staging
 *    means the plan-owned one, which is safe only for calls serialised on one
 *    stream.
 */
#ifndef LEGCHEB_H_
#define LEGCHEB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lc_plan lc_plan; /* opaque; immutable after create */

typedef enum { LC_LEG2CHEB = 0, LC_CHEB2LEG = 1 } lc_direction;

/* Batch layouts of in/out.  VEC: in[v*ld + j] (vector-contiguous, default);
 * BATCH: in[j*ld + v] (batch-contiguous, e.g. the second pass of a 2-D
 * tensor-product transform). */
typedef enum { LC_VEC_CONTIGUOUS = 0, LC_BATCH_CONTIGUOUS = 1 } lc_layout;

typedef enum {
  LC_OK = 0,
  LC_ERR_INVALID_ARG = 1,
  LC_ERR_UNSUPPORTED_DEVICE = 2,
  LC_ERR_OUT_OF_MEMORY = 3,
  LC_ERR_CUDA = 4,
  LC_ERR_ALIASING = 5,
  LC_ERR_INTERNAL = 6
} lc_status;

typedef struct {
  int64_t s_hat;    /* preferred smallest-submatrix half size s_hat (eq:numlevels); 0 -> 40 */
  int32_t M;        /* Chebyshev modes per axis; only 18 is supported; 0 -> 18 */
  int32_t layout;   /* lc_layout of in/out */
  int64_t ld_in;    /* leading dimension of in  (elements); 0 -> n (VEC) or batch (BATCH) */
  int64_t ld_out;   /* leading dimension of out (elements); 0 -> n (VEC) or batch (BATCH) */
  int32_t device;   /* CUDA device ordinal; -1 -> current device */
  int32_t vt;       /* vectors per CTA tile; 0 -> automatic */
  int32_t subtree;  /* subtree depth k of the execution kernels; 0 -> automatic */
  int32_t stage_blocks; /* FMM blocks (3 A_hat each) per TMA bulk-copy stage; 0 -> automatic */
  int32_t stages;   /* bulk-copy ring depth; 0 -> automatic */
  int32_t up_subtree; /* subtree depth of the upward (leaf projection + M2M) kernel; 0 -> automatic */
  int32_t engine;   /* 0 -> automatic; 1 -> level-pipelined kernels (up / streaming / down);
                       2 -> per-tile streaming kernel (one CTA per 8-vector tile, whole Alg. 4 on chip;
                       needs L >= 1 and s <= 40; automatic choice from about one tile per SM, or a third of that for n <= 2048);
                       3 -> up kernel of 8-vector tiles + the per-tile pass over leaf ranges (needs L >= 1, s <= 40;
                       automatic for L >= 7 with >= 8 vectors and >= 1.6e6 coefficients in all, and fewer tiles than SMs) */
  int32_t part_index; /* partitioned plan (NEXT-2, one long transform over several GPUs): this plan computes */
  int32_t part_count; /* output rows [row_lo, row_hi) of part part_index of part_count (lc_partition); 0/1 -> all.
                         The input is the whole vector (the upward pass -- leaf projection and M2M, PAPER.md:363-379
                         -- runs whole on every part); the M2L of the rows of the part and of their ancestor
                         segments, the band of its rows and the downward pass of its subtrees run here
                         (eq:fgamma, eq:flevels, eq:zlevels).  Rows outside the part are not
                         written.  Engine 1 only. */
  int32_t part_up;    /* partitioned plans: 1 -> the upward pass is partitioned too: each part projects and
                         merges only its own subtrees; run with lc_execute_part: phase 0 (upward pass), then the
                         caller exchanges the subtree roots of all parts and the w halo (2 segments per fine
                         level) of the next part in the workspace (lc_plan_kernel_info: kup, grup, part_lo,
                         part_hi), then phase 1 (coarse levels, M2L, band, downward pass).  0 -> replicated.
                         part_up needs batch = 1 (INVALID_ARG otherwise). */
  int64_t out_block;  /* > 0: column-blocked output, out[(i / B) * batch * B + v * B + i % B] with B = out_block:
                         the blocks of B output coefficients of all vectors are contiguous, i.e. the first pass of
                         a 2-D transform over G ranks writes its rows already packed by destination rank
                         ([G][rows][n/G], the send buffer of the all-to-all) when B = n / G.  VEC input layout,
                         engines 2/3 (chosen automatically; INVALID_ARG where neither applies), ld_out ignored. */
} lc_plan_opts;

/* Geometry and algorithmic work of a plan (per vector unless stated). */
typedef struct {
  int64_t n;          /* user length */
  int64_t N;          /* padded length s*2^(L+2)                 (eq:Ntot) */
  int64_t L;          /* number of levels                          (eq:numlevels) */
  int64_t s;          /* smallest half size h_{L-1} */
  int64_t M;          /* modes per axis (18) */
  int64_t batch;      /* vectors per execute */
  int64_t nc;         /* number of A_hat matrices N_c = 3(N/2s-L-2) (eq:total_blocks_and_mats) */
  int64_t direction;  /* lc_direction */
  int64_t band_nnz;   /* nonzeros of A in the direct band (exact count) */
  size_t plan_bytes;  /* device bytes owned by the plan (A_hat arena, tables) */
  size_t workspace_bytes; /* bytes lc_execute needs as workspace */
  double flops_alg;   /* algorithmic flops per vector: 2 nnz_band + 16 b_{L-1} s M + 4 N_c M^2 + 8(M^2+2M)(2^L-L-1) + n */
  double bytes_alg;   /* algorithmic HBM bytes per execute: 16 n batch + 8 M^2 N_c + 8 N */
  int32_t vt, subtree, stage_blocks, stages; /* chosen kernel configuration */
  int32_t kernels_per_execute;               /* kernel launches per lc_execute */
  double plan_device_ms;                     /* device time of the planning kernels at create (CUDA events) */
  int64_t row_lo, row_hi;                    /* output rows this plan computes ([0, n) unless partitioned) */
} lc_plan_desc;

/* Host-only: output rows [*row_lo, *row_hi) of part part_index of part_count for length n (s_hat <= 0
 * -> 40).  Parts are contiguous runs of whole groups of 64 leaf segments of 2s rows,
 * balanced over the segments that hold outputs; a part may be empty.  Errors: INVALID_ARG. */
lc_status lc_partition(int64_t n, int64_t s_hat, int32_t part_index, int32_t part_count, int64_t* row_lo,
                       int64_t* row_hi);

/* Host-only geometry (no GPU needed): fills n, N, L, s, M, nc, band_nnz,
 * flops_alg (batch = 1), bytes_alg (batch = 1).  s_hat <= 0 -> 40.
 * Errors: LC_ERR_INVALID_ARG if n < 1 or out == NULL. */
lc_status lc_geometry(int64_t n, int64_t s_hat, lc_plan_desc* out);

/* Create a plan: precomputes on the device lambda (and for C2L the band
 * tables), the level/block hierarchy, B(0) (App. A3, exact), the
 * finest-level Vandermonde T(sigma) (eq:Xs) and the N_c A_hat matrices
 * (eq:aklmore, sampled at Chebyshev-Gauss points, 2-D DCT-II), level-major
 * in (level, block, r) order (eq:cfrompq).  batch >= 1 vectors per execute.
 * opts may be NULL (defaults).  Allocates a plan-owned workspace.
 * Errors: INVALID_ARG (n < 1, batch < 1, M != 18, bad layout/ld),
 * UNSUPPORTED_DEVICE (not compute capability 10.x), OUT_OF_MEMORY, CUDA. */
lc_status lc_plan_create(lc_plan** out, int64_t n, lc_direction dir, int64_t batch, const lc_plan_opts* opts);

lc_status lc_plan_describe(const lc_plan* p, lc_plan_desc* out);

/* Bytes of workspace lc_execute needs. */
size_t lc_workspace_bytes(const lc_plan* p);

/* Zero-initialise a caller-owned workspace before its first use with any
 * plan (enqueued on stream).  Plan-owned workspaces are initialised at create. */
lc_status lc_workspace_init(const lc_plan* p, void* workspace, void* stream);

/* Execute the transform of `batch` vectors: out = T(in), enqueue-only on
 * `stream` (a cudaStream_t; NULL = legacy default stream).
 *   T = C^{-1} A (leg2cheb) or A^{-1} C (cheb2leg) of PAPER.md:29-32 (eq:directmv),
 *   evaluated by Alg. 4 (alg:fastercomplete) with the plan's
 *   hierarchy; the result equals the plain definition within the FMM's
 *   accuracy (relative max norm <= 1e-12 for n <= 1e6, PAPER.md:527 eq:Einf).
 *   in:  device, batch vectors of n doubles in the plan's layout; unmodified.
 *   out: device, same shape; must not overlap in (LC_ERR_ALIASING).
 *   workspace: device, >= lc_workspace_bytes(p), zero-initialised once, or
 *              NULL for the plan-owned workspace.
 * Outputs are the first n entries of the transform of the zero-padded input. */
lc_status lc_execute(const lc_plan* p, const double* in, double* out, void* workspace, void* stream);

/* Two-phase execution of a plan created with opts.part_up = 1 (NEXT-2): phase 0 enqueues the upward
 * pass of the part's subtrees, phase 1 the coarse levels of step 2, the M2L, band and downward passes.
 * Between them the caller makes w of the workspace complete for this part: all subtree roots (level
 * grup) and, on every level g >= grup, the 2 segments following the part (from the next part).
 * workspace must be caller-owned (its layout: DESIGN.md section 5).  Errors: INVALID_ARG (not a
 * part_up plan, bad phase, NULL workspace), CUDA.  lc_execute rejects part_up plans. */
lc_status lc_execute_part(const lc_plan* p, int32_t phase, const double* in, double* out, void* workspace,
                          void* stream);

/* As lc_execute, and records ev[0] before the first kernel, ev[i] after
 * kernel i (i = 1..kernels_per_execute).  ev are cudaEvent_t handles; nev
 * must be >= kernels_per_execute + 1.  Used by bench.py for per-kernel times. */
lc_status lc_execute_timed(const lc_plan* p, const double* in, double* out, void* workspace, void* stream,
                           void* const* ev, int32_t nev);

/* Bytes of the device staging buffer lc_execute_host needs (input and
 * output staging, each rounded up to 256 bytes). */
size_t lc_host_stage_bytes(const lc_plan* p);

/* End-to-end call with HOST buffers (the transform of lc_execute): copies
 * h_in (batch vectors, layout and leading dimensions of the plan) to device
 * staging, executes, copies the result to h_out, all enqueued on stream (no
 * host sync; h_out is valid after the stream is synchronised).
 *   d_stage: device, >= lc_host_stage_bytes(p), caller-owned; or NULL for the
 *            plan-owned staging (allocated once on first use, under the plan's
 *            mutex; calls with NULL must be serialised on one stream).
 *   workspace: as for lc_execute (NULL = plan-owned).
 * Host buffers should be page-locked for asynchronous copies (pageable ones
 * make the copies synchronous).  Errors: INVALID_ARG, OUT_OF_MEMORY (staging),
 * CUDA. */
lc_status lc_execute_host(const lc_plan* p, const double* h_in, double* h_out, void* d_stage, void* workspace,
                          void* stream);

/* Bytes of the device staging lc_execute_host_chain needs for plans[0..nplans):
 * two ping-pong halves, each the largest input or output extent of the plans
 * (rounded up to 256 bytes).  0 if plans is NULL, nplans < 1 or a plan is NULL. */
size_t lc_host_chain_stage_bytes(const lc_plan* const* plans, int nplans);

/* A chain of transforms on HOST data with one copy each way: h_in (the input
 * of plans[0]) is copied to device staging, plans[0], ..., plans[nplans-1] are
 * executed one after another on the device (the output array of plan k, as
 * that plan lays it out, is the input array of plan k+1), and the output of
 * the last plan is copied to h_out; all enqueued on stream, no host sync.
 * Examples: a round trip (leg2cheb then cheb2leg of the same n and batch), or
 * the two passes of a 2-D tensor-product transform (a vector-layout plan over
 * the rows, then a batch-layout plan over the columns of the same array).
 * Applies Alg. 4 per plan, as lc_execute does.
 *   plans: nplans >= 1 plans of one device, none with part_up; the output
 *          extent of plan k must cover the input extent of plan k+1.
 *   d_stage: device, >= lc_host_chain_stage_bytes(plans, nplans), caller-owned
 *            (required).
 *   workspaces: NULL (every plan's own workspace; calls must then be
 *            serialised on one stream) or nplans workspaces, one per plan.
 * Host buffers should be page-locked (lc_host_alloc).  Errors: INVALID_ARG,
 * ALIASING, CUDA. */
lc_status lc_execute_host_chain(const lc_plan* const* plans, int nplans, const double* h_in, double* h_out,
                                void* d_stage, void* const* workspaces, void* stream);

/* Page-locked host memory for lc_execute_host's buffers: an anonymous mapping
 * aligned to 2 MiB, advised for transparent huge pages, touched (zeroed) and
 * registered with cudaHostRegister.  Huge pages keep the DMA engines' address
 * translations few: measured on this pool's B200 boxes, 8-16 MiB host-to-device
 * copies run at 54-55 GB/s from such buffers against 12-15 GB/s from
 * cudaHostAlloc memory (tools/h2d_sizes.py).  Where huge pages are not
 * available the same mapping is registered with 4 KiB pages.
 *   bytes: > 0.  *ptr receives the buffer (16-byte aligned, zero-filled).
 * The caller owns the buffer and releases it with lc_host_free (not free or
 * cudaFreeHost).  Errors: INVALID_ARG (bytes == 0, ptr NULL), OUT_OF_MEMORY
 * (mapping failed), CUDA (registration failed; nothing is leaked). */
lc_status lc_host_alloc(size_t bytes, void** ptr);

/* Unregister and unmap a buffer from lc_host_alloc.  The caller makes sure no
 * enqueued copy still uses it (e.g. synchronises the streams that do).
 * Errors: INVALID_ARG (not a live lc_host_alloc buffer), CUDA. */
lc_status lc_host_free(void* ptr);

/* Copy plan data to host memory (synchronous; test/diagnostic use).
 * what: 0 band table B (length N: lambda_m for L2C, rho_m for C2L),
 *       1 band table A (length 2s: lambda_k for L2C, kappa_k for C2L),
 *       2 A_hat arena (nc*M*M, row-major per matrix, level-major order),
 *       3 B(0) (M*M row-major), 4 T(sigma) (2*s*M, [sigma][m][k]).
 * count = number of doubles host_out can hold; returns INVALID_ARG if short. */
lc_status lc_plan_export(const lc_plan* p, int32_t what, double* host_out, int64_t count);

/* Kernel configuration chosen for the plan (diagnostic; host only, no device work).
 * out[0..] = stream_grid, smem_stream, smem_up, kup (up-kernel subtree depth), grup,
 * kb (band/down unit depth), cb (blocks per A_hat stage), nst (stages), vt, stream CTAs per
 * SM, m2l_units, band_units, up_grid (CTAs), kd (down-kernel subtree depth), smem_down, engine (1, 2 or 3),
 * tile_grid and smem_tile (per-tile kernel, engine 2; range kernel, engine 3), ranges and range_len
 * (engine 3), up_ksub, part_lo, part_hi, part_up.  count = capacity of out; returns the number of
 * values written through *written (may be NULL).  Errors: INVALID_ARG on NULL p or out. */
lc_status lc_plan_kernel_info(const lc_plan* p, int64_t* out, int32_t count, int32_t* written);

/* Frees the plan's device arrays, its own workspace and staging.  The frees
 * are stream-ordered after the last lc_execute / lc_execute_host of the plan
 * on every stream it was used on (the plan records one event per stream), and
 * the call returns when that work is done; unrelated streams are not waited
 * for (beyond 64 distinct streams it falls back to a device synchronisation).
 * Executions captured into CUDA graphs are not tracked: the caller must
 * finish such graph launches first.  Caller-owned workspaces are the caller's.
 * Errors: INVALID_ARG on NULL p. */
lc_status lc_plan_destroy(lc_plan* p);

const char* lc_status_string(lc_status s);

/* Version string of the library. */
const char* lc_version(void);

/* Name and description of the last CUDA error seen by this thread inside the
 * library (for messages accompanying LC_ERR_CUDA / LC_ERR_OUT_OF_MEMORY). */
const char* lc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* LEGCHEB_H_ */
