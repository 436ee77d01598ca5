// lc_plan.cu -- planning stage on the B200: lambda tables, A_hat arena (device
// kernels), exact B(0) and Vandermonde T(sigma) (host, tiny), plan lifetime,
// host-only geometry, plan export.
//
// Paper references (PAPER.md = arXiv 2411.00033 LaTeX source):
//   Lambda(z) by the tau series, eq:tau, with an upward
//     integer shift below z = 20 (reading R5);
//   lambda vector: every 8th value from eq:tau, the other 7 from the
//     recurrence eq:Lambdaint;
//   A_hat(g,b,r): kernel sampled on the Chebyshev-Gauss grid of the
//     submatrix and 2-D DCT-II, eq:aklmore, with corners
//     eq:globalij and the affine map eq:Xfromx;
//     L2C kernel A(x,y) = Lambda((y-x)/2) Lambda((y+x)/2),
//     C2L kernel L(x,y) eq:Lxymod;
//   B(0): T_n((Y-1)/2) = sum_k b_nk T_k(Y), eq:Tky, built
//     exactly (dyadic rationals, App. A3);
//   T(sigma)[m][k] = T_k(-1 + (2m+sigma)/s), eq:Xs.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <chrono>
#include <mutex>
#include <unordered_map>
#include <utility>
#include <vector>

#include <sys/mman.h>

#include "lc_internal.h"

// Host-side synchronisation state of a plan: a mutex for the lazily allocated lc_execute_host
// staging and the last-execute event of every stream the plan was executed on, so that
// lc_plan_destroy waits for the plan's own work only (never for the whole device).
struct lc_plan_sync {
  std::mutex mu;
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> seen;
  bool overflow = false;  // more than kMaxStreams streams: destroy falls back to a device synchronisation
};
static constexpr size_t kMaxStreams = 64;

namespace lc {

// ---------------------------------------------------------------- device Lambda
// Lambda(z) = tau(z + 1/4) / sqrt(z + 1/4), tau(x) = 1 - 1/(2^6 x^2) + 21/(2^13 x^4)
// - 671/(2^19 x^6) + 180323/(2^27 x^8)  (eq:tau; all five coefficients are exact
// dyadics).  Below z = 20 the argument is shifted up by whole steps using
// Lambda(z) = Lambda(z+1) (z+1)/(z+1/2)  (eq:Lambdaint generalised).
__device__ __forceinline__ double Lambda_dev(double z) {
  double prod = 1.0;
  while (z < 20.0) {
    prod *= (z + 1.0) / (z + 0.5);
    z += 1.0;
  }
  const double x = z + 0.25;
  const double y = 1.0 / (x * x);
  const double tau =
      1.0 + y * (-1.0 / 64.0 + y * (21.0 / 8192.0 + y * (-671.0 / 524288.0 + y * (180323.0 / 134217728.0))));
  return prod * tau / sqrt(x);
}

constexpr double kSqrtPi = 1.7724538509055160272981674833411452;

// lambda_m for m in [8t, 8t+8): anchor from eq:tau, then 7 recurrence steps.
// dir 0 (L2C): tabB[m] = lambda_m.  dir 1 (C2L): tabB[m] = rho_m = 1/(2m(2m+1) lambda_m), rho_0 = 0
// (the band factorisation of DESIGN.md "C2L band").
__global__ void plan_lambda_kernel(double* tabB, int64_t N, int dir) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t m0 = t * 8;
  if (m0 >= N) return;
  double lam;
  int64_t m = m0;
  if (m0 < 24) {  // small arguments: recurrence from Lambda(0) = sqrt(pi)
    lam = kSqrtPi;
    for (int64_t i = 1; i <= m0; ++i) lam *= (double(i) - 0.5) / double(i);
  } else {
    lam = Lambda_dev(double(m0));
  }
  for (int q = 0; q < 8 && m < N; ++q, ++m) {
    if (q > 0) lam *= (double(m) - 0.5) / double(m);
    if (dir == 0) {
      tabB[m] = lam;
    } else {
      const double dm = double(m);
      tabB[m] = (m == 0) ? 0.0 : 1.0 / ((2.0 * dm) * (2.0 * dm + 1.0) * lam);
    }
  }
}

__global__ void plan_taba_kernel(double* tabA, int64_t n2s, int dir) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double lam = kSqrtPi;
  for (int64_t k = 0; k < n2s; ++k) {
    if (k > 0) lam *= (double(k) - 0.5) / double(k);
    tabA[k] = dir == 0 ? lam : lam / (1.0 - 2.0 * double(k));
  }
}

// Lambda with the number of eq:tau terms chosen from the smallest argument zmin the caller will pass
// (5 terms to machine precision for z > 19.88, 4 for z > 40, 3 for z > 134, 2 for
// z > 1844).  Arguments below 20 are shifted up as in Lambda_dev (5 terms then).
__device__ __forceinline__ int tau_terms(double zmin) {
  return zmin > 1844.0 ? 2 : (zmin > 134.0 ? 3 : (zmin > 40.0 ? 4 : 5));
}
__device__ __forceinline__ double Lambda_terms(double z, int K) {
  if (K == 5) return Lambda_dev(z);
  const double x = z + 0.25;
  const double y = 1.0 / (x * x);
  double tau;
  if (K == 2) tau = 1.0 + y * (-1.0 / 64.0);
  else if (K == 3) tau = 1.0 + y * (-1.0 / 64.0 + y * (21.0 / 8192.0));
  else tau = 1.0 + y * (-1.0 / 64.0 + y * (21.0 / 8192.0 + y * (-671.0 / 524288.0)));
  return tau / sqrt(x);
}

// Chebyshev-Gauss nodes and DCT-II table in constant memory (host-filled in long double):
// c_cos[k][m] = cos(k (m + 1/2) pi / M), X_m = c_cos[1][m] (decreasing; X_{M-1-m} = -X_m);
// c_tri[u] = (m, n), m <= n, the (M^2 + M)/2 = 171 upper-triangle index pairs.
__constant__ double c_cos[kMM];
__constant__ unsigned char c_tri[2 * (kMM + kM) / 2];
constexpr int kTri = (kMM + kM) / 2;  // 171

// Lambda^- of every level (sec:fastinit): Lambda((y_n - x_m)/2) depends on the block only
// through the corner distance j0 - i0 = d h, d = 4 (r = 0, 2) or 6 (r = 1), so two M x M matrices per
// level serve every submatrix of the level; each is persymmetric ((m,n) ~ (M-1-n, M-1-m)), so only
// 171 entries are evaluated.  Out: Lm[(g*2 + t)*M*M + m*M + n], t = 0 for d = 4, 1 for d = 6.
__global__ void plan_lminus_kernel(double* Lm, int L, int64_t s) {
  const int g = blockIdx.x >> 1, t = blockIdx.x & 1;
  const int64_t h = s << (L - g - 1);
  const double dh = double((t ? 6 : 4) * h);
  double* out = Lm + int64_t(blockIdx.x) * kMM;
  for (int o = threadIdx.x; o < kMM; o += blockDim.x) {
    const int m = o / kM, n = o % kM;
    if (m + n > kM - 1) continue;  // orbit representatives of (m, n) -> (M-1-n, M-1-m): 171 of 324
    const double hx = double(h) * (c_cos[kM + m] + 1.0), hy = double(h) * (c_cos[kM + n] + 1.0);
    const double v = Lambda_dev(0.5 * dh + 0.5 * (hy - hx));  // (y_n - x_m)/2 (eq:Xfromx, eq:globalij)
    out[m * kM + n] = v;
    out[(kM - 1 - n) * kM + (kM - 1 - m)] = v;
  }
}

// A_hat(g, b, r) for the arena indices [q0, q0 + count), one warp per matrix (grid-stride):
//   G(m, n) = kernel at (x_m, y_n) (eq:aklmore), x = i0 + h(X_m + 1), y = j0 + h(X_n + 1) (eq:Xfromx),
//     L2C: A = Lambda^- o Lambda^+, C2L: L(x, y) of eq:Lxymod = prefactor * Lambda^- / Lambda^+;
//   Lambda^+ = Lambda((x_m + y_n)/2) is symmetric in (m, n): 171 evaluations per block with the eq:tau
//     term count of the block's smallest argument (i0 + j0)/2;
//   A_hat = 4/(c_k c_l M^2) C G C^T (2-D DCT-II), each 1-D pass folded by the even/odd symmetry of the
//     DCT matrix, C[k][M-1-m] = (-1)^k C[k][m] (one radix-2 stage of the mixed-radix DCT):
//     M/2 = 9 products per output instead of 18.
constexpr int kAhatWarps = 8;
__global__ void __launch_bounds__(32 * kAhatWarps) plan_ahat_kernel(double* A, const double* __restrict__ Lm,
                                                                  int64_t q0, int64_t count, int L, int64_t s,
                                                                  int dir) {
  __shared__ double Gs[kAhatWarps][kMM];
  __shared__ double Hs[kAhatWarps][kMM];
  __shared__ double Cs[kMM];             // the DCT table, from constant memory once per CTA: lanes read
  __shared__ unsigned char Ts[2 * kTri]; // different entries, which the constant cache would serialise
  for (int i = threadIdx.x; i < kMM; i += blockDim.x) Cs[i] = c_cos[i];
  for (int i = threadIdx.x; i < 2 * kTri; i += blockDim.x) Ts[i] = c_tri[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  double* G = Gs[wq];
  double* H = Hs[wq];
  const int64_t nwarps = int64_t(gridDim.x) * kAhatWarps;
  for (int64_t qi = int64_t(blockIdx.x) * kAhatWarps + wq; qi < count; qi += nwarps) {
    const int64_t q = q0 + qi;
    int g = 0;
    while (g + 1 < L && ahat_level_offset(g + 1) <= q) ++g;
    const int64_t loc = q - ahat_level_offset(g);
    const int64_t b = loc / 3;
    const int r = int(loc % 3);
    const int p = (r == 2) ? 1 : 0;  // eq:cfrompq: r = 0,1,2 <-> (p,q) = (0,0),(0,1),(1,1)
    const int qq = (r >= 1) ? 1 : 0;
    const int64_t h = s << (L - g - 1);
    const int64_t i0 = 2 * h * (2 * b + p);  // eq:globalij
    const int64_t j0 = 2 * h * (2 * b + qq + 2);
    const double* Lmg = Lm + int64_t(2 * g + (r == 1 ? 1 : 0)) * kMM;
    const int K = tau_terms(0.5 * double(i0 + j0));
    const double xy0 = 0.5 * double(i0 + j0);
    for (int u = lane; u < kTri; u += 32) {
      const int m = Ts[2 * u], n = Ts[2 * u + 1];
      const double hx = double(h) * (Cs[kM + m] + 1.0), hy = double(h) * (Cs[kM + n] + 1.0);
      const double lp = Lambda_terms(xy0 + 0.5 * (hx + hy), K);  // symmetric: hx + hy == hy + hx
      if (dir == 0) {
        G[m * kM + n] = __ldg(Lmg + m * kM + n) * lp;
        G[n * kM + m] = __ldg(Lmg + n * kM + m) * lp;
      } else {
        // L(x,y) = 2(x+1/2) y / ((x+y)(x+y+1)(x-y+1)) Lambda((y-x)/2)/Lambda((x+y)/2)   (eq:Lxymod)
        const double x = double(i0) + hx, y = double(j0) + hy, xs = 2.0 * (xy0 + 0.5 * (hx + hy));
        const double ymx = 0.5 * double(j0 - i0) + 0.5 * (hy - hx);
        G[m * kM + n] = (2.0 * (x + 0.5) * y) / (xs * (xs + 1.0) * (1.0 - 2.0 * ymx)) * (__ldg(Lmg + m * kM + n) / lp);
        if (m != n) {
          const double x2 = double(i0) + hy, y2 = double(j0) + hx;
          const double ymx2 = 0.5 * double(j0 - i0) + 0.5 * (hx - hy);
          G[n * kM + m] = (2.0 * (x2 + 0.5) * y2) / (xs * (xs + 1.0) * (1.0 - 2.0 * ymx2)) *
                          (__ldg(Lmg + n * kM + m) / lp);
        }
      }
    }
    __syncwarp();
    // H = C G along x (rows m), folded: H[k][n] = sum_{m < 9} C[k][m] (G[m][n] +- G[M-1-m][n])
    for (int o = lane; o < kMM; o += 32) {
      const int k = o / kM, n = o % kM;
      const double sg = (k & 1) ? -1.0 : 1.0;
      double acc = 0.0;
#pragma unroll
      for (int m = 0; m < kM / 2; ++m) acc = fma(Cs[k * kM + m], G[m * kM + n] + sg * G[(kM - 1 - m) * kM + n], acc);
      H[o] = acc;
    }
    __syncwarp();
    // A_hat[k][l] = 4/(c_k c_l M^2) sum_{n < 9} C[l][n] (H[k][n] +- H[k][M-1-n])   (eq:aklmore)
    double* Aq = A + q * kMM;
    for (int o = lane; o < kMM; o += 32) {
      const int k = o / kM, l = o % kM;
      const double sg = (l & 1) ? -1.0 : 1.0;
      double acc = 0.0;
#pragma unroll
      for (int n = 0; n < kM / 2; ++n) acc = fma(Cs[l * kM + n], H[k * kM + n] + sg * H[k * kM + kM - 1 - n], acc);
      const double ck = k == 0 ? 2.0 : 1.0, cl = l == 0 ? 2.0 : 1.0;
      Aq[o] = acc * (4.0 / (ck * cl * double(kM) * double(kM)));
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- host pieces
// B(0) exactly: P_n(Y) = T_n((Y-1)/2) satisfies P_{n+1} = (Y-1) P_n - P_{n-1};
// in the Chebyshev basis Y T_0 = T_1, Y T_k = (T_{k+1} + T_{k-1})/2.  Every
// operation is a halving/sum of dyadic rationals far inside 53 bits, so the
// doubles are exact (App. A3: "represented exactly in double precision").
static void build_B0(double* B) {
  std::memset(B, 0, sizeof(double) * kMM);
  B[0] = 1.0;
  B[1 * kM + 0] = -0.5;
  B[1 * kM + 1] = 0.5;
  for (int n = 1; n + 1 < kM; ++n) {
    double y[kM] = {0};
    for (int k = 0; k <= n; ++k) {
      const double c = B[n * kM + k];
      if (k == 0) {
        y[1] += c;
      } else {
        y[k + 1] += 0.5 * c;
        y[k - 1] += 0.5 * c;
      }
    }
    for (int k = 0; k < kM; ++k) B[(n + 1) * kM + k] = y[k] - B[n * kM + k] - B[(n - 1) * kM + k];
  }
}

// T(sigma)[m][k] = T_k(X), X = -1 + (2m+sigma)/s (eq:Xs), three-term recurrence in long double.
static void build_T(int64_t s, std::vector<double>& T, std::vector<double>& Tt) {
  T.assign(size_t(2 * s * kM), 0.0);
  Tt.assign(size_t(2 * s * kM), 0.0);
  for (int sg = 0; sg < 2; ++sg)
    for (int64_t m = 0; m < s; ++m) {
      const long double X = -1.0L + (long double)(2 * m + sg) / (long double)s;
      long double t0 = 1.0L, t1 = X;
      for (int k = 0; k < kM; ++k) {
        long double v;
        if (k == 0) v = t0;
        else if (k == 1) v = t1;
        else {
          v = 2.0L * X * t1 - t0;
          t0 = t1;
          t1 = v;
        }
        T[size_t((sg * s + m) * kM + k)] = double(v);
        Tt[size_t((sg * kM + k) * s + m)] = double(v);
      }
    }
}

int64_t band_nnz(int64_t N, int64_t s) {
  // nonzeros (i, i+2k) of A with i <= j < j_end(i) = min(N, 2s(floor(i/2s)+2)).  Every segment u whose
  // window ends inside the matrix (2s(u+2) <= N) has the same count, so only one of them and the last
  // (at most two) segments are summed row by row: O(s) instead of O(N) on the host.
  const int64_t seg = 2 * s;
  auto seg_sum = [&](int64_t u) {
    int64_t tot = 0;
    const int64_t je = std::min<int64_t>(N, seg * (u + 2));
    for (int64_t r = 0; r < seg && u * seg + r < N; ++r) tot += (je - (u * seg + r) + 1) / 2;
    return tot;
  };
  const int64_t nu = (N + seg - 1) / seg;
  const int64_t nfull = std::max<int64_t>(0, N / seg - 1);
  int64_t tot = nfull > 0 ? nfull * seg_sum(0) : 0;
  for (int64_t u = nfull; u < nu; ++u) tot += seg_sum(u);
  return tot;
}

// leaf segments [lo, hi) of part `pidx` of `pcnt`: whole groups of 2^part_align_log2(L) leaves, balanced
// over the groups that hold outputs (rows < n)
static void part_leaves(int64_t n, const Geometry& G, int pidx, int pcnt, int64_t* lo, int64_t* hi) {
  const int64_t nls = G.L > 0 ? (int64_t(2) << G.L) : 2;
  const int64_t align = int64_t(1) << part_align_log2(G.L);
  const int64_t nreal = (n + 2 * G.s - 1) / (2 * G.s);
  const int64_t nch = (nreal + align - 1) / align;
  *lo = std::min(nls, (int64_t(pidx) * nch / pcnt) * align);
  *hi = std::min(nls, (int64_t(pidx + 1) * nch / pcnt) * align);
  // the groups past the last output row (zero padding) belong to no part: their w is 0
  // and their rows are not returned, so no part projects, merges or evaluates them
}

static void fill_work(lc_plan_desc* d, int64_t batch) {
  const double M = kM;
  const int64_t L = d->L;
  const double b_last = L > 0 ? double((int64_t(2) << (L - 1)) - 1) : 0.0;  // b_{L-1}
  const double m2m = L > 0 ? double((int64_t(1) << L) - L - 1) : 0.0;
  d->flops_alg = 2.0 * double(d->band_nnz) + 16.0 * b_last * double(d->s) * M + 4.0 * double(d->nc) * M * M +
                 8.0 * (M * M + 2 * M) * m2m + double(d->n);
  d->bytes_alg = 16.0 * double(d->n) * double(batch) + 8.0 * M * M * double(d->nc) + 8.0 * double(d->N);
}

}  // namespace lc

using namespace lc;

namespace lc {
static thread_local char g_last_error[256] = "no error";
lc_status record_cuda_error(cudaError_t e) {
  std::snprintf(g_last_error, sizeof(g_last_error), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? LC_ERR_OUT_OF_MEMORY : LC_ERR_CUDA;
}
}  // namespace lc

#define LC_CUDA_TRY(expr)                                   \
  do {                                                      \
    cudaError_t e_ = (expr);                                \
    if (e_ != cudaSuccess) return record_cuda_error(e_);    \
  } while (0)

extern "C" {

const char* lc_version(void) { return "legcheb-b200 0.1 (sm_100a)"; }

const char* lc_last_error(void) { return lc::g_last_error; }

const char* lc_status_string(lc_status s) {
  switch (s) {
    case LC_OK: return "ok";
    case LC_ERR_INVALID_ARG: return "invalid argument";
    case LC_ERR_UNSUPPORTED_DEVICE: return "unsupported device (needs compute capability 10.x, sm_100a)";
    case LC_ERR_OUT_OF_MEMORY: return "out of device memory";
    case LC_ERR_CUDA: return "CUDA error";
    case LC_ERR_ALIASING: return "input and output overlap";
    case LC_ERR_INTERNAL: return "internal error";
  }
  return "unknown status";
}

lc_status lc_partition(int64_t n, int64_t s_hat, int32_t part_index, int32_t part_count, int64_t* row_lo,
                       int64_t* row_hi) {
  if (n < 1 || !row_lo || !row_hi || part_count < 1 || part_index < 0 || part_index >= part_count)
    return LC_ERR_INVALID_ARG;
  if (s_hat <= 0) s_hat = kSHatDefault;
  if (s_hat < 2 || s_hat > 64) return LC_ERR_INVALID_ARG;
  const Geometry G = geometry(n, s_hat);
  int64_t llo = 0, lhi = 0;
  part_leaves(n, G, part_index, part_count, &llo, &lhi);
  *row_lo = std::min(n, llo * 2 * G.s);
  *row_hi = std::min(n, lhi * 2 * G.s);
  return LC_OK;
}

lc_status lc_geometry(int64_t n, int64_t s_hat, lc_plan_desc* out) {
  if (n < 1 || out == nullptr) return LC_ERR_INVALID_ARG;
  if (s_hat <= 0) s_hat = kSHatDefault;
  if (s_hat < 2 || s_hat > 64) return LC_ERR_INVALID_ARG;
  std::memset(out, 0, sizeof(*out));
  const Geometry G = geometry(n, s_hat);
  out->n = n;
  out->N = G.N;
  out->L = G.L;
  out->s = G.s;
  out->M = kM;
  out->batch = 1;
  out->nc = G.nc;
  out->band_nnz = band_nnz(G.N, G.s);
  fill_work(out, 1);
  return LC_OK;
}

}  // extern "C"

namespace lc {
lc_status configure_kernels(lc_plan* p);  // lc_exec.cu
}

extern "C" lc_status lc_plan_create(lc_plan** out, int64_t n, lc_direction dir, int64_t batch,
                                    const lc_plan_opts* opts) {
  const auto t_create = std::chrono::steady_clock::now();
  if (out == nullptr || n < 1 || batch < 1) return LC_ERR_INVALID_ARG;
  *out = nullptr;
  if (dir != LC_LEG2CHEB && dir != LC_CHEB2LEG) return LC_ERR_INVALID_ARG;
  lc_plan_opts o{};
  if (opts) o = *opts;
  if (o.s_hat <= 0) o.s_hat = kSHatDefault;
  if (o.M <= 0) o.M = kM;
  if (o.M != kM || o.s_hat < 2 || o.s_hat > 64) return LC_ERR_INVALID_ARG;
  if (o.engine < 0 || o.engine > 3) return LC_ERR_INVALID_ARG;
  if (o.layout != LC_VEC_CONTIGUOUS && o.layout != LC_BATCH_CONTIGUOUS) return LC_ERR_INVALID_ARG;
  if (o.out_block < 0 || (o.out_block > 0 && (o.layout != LC_VEC_CONTIGUOUS || o.part_count > 1)))
    return LC_ERR_INVALID_ARG;
  const int64_t def_ld = o.layout == LC_VEC_CONTIGUOUS ? n : batch;
  if (o.ld_in == 0) o.ld_in = def_ld;
  if (o.ld_out == 0) o.ld_out = def_ld;
  if (o.ld_in < def_ld || o.ld_out < def_ld) return LC_ERR_INVALID_ARG;

  int dev = o.device;
  if (dev < 0) LC_CUDA_TRY(cudaGetDevice(&dev));
  // two attribute queries (microseconds) instead of cudaGetDeviceProperties (it fills the whole structure)
  int cc_major = 0, sm_count = 0;
  LC_CUDA_TRY(cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, dev));
  LC_CUDA_TRY(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev));
  if (cc_major != 10) return LC_ERR_UNSUPPORTED_DEVICE;
  int prev_dev = 0;
  LC_CUDA_TRY(cudaGetDevice(&prev_dev));
  LC_CUDA_TRY(cudaSetDevice(dev));

  // LC_PLAN_TRACE=1: host wall time of the stages of plan creation on stderr (tools/plan_wall.py)
  static const bool trace = std::getenv("LC_PLAN_TRACE") != nullptr;
  auto mark = [&](const char* what) {
    if (trace)
      std::fprintf(stderr, "lc_plan_create %-12s %8.3f ms\n", what,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_create).count());
  };
  mark("device");
  lc_plan* p = new lc_plan();
  std::memset(p, 0, sizeof(*p));
  const Geometry G = geometry(n, o.s_hat);
  p->n = n; p->N = G.N; p->L = G.L; p->s = G.s; p->M = kM; p->batch = batch; p->nc = G.nc;
  p->dir = int(dir); p->layout = o.layout; p->ld_in = o.ld_in; p->ld_out = o.ld_out;
  p->device = dev; p->sm_count = sm_count;
  p->vt = o.vt; p->k = o.subtree; p->bps = o.stage_blocks; p->nst = o.stages; p->kup = o.up_subtree;
  p->engine = o.engine;
  p->out_block = o.out_block;
  if (o.part_count > 1) {
    if (o.part_index < 0 || o.part_index >= o.part_count || G.L < 1 || (o.engine != 0 && o.engine != 1)) {
      delete p;
      cudaSetDevice(prev_dev);
      return LC_ERR_INVALID_ARG;
    }
    p->part_index = o.part_index;
    p->part_count = o.part_count;
    if (o.part_up && batch != 1) {  // the exchange layout (PartExchange) is that of one vector
      delete p;
      cudaSetDevice(prev_dev);
      return LC_ERR_INVALID_ARG;
    }
    p->part_up = (o.part_up && G.L >= 2) ? 1 : 0;
    part_leaves(n, G, o.part_index, o.part_count, &p->part_lo, &p->part_hi);
    p->row_lo = std::min(n, p->part_lo * 2 * G.s);
    p->row_hi = std::min(n, p->part_hi * 2 * G.s);
  } else {
    p->part_count = 1;
    p->row_lo = 0;
    p->row_hi = n;
  }

  auto fail = [&](lc_status st) {
    lc_plan_destroy(p);
    cudaSetDevice(prev_dev);
    return st;
  };
#define LC_PTRY(expr)                                                         \
  do {                                                                        \
    cudaError_t e_ = (expr);                                                  \
    if (e_ != cudaSuccess) return fail(record_cuda_error(e_));                \
  } while (0)

  const int64_t s = p->s;
  p->sync = new (std::nothrow) lc_plan_sync();
  if (!p->sync) return fail(LC_ERR_OUT_OF_MEMORY);
  // every device array of the plan is stream-ordered memory of `own`, so that destroy can free it
  // after the plan's own work without the device-wide synchronisation of cudaFree
  LC_PTRY(cudaStreamCreateWithFlags(&p->own, cudaStreamNonBlocking));
  cudaStream_t os = p->own;
  LC_PTRY(cudaMallocAsync(reinterpret_cast<void**>(&p->d_tabB), sizeof(double) * size_t(p->N), os));
  LC_PTRY(cudaMallocAsync(reinterpret_cast<void**>(&p->d_tabA), sizeof(double) * size_t(2 * s), os));
  LC_PTRY(cudaMallocAsync(reinterpret_cast<void**>(&p->d_T), sizeof(double) * size_t(2 * s * kM), os));
  LC_PTRY(cudaMallocAsync(reinterpret_cast<void**>(&p->d_Tt), sizeof(double) * size_t(2 * s * kM), os));
  LC_PTRY(cudaMallocAsync(reinterpret_cast<void**>(&p->d_B), sizeof(double) * kMM, os));
  if (p->nc > 0) LC_PTRY(cudaMallocAsync(reinterpret_cast<void**>(&p->d_A), sizeof(double) * size_t(p->nc) * kMM, os));
  p->plan_bytes = sizeof(double) * (size_t(p->N) + size_t(2 * s) + size_t(4 * s * kM) + kMM + size_t(p->nc) * kMM);

  mark("malloc");
  double B[kMM];
  build_B0(B);
  std::vector<double> T, Tt;
  build_T(s, T, Tt);
  double Cc[kMM];
  for (int k = 0; k < kM; ++k)
    for (int m = 0; m < kM; ++m)
      Cc[k * kM + m] = double(cosl((long double)k * ((long double)m + 0.5L) *
                                   3.141592653589793238462643383279502884L / (long double)kM));
  unsigned char tri[2 * kTri];
  for (int m = 0, u = 0; m < kM; ++m)
    for (int nn = m; nn < kM; ++nn, ++u) {
      tri[2 * u] = (unsigned char)m;
      tri[2 * u + 1] = (unsigned char)nn;
    }
  mark("host tables");
  double* d_Lm = nullptr;  // Lambda^- of every level: L x 2 x M x M
  if (p->L > 0) LC_PTRY(cudaMallocAsync(reinterpret_cast<void**>(&d_Lm), sizeof(double) * size_t(2 * p->L) * kMM, os));
  // pageable sources: these copies return once the host data has been staged
  LC_PTRY(cudaMemcpyAsync(p->d_B, B, sizeof(B), cudaMemcpyHostToDevice, os));
  LC_PTRY(cudaMemcpyAsync(p->d_T, T.data(), sizeof(double) * T.size(), cudaMemcpyHostToDevice, os));
  LC_PTRY(cudaMemcpyAsync(p->d_Tt, Tt.data(), sizeof(double) * Tt.size(), cudaMemcpyHostToDevice, os));
  {
    static std::mutex const_mu;  // the constant tables are per device; writing the same values is idempotent
    std::lock_guard<std::mutex> lk(const_mu);
    LC_PTRY(cudaMemcpyToSymbolAsync(c_cos, Cc, sizeof(Cc), 0, cudaMemcpyHostToDevice, os));
    LC_PTRY(cudaMemcpyToSymbolAsync(c_tri, tri, sizeof(tri), 0, cudaMemcpyHostToDevice, os));
    LC_PTRY(cudaStreamSynchronize(os));
  }

  mark("copies");
  {
    cudaEvent_t pe[2] = {nullptr, nullptr};
    LC_PTRY(cudaEventCreate(&pe[0]));
    LC_PTRY(cudaEventCreate(&pe[1]));
    cudaEventRecord(pe[0], os);
    const int64_t groups = (p->N + 7) / 8;
    const int tpb = 256;
    plan_lambda_kernel<<<unsigned((groups + tpb - 1) / tpb), tpb, 0, os>>>(p->d_tabB, p->N, p->dir);
    plan_taba_kernel<<<1, 32, 0, os>>>(p->d_tabA, 2 * s, p->dir);
    if (p->L > 0) {
      plan_lminus_kernel<<<unsigned(2 * p->L), 96, 0, os>>>(d_Lm, int(p->L), s);
      const int64_t grid = std::min<int64_t>((p->nc + kAhatWarps - 1) / kAhatWarps, int64_t(p->sm_count) * 8);
      plan_ahat_kernel<<<unsigned(grid), 32 * kAhatWarps, 0, os>>>(p->d_A, d_Lm, 0, p->nc, int(p->L), s, p->dir);
    }
    cudaEventRecord(pe[1], os);
    const cudaError_t ek = cudaGetLastError();
    const cudaError_t es = cudaEventSynchronize(pe[1]);
    float ms = 0.f;
    if (ek == cudaSuccess && es == cudaSuccess) cudaEventElapsedTime(&ms, pe[0], pe[1]);
    p->plan_ms = ms;
    cudaEventDestroy(pe[0]);
    cudaEventDestroy(pe[1]);
    LC_PTRY(ek);
    LC_PTRY(es);
  }
  if (d_Lm) cudaFreeAsync(d_Lm, os);
  mark("kernels");

  p->band_nnz = band_nnz(p->N, s);
  {
    lc_plan_desc d{};
    d.n = n; d.N = p->N; d.L = p->L; d.s = s; d.nc = p->nc; d.band_nnz = p->band_nnz;
    fill_work(&d, batch);
    p->flops_alg = d.flops_alg;
    p->bytes_alg = d.bytes_alg;
  }

  p->h_Tpad = static_cast<double*>(std::calloc(size_t(2) * 64 * kM, sizeof(double)));
  if (!p->h_Tpad) return fail(LC_ERR_OUT_OF_MEMORY);
  {
    const int smax_rows = s <= 32 ? 32 : 64;  // [2][smax][M], rows m >= s zero (kernel-parameter copy)
    for (int sg = 0; sg < 2; ++sg)
      for (int64_t m = 0; m < s; ++m)
        for (int k = 0; k < kM; ++k) p->h_Tpad[(sg * smax_rows + m) * kM + k] = T[size_t((sg * s + m) * kM + k)];
  }
  {
    const int smax_rows = s <= 32 ? 32 : 64;
    LC_PTRY(cudaMallocAsync(reinterpret_cast<void**>(&p->d_Tpad), sizeof(double) * size_t(2 * smax_rows * kM), os));
    LC_PTRY(cudaMemcpyAsync(p->d_Tpad, p->h_Tpad, sizeof(double) * size_t(2 * smax_rows * kM), cudaMemcpyHostToDevice,
                            os));
  }
  mark("Tpad");
  const lc_status cs = configure_kernels(p);
  if (cs != LC_OK) return fail(cs);
  mark("configure");
  {
    p->stage_bytes = size_t(align_up(in_extent(p) * 8, 256) + align_up(out_extent(p) * 8, 256));
  }
  LC_PTRY(cudaMallocAsync(&p->d_ws, p->ws_bytes > 0 ? p->ws_bytes : 16, os));
  LC_PTRY(cudaMemsetAsync(p->d_ws, 0, p->ws_bytes > 0 ? p->ws_bytes : 16, os));
  // the plan's arrays are complete before any caller stream can see the plan
  LC_PTRY(cudaStreamSynchronize(os));
  mark("workspace");
  cudaSetDevice(prev_dev);
  *out = p;
  return LC_OK;
#undef LC_PTRY
}

namespace lc {
void note_execute(const lc_plan* p, cudaStream_t st) {
  if (!p || !p->sync) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return;
  }
  std::lock_guard<std::mutex> lk(p->sync->mu);
  for (auto& e : p->sync->seen)
    if (e.first == st) {
      cudaEventRecord(e.second, st);
      return;
    }
  if (p->sync->seen.size() >= kMaxStreams) {
    p->sync->overflow = true;
    return;
  }
  cudaEvent_t ev = nullptr;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    p->sync->overflow = true;
    return;
  }
  cudaEventRecord(ev, st);
  p->sync->seen.emplace_back(st, ev);
}

double* plan_stage(const lc_plan* p_) {
  lc_plan* p = const_cast<lc_plan*>(p_);  // the staging pointer is set once, under the plan's mutex
  std::lock_guard<std::mutex> lk(p->sync->mu);
  if (!p->d_stage) {
    void* d = nullptr;
    if (cudaMallocAsync(&d, p->stage_bytes, p->own) != cudaSuccess || cudaStreamSynchronize(p->own) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    p->d_stage = static_cast<double*>(d);
  }
  return p->d_stage;
}
}  // namespace lc

extern "C" size_t lc_host_stage_bytes(const lc_plan* p) { return p ? p->stage_bytes : 0; }

// Page-locked host buffers on transparent huge pages (legcheb.h): the mapping of every live buffer,
// for lc_host_free
namespace {
struct HostMapping {
  void* base;
  size_t len;
};
std::mutex g_host_mu;
std::unordered_map<void*, HostMapping>& host_maps() {
  static std::unordered_map<void*, HostMapping> m;
  return m;
}
}  // namespace

extern "C" lc_status lc_host_alloc(size_t bytes, void** ptr) {
  if (bytes == 0 || !ptr) return LC_ERR_INVALID_ARG;
  *ptr = nullptr;
  constexpr size_t kHuge = size_t(1) << 21;
  const size_t len = (bytes + kHuge - 1) / kHuge * kHuge;
  void* base = mmap(nullptr, len + kHuge, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (base == MAP_FAILED) return LC_ERR_OUT_OF_MEMORY;
  char* a = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(base) + kHuge - 1) & ~uintptr_t(kHuge - 1));
#ifdef MADV_HUGEPAGE
  madvise(a, len, MADV_HUGEPAGE);  // advisory: without THP the 4 KiB pages serve
#endif
  std::memset(a, 0, len);  // fault the pages in (as huge pages where granted) before registration
  const cudaError_t e = cudaHostRegister(a, len, cudaHostRegisterDefault);
  if (e != cudaSuccess) {
    munmap(base, len + kHuge);
    return lc::record_cuda_error(e);
  }
  {
    std::lock_guard<std::mutex> lk(g_host_mu);
    host_maps()[a] = HostMapping{base, len + kHuge};
  }
  *ptr = a;
  return LC_OK;
}

extern "C" lc_status lc_host_free(void* ptr) {
  HostMapping m{};
  {
    std::lock_guard<std::mutex> lk(g_host_mu);
    auto it = host_maps().find(ptr);
    if (!ptr || it == host_maps().end()) return LC_ERR_INVALID_ARG;
    m = it->second;
    host_maps().erase(it);
  }
  const cudaError_t e = cudaHostUnregister(ptr);
  munmap(m.base, m.len);
  return e == cudaSuccess ? LC_OK : lc::record_cuda_error(e);
}

extern "C" lc_status lc_plan_destroy(lc_plan* p) {
  if (!p) return LC_ERR_INVALID_ARG;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  cudaStream_t os = p->own;
  if (p->sync) {
    // executions still in flight may read the plan's arrays and workspace: order the frees after the
    // last execution on every stream the plan was used on (and only those streams)
    std::lock_guard<std::mutex> lk(p->sync->mu);
    for (auto& e : p->sync->seen)
      if (os) cudaStreamWaitEvent(os, e.second, 0);
    if (p->sync->overflow) cudaDeviceSynchronize();  // untracked streams: wait for everything
  }
  void* bufs[] = {p->d_A, p->d_tabB, p->d_tabA, p->d_T, p->d_Tt, p->d_B, p->d_ws, p->d_stage, p->d_Tpad};
  for (void* b : bufs)
    if (b && os) cudaFreeAsync(b, os);
  if (os) {
    cudaStreamSynchronize(os);
    cudaStreamDestroy(os);
  }
  if (p->sync) {
    for (auto& e : p->sync->seen) cudaEventDestroy(e.second);
    delete p->sync;
  }
  std::free(p->h_Tpad);
  cudaGetLastError();  // errors of earlier asynchronous work are reported by the caller's synchronisation
  cudaSetDevice(prev);
  delete p;
  return LC_OK;
}

extern "C" lc_status lc_plan_describe(const lc_plan* p, lc_plan_desc* d) {
  if (!p || !d) return LC_ERR_INVALID_ARG;
  std::memset(d, 0, sizeof(*d));
  d->n = p->n; d->N = p->N; d->L = p->L; d->s = p->s; d->M = p->M; d->batch = p->batch; d->nc = p->nc;
  d->direction = p->dir; d->band_nnz = p->band_nnz;
  d->plan_bytes = p->plan_bytes; d->workspace_bytes = p->ws_bytes;
  d->flops_alg = p->flops_alg; d->bytes_alg = p->bytes_alg;
  d->vt = p->vt; d->subtree = p->k; d->stage_blocks = p->bps; d->stages = p->nst;
  d->kernels_per_execute = kernels_per_execute(p);
  d->plan_device_ms = p->plan_ms;
  d->row_lo = p->row_lo;
  d->row_hi = p->row_hi;
  return LC_OK;
}

extern "C" size_t lc_workspace_bytes(const lc_plan* p) { return p ? p->ws_bytes : 0; }

extern "C" lc_status lc_workspace_init(const lc_plan* p, void* ws, void* stream) {
  if (!p || !ws) return LC_ERR_INVALID_ARG;
  if (p->ws_bytes == 0) return LC_OK;
  return cudaMemsetAsync(ws, 0, p->ws_bytes, (cudaStream_t)stream) == cudaSuccess ? LC_OK : LC_ERR_CUDA;
}

extern "C" lc_status lc_plan_export(const lc_plan* p, int32_t what, double* host_out, int64_t count) {
  if (!p || !host_out) return LC_ERR_INVALID_ARG;
  const double* src = nullptr;
  int64_t len = 0;
  switch (what) {
    case 0: src = p->d_tabB; len = p->N; break;
    case 1: src = p->d_tabA; len = 2 * p->s; break;
    case 2: src = p->d_A; len = p->nc * kMM; break;
    case 3: src = p->d_B; len = kMM; break;
    case 4: src = p->d_T; len = 2 * p->s * kM; break;
    default: return LC_ERR_INVALID_ARG;
  }
  if (count < len) return LC_ERR_INVALID_ARG;
  if (len == 0) return LC_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  const cudaError_t e = cudaMemcpy(host_out, src, sizeof(double) * size_t(len), cudaMemcpyDeviceToHost);
  cudaSetDevice(prev);
  return e == cudaSuccess ? LC_OK : record_cuda_error(e);
}
