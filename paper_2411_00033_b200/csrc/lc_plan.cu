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
#include <vector>

#include "lc_internal.h"

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

// One CTA per A_hat matrix (global arena index q = blockIdx.x + q0).
// Ccos[k][m] = cos(k (m+1/2) pi / M); Gauss nodes X_m = Ccos[1][m].
__global__ void __launch_bounds__(384) plan_ahat_kernel(double* A, const double* __restrict__ Ccos, int64_t q0,
                                                        int L, int64_t s, int dir) {
  __shared__ double Cs[kMM];
  __shared__ double G[kMM];
  __shared__ double H[kMM];
  const int tid = threadIdx.x;
  const int64_t q = q0 + blockIdx.x;
  for (int i = tid; i < kMM; i += blockDim.x) Cs[i] = Ccos[i];
  int g = 0;
  while (g + 1 < L && ahat_level_offset(g + 1) <= q) ++g;
  const int64_t loc = q - ahat_level_offset(g);
  const int64_t b = loc / 3;
  const int r = int(loc % 3);
  const int p = (r == 2) ? 1 : 0;   // eq:cfrompq: r = 0,1,2 <-> (p,q) = (0,0),(0,1),(1,1)
  const int qq = (r >= 1) ? 1 : 0;
  const int64_t h = s << (L - g - 1);
  const int64_t i0 = 2 * h * (2 * b + p);       // eq:globalij
  const int64_t j0 = 2 * h * (2 * b + qq + 2);
  __syncthreads();
  if (tid < kMM) {
    const int m = tid / kM, nn = tid % kM;
    const double hx = double(h) * (Cs[kM + m] + 1.0);   // x - i0 = h (X_m + 1)   (eq:Xfromx)
    const double hy = double(h) * (Cs[kM + nn] + 1.0);  // y - j0 = h (Y_n + 1)
    // (y-x)/2 and (x+y)/2 from the exact integer corner offsets (no cancellation)
    const double ymx = 0.5 * double(j0 - i0) + 0.5 * (hy - hx);
    const double xpy = 0.5 * double(i0 + j0) + 0.5 * (hx + hy);
    const double lm = Lambda_dev(ymx), lp = Lambda_dev(xpy);
    double val;
    if (dir == 0) {
      val = lm * lp;  // A(x,y) = Lambda((y-x)/2) Lambda((y+x)/2)
    } else {
      // L(x,y) = 2(x+1/2) y / ((x+y)(x+y+1)(x-y+1)) Lambda((y-x)/2)/Lambda((x+y)/2)   (eq:Lxymod)
      const double x = double(i0) + hx, y = double(j0) + hy;
      val = (2.0 * (x + 0.5) * y) / ((2.0 * xpy) * (2.0 * xpy + 1.0) * (1.0 - 2.0 * ymx)) * (lm / lp);
    }
    G[m * kM + nn] = val;
  }
  __syncthreads();
  if (tid < kMM) {  // H = C G  (DCT-II along x)
    const int k = tid / kM, nn = tid % kM;
    double acc = 0.0;
    for (int m = 0; m < kM; ++m) acc += Cs[k * kM + m] * G[m * kM + nn];
    H[k * kM + nn] = acc;
  }
  __syncthreads();
  if (tid < kMM) {  // A_hat = 4/(c_k c_l M^2) H C^T  (eq:aklmore)
    const int k = tid / kM, l = tid % kM;
    double acc = 0.0;
    for (int nn = 0; nn < kM; ++nn) acc += H[k * kM + nn] * Cs[l * kM + nn];
    const double ck = k == 0 ? 2.0 : 1.0, cl = l == 0 ? 2.0 : 1.0;
    A[q * kMM + tid] = acc * (4.0 / (ck * cl * double(kM) * double(kM)));
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
  // nonzeros (i, i+2k) of A with i <= j < j_end(i) = min(N, 2s(floor(i/2s)+2))
  int64_t tot = 0;
  const int64_t seg = 2 * s;
  for (int64_t u = 0; u * seg < N; ++u) {
    const int64_t je = std::min<int64_t>(N, seg * (u + 2));
    for (int64_t r = 0; r < seg && u * seg + r < N; ++r) {
      const int64_t i = u * seg + r;
      tot += (je - i + 1) / 2;
    }
  }
  return tot;
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

lc_status lc_geometry(int64_t n, int64_t s_hat, lc_plan_desc* out) {
  if (n < 1 || out == nullptr) return LC_ERR_INVALID_ARG;
  if (s_hat <= 0) s_hat = 32;
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
  if (out == nullptr || n < 1 || batch < 1) return LC_ERR_INVALID_ARG;
  *out = nullptr;
  if (dir != LC_LEG2CHEB && dir != LC_CHEB2LEG) return LC_ERR_INVALID_ARG;
  lc_plan_opts o{};
  if (opts) o = *opts;
  if (o.s_hat <= 0) o.s_hat = 32;
  if (o.M <= 0) o.M = kM;
  if (o.M != kM || o.s_hat < 2 || o.s_hat > 64) return LC_ERR_INVALID_ARG;
  if (o.engine < 0 || o.engine > 3) return LC_ERR_INVALID_ARG;
  if (o.layout != LC_VEC_CONTIGUOUS && o.layout != LC_BATCH_CONTIGUOUS) return LC_ERR_INVALID_ARG;
  const int64_t def_ld = o.layout == LC_VEC_CONTIGUOUS ? n : batch;
  if (o.ld_in == 0) o.ld_in = def_ld;
  if (o.ld_out == 0) o.ld_out = def_ld;
  if (o.ld_in < def_ld || o.ld_out < def_ld) return LC_ERR_INVALID_ARG;

  int dev = o.device;
  if (dev < 0) LC_CUDA_TRY(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  LC_CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10) return LC_ERR_UNSUPPORTED_DEVICE;
  int prev_dev = 0;
  LC_CUDA_TRY(cudaGetDevice(&prev_dev));
  LC_CUDA_TRY(cudaSetDevice(dev));

  lc_plan* p = new lc_plan();
  std::memset(p, 0, sizeof(*p));
  const Geometry G = geometry(n, o.s_hat);
  p->n = n; p->N = G.N; p->L = G.L; p->s = G.s; p->M = kM; p->batch = batch; p->nc = G.nc;
  p->dir = int(dir); p->layout = o.layout; p->ld_in = o.ld_in; p->ld_out = o.ld_out;
  p->device = dev; p->sm_count = prop.multiProcessorCount;
  p->vt = o.vt; p->k = o.subtree; p->bps = o.stage_blocks; p->nst = o.stages; p->kup = o.up_subtree;
  p->engine = o.engine;

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
  LC_PTRY(cudaMalloc(&p->d_tabB, sizeof(double) * size_t(p->N)));
  LC_PTRY(cudaMalloc(&p->d_tabA, sizeof(double) * size_t(2 * s)));
  LC_PTRY(cudaMalloc(&p->d_T, sizeof(double) * size_t(2 * s * kM)));
  LC_PTRY(cudaMalloc(&p->d_Tt, sizeof(double) * size_t(2 * s * kM)));
  LC_PTRY(cudaMalloc(&p->d_B, sizeof(double) * kMM));
  if (p->nc > 0) LC_PTRY(cudaMalloc(&p->d_A, sizeof(double) * size_t(p->nc) * kMM));
  p->plan_bytes = sizeof(double) * (size_t(p->N) + size_t(2 * s) + size_t(4 * s * kM) + kMM + size_t(p->nc) * kMM);

  double B[kMM];
  build_B0(B);
  std::vector<double> T, Tt;
  build_T(s, T, Tt);
  double Cc[kMM];
  for (int k = 0; k < kM; ++k)
    for (int m = 0; m < kM; ++m)
      Cc[k * kM + m] = double(cosl((long double)k * ((long double)m + 0.5L) *
                                   3.141592653589793238462643383279502884L / (long double)kM));
  double* d_C = nullptr;
  LC_PTRY(cudaMalloc(&d_C, sizeof(double) * kMM));
  LC_PTRY(cudaMemcpy(p->d_B, B, sizeof(B), cudaMemcpyHostToDevice));
  LC_PTRY(cudaMemcpy(p->d_T, T.data(), sizeof(double) * T.size(), cudaMemcpyHostToDevice));
  LC_PTRY(cudaMemcpy(p->d_Tt, Tt.data(), sizeof(double) * Tt.size(), cudaMemcpyHostToDevice));
  LC_PTRY(cudaMemcpy(d_C, Cc, sizeof(Cc), cudaMemcpyHostToDevice));

  {
    const int64_t groups = (p->N + 7) / 8;
    const int tpb = 256;
    plan_lambda_kernel<<<unsigned((groups + tpb - 1) / tpb), tpb>>>(p->d_tabB, p->N, p->dir);
    plan_taba_kernel<<<1, 32>>>(p->d_tabA, 2 * s, p->dir);
    for (int64_t q0 = 0; q0 < p->nc; q0 += (int64_t(1) << 30)) {
      const int64_t cnt = std::min<int64_t>(p->nc - q0, int64_t(1) << 30);
      plan_ahat_kernel<<<unsigned(cnt), 352>>>(p->d_A, d_C, q0, int(p->L), s, p->dir);
    }
    LC_PTRY(cudaGetLastError());
    LC_PTRY(cudaDeviceSynchronize());
  }
  cudaFree(d_C);

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
    LC_PTRY(cudaMalloc(&p->d_Tpad, sizeof(double) * size_t(2 * smax_rows * kM)));
    LC_PTRY(cudaMemcpy(p->d_Tpad, p->h_Tpad, sizeof(double) * size_t(2 * smax_rows * kM), cudaMemcpyHostToDevice));
  }
  const lc_status cs = configure_kernels(p);
  if (cs != LC_OK) return fail(cs);
  LC_PTRY(cudaMalloc(&p->d_ws, p->ws_bytes > 0 ? p->ws_bytes : 16));
  LC_PTRY(cudaMemset(p->d_ws, 0, p->ws_bytes > 0 ? p->ws_bytes : 16));
  LC_PTRY(cudaDeviceSynchronize());
  cudaSetDevice(prev_dev);
  *out = p;
  return LC_OK;
#undef LC_PTRY
}

extern "C" lc_status lc_plan_destroy(lc_plan* p) {
  if (!p) return LC_ERR_INVALID_ARG;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  // executions still in flight on any stream may read the plan's arrays and workspace: finish them
  // before the memory can be handed to another allocation
  cudaDeviceSynchronize();
  cudaFree(p->d_A);
  cudaFree(p->d_tabB);
  cudaFree(p->d_tabA);
  cudaFree(p->d_T);
  cudaFree(p->d_Tt);
  cudaFree(p->d_B);
  cudaFree(p->d_ws);
  cudaFree(p->d_stage_in);
  cudaFree(p->d_stage_out);
  std::free(p->h_Tpad);
  cudaFree(p->d_Tpad);
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
  d->kernels_per_execute = p->engine == 2 ? 1 : (p->engine == 3 ? 2 : (p->L > 0 ? 3 : 2));
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
