/* cpu_fmm.c -- CPU baseline of the SAME O(N) algorithm as the GPU path (Alg. 4 of arXiv 2411.00033,
 * alg:fastercomplete), in plain C with OpenMP over the blocks of each step.
 *
 * REPORTED BASELINE ONLY (BASELINE.json north_star: "a CPU implementation of the same O(N)
 * algorithm ... timed on the box's host cores").  It is neither the oracle (oracle/ is the direct
 * O(n^2) definition) nor part of the product: bench.py times it next to the GPU, and a GPU test
 * checks it against the oracle.  It takes the plan's tables (lambda / rho, kappa, A_hat, B(0), T)
 * exported from a GPU plan through lc_plan_export, so it measures the execution stage only, like
 * the GPU numbers.  Segment indexing as in DESIGN.md "Data layout": on level g the padded vector is
 * cut into 2^(g+2) segments of 2h_g = s 2^(L-g) coefficients; block b of level g has rows u = 2b, 2b+1
 * and columns t = 2b+2, 2b+3 (eq:globalij); segment t of level g is segments 2t, 2t+1 of level g+1.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define M 18

static int64_t nseg(int g) { return (int64_t)4 << g; }
static int64_t ahat_off(int g) { return 3 * (((int64_t)2 << g) - 2 - g); }

/* one transform of one vector: dir 0 = leg2cheb (C^{-1} A f), 1 = cheb2leg (A^{-1} C f) */
int cpu_fmm_execute(int dir, int64_t n, int64_t N, int L, int s, const double* Ahat, const double* tabA,
                    const double* tabB, const double* T, const double* B, const double* f, double* z) {
  double* fp = (double*)calloc((size_t)N, sizeof(double));
  double* zp = (double*)calloc((size_t)N, sizeof(double));
  if (!fp || !zp) { free(fp); free(zp); return 1; }
  memcpy(fp, f, (size_t)n * sizeof(double));
  const int64_t seg = 2 * (int64_t)s;

  if (L > 0) {
    /* w, c: per level g, [sigma][segment][M] */
    int64_t off[64];
    int64_t tot = 0;
    for (int g = 0; g < L; ++g) { off[g] = tot; tot += 2 * nseg(g) * M; }
    double* w = (double*)calloc((size_t)tot, sizeof(double));
    double* c = (double*)calloc((size_t)tot, sizeof(double));
    if (!w || !c) { free(w); free(c); free(fp); free(zp); return 1; }
#define W(g, sg, t) (w + off[g] + ((int64_t)(sg) * nseg(g) + (t)) * M)
#define CC(g, sg, t) (c + off[g] + ((int64_t)(sg) * nseg(g) + (t)) * M)
    const int64_t nleaf = nseg(L - 1);
    /* step 1 (eq:wMM): w(L-1)[t][k] = sum_m f[2s t + 2m + sigma] T(sigma)[m][k] */
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < nleaf; ++t)
      for (int sg = 0; sg < 2; ++sg) {
        double* o = W(L - 1, sg, t);
        for (int k = 0; k < M; ++k) o[k] = 0.0;
        for (int m = 0; m < s; ++m) {
          const double x = fp[seg * t + 2 * m + sg];
          const double* tr = T + ((int64_t)sg * s + m) * M;
          for (int k = 0; k < M; ++k) o[k] += x * tr[k];
        }
      }
    /* step 2 (Alg. a.1): parent[n] = sum_{k<=n} b_nk (x0_k + (-1)^(n-k) x1_k) */
    for (int g = L - 1; g >= 1; --g) {
#pragma omp parallel for schedule(static)
      for (int64_t t = 0; t < nseg(g - 1); ++t)
        for (int sg = 0; sg < 2; ++sg) {
          const double* x0 = W(g, sg, 2 * t);
          const double* x1 = W(g, sg, 2 * t + 1);
          double* o = W(g - 1, sg, t);
          for (int nn = 0; nn < M; ++nn) {
            double acc = 0.0;
            for (int k = 0; k <= nn; ++k) acc += B[nn * M + k] * (((nn - k) & 1) ? x0[k] - x1[k] : x0[k] + x1[k]);
            o[nn] = acc;
          }
        }
    }
    /* step 3 (M2L): c(u=2b) = A_hat(b,0) w(2b+2) + A_hat(b,1) w(2b+3); c(2b+1) = A_hat(b,2) w(2b+3) */
    for (int g = 0; g < L; ++g) {
      const int64_t bg = ((int64_t)2 << g) - 1;
#pragma omp parallel for schedule(static)
      for (int64_t b = 0; b < bg; ++b)
        for (int sg = 0; sg < 2; ++sg)
          for (int r = 0; r < 3; ++r) {
            const int64_t u = 2 * b + (r == 2), t = 2 * b + 2 + (r > 0);
            const double* A = Ahat + (ahat_off(g) + 3 * b + r) * M * M;
            const double* x = W(g, sg, t);
            double* o = CC(g, sg, u);
            for (int k = 0; k < M; ++k) {
              double acc = 0.0;
              for (int l = 0; l < M; ++l) acc += A[k * M + l] * x[l];
              o[k] += acc;
            }
          }
    }
    /* step 4: c(g, u)[k] += (-1)^(pk) sum_{n>=k} b_nk (-1)^(pn) c(g-1, u/2)[n], p = u & 1 */
    for (int g = 1; g < L; ++g) {
#pragma omp parallel for schedule(static)
      for (int64_t u = 0; u < nseg(g); ++u)
        for (int sg = 0; sg < 2; ++sg) {
          const int p = (int)(u & 1);
          const double* x = CC(g - 1, sg, u >> 1);
          double* o = CC(g, sg, u);
          for (int k = 0; k < M; ++k) {
            double acc = 0.0;
            for (int nn = k; nn < M; ++nn) acc += B[nn * M + k] * ((p && (nn & 1)) ? -x[nn] : x[nn]);
            o[k] += (p && (k & 1)) ? -acc : acc;
          }
        }
    }
    /* step 5 (eq:step5): z[2s U + 2m + sigma] = sum_k T(sigma)[m][k] c(L-1, U)[k] */
#pragma omp parallel for schedule(static)
    for (int64_t U = 0; U < nleaf; ++U)
      for (int sg = 0; sg < 2; ++sg) {
        const double* x = CC(L - 1, sg, U);
        for (int m = 0; m < s; ++m) {
          const double* tr = T + ((int64_t)sg * s + m) * M;
          double acc = 0.0;
          for (int k = 0; k < M; ++k) acc += tr[k] * x[k];
          zp[seg * U + 2 * m + sg] = acc;
        }
      }
#undef W
#undef CC
    free(w);
    free(c);
  }
  /* step 6: direct band, j = i + 2k < j_end(i) = min(N, 2s(floor(i/2s) + 2)) (L = 0: N);
   * L2C: a_k b_m f_j (a = lambda_k, b = lambda_m, m = i + k); C2L: (2i+1) kappa_k rho_m j f_j, z_0 += f_0 */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    int64_t je = L > 0 ? seg * (i / seg + 2) : N;
    if (je > N) je = N;
    double acc = 0.0;
    for (int64_t k = 0; i + 2 * k < je; ++k) {
      const int64_t j = i + 2 * k;
      const double g = dir == 1 ? (double)j * fp[j] : fp[j];
      acc += tabA[k] * tabB[i + k] * g;
    }
    if (dir == 1) {
      acc *= (double)(2 * i + 1);
      if (i == 0) acc += fp[0];
    }
    zp[i] += acc;
  }
  /* step 7: C^{-1} (L2C) and stage-out */
  const double inv_pi = 0.318309886183790671537767526745028724;
  for (int64_t i = 0; i < n; ++i) z[i] = dir == 0 ? zp[i] * (i == 0 ? inv_pi : 2.0 * inv_pi) : zp[i];
  free(fp);
  free(zp);
  return 0;
}

int cpu_fmm_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* thread count of the following cpu_fmm_execute calls (bench.py: 1 core and all cores) */
void cpu_fmm_set_threads(int t) {
#ifdef _OPENMP
  extern void omp_set_num_threads(int);
  omp_set_num_threads(t > 0 ? t : 1);
#else
  (void)t;
#endif
}
