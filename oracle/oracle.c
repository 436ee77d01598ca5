/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for the Legendre<->Chebyshev
 * connection problem of arXiv 2411.00033, written from the paper's
 * definitions in x87 `long double` (64-bit mantissa) with Neumaier-compensated
 * accumulation.  It shares no code, header, table or constant generator with
 * the CUDA product path (paper_2411_00033_b200/csrc).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.
 *
 * What it computes (the plain definitions; no FMM, no blocking, no reordering):
 *
 *   lambda_k = Lambda(k) = Gamma(k+1/2)/Gamma(k+1)                PAPER.md:38-40 (eq:Lambda)
 *     by Lambda(0) = sqrt(pi) and Lambda(i) = Lambda(i-1)(i-1/2)/i   PAPER.md:501-503 (eq:Lambdaint)
 *
 *   L2C:  z = C^{-1} A f,  a_{i,i+2k} = lambda_k lambda_{i+k},       PAPER.md:24-46 (eq:AfCf, eq:directmv, eq:hik)
 *         C = diag(c_i pi/2), c_0 = 2, c_i = 1
 *         i.e. Alg. 1 (DIRECTL2C) evaluated row by row.
 *
 *   C2L:  z = A^{-1} C f                                              PAPER.md:31 (eq:directmv)
 *         (a) back-substitution on A x = C f using only the definition above;
 *         (b) row formula with the entries of the C2L kernel
 *             L(x,y) = 2(x+1/2)y/((x+y)(x+y+1)(x-y+1)) Lambda((y-x)/2)/Lambda((x+y)/2)
 *             at integer points (x,y) = (i, i+2k), and entry (0,0) = 1      PAPER.md:509-514 (eq:Lxymod)
 *             (reading R2: the (0,0) entry of A^{-1}C is 1; eq:Lxymod is 0/0 there).
 *
 * Pins that tie this file to something other than itself live in
 * tests/test_oracle_pins.py (exact-rational Chebyshev/Legendre expansions,
 * Gauss-Chebyshev quadrature, mpmath Gamma ratios, printed values).
 *
 * Build: gcc -O2 -fno-fast-math -fopenmp -shared -fPIC oracle.c -o liboracle.so
 * (never -ffast-math: it deletes the compensation terms).
 */
#include <math.h>
#include <quadmath.h>
#include <stdlib.h>
#include <string.h>

#define ORC_SQRT_PI 1.772453850905516027298167483341145182797549456122387128213807789852911284591025L
#define ORC_PI 3.141592653589793238462643383279502884197169399375105820974944592307816406286209L

/* Neumaier compensated accumulator (long double). */
typedef struct { long double s, c; } orc_acc;
static inline void acc_add(orc_acc* a, long double x) {
  long double t = a->s + x;
  if (fabsl(a->s) >= fabsl(x)) a->c += (a->s - t) + x;
  else a->c += (x - t) + a->s;
  a->s = t;
}
static inline long double acc_get(const orc_acc* a) { return a->s + a->c; }

/* lambda_k for k < n: lambda_0 = sqrt(pi), lambda_i = lambda_{i-1} (i - 1/2)/i. */
void orc_lambda(long n, long double* out) {
  if (n <= 0) return;
  out[0] = ORC_SQRT_PI;
  for (long i = 1; i < n; ++i) out[i] = out[i - 1] * ((long double)i - 0.5L) / (long double)i;
}

/* L2C rows: z_i = (2 - delta_{i0})/pi * sum_{k>=0, i+2k<n} lambda_k lambda_{i+k} f_{i+2k}
 * (Alg. 1 PAPER.md:75-98 restricted to row i).
 * absrow_i = (2 - delta_{i0})/pi * sum_k |lambda_k lambda_{i+k} f_{i+2k}|  (per-row error scale). */
int orc_l2c_rows(const long double* f, long n, const long* rows, long R,
                 long double* out, long double* absrow) {
  if (n <= 0) return 1;
  long double* lam = (long double*)malloc(sizeof(long double) * (size_t)n);
  if (!lam) return 2;
  orc_lambda(n, lam);
#pragma omp parallel for schedule(dynamic, 4)
  for (long r = 0; r < R; ++r) {
    long i = rows[r];
    orc_acc a = {0.0L, 0.0L}, b = {0.0L, 0.0L};
    for (long k = 0; i + 2 * k < n; ++k) {
      long double term = lam[k] * lam[i + k] * f[i + 2 * k];
      acc_add(&a, term);
      acc_add(&b, fabsl(term));
    }
    long double scale = (i == 0) ? 1.0L / ORC_PI : 2.0L / ORC_PI;
    out[r] = scale * acc_get(&a);
    if (absrow) absrow[r] = scale * acc_get(&b);
  }
  free(lam);
  return 0;
}

/* Entry M_{i,i+2k} of M = A^{-1} C from eq:Lxymod at (x,y) = (i, i+2k),
 * written with Lambda((y-x)/2) = lambda_k and Lambda((x+y)/2) = lambda_{i+k}. (0,0) -> 1. */
static inline long double c2l_entry(long i, long k, const long double* lam) {
  if (i == 0 && k == 0) return 1.0L;
  long double x = (long double)i, y = (long double)(i + 2 * k);
  long double num = 2.0L * (x + 0.5L) * y;
  long double den = (x + y) * (x + y + 1.0L) * (x - y + 1.0L);
  return num / den * (lam[k] / lam[i + k]);
}

/* C2L rows by the row formula (b). */
int orc_c2l_rows(const long double* f, long n, const long* rows, long R,
                 long double* out, long double* absrow) {
  if (n <= 0) return 1;
  long double* lam = (long double*)malloc(sizeof(long double) * (size_t)n);
  if (!lam) return 2;
  orc_lambda(n, lam);
#pragma omp parallel for schedule(dynamic, 4)
  for (long r = 0; r < R; ++r) {
    long i = rows[r];
    orc_acc a = {0.0L, 0.0L}, b = {0.0L, 0.0L};
    for (long k = 0; i + 2 * k < n; ++k) {
      long double term = c2l_entry(i, k, lam) * f[i + 2 * k];
      acc_add(&a, term);
      acc_add(&b, fabsl(term));
    }
    out[r] = acc_get(&a);
    if (absrow) absrow[r] = acc_get(&b);
  }
  free(lam);
  return 0;
}

/* C2L by back-substitution (a): solve A x = C f (eq:AfCf) with
 * a_{i,i+2k} = lambda_k lambda_{i+k}; b = C f, b_0 = pi f_0, b_i = (pi/2) f_i;
 * x_i = (b_i - sum_{k>=1, i+2k<n} lambda_k lambda_{i+k} x_{i+2k}) / (lambda_0 lambda_i). O(n^2). */
int orc_c2l_backsub(const long double* f, long n, long double* out) {
  if (n <= 0) return 1;
  long double* lam = (long double*)malloc(sizeof(long double) * (size_t)n);
  if (!lam) return 2;
  orc_lambda(n, lam);
  for (long i = n - 1; i >= 0; --i) {
    long double bi = (i == 0 ? ORC_PI : 0.5L * ORC_PI) * f[i];
    orc_acc a = {bi, 0.0L};
    for (long k = 1; i + 2 * k < n; ++k) acc_add(&a, -(lam[k] * lam[i + k] * out[i + 2 * k]));
    out[i] = acc_get(&a) / (lam[0] * lam[i]);
  }
  free(lam);
  return 0;
}

/* Convenience: all rows of one direction (dir 0 = L2C, 1 = C2L rows formula). */
int orc_transform(int dir, const long double* f, long n, long double* out) {
  long* rows = (long*)malloc(sizeof(long) * (size_t)n);
  if (!rows) return 2;
  for (long i = 0; i < n; ++i) rows[i] = i;
  int rc = dir == 0 ? orc_l2c_rows(f, n, rows, n, out, NULL) : orc_c2l_rows(f, n, rows, n, out, NULL);
  free(rows);
  return rc;
}

/* ---------------------------------------------------------------------------
 * Cross-check tier ("oracle summation" pin): the same row
 * definitions as orc_l2c_rows / orc_c2l_rows, evaluated in __float128
 * (libquadmath, 113-bit significand) with plain sums -- no compensation -- so
 * that the compensated long-double sums above can be checked at n >= 1e6.
 * lambda by the same recurrence from sqrt(pi), either in
 * quad (lam_ld = 0: pins the whole long-double oracle, lambda error included)
 * or widened from the long-double recurrence (lam_ld = 1: both sides use the
 * same lambda, isolating the summation).  Results are rounded to long double.
 * ------------------------------------------------------------------------- */
static __float128* orc_lambda_q(long n, int lam_ld) {
  __float128* lam = (__float128*)malloc(sizeof(__float128) * (size_t)n);
  if (!lam) return NULL;
  if (lam_ld) {
    long double* l = (long double*)malloc(sizeof(long double) * (size_t)n);
    if (!l) { free(lam); return NULL; }
    orc_lambda(n, l);
    for (long i = 0; i < n; ++i) lam[i] = (__float128)l[i];
    free(l);
    return lam;
  }
  lam[0] = sqrtq(M_PIq);
  for (long i = 1; i < n; ++i) lam[i] = lam[i - 1] * ((__float128)i - 0.5Q) / (__float128)i;
  return lam;
}

int orc_l2c_rows_q(const long double* f, long n, const long* rows, long R, long double* out, int lam_ld) {
  if (n <= 0) return 1;
  __float128* lam = orc_lambda_q(n, lam_ld);
  if (!lam) return 2;
#pragma omp parallel for schedule(dynamic, 1)
  for (long r = 0; r < R; ++r) {
    long i = rows[r];
    __float128 a = 0;
    for (long k = 0; i + 2 * k < n; ++k) a += lam[k] * lam[i + k] * (__float128)f[i + 2 * k];
    out[r] = (long double)((i == 0 ? 1.0Q : 2.0Q) / M_PIq * a);
  }
  free(lam);
  return 0;
}

int orc_c2l_rows_q(const long double* f, long n, const long* rows, long R, long double* out, int lam_ld) {
  if (n <= 0) return 1;
  __float128* lam = orc_lambda_q(n, lam_ld);
  if (!lam) return 2;
#pragma omp parallel for schedule(dynamic, 1)
  for (long r = 0; r < R; ++r) {
    long i = rows[r];
    __float128 a = 0;
    for (long k = 0; i + 2 * k < n; ++k) {
      __float128 e;
      if (i == 0 && k == 0) {
        e = 1;
      } else {
        __float128 x = i, y = i + 2 * k;  /* eq:Lxymod at (x, y) = (i, i+2k) */
        e = 2 * (x + 0.5Q) * y / ((x + y) * (x + y + 1) * (x - y + 1)) * (lam[k] / lam[i + k]);
      }
      a += e * (__float128)f[i + 2 * k];
    }
    out[r] = (long double)a;
  }
  free(lam);
  return 0;
}
