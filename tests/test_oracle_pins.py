"""Pins for the CPU oracle (oracle/): tie it to things other than itself.

Each test states the passage it follows.  A plausible mistake anywhere in
oracle.c (a dropped C^{-1} factor, a wrong lambda index, a transposed entry,
a sign slip in the C2L kernel, a broken compensated sum) fails at least one:

* L2C columns == exact-rational Chebyshev coefficients of each Legendre
  polynomial L_j (Legendre recurrence + x T_k = (T_{k+1}+T_{|k-1|})/2):
  shares nothing with the Lambda formula.
* a_ij == Gauss-Chebyshev quadrature of (T_i, L_j)_w.
* C2L columns == exact-rational Legendre coefficients of T_j.
* lambda vs mpmath Gamma ratios (40 digits) and printed values. PAPER.md:38-40, 501-503
* L2C rows vs an exact Fraction evaluation (lambda_k/sqrt(pi) rational).
* back-substitution == eq:Lxymod rows; A^{-1}C C^{-1}A = I.
"""
from fractions import Fraction

import mpmath
import numpy as np
import pytest

import oracle
from lc_inputs import vector

LD = np.longdouble


# ---------------------------------------------------------------- exact helpers
def legendre_in_chebyshev(jmax):
    """cheb[j][i] = coefficient of T_i in L_j, exact Fractions.
    (n+1)L_{n+1} = (2n+1) x L_n - n L_{n-1};  x T_0 = T_1, x T_k = (T_{k+1}+T_{k-1})/2."""
    def xtimes(c):
        out = [Fraction(0)] * (len(c) + 1)
        for k, a in enumerate(c):
            if a == 0:
                continue
            if k == 0:
                out[1] += a
            else:
                out[k + 1] += a / 2
                out[k - 1] += a / 2
        return out
    polys = [[Fraction(1)], [Fraction(0), Fraction(1)]]
    for n in range(1, jmax):
        xl = xtimes(polys[n])
        prev = polys[n - 1] + [Fraction(0)] * (len(xl) - len(polys[n - 1]))
        polys.append([((2 * n + 1) * a - n * b) / (n + 1) for a, b in zip(xl, prev)])
    return polys[: jmax + 1]


def chebyshev_in_legendre(jmax):
    """leg[j][i] = coefficient of L_i in T_j, exact Fractions.
    x L_k = ((k+1) L_{k+1} + k L_{k-1})/(2k+1);  T_{j+1} = 2x T_j - T_{j-1}."""
    def xtimes(c):
        out = [Fraction(0)] * (len(c) + 1)
        for k, a in enumerate(c):
            if a == 0:
                continue
            out[k + 1] += a * Fraction(k + 1, 2 * k + 1)
            if k > 0:
                out[k - 1] += a * Fraction(k, 2 * k + 1)
        return out
    polys = [[Fraction(1)], [Fraction(0), Fraction(1)]]
    for n in range(1, jmax):
        xt = xtimes(polys[n])
        prev = polys[n - 1] + [Fraction(0)] * (len(xt) - len(polys[n - 1]))
        polys.append([2 * a - b for a, b in zip(xt, prev)])
    return polys[: jmax + 1]


def frac_ld(q):
    mpmath.mp.dps = 30
    return LD(mpmath.nstr(mpmath.mpf(q.numerator) / q.denominator, 25))


def unit(n, j):
    e = np.zeros(n, dtype=LD)
    e[j] = 1
    return e


# ---------------------------------------------------------------- lambda pins
def test_lambda_printed_values():
    # PAPER.md:501 Lambda(0)=sqrt(pi); one and two steps of eq:Lambdaint
    mpmath.mp.dps = 40
    lam = oracle.lam(3)
    sp = mpmath.sqrt(mpmath.pi)
    for got, exact in zip(lam, [sp, sp / 2, 3 * sp / 8]):
        assert abs(float((mpmath.mpf(str(got)) - exact) / exact)) < 2e-19


@pytest.mark.parametrize("k", [1, 7, 19, 20, 100, 1000, 123457, 1000000, 9999999])
def test_lambda_vs_mpmath_gamma_ratio(k):
    # Lambda(x) = Gamma(x+1/2)/Gamma(x+1), PAPER.md:38-40 (eq:Lambda)
    mpmath.mp.dps = 40
    exact = mpmath.exp(mpmath.loggamma(k + mpmath.mpf(1) / 2) - mpmath.loggamma(k + 1))
    got = oracle.lam(k + 1)[k]
    rel = abs((mpmath.mpf(str(got)) - exact) / exact)
    # long-double recurrence: <= ~1e-16 up to 1e7 (SURVEY F2 measured 7.7e-17); far below the 1e-12 gate
    assert rel < 2e-16, (k, float(rel))


def test_lambda_asymptote():
    # Lambda(z) sqrt(z) -> 1, monotonically from below
    lam = oracle.lam(2_000_001)
    prev = 0.0
    for z in [10, 100, 1000, 10**4, 10**5, 10**6, 2 * 10**6]:
        v = float(lam[z] * np.sqrt(LD(z)))
        assert v < 1.0 and v > prev
        prev = v
    assert abs(prev - 1) < 1e-7


# ---------------------------------------------------------------- L2C pins
def test_l2c_columns_are_legendre_chebyshev_coefficients():
    # f_leg = e_j  <=>  f(x) = L_j(x) = sum_i f_cheb_i T_i(x)   (eq:fx)
    jmax = 64
    n = jmax + 1
    cheb = legendre_in_chebyshev(jmax)
    for j in range(jmax + 1):
        z = oracle.l2c(unit(n, j))
        exact = np.array([frac_ld(c) for c in cheb[j]] + [LD(0)] * (n - len(cheb[j])), dtype=LD)
        assert np.max(np.abs(z - exact)) < 1e-18, j
    # printed special cases L2 = T0/4 + 3T2/4, L3 = 3T1/8 + 5T3/8 (SURVEY pins)
    assert cheb[2][:3] == [Fraction(1, 4), 0, Fraction(3, 4)]
    assert cheb[3][:4] == [0, Fraction(3, 8), 0, Fraction(5, 8)]


def test_l2c_unit_vectors_e0_e1():
    # L0 = T0, L1 = T1
    for j in (0, 1):
        z = oracle.l2c(unit(16, j))
        assert np.max(np.abs(z - unit(16, j))) < 1e-18


def test_a_matrix_by_gauss_chebyshev_quadrature():
    # a_ij = (T_i, L_j)_w with w = (1-x^2)^{-1/2}; A = C * (C^{-1} A)
    n = 24
    Q = n + 2  # exact for deg < 2Q
    mpmath.mp.dps = 30
    xs = [mpmath.cos((q + mpmath.mpf(1) / 2) * mpmath.pi / Q) for q in range(Q)]
    for j in range(n):
        z = oracle.l2c(unit(n, j))
        for i in range(n):
            quad = mpmath.pi / Q * sum(mpmath.chebyt(i, x) * mpmath.legendre(j, x) for x in xs)
            ci = 2 if i == 0 else 1
            a = float(quad)
            got = float(z[i]) * ci * np.pi / 2
            assert abs(got - a) < 1e-15 * max(1.0, abs(a)), (i, j, got, a)


def test_l2c_rows_exact_rational():
    # lambda_k = sqrt(pi) r_k with r_k = prod_{j<=k} (j-1/2)/j rational, so
    # z_i = (2-delta_i0)/pi * sum pi r_k r_{i+k} f_{i+2k} is an exact rational of the fp64 input.
    n = 150
    f = vector("normal", n, seed=3)
    r = [Fraction(1)]
    for k in range(1, n):
        r.append(r[-1] * Fraction(2 * k - 1, 2 * k))
    fq = [Fraction(float(x)) for x in f]
    z, ab = oracle.l2c_rows(f, with_abs=True)
    for i in range(n):
        s = sum(r[k] * r[i + k] * fq[i + 2 * k] for k in range((n - 1 - i) // 2 + 1))
        s *= 1 if i == 0 else 2
        mpmath.mp.dps = 40
        err = abs(mpmath.mpf(str(z[i])) - mpmath.mpf(s.numerator) / s.denominator)
        assert err <= 1e-18 * float(ab[i]) + 1e-300, (i, float(err))


def test_l2c_parity_separation_and_linearity():
    n = 257
    f = vector("normal", n, seed=5)
    fe = f.copy()
    fe[1::2] = 0
    z = oracle.l2c(fe)
    assert np.all(z[1::2] == 0)
    g = vector("normal", n, seed=6)
    f, g = f.astype(LD), g.astype(LD)
    lhs = oracle.l2c(2.5 * f - 0.75 * g)
    rhs = 2.5 * oracle.l2c(f) - 0.75 * oracle.l2c(g)
    assert oracle.einf(lhs, rhs) < 1e-17


# ---------------------------------------------------------------- C2L pins
def test_c2l_columns_are_chebyshev_legendre_coefficients():
    # f_cheb = e_j <=> f = T_j = sum_i f_leg_i L_i
    jmax = 64
    n = jmax + 1
    leg = chebyshev_in_legendre(jmax)
    for j in range(jmax + 1):
        exact = np.array([frac_ld(c) for c in leg[j]] + [LD(0)] * (n - len(leg[j])), dtype=LD)
        for z in (oracle.c2l(unit(n, j)), oracle.c2l_backsub(unit(n, j))):
            assert np.max(np.abs(z - exact)) < 1e-18 * max(1, np.max(np.abs(exact))), j


def test_c2l_unit_cases():
    # T2 = -1/3 L0 + 4/3 L2;  T0 = L0
    z = oracle.c2l(unit(8, 2))
    assert abs(float(z[0]) + 1 / 3) < 1e-18 and abs(float(z[2]) - 4 / 3) < 1e-18 and z[1] == 0
    z0 = oracle.c2l(unit(8, 0))
    assert np.max(np.abs(z0 - unit(8, 0))) < 1e-19


@pytest.mark.parametrize("n", [64, 1000, 4096])
def test_c2l_backsub_equals_row_formula(n):
    # (a) back-substitution uses only A f = C f_cheb; (b) eq:Lxymod rows
    f = vector("normal", n, seed=7)
    za = oracle.c2l_backsub(f)
    zb = oracle.c2l(f)
    assert oracle.einf(zb, za) < 1e-17


@pytest.mark.parametrize("n,kind", [(1024, "uniform_r0"), (4096, "uniform_r0"), (4096, "normal_exp1000")])
def test_oracle_round_trip_identity(n, kind):
    # A^{-1} C (C^{-1} A) = I, in long double end to end
    f = vector(kind, n, seed=11)
    z = oracle.l2c(f)
    back = oracle.c2l(z)
    assert oracle.einf(back, f) < 1e-16
    back2 = oracle.c2l_backsub(z)
    assert oracle.einf(back2, f) < 1e-16


@pytest.mark.parametrize("direction", ["leg2cheb", "cheb2leg"])
def test_compensated_sum_vs_float128(direction):
    """SURVEY.md 8(c) "oracle summation" pin: at n = 1e6 the compensated long-double row sums agree
    with plain __float128 sums of the same terms (same lambda) to ~1e-19 of the row scale
    sum_k |K_ik f_k|, far tighter than a plain long-double sum achieves (the control below), and with
    quad lambda the whole oracle is within 2e-16 of the row scale (the long-double lambda recurrence,
    SURVEY F2: <= 7.7e-17 per factor) -- four orders inside the 1e-12 parity gate."""
    n = 1_000_000
    f = vector("normal", n, seed=3)
    rng = np.random.default_rng(5)
    rows = np.unique(np.r_[0, 1, 2, n - 2, n - 1, rng.integers(0, n, 24)])
    rows_fn = oracle.l2c_rows if direction == "leg2cheb" else oracle.c2l_rows
    q_fn = oracle.l2c_rows_q if direction == "leg2cheb" else oracle.c2l_rows_q
    z, ab = rows_fn(f, rows, with_abs=True)
    q_same = q_fn(f, rows, lam_ld=True)
    q_quad = q_fn(f, rows)
    assert np.max(np.abs(z - q_same) / ab) < 1e-18
    assert np.max(np.abs(z - q_quad) / ab) < 2e-16
    # control: a plain (uncompensated) long-double sum of the same terms misses the 1e-18 bound
    lam = oracle.lam(n)
    fl = f.astype(LD)
    worst = 0.0
    for r, i in enumerate(rows[rows < n // 4][:4]):
        k = np.arange((n - 1 - i) // 2 + 1)
        if direction == "leg2cheb":
            terms = lam[k] * lam[i + k] * fl[i + 2 * k] * LD(1 if i == 0 else 2) / LD(np.pi)
        else:
            x, y = LD(i), (i + 2 * k).astype(LD)
            with np.errstate(invalid="ignore", divide="ignore"):  # (0,0) is 0/0; set to 1 below
                terms = (2 * (x + LD(0.5)) * y / ((x + y) * (x + y + 1) * (x - y + 1)) * (lam[k] / lam[i + k])
                         * fl[i + 2 * k])
            if i == 0:
                terms[0] = fl[0]
        plain = LD(0)
        for t in np.array_split(terms, 64):  # sequential accumulation in long double
            for v in t:
                plain += v
        rr = int(np.nonzero(rows == i)[0][0])
        worst = max(worst, float(abs(plain - q_same[rr]) / ab[rr]))
    assert worst > 1e-18, worst


@pytest.mark.parametrize("direction", ["leg2cheb", "cheb2leg"])
def test_absrow_is_row_sum_of_abs_entries(direction):
    """absrow_i = sum_j |K_ij f_j| (the per-row diagnostic scale of SURVEY C-5), with K from the
    exact-rational expansions (L2C: Chebyshev coefficients of L_j; C2L: Legendre coefficients of T_j),
    which share nothing with the oracle's lambda formula."""
    jmax = 48
    n = jmax + 1
    cols = legendre_in_chebyshev(jmax) if direction == "leg2cheb" else chebyshev_in_legendre(jmax)
    K = np.zeros((n, n), dtype=LD)
    for j in range(n):
        for i, c in enumerate(cols[j]):
            K[i, j] = frac_ld(c)
    f = vector("normal", n, seed=17).astype(LD)
    rows = np.arange(n)
    z, ab = oracle.transform_rows(direction, f, rows, with_abs=True)
    exact_abs = np.abs(K * f[None, :]).sum(axis=1)
    exact = (K * f[None, :]).sum(axis=1)
    assert np.max(np.abs(ab - exact_abs) / exact_abs) < 1e-17
    assert np.max(np.abs(z - exact) / exact_abs) < 1e-17
    assert np.all(ab >= np.abs(z) * (1 - 1e-18))  # triangle inequality


# ---------------------------------------------------------------- metric
def test_einf_examples():
    # SPEC.md:441-443 (eq:Einf)
    assert oracle.einf([1.0, 2.0], [1.0, 2.0]) == 0
    assert abs(oracle.einf([1.0, 2.0000002], [1.0, 2.0]) - 1e-7) < 1e-15
    assert oracle.einf([1.0, 0.0], [0.0, 1.0]) == 1.0
