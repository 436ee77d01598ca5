"""CPU tests of the host logic: the C ABI library loads and exports what include/legcheb.h declares,
the host-only geometry and work model, the decomposition readings (exact cover, staircase band),
the exact B(l) construction, and the paper-notation FMM model against the oracle.

None of these launches a kernel (no GPU here)."""
import ctypes
import math
import os
import re
from fractions import Fraction

import numpy as np
import pytest

import oracle
from lc_inputs import vector

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "legcheb.h")


def _lib():
    from paper_2411_00033_b200 import _lib as L
    return L


# ---------------------------------------------------------------- the C ABI boundary
def test_library_exports_every_declared_symbol():
    text = open(HEADER).read()
    declared = set(re.findall(r"^\s*(?:const\s+)?[a-z_]+\*?\s+\**(lc_[a-z_]+)\s*\(", text, re.M))
    assert {"lc_plan_create", "lc_execute", "lc_plan_destroy", "lc_geometry"} <= declared
    lib = ctypes.CDLL(_lib().LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), name
    # the binding declares exactly the header's functions
    assert set(_lib().SIGNATURES) == declared


def test_status_strings_and_version():
    lib = _lib().load()
    assert lib.lc_status_string(0) == b"ok"
    assert b"overlap" in lib.lc_status_string(5)
    assert b"sm_100a" in lib.lc_version()


def test_geometry_rejects_bad_arguments():
    L = _lib()
    d = L.PlanDesc()
    assert L.load().lc_geometry(0, 32, ctypes.byref(d)) == 1
    assert L.load().lc_geometry(10, 32, None) == 1


# ---------------------------------------------------------------- decomposition
@pytest.mark.parametrize("s_hat,n,L,s,N", [
    (32, 1000, 3, 32, 1024), (32, 1024, 3, 32, 1024), (32, 4096, 5, 32, 4096), (32, 10**6, 13, 31, 1015808),
    (32, 1 << 20, 13, 32, 1 << 20), (32, 10**7, 17, 20, 10485760), (32, 8192, 6, 32, 8192),
    # the library default s_hat = 40 (R17): the BASELINE configs keep their s but for 10^7
    (0, 1024, 3, 32, 1024), (0, 4096, 5, 32, 4096), (0, 8192, 6, 32, 8192), (0, 10**6, 13, 31, 1015808),
    (0, 1 << 20, 13, 32, 1 << 20), (0, 10**7, 16, 39, 10223616), (0, 640, 2, 40, 640), (40, 641, 3, 21, 672)])
def test_geometry_eq_numlevels(s_hat, n, L, s, N):
    from paper_2411_00033_b200 import geometry
    g = geometry(n, s_hat)
    assert (g["L"], g["s"], g["N"]) == (L, s, N)
    # eq:Ntot N = s 2^(L+2);  s in [s_hat/2, s_hat]
    sh = s_hat or 40
    assert g["N"] == g["s"] << (g["L"] + 2) and sh // 2 <= g["s"] <= sh
    # eq:total_blocks_and_mats: N_b = N/2s - L - 2, N_c = 3 N_b
    assert g["nc"] == 3 * (N // (2 * s) - L - 2)
    assert g["nc"] == 3 * sum((1 << (gg + 1)) - 1 for gg in range(L))  # eq:Nb summed


def test_geometry_fig1_and_spec_examples():
    from paper_2411_00033_b200 import geometry
    g = geometry(1024)
    # Fig. 1: 1 + 3 + 7 = 11 blocks, N_c = 33
    assert [(1 << (gg + 1)) - 1 for gg in range(g["L"])] == [1, 3, 7] and g["nc"] == 33
    assert geometry(4096)["nc"] // 3 == 57
    # small n: band only (reading R6)
    assert geometry(100)["L"] == 0 and geometry(1)["N"] == 4


def j_end(i, s, N):
    return min(N, 2 * s * (i // (2 * s) + 2))


def test_j_end_spec_examples():
    # SPEC.md:131-134 (s=32): i=0,70,130 -> 128, 192, 256
    assert [j_end(i, 32, 4096) for i in (0, 70, 130)] == [128, 192, 256]


@pytest.mark.parametrize("n,s_hat,s_expect", [(1024, 0, 32), (2048, 0, 32), (4096, 0, 32), (640, 32, 20),
                                               (1984, 0, 31), (1300, 0, 21), (1200, 0, 38)])
def test_exact_cover_of_submatrices_and_band(n, s_hat, s_expect):
    # every (i, j), j >= i, is covered exactly once: by the band (j < j_end(i)) or by exactly one
    # submatrix (g, b, r) with corners eq:globalij and size 2h_g
    from paper_2411_00033_b200 import geometry
    g = geometry(n, s_hat)
    L, s, N = g["L"], g["s"], g["N"]
    assert s == s_expect
    cover = np.zeros((N, N), dtype=np.int32)
    for i in range(N):
        cover[i, i:j_end(i, s, N)] += 1
    for gg in range(L):
        h = s << (L - gg - 1)
        for b in range((1 << (gg + 1)) - 1):
            for p, q in ((0, 0), (0, 1), (1, 1)):
                i0, j0 = 2 * h * (2 * b + p), 2 * h * (2 * b + q + 2)
                cover[i0:i0 + 2 * h, j0:j0 + 2 * h] += 1
    upper = np.triu(np.ones((N, N), dtype=bool))
    assert np.all(cover[upper] == 1) and np.all(cover[~upper] == 0)


def test_band_nnz_is_about_1p5_sN():
    from paper_2411_00033_b200 import geometry
    for n in (4096, 1 << 16, 10**6):
        g = geometry(n)
        assert abs(g["band_nnz"] / (1.5 * g["s"] * g["N"]) - 1) < 0.05
    # exact against brute force over every row (the library sums one interior segment and the last two)
    for n, s_hat in ((4096, 0), (1, 0), (37, 0), (130, 16), (1000, 24), (5001, 64), (65537, 0), (30000, 48)):
        g = geometry(n, s_hat)
        N, s = g["N"], g["s"]
        brute = sum((j_end(i, s, N) - i + 1) // 2 for i in range(N))
        assert g["band_nnz"] == brute, (n, s_hat)


def test_flop_model_lemma2():
    # eq:totalnumflopsnew: (mu s + 4M + 8M^2/s) N; 249N at s=32, M=18, mu=3; optimum s=29
    M, mu = 18, 3
    f = lambda s: mu * s + 4 * M + 8 * M * M / s
    assert round(f(32)) == 249
    assert min(range(8, 80), key=f) == 29
    nodal = lambda s: mu * s + 4 * M + 14 * M * M / s
    assert 300 <= nodal(32) <= 320
    # the library's per-vector algorithmic flops at 2^20: same order (exact nnz, exact block counts)
    from paper_2411_00033_b200 import geometry
    g = geometry(1 << 20)
    assert 230 <= g["flops_alg"] / g["N"] <= 260


# ---------------------------------------------------------------- B(l) exactly (App. A3)
def B_from_W(l, M=18):
    """B(l) = W^{-1} V(l) W with the closed forms of App. A3, in exact rationals."""
    W = [[Fraction(0)] * M for _ in range(M)]
    Wi = [[Fraction(0)] * M for _ in range(M)]
    V = [[Fraction(0)] * M for _ in range(M)]
    for n in range(M):
        for j in range(n + 1):
            if (n - j) % 2 == 0:
                cj = 2 if j == 0 else 1
                W[n][j] = Fraction(2, cj * 2 ** n) * math.comb(n, (n - j) // 2)
                Wi[n][j] = Fraction(1) if n == j == 0 else Fraction(n * (-1) ** ((n - j) // 2) * 2 ** j, n + j) * \
                    math.comb((n + j) // 2, (n - j) // 2)
            V[n][j] = Fraction(math.comb(n, n - j) * (2 * l - 1) ** (n - j), 2 ** n)
    mul = lambda X, Y: [[sum(X[i][k] * Y[k][j] for k in range(M)) for j in range(M)] for i in range(M)]
    I = mul(W, Wi)
    assert all(I[i][j] == (1 if i == j else 0) for i in range(M) for j in range(M))  # W W^{-1} = I
    return mul(mul(Wi, V), W)


def test_B_matrices_exact_and_printed_rows():
    B0, B1 = B_from_W(0), B_from_W(1)
    # printed rows 0-3 (tests/golden/paper_printed_values.txt)
    F = Fraction
    assert B0[1][:2] == [F(-1, 2), F(1, 2)] and B0[2][:3] == [F(-1, 4), -1, F(1, 4)]
    assert B0[3][:4] == [F(1, 4), F(3, 8), F(-3, 4), F(1, 8)]
    assert B1[1][:2] == [F(1, 2), F(1, 2)] and B1[2][:3] == [F(-1, 4), 1, F(1, 4)]
    assert B1[3][:4] == [F(-1, 4), F(3, 8), F(3, 4), F(1, 8)]
    # B(1) = B(0) with the odd diagonals negated; lower triangular; dyadic (exact in fp64)
    for n in range(18):
        for k in range(18):
            assert B1[n][k] == (-1) ** (n - k) * B0[n][k]
            assert k <= n or B0[n][k] == 0
            assert B0[n][k].denominator & (B0[n][k].denominator - 1) == 0
            assert float(B0[n][k]) == B0[n][k]
    # eq:Tky at a random point: T_n((Y-1)/2) = sum_k b_nk T_k(Y)
    Y = 0.3
    T = lambda k, x: math.cos(k * math.acos(x))
    for n in range(18):
        assert abs(sum(float(B0[n][k]) * T(k, Y) for k in range(18)) - T(n, (Y - 1) / 2)) < 1e-13


def test_library_B0_equals_exact_construction():
    # the library builds B(0) with the Chebyshev-basis recurrence (lc_plan.cu build_B0);
    # the fmm_model uses the same recurrence in numpy: both must equal W^{-1} V W exactly
    import fmm_model
    B0 = B_from_W(0)
    Bm = fmm_model.B0()
    assert all(Bm[n, k] == B0[n][k] for n in range(18) for k in range(18))


# ---------------------------------------------------------------- Lambda: eq:tau
def test_tau_series_thresholds():
    import mpmath
    mpmath.mp.dps = 40
    c = [1, -1 / 2**6, 21 / 2**13, -671 / 2**19, 180323 / 2**27]
    assert all(float(mpmath.mpf(x)) == x for x in c)  # all five exact dyadics (reading R5)

    def tau_exact(z):
        z = mpmath.mpf(z)
        return mpmath.sqrt(z) * mpmath.gamma(z + mpmath.mpf(1) / 4) / mpmath.gamma(z + mpmath.mpf(3) / 4)

    for nterms, zmin in ((5, 19.88), (4, 40), (3, 134), (2, 1844)):
        z = mpmath.mpf(zmin) + mpmath.mpf(1) / 4  # tau(z + 1/4): argument of Lambda(zmin)
        approx = sum(c[i] / z ** (2 * i) for i in range(nterms))
        assert abs(approx / tau_exact(z) - 1) < 2.3e-16, (nterms, zmin)


# ---------------------------------------------------------------- readings, via the paper-notation model
@pytest.mark.parametrize("n", [5, 129, 1000, 3000])
@pytest.mark.parametrize("direction", ["l2c", "c2l"])
def test_fmm_model_matches_oracle(n, direction):
    # the readings R1-R6 of DESIGN.md (band staircase, skipped blocks, C2L kernel, padding),
    # exercised in the segment indexing of the CUDA kernels, reproduce the direct definition
    import fmm_model
    f = vector("uniform_r0", n, seed=1)
    z = fmm_model.execute(fmm_model.plan(n, direction), f)
    tol = 5e-15 if direction == "l2c" else 5e-13  # Table 1 magnitudes (tests/golden/paper_table1.txt)
    assert oracle.einf(z, oracle.transform_rows(direction, f)) < tol
