"""Independent O(N log N) modal FMM of the paper's Sec. 3 (Alg. 2 MATVECBLOCK + Alg. 3),
in numpy fp64, with its OWN Chebyshev coefficient matrices A_hat -- test infrastructure (NEXT-3).

It shares nothing with the CUDA path (no plan export, no kernel code): A_hat(g, b, r) is built here
from eq:aklmore -- the kernel sampled on the Chebyshev-Gauss grid of each submatrix
(corners eq:globalij, affine map eq:Xfromx) with Lambda(z) = Gamma(z+1/2)/Gamma(z+1) evaluated by
mpmath (30 digits, from the exact integer corners) and a library 2-D DCT-II (scipy.fft.dctn) -- and the matrix-vector product runs
level by level, block by block, parity by parity exactly as Alg. 3 / Alg. 2 state (no step 2/4
transfers, no tiles, no fusion), plus the direct band of Alg. 1 restricted to j < j_end(i)
(reading R4) and C^{-1} (L2C).  The entries of the band come from the oracle's
long-double lambda (the plain definition, PAPER.md:34-46 / eq:Lxymod).

Because the fast O(N) engines of the library restructure steps 2-4 and build A_hat
on the GPU, agreement of three things -- this model vs the oracle, the GPU plan's A_hat vs this
model's, and the GPU output vs this model -- checks the planner and step 3 independently of the GPU
path's own arithmetic.
"""
from __future__ import annotations

import mpmath
import numpy as np
from scipy.fft import dctn

import oracle

M = 18


def geometry(n: int, s_hat: int = 32):
    """eq:numlevels and eq:Ntot: L, s, N (L clamped at 0 for small n)."""
    lp = 0
    while (s_hat << lp) < n:
        lp += 1
    L = lp - 2 if lp >= 2 else 0
    s = -(-n // (1 << (L + 2)))
    return L, s, s << (L + 2)


def Lambda(z) -> mpmath.mpf:
    """Gamma(z+1/2)/Gamma(z+1) (eq:Lambda) by mpmath (caller's working precision)."""
    zz = mpmath.mpf(z)
    return mpmath.exp(mpmath.loggamma(zz + 0.5) - mpmath.loggamma(zz + 1))


def kernel(direction: str, i0: int, j0: int, h: int, X: float, Y: float) -> float:
    """The kernel at x = i0 + h(X+1), y = j0 + h(Y+1) (eq:Xfromx), evaluated at 30 digits from the exact
    integer corners (no cancellation in y - x for large i0, j0):
    L2C: A(x,y) = Lambda((y-x)/2) Lambda((y+x)/2);
    C2L: L(x,y) = 2(x+1/2)y / ((x+y)(x+y+1)(x-y+1)) Lambda((y-x)/2)/Lambda((x+y)/2) (eq:Lxymod)."""
    with mpmath.workdps(30):
        x = mpmath.mpf(i0) + mpmath.mpf(h) * (mpmath.mpf(float(X)) + 1)
        y = mpmath.mpf(j0) + mpmath.mpf(h) * (mpmath.mpf(float(Y)) + 1)
        lm, lp = Lambda((y - x) / 2), Lambda((y + x) / 2)
        if direction == "leg2cheb":
            return float(lm * lp)
        return float(2 * (x + mpmath.mpf(0.5)) * y / ((x + y) * (x + y + 1) * (x - y + 1)) * lm / lp)


def gauss_nodes() -> np.ndarray:
    """X^G_m = cos((m + 1/2) pi / M)."""
    return np.cos((np.arange(M) + 0.5) * np.pi / M)


def ahat(direction: str, L: int, s: int) -> dict:
    """{(g, b, r): A_hat} for every submatrix (eq:aklmore); sampled kernel -> 2-D DCT-II."""
    XG = gauss_nodes()
    ck = np.where(np.arange(M) == 0, 2.0, 1.0)
    scale = 1.0 / (np.outer(ck, ck) * M * M)  # 4/(c_k c_l M^2) with scipy's unnormalised DCT-II (factor 2 per axis)
    out = {}
    for g in range(L):
        h = s << (L - g - 1)
        for b in range((2 << g) - 1):
            for r, (p, q) in enumerate(((0, 0), (0, 1), (1, 1))):  # eq:cfrompq
                i0, j0 = 2 * h * (2 * b + p), 2 * h * (2 * b + q + 2)  # eq:globalij
                G = np.array([[kernel(direction, i0, j0, h, X, Y) for Y in XG] for X in XG])
                out[(g, b, r)] = dctn(G, type=2) * scale
    return out


def vandermonde(sigma: int, h: int) -> np.ndarray:
    """T(sigma, gamma)[m, k] = T_k(-1 + (2m + sigma)/h_gamma) (eq:Xs)."""
    X = -1.0 + (2 * np.arange(h) + sigma) / h
    return np.cos(np.outer(np.arccos(np.clip(X, -1, 1)), np.arange(M)))


def band_entries(direction: str, N: int, s: int, lam: np.ndarray):
    """(rows, cols, values) of A (L2C, before C^{-1}) or A^{-1}C (C2L) with i <= j < j_end(i)."""
    I, J, V = [], [], []
    seg = 2 * s
    for i in range(N):
        je = min(N, seg * (i // seg + 2))
        for j in range(i, je, 2):
            k, m = (j - i) // 2, (j + i) // 2
            if direction == "leg2cheb":
                v = lam[k] * lam[m]
            elif i == 0 and j == 0:
                v = 1.0
            else:
                v = 2 * (i + 0.5) * j / ((i + j) * (i + j + 1) * (i - j + 1)) * lam[k] / lam[m]
            I.append(i)
            J.append(j)
            V.append(float(v))
    return np.array(I), np.array(J), np.array(V)


class Alg3:
    """z = C^{-1} A f (leg2cheb) or A^{-1} C f (cheb2leg) by Alg. 3 (+ the direct band)."""

    def __init__(self, n: int, direction: str, s_hat: int = 32):
        self.n, self.direction = n, direction
        self.L, self.s, self.N = geometry(n, s_hat)
        self.A = ahat(direction, self.L, self.s)
        lam = oracle.lam(self.N + 1).astype(np.longdouble)
        self.band = band_entries(direction, self.N, self.s, lam)

    def __call__(self, f: np.ndarray) -> np.ndarray:
        N, L, s = self.N, self.L, self.s
        fp = np.zeros(N)
        fp[: self.n] = f
        z = np.zeros(N)
        I, J, V = self.band  # step 6 (Alg. 1 restricted to the band)
        np.add.at(z, I, V * fp[J])
        for sigma in (0, 1):  # Alg. 3
            for g in range(L):
                h = s << (L - g - 1)
                T = vandermonde(sigma, h)
                for b in range((2 << g) - 1):  # Alg. 2, MATVECBLOCK
                    c = np.zeros((2, M))
                    for q in (0, 1):
                        j0 = 2 * h * (2 * b + q + 2)
                        w = T.T @ fp[j0 + sigma: j0 + 2 * h: 2]  # w = T^T f^sigma(q)
                        for p in range(q + 1):
                            r = p + q * (q + 1) // 2
                            c[p] += self.A[(g, b, r)] @ w
                    for p in (0, 1):
                        i0 = 2 * h * (2 * b + p)
                        z[i0 + sigma: i0 + 2 * h: 2] += T @ c[p]
        if self.direction == "leg2cheb":  # C^{-1}
            z[0] /= np.pi
            z[1:] *= 2 / np.pi
        return z[: self.n]
