"""Test-side numpy model of the paper's O(N) modal FMM (Alg. 4).

TEST INFRASTRUCTURE ONLY (never imported by the product).  It is NOT the
oracle: the oracle (oracle/) is the direct O(n^2) definition.  This model
exists to (1) check on CPU, against the oracle, the readings DESIGN.md takes of
the paper (staircase band, skipped blocks, C2L kernel, padding) in the same
"segment" indexing the CUDA kernels use, and (2) provide intermediates (w, c)
for debugging the GPU path.  Written from the paper in numpy, sharing no code
with paper_2411_00033_b200/csrc.

Segment indexing: on level g (0..L-1) the padded
vector is cut into 2^(g+2) segments of length 2h_g = s 2^(L-g).  Column block
(g,b,q) of eq:globalij is segment t = 2b+q+2 and row block (g,b,p) is segment
u = 2b+p; the three submatrices r=0,1,2 of block b are (u,t) = (2b,2b+2),
(2b,2b+3), (2b+1,2b+3).  eq:flevels / eq:zlevels make segment t of level g
the union of segments 2t, 2t+1 of level g+1.
"""
from __future__ import annotations

import math

import numpy as np

M_DEFAULT = 18


def decomposition(n: int, s_hat: int = 32):
    """eq:numlevels: L = ceil(log2(n/s_hat)) - 2, s = ceil(n/2^(L+2)), N = s 2^(L+2).
    L is clamped at 0 (band-only) for n <= 4 s_hat (reading R6)."""
    lp = 0
    while (s_hat << lp) < n:
        lp += 1
    L = max(0, lp - 2)
    s = -(-n // (1 << (L + 2)))
    return L, s, s << (L + 2)


def Lambda(z):
    """Lambda(z) = tau(z+1/4)/sqrt(z+1/4), eq:tau, upward shift below 20."""
    z = np.asarray(z, dtype=np.float64)
    m = np.maximum(0, np.ceil(20.0 - z)).astype(np.int64)
    zz = z + m
    x = zz + 0.25
    y = 1.0 / (x * x)
    tau = 1 + y * (-1 / 2**6 + y * (21 / 2**13 + y * (-671 / 2**19 + y * 180323 / 2**27)))
    val = tau / np.sqrt(x)
    for i in range(int(m.max()) if m.size else 0):
        act = m > i
        # Lambda(w) = Lambda(w+1) (w+1)/(w+1/2),  w = zz - i - 1
        w = zz - i - 1
        val = np.where(act, val * (w + 1) / (w + 0.5), val)
    return val


def lambda_vec(n):
    lam = np.empty(n)
    lam[0] = math.sqrt(math.pi)
    for k in range(1, n):
        lam[k] = lam[k - 1] * (k - 0.5) / k
    return lam


def B0(M=M_DEFAULT):
    """T_n((Y-1)/2) = sum_k b_nk T_k(Y) (eq:Tky, l=0). P_{n+1} = (Y-1) P_n - P_{n-1} in the Chebyshev basis."""
    B = np.zeros((M, M))
    B[0, 0] = 1.0
    if M > 1:
        B[1, 0], B[1, 1] = -0.5, 0.5
    for n in range(1, M - 1):
        y = np.zeros(M)
        for k in range(n + 1):
            c = B[n, k]
            if k == 0:
                y[1] += c
            else:
                y[k + 1] += c / 2
                y[k - 1] += c / 2
        B[n + 1] = y - B[n] - B[n - 1]
    return B


def vandermonde(s, sigma, M=M_DEFAULT):
    X = -1.0 + (2 * np.arange(s) + sigma) / s
    return np.cos(np.outer(np.arccos(np.clip(X, -1, 1)), np.arange(M)))


def kernel(direction, i0, j0, h, M=M_DEFAULT):
    """Kernel samples on the Gauss grid of the submatrix with corner (i0, j0), half size h."""
    xg = np.cos((np.arange(M) + 0.5) * np.pi / M)
    dx = h * (xg + 1.0)
    # (y-x)/2 and (x+y)/2 formed from exact integer corner offsets (no cancellation)
    ymx = (j0 - i0) / 2 + (dx[None, :] - dx[:, None]) / 2
    xpy = (i0 + j0) / 2 + (dx[None, :] + dx[:, None]) / 2
    lm, lp = Lambda(ymx), Lambda(xpy)
    if direction == "l2c":
        return lm * lp
    x = i0 + dx[:, None]
    y = j0 + dx[None, :]
    # eq:Lxymod with x-y+1 = -(2 ymx) + 1 and x+y = 2 xpy
    return 2 * (x + 0.5) * y / ((2 * xpy) * (2 * xpy + 1) * (1 - 2 * ymx)) * lm / lp


def ahat(G, M=M_DEFAULT):
    """eq:aklmore: a_kl = 4/(c_k c_l M^2) sum_mn G_mn cos(k(m+1/2)pi/M) cos(l(n+1/2)pi/M)."""
    C = np.cos(np.outer(np.arange(M), np.arange(M) + 0.5) * np.pi / M)
    c = np.ones(M)
    c[0] = 2
    return 4.0 / (M * M) * (C @ G @ C.T) / np.outer(c, c)


def plan(n, direction, s_hat=32, M=M_DEFAULT):
    L, s, N = decomposition(n, s_hat)
    A = []
    for g in range(L):
        h = s << (L - g - 1)
        for b in range((1 << (g + 1)) - 1):
            for (p, q) in ((0, 0), (0, 1), (1, 1)):
                i0 = 2 * h * (2 * b + p)
                j0 = 2 * h * (2 * b + q + 2)
                A.append(ahat(kernel(direction, i0, j0, h, M), M))
    return dict(L=L, s=s, N=N, M=M, n=n, dir=direction, A=np.array(A).reshape(-1, M, M),
                B=B0(M), T=[vandermonde(s, 0, M), vandermonde(s, 1, M)], lam=lambda_vec(N))


def execute(P, f, return_work=False):
    L, s, N, M, n = P["L"], P["s"], P["N"], P["M"], P["n"]
    fp = np.zeros(N)
    fp[:n] = f
    z = np.zeros(N)
    B = P["B"]
    sgn = (-1.0) ** np.subtract.outer(np.arange(M), np.arange(M))
    Bl = [B, B * sgn]
    aoff = [3 * ((1 << (g + 1)) - 2 - g) for g in range(L + 1)]
    work = []
    for sig in (0, 1):
        if L == 0:
            break
        w = [None] * L
        c = [None] * L
        nseg = 1 << (L + 1)
        fs = fp.reshape(nseg, 2 * s)[:, sig::2]                      # f^sigma per leaf segment
        w[L - 1] = fs @ P["T"][sig]                                    # step 1 (eq:wMM), all segments
        for g in range(L - 1, 0, -1):                                  # step 2 (eq:wtk)
            ch = w[g].reshape(-1, 2, M)
            w[g - 1] = ch[:, 0] @ Bl[0].T + ch[:, 1] @ Bl[1].T
        for g in range(L):                                             # step 3 (M2L)
            nr = (1 << (g + 2)) - 2
            cg = np.zeros((1 << (g + 2), M))
            A = P["A"][aoff[g]: aoff[g + 1]].reshape(-1, 3, M, M)
            u = np.arange(0, nr, 2)
            cg[u] += np.einsum("bkl,bl->bk", A[:, 0], w[g][u + 2]) + np.einsum("bkl,bl->bk", A[:, 1], w[g][u + 3])
            cg[u + 1] += np.einsum("bkl,bl->bk", A[:, 2], w[g][u + 3])
            c[g] = cg
        for g in range(L - 1):                                         # step 4 (L2L)
            par = c[g][: (1 << (g + 2)) - 2]
            c[g + 1][0: 2 * len(par): 2] += par @ Bl[0]
            c[g + 1][1: 2 * len(par): 2] += par @ Bl[1]
        zs = c[L - 1] @ P["T"][sig].T                                  # step 5 (eq:step5)
        z.reshape(nseg, 2 * s)[:, sig::2] += zs
        work.append((w, c))
    # step 6: direct band i <= j < j_end(i) = min(N, 2s(floor(i/2s)+2))
    lam = P["lam"]
    for i in range(N):
        je = min(N, 2 * s * (i // (2 * s) + 2))
        k = np.arange((je - i + 1) // 2)
        j = i + 2 * k
        if P["dir"] == "l2c":
            z[i] += np.sum(lam[k] * lam[i + k] * fp[j])
        else:
            if i == 0:
                ent = np.empty(len(k))
                ent[0] = 1.0
                kk = k[1:]
                ent[1:] = (2 * i + 1) * j[1:] / (2.0 * (i + kk) * (2 * i + 2 * kk + 1) * (1 - 2 * kk)) * lam[kk] / lam[i + kk]
            else:
                ent = (2 * i + 1) * j / (2.0 * (i + k) * (2 * i + 2 * k + 1) * (1 - 2 * k)) * lam[k] / lam[i + k]
            z[i] += np.sum(ent * fp[j])
    if P["dir"] == "l2c":                                              # step 7: C^{-1}
        z[0] /= np.pi
        z[1:] *= 2 / np.pi
    out = z[:n]
    return (out, work) if return_work else out
