"""The device planner (NEXT-1) pinned directly: every sampled A_hat(g, b, r) reconstructs the exact
matrix entries of its submatrix, sum_kl A_hat_kl T_k(X) T_l(Y) = a_xy (eq:aklmore, PAPER.md:232-238,
with X = (x - i0)/h - 1, Y = (y - j0)/h - 1, eq:Xfromx, corners eq:globalij), for L2C (a_xy =
Lambda((y-x)/2) Lambda((y+x)/2)) and C2L (eq:Lxymod); exact entries come from the CPU oracle's rows
of unit vectors.  Also: lambda (every 8th from eq:tau) and the planner's device time.
"""
import numpy as np
import pytest
import torch

import oracle
from alg3_model import gauss_nodes, kernel

pytestmark = pytest.mark.gpu

M = 18


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


def _plan(*a, **k):
    from paper_2411_00033_b200 import Plan
    return Plan(*a, **k)


def _cheb(X):
    T = np.empty(M)
    T[0], T[1] = 1.0, X
    for k in range(2, M):
        T[k] = 2 * X * T[k - 1] - T[k - 2]
    return T


def _blocks(L, rng, per_level=6):
    """(g, b, r, arena index) samples: every block of levels 0-2, `per_level` random ones elsewhere,
    always including the first and last block of a level."""
    out = []
    for g in range(L):
        nb = (2 << g) - 1
        off = 3 * ((2 << g) - 2 - g)
        bs = range(nb) if g <= 2 else sorted({0, nb - 1} | set(rng.integers(0, nb, per_level).tolist()))
        for b in bs:
            for r in range(3):
                out.append((g, b, r, off + 3 * b + r))
    return out


def _exact_oracle(direction, x, y):
    """a_xy (L2C, before C^{-1}) or M_xy (C2L) as a row of the oracle applied to the unit vector e_y."""
    e = np.zeros(y + 1)
    e[y] = 1.0
    if direction == "leg2cheb":
        v = float(oracle.l2c_rows(e, [x])[0])
        return v * np.pi / (1.0 if x == 0 else 2.0)  # undo C^{-1}: a_xy itself
    return float(oracle.c2l_rows(e, [x])[0])


def _exact_lam(direction, x, y, lam):
    """The same entries from the oracle's long-double lambda table (PAPER.md:34-46 and eq:Lxymod), for
    large n where a full oracle row per entry is too slow; cross-checked against _exact_oracle."""
    k, m = (y - x) // 2, (y + x) // 2
    if direction == "leg2cheb":
        return float(lam[k] * lam[m])
    X, Y = np.longdouble(x), np.longdouble(y)
    return float(2 * (X + np.longdouble(0.5)) * Y / ((X + Y) * (X + Y + 1) * (X - Y + 1)) * (lam[k] / lam[m]))


# Chebyshev approximation error of M = 18 modes on a submatrix, at integer points including the block
# edges (X, Y = -1 and near +1), relative to the block's largest entry.  Measured (round 2): L2C <= 8e-15
# ("M = 18 is sufficient for full double precision"); C2L <= 2.3e-13 -- the kernel of
# eq:Lxymod is less smooth near the diagonal, cf. the C2L errors of Table 1.
APPROX = {"leg2cheb": 2e-14, "cheb2leg": 1e-12}


@pytest.mark.parametrize("direction", ["leg2cheb", "cheb2leg"])
@pytest.mark.parametrize("n", [4096, 1_000_000, 10_000_000])
def test_ahat_pins(direction, n):
    """(a) DCT exactness: T A_hat T^T at the Chebyshev-Gauss nodes reproduces the sampled kernel
    (eq:aklmore is the inverse of that evaluation), with the kernel evaluated independently by mpmath;
    (b) approximation: at integer points of the submatrix it reproduces the exact entries a_xy."""
    dev = _dev()
    p = _plan(n, direction, device=dev)
    d = p.desc
    L, s = int(d["L"]), int(d["s"])
    A = p.export("ahat").reshape(-1, M, M)
    assert A.shape[0] == d["nc"]
    rng = np.random.default_rng(n % 1009 + (0 if direction == "leg2cheb" else 1))
    lam = oracle.lam(d["N"] + 1)
    XG = gauss_nodes()
    TG = np.stack([_cheb(X) for X in XG])  # TG[m, k] = T_k(X_m)
    worst_nodes = worst_int = 0.0
    for g, b, r, q in _blocks(L, rng, per_level=2 if n > 10**6 else 4):
        pp, qq = (0, 0) if r == 0 else ((0, 1) if r == 1 else (1, 1))  # eq:cfrompq
        h = s << (L - g - 1)
        i0, j0 = 2 * h * (2 * b + pp), 2 * h * (2 * b + qq + 2)  # eq:globalij
        # (a) at the Gauss nodes x_m = i0 + h(X_m + 1), y_n = j0 + h(X_n + 1) (eq:Xfromx)
        if g <= 2 or rng.random() < 0.5:
            G = np.array([[kernel(direction, i0, j0, h, X, Y) for Y in XG] for X in XG])
            e = np.max(np.abs(TG @ A[q] @ TG.T - G)) / np.max(np.abs(G))
            worst_nodes = max(worst_nodes, e)
            assert e < 1e-14, ("nodes", direction, n, g, b, r, e)
        # (b) at integer points, block edges included
        xs = np.r_[i0, i0 + 2 * h - 1, rng.integers(i0, i0 + 2 * h, 2)]
        vals, refs = [], []
        for x in xs:
            for y in (j0, j0 + 2 * h - 1, int(rng.integers(j0, j0 + 2 * h))):
                y = int(y) + ((int(y) - int(x)) % 2)  # same parity as x (a nonzero entry of A)
                if y >= j0 + 2 * h:
                    y -= 2
                X, Y = (x - i0) / h - 1.0, (y - j0) / h - 1.0
                vals.append(_cheb(X) @ A[q] @ _cheb(Y))
                refs.append(_exact_lam(direction, int(x), y, lam))
                if n <= 4096:
                    assert abs(refs[-1] - _exact_oracle(direction, int(x), y)) <= 1e-15 * abs(refs[-1])
        vals, refs = np.array(vals), np.array(refs)
        err = np.max(np.abs(vals - refs)) / np.max(np.abs(refs))
        worst_int = max(worst_int, err)
        assert err < APPROX[direction], ("integer points", direction, n, g, b, r, err)
    print(f"{direction} n={n}: Gauss-node reconstruction {worst_nodes:.2e}, integer points {worst_int:.2e}")


def test_plan_time_reported():
    dev = _dev()
    p = _plan(1_000_000, "leg2cheb", device=dev)
    # the planner moves ~127 MB of A_hat for 1e6 (~20 us at HBM speed); 2 ms is a loose upper bound
    assert 0.0 < p.plan_device_ms < 2.0, p.plan_device_ms
