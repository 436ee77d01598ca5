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


@pytest.mark.parametrize("direction", ["leg2cheb", "cheb2leg"])
@pytest.mark.parametrize("n", [4096, 1_000_000, 10_000_000])
def test_ahat_reconstructs_exact_entries(direction, n):
    dev = _dev()
    p = _plan(n, direction, device=dev)
    d = p.desc
    L, s = int(d["L"]), int(d["s"])
    A = p.export("ahat").reshape(-1, M, M)
    assert A.shape[0] == d["nc"]
    rng = np.random.default_rng(n % 1009 + (0 if direction == "leg2cheb" else 1))
    lam = oracle.lam(d["N"] + 1)
    worst = 0.0
    for g, b, r, q in _blocks(L, rng, per_level=4 if n > 10**6 else 6):
        pp, qq = (0, 0) if r == 0 else ((0, 1) if r == 1 else (1, 1))  # eq:cfrompq
        h = s << (L - g - 1)
        i0, j0 = 2 * h * (2 * b + pp), 2 * h * (2 * b + qq + 2)  # eq:globalij
        xs = rng.integers(i0, i0 + 2 * h, 3)
        vals, refs = [], []
        for x in xs:
            for y in (j0 + (x - i0) % 2, j0 + 2 * h - 2 + (x - i0) % 2, int(rng.integers(j0, j0 + 2 * h))):
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
        worst = max(worst, err)
        # M = 18 modes are "sufficient for full double precision"
        assert err < 5e-15, (direction, n, g, b, r, err)
    print(f"{direction} n={n}: worst block-relative reconstruction error {worst:.2e}")


def test_plan_time_reported():
    dev = _dev()
    p = _plan(1_000_000, "leg2cheb", device=dev)
    assert 0.0 < p.plan_device_ms < 50.0, p.plan_device_ms
