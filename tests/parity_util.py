"""Shared checks of the GPU parity tests (test infrastructure; no arithmetic of the method).

* `c4_rows`  -- SURVEY.md 8(c) C-4 row sample, with the tile boundaries at the plan's OWN s
               (2s-row tiles: s = 31 at n = 1e6, 20 at 1e7), plus every row of a few whole leaf
               tiles in the last 10% of the vector (so a wrong tail block is sampled whole).
* `check_rows` -- E_inf gate (eq:Einf) and the per-row diagnostic of SURVEY C-5,
               |z_i - z*_i| / sum_k |K_ik f_k|, asserted at DIAG.
* `blockwise_einf` -- E_inf per block of consecutive entries (each block normalised by its own
               max), so that errors in the tail of a decaying vector are not hidden by |x_0|.

Measured values are appended to $LC_PARITY_LOG (json lines) when that variable is set.
"""
from __future__ import annotations

import json
import os

import numpy as np

import oracle

# north-star gate (BASELINE.json): relative max norm <= 1e-12 for n <= 1e6, <= 1e-11 beyond
def gate(n: int) -> float:
    return 1e-12 if n <= 1_000_000 else 1e-11


# per-row diagnostic bound: error relative to the row's own scale sum_k |K_ik f_k|.  The FMM's
# low-rank blocks are accurate to ~1e-16 of their block scale and fp64 accumulation adds ~1e-16 per
# level, so ~1e-15 is expected (measured <= 1.4e-14 over every config, engine and s_hat, round 2);
# 1e-13 still flags any block whose result is wrong by more than 1e-13 of its own magnitude.
DIAG = 1e-13


def log(**kw):
    path = os.environ.get("LC_PARITY_LOG")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps(kw) + "\n")


def c4_rows(n: int, s: int, seed: int = 1, uniform: int = 2048, tiles: int = 256, tail_tiles: int = 4):
    """C-4 rows: `uniform` seeded rows, the first and last 256, both sides of `tiles` random 2s-tile
    boundaries {2su-1, 2su}, and all rows of `tail_tiles` random whole tiles in the last 10%."""
    rng = np.random.default_rng(seed)
    r = set(rng.choice(n, size=min(n, uniform), replace=False).tolist())
    r |= set(range(min(n, 256))) | set(range(max(0, n - 256), n))
    nt = max(1, n // (2 * s))
    for u in rng.integers(1, max(2, nt), size=tiles):
        r |= {int(2 * s * u - 1), int(2 * s * u)}
    lo = int(0.9 * nt)
    for u in rng.integers(lo, max(lo + 1, nt), size=tail_tiles):
        r |= set(range(int(2 * s * u), int(min(n, 2 * s * (u + 1)))))
    return np.array(sorted(x for x in r if 0 <= x < n), dtype=np.int64)


def check_rows(direction: str, f: np.ndarray, z: np.ndarray, rows: np.ndarray, tag: str = "",
               g: float | None = None, diag: float = DIAG):
    """z (the GPU output, full vector) against the oracle on `rows`: E_inf <= gate and per-row
    diagnostic <= diag.  Returns (einf, max diagnostic)."""
    n = f.shape[0]
    ref, ab = oracle.transform_rows(direction, f, rows, with_abs=True)
    zr = np.asarray(z)[rows]
    e = oracle.einf(zr, ref)
    d = float(np.max(np.abs(zr.astype(np.longdouble) - ref) / np.maximum(ab, np.longdouble(1e-300))))
    log(tag=tag, direction=direction, n=int(n), rows=int(rows.size), einf=e, diag=d)
    g = gate(n) if g is None else g
    assert e <= g, (tag, direction, "E_inf", e, g)
    assert d <= diag, (tag, direction, "per-row diagnostic", d, diag)
    return e, d


def blockwise_einf(y: np.ndarray, x: np.ndarray, block: int) -> float:
    """max over blocks of consecutive entries of ||y - x||_inf,b / ||x||_inf,b (blocks with x = 0 skipped)."""
    n = x.shape[0]
    nb = n // block
    yb = np.asarray(y[: nb * block], dtype=np.float64).reshape(nb, block)
    xb = np.asarray(x[: nb * block], dtype=np.float64).reshape(nb, block)
    den = np.abs(xb).max(axis=1)
    num = np.abs(yb - xb).max(axis=1)
    ok = den > 0
    worst = float(np.max(num[ok] / den[ok])) if ok.any() else 0.0
    if nb * block < n:
        xt, yt = np.asarray(x[nb * block:]), np.asarray(y[nb * block:])
        if np.abs(xt).max() > 0:
            worst = max(worst, float(np.abs(yt - xt).max() / np.abs(xt).max()))
    return worst


# round-trip bounds: global E_inf at the north-star gate; per 2s-block E_inf (each block relative to its
# own max) at BLOCK_RT.  Measured on the B200 (round 2, tests/test_gpu_fullsize.py): <= 1.4e-14 for
# inputs with random signs (normal, sign/(j+1), cfg3/cfg4), up to 3.2e-12 for the all-positive
# u_k/(k+1)^0.5 of PAPER.md:531 at n = 1e7 (the tail of the C2L sum cancels large positive partial sums,
# cf. the r = 0 round-trip remark of PAPER.md:553); 1e-10 keeps 30x margin and still flags a tail block
# that is wrong at 1e-10 of its own scale (tests/test_gpu_fullsize.py plants one at 1e-9).
BLOCK_RT = 1e-10
BLOCK_RT_SIGNED = 1e-13  # inputs with random signs
DIAG_MEASURED = 2.6e-14  # largest per-row diagnostic seen (tools/fuzz_parity.py, 3360 cases; the suite: 1.4e-14, C2L, s_hat = 24, n = 70001)


def check_round_trip(x: np.ndarray, y: np.ndarray, s: int, tag: str = "", block_bound: float = BLOCK_RT):
    n = x.shape[0]
    e = oracle.einf(y, x)
    eb = blockwise_einf(y, x, 2 * s)
    log(tag=tag, direction="round_trip", n=int(n), einf=e, block_einf=eb)
    assert e <= gate(n), (tag, "round trip E_inf", e)
    assert eb <= block_bound, (tag, "round trip per-block E_inf", eb)
    return e, eb
