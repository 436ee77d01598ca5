"""Full-size parity that can fail ("next round" item 1).

* Non-decaying inputs (`normal`, `uniform_r0.5`) at L = 13 .. 17 for the single-vector engine
  (engine 1) and the long-vector batch engine (engine 3), so that every block of the hierarchy
  carries a result of the same magnitude as row 0 and an error anywhere shows in E_inf.
* Rows per SURVEY C-4 with the tile boundaries at the plan's own s (31, 32, 20, ...), plus whole
  tiles in the last 10% (tests/parity_util.c4_rows).
* The per-row diagnostic |z_i - z*_i| / sum_k |K_ik f_k| (SURVEY C-5) on every sampled row.
* Round trips over ALL entries, globally and per 2s-block (each block against its own scale).
* A planted tail-block error must make these checks fail (the checks can fail).

Gates: the north-star relative max norm (1e-12 for n <= 1e6, 1e-11 beyond) and DIAG (parity_util).
"""
import numpy as np
import pytest
import torch

from lc_inputs import batch, vector
from parity_util import BLOCK_RT, BLOCK_RT_SIGNED, blockwise_einf, c4_rows, check_round_trip, check_rows

pytestmark = pytest.mark.gpu


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


def _plan(*a, **k):
    from paper_2411_00033_b200 import Plan
    return Plan(*a, **k)


# (n, L, s) at the default s_hat = 40: 1e6 -> L 13, s 31; 2^20 -> L 13, s 32; 4e6+17 -> L 15, s 31;
# 1e7 -> L 16, s 39 (s_hat = 32: L 17, s 20)
@pytest.mark.parametrize("kind", ["normal", "uniform_r0.5"])
@pytest.mark.parametrize("n,s_hat", [(1_000_000, 0), (1 << 20, 0), (4_000_017, 0), (10_000_000, 0), (10_000_000, 32)])
def test_single_vector_nondecaying(n, s_hat, kind):
    dev = _dev()
    f = vector(kind, n, seed=101)
    x = torch.from_numpy(f).reshape(1, -1).to(dev)
    pl, pc = _plan(n, "leg2cheb", device=dev, s_hat=s_hat), _plan(n, "cheb2leg", device=dev, s_hat=s_hat)
    assert pl.kernel_info["engine"] == 1
    s = pl.desc["s"]
    z = pl.execute(x)
    y = pc.execute(z)
    w = pc.execute(x)  # cheb2leg of the same non-decaying input
    zh, yh, wh = (t.cpu().numpy()[0] for t in (z, y, w))
    rows = c4_rows(n, s)
    tag = f"engine1 n={n} L={pl.desc['L']} s={s} {kind}"
    check_rows("leg2cheb", f, zh, rows, tag)
    check_rows("cheb2leg", f, wh, rows, tag)
    check_round_trip(f, yh, s, tag, BLOCK_RT_SIGNED if kind == "normal" else BLOCK_RT)


# engine 3 (8-vector tiles: up pass + per-range pass) on long non-decaying vectors
@pytest.mark.parametrize("n,V,kind,s_hat", [(2_000_000, 16, "normal", 0), (10_000_000, 8, "uniform_r0.5", 0),
                                             (10_000_000, 8, "normal", 32), (3_000_005, 11, "normal", 0)])
def test_engine3_long_vectors_nondecaying(n, V, kind, s_hat):
    dev = _dev()
    xh = batch(kind, n, V, seed=202)
    x = xh.to(dev)
    pl = _plan(n, "leg2cheb", batch=V, device=dev, engine=3, s_hat=s_hat)
    pc = _plan(n, "cheb2leg", batch=V, device=dev, engine=3, s_hat=s_hat)
    assert pl.kernel_info["engine"] == 3 and pc.kernel_info["engine"] == 3
    s = pl.desc["s"]
    z = pl.execute(x)
    y = pc.execute(z)
    w = pc.execute(x)
    torch.cuda.synchronize()
    rows = c4_rows(n, s)
    vs = (0, V - 1) if n >= 10_000_000 else (0, V // 2, V - 1)
    for v in vs:
        tag = f"engine3 n={n} V={V} v={v} L={pl.desc['L']} s={s} {kind}"
        check_rows("leg2cheb", xh[v].numpy(), z[v].cpu().numpy(), rows, tag)
        check_rows("cheb2leg", xh[v].numpy(), w[v].cpu().numpy(), rows, tag)
    yh = y.cpu().numpy()
    for v in range(V):
        check_round_trip(xh[v].numpy(), yh[v], s, f"engine3 n={n} V={V} v={v} {kind}",
                         BLOCK_RT_SIGNED if kind == "normal" else BLOCK_RT)


@pytest.mark.parametrize("engine", [1, 2, 3])
@pytest.mark.parametrize("s_hat", [16, 24, 32, 48, 64])
def test_s_hat_variants(engine, s_hat):
    """opts.s_hat in [2, 64] changes s, L and the band blocking (SMAX = 64 instantiations for s > 32);
    engines 2 and 3 take s <= 40 (5 row tiles) and reject larger s at plan time."""
    from paper_2411_00033_b200 import geometry
    from paper_2411_00033_b200._lib import LegChebError
    dev = _dev()
    for n, V in ((5000, 9), (70001, 8), (600, 9)):
        xh = batch("normal", n, V, seed=s_hat + n)
        try:
            pl = _plan(n, "leg2cheb", batch=V, device=dev, engine=engine, s_hat=s_hat)
            pc = _plan(n, "cheb2leg", batch=V, device=dev, engine=engine, s_hat=s_hat)
        except LegChebError:
            assert engine in (2, 3) and geometry(n, s_hat)["s"] > 40
            continue
        s = pl.desc["s"]
        assert s_hat // 2 <= s <= s_hat or pl.desc["L"] == 0
        z = pl.execute(xh.to(dev)).cpu().numpy()
        w = pc.execute(xh.to(dev)).cpu().numpy()
        rows = np.arange(n) if n <= 5000 else c4_rows(n, s, uniform=512, tiles=64)
        for v in (0, V - 1):
            tag = f"s_hat={s_hat} engine={engine} n={n} s={s} L={pl.desc['L']}"
            check_rows("leg2cheb", xh[v].numpy(), z[v], rows, tag)
            check_rows("cheb2leg", xh[v].numpy(), w[v], rows, tag)


# engines 2 and 3 at s in (32, 40] (row tile 4 of the band and of step 5; T(sigma) staged with 40 rows;
# the up pass with the 64-row T copy and subtrees of 4 leaves packing two vectors per MMA item), against
# engine 1 and the oracle, both directions, ragged tiles and tails; s = 33 / 36 / 39 / 40
@pytest.mark.parametrize("engine", [1, 2, 3])
@pytest.mark.parametrize("n,V", [(2105, 9), (9215, 16), (39836, 11), (163840, 8), (1_277_951, 8)])
def test_s_above_32(engine, n, V):
    from paper_2411_00033_b200._lib import LegChebError
    dev = _dev()
    xh = batch("normal", n, V, seed=n % 1000 + V)
    x = xh.to(dev)
    try:
        pl = _plan(n, "leg2cheb", batch=V, device=dev, engine=engine)
        pc = _plan(n, "cheb2leg", batch=V, device=dev, engine=engine)
    except LegChebError:
        assert engine == 3 and n < 100_000  # engine 3 wants L >= 1 and ranges; small cases may be refused
        return
    s, L = pl.desc["s"], pl.desc["L"]
    assert 32 < s <= 40, s
    assert pl.kernel_info["engine"] == engine
    z = pl.execute(x)
    w = pc.execute(x)
    y = pc.execute(z)
    torch.cuda.synchronize()
    rows = np.arange(n) if n <= 10000 else c4_rows(n, s, uniform=512, tiles=32)
    zh, wh, yh = z.cpu().numpy(), w.cpu().numpy(), y.cpu().numpy()
    for v in sorted({0, V // 2, V - 1}):
        tag = f"s>32 engine={engine} n={n} V={V} v={v} s={s} L={L}"
        check_rows("leg2cheb", xh[v].numpy(), zh[v], rows, tag)
        check_rows("cheb2leg", xh[v].numpy(), wh[v], rows, tag)
        check_round_trip(xh[v].numpy(), yh[v], s, tag, BLOCK_RT_SIGNED)


def test_planted_tail_block_error_is_caught():
    """The checks above can fail: perturb one 2s-row block in the last 5% of one vector's leg2cheb
    output by 1e-9 of its magnitude (a plausible tail-block bug) and the round-trip checks must flag
    it (it need not be among the sampled rows)."""
    dev = _dev()
    n, V = 2_000_000, 16
    xh = batch("normal", n, V, seed=202)
    x = xh.to(dev)
    pl = _plan(n, "leg2cheb", batch=V, device=dev, engine=3)
    pc = _plan(n, "cheb2leg", batch=V, device=dev, engine=3)
    s = pl.desc["s"]
    z = pl.execute(x)
    rng = np.random.default_rng(7)
    u = int(rng.integers(int(0.95 * n) // (2 * s), n // (2 * s) - 1))
    v = 5
    blk = z[v, 2 * s * u: 2 * s * (u + 1)]
    blk += 1e-9 * blk.abs().max()  # the planted error
    y = pc.execute(z).cpu().numpy()
    with pytest.raises(AssertionError):
        check_round_trip(xh[v].numpy(), y[v], s, "planted")
    # the per-block check alone catches it too, even at the loose (all-positive input) bound
    assert blockwise_einf(y[v], xh[v].numpy(), 2 * s) > BLOCK_RT
    # and the untouched vectors still pass
    check_round_trip(xh[4].numpy(), y[4], s, "planted-neighbour", BLOCK_RT_SIGNED)


# the engine-3 up pass with one f buffer (8-leaf subtrees at s > 32 when two double-buffered CTAs do not
# fit) and with two (forced by LC_UP3_NBUF, read at plan creation): bit-identical results, oracle rows
@pytest.mark.parametrize("n,V", [(1_277_951, 8), (400_001, 16), (2_000_000, 9)])
def test_engine3_up_pass_buffering(n, V, monkeypatch):
    dev = _dev()
    xh = batch("normal", n, V, seed=31 + V)
    x = xh.to(dev)
    outs, infos = {}, {}
    for nbuf in ("1", "2"):
        monkeypatch.setenv("LC_UP3_NBUF", nbuf)
        p = _plan(n, "leg2cheb", batch=V, device=dev, engine=3)
        infos[nbuf] = p.kernel_info
        outs[nbuf] = p.execute(x).cpu().numpy()
        p.close()
    monkeypatch.delenv("LC_UP3_NBUF")
    assert np.array_equal(outs["1"], outs["2"])  # same arithmetic, different staging
    s = _plan(n, "leg2cheb", batch=V, device=dev, engine=3).desc["s"]
    rows = c4_rows(n, s, uniform=256, tiles=16)
    for v in (0, V - 1):
        check_rows("leg2cheb", xh[v].numpy(), outs["1"][v], rows, f"engine3 up nbuf n={n} V={V} v={v}")
