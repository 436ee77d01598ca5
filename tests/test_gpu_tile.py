"""GPU parity of the per-tile streaming kernel (engine 2: one CTA per 8-vector tile runs the whole
of Alg. 4 in one right-to-left pass over the leaf segments) against the CPU oracle.

Cases span L = 1 .. 8, odd and even s, ragged batches (not a multiple of the 8-vector tile), both
layouts, both directions and round trips; the gate is the north-star 1e-12 relative max norm.
"""
import numpy as np
import pytest
import torch

import oracle
from lc_inputs import batch

pytestmark = pytest.mark.gpu

GATE = 1e-12


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


def _plan(*a, **k):
    from paper_2411_00033_b200 import Plan
    return Plan(*a, **k)


# (n, V) at the default s_hat = 40: n = 161 -> L = 1, s = 21; 1500 -> s = 24, L = 4; 3900 -> s = 31 (odd);
# 4096 -> L = 5, s = 32; 5000 -> L = 5, s = 40; 8192 -> L = 6; 20000 -> L = 7, s = 40; 39836 -> s = 39
CASES = [(161, 8), (200, 13), (1000, 9), (1500, 3), (3900, 17), (4096, 8), (5000, 11), (8192, 10), (20000, 5),
         (39836, 9)]


@pytest.mark.parametrize("direction", ["leg2cheb", "cheb2leg"])
@pytest.mark.parametrize("n,V", CASES)
def test_tile_engine_vs_oracle(direction, n, V):
    dev = _dev()
    x = batch("normal_exp1000", n, V, seed=11)
    p = _plan(n, direction, batch=V, device=dev, engine=2)
    assert p.kernel_info["engine"] == 2 and p.kernels_per_execute == 1
    z = p.execute(x.to(dev)).cpu().numpy()
    for v in range(V):
        e = oracle.einf(z[v], oracle.transform_rows(direction, x[v].numpy()))
        assert e <= GATE, (n, V, v, direction, e, p.desc)


@pytest.mark.parametrize("direction", ["leg2cheb", "cheb2leg"])
def test_tile_engine_batch_layout_and_ld(direction):
    dev = _dev()
    n, V = 3000, 12
    x = batch("normal", n, V, seed=5)
    pv = _plan(n, direction, batch=V, device=dev, engine=2)
    pb = _plan(n, direction, batch=V, device=dev, layout="batch", engine=2)
    zv = pv.execute(x.to(dev))
    zb = pb.execute(x.t().contiguous().to(dev))
    assert torch.equal(zv, zb.t().contiguous())  # same arithmetic, only the addressing differs
    # padded leading dimensions (VEC layout): ld_in = n + 7, ld_out = n + 3
    xin = torch.zeros(V, n + 7, dtype=torch.float64)
    xin[:, :n] = x
    pl = _plan(n, direction, batch=V, device=dev, engine=2, ld_in=n + 7, ld_out=n + 3)
    out = torch.full((V, n + 3), 7.0, dtype=torch.float64, device=dev)
    pl.execute(xin.to(dev), out=out)
    assert torch.equal(out[:, :n], zv)
    assert torch.all(out[:, n:] == 7.0)  # nothing written past n


def test_tile_engine_matches_level_pipeline():
    dev = _dev()
    n, V = 4096, 24
    xh = batch("normal_exp1000", n, V, seed=6)
    x = xh.to(dev)
    for direction in ("leg2cheb", "cheb2leg"):
        p1 = _plan(n, direction, batch=V, device=dev, engine=1)
        p2 = _plan(n, direction, batch=V, device=dev, engine=2)
        # outputs pre-filled with NaN: every row must be written by either engine
        z1 = torch.full_like(x, float("nan"))
        z2 = torch.full_like(x, float("nan"))
        p1.execute(x, out=z1)
        p2.execute(x, out=z2)
        torch.cuda.synchronize()
        e = (z1 - z2).abs().max().item() / z1.abs().max().item()
        if not e <= 1e-13:
            zs = [oracle.transform_rows(direction, xh[v].numpy()) for v in range(V)]
            e1 = [oracle.einf(z1[v].cpu().numpy(), zs[v]) for v in range(V)]
            e2 = [oracle.einf(z2[v].cpu().numpy(), zs[v]) for v in range(V)]
            raise AssertionError((direction, e, "engine1 vs oracle", max(e1), "engine2 vs oracle", max(e2)))


@pytest.mark.parametrize("n", [1000, 4096])
def test_tile_engine_round_trip(n):
    dev = _dev()
    V = 16
    x = batch("normal_exp1000", n, V, seed=7).to(dev)
    a = _plan(n, "leg2cheb", batch=V, device=dev, engine=2)
    b = _plan(n, "cheb2leg", batch=V, device=dev, engine=2)
    back = b.execute(a.execute(x)).cpu().numpy()
    xs = x.cpu().numpy()
    for v in range(V):
        assert oracle.einf(back[v], xs[v]) <= GATE


def test_tile_engine_automatic_choice():
    dev = _dev()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    big = _plan(4096, "leg2cheb", batch=4096, device=dev)  # cfg3: 512 tiles >= 2 per SM
    assert big.kernel_info["engine"] == 2 and big.kernel_info["tile_grid"] <= 512
    assert big.kernel_info["tile_grid"] <= 2 * sms * 2
    few = _plan(4096, "leg2cheb", batch=16, device=dev)  # 2 tiles: level-pipelined kernels
    assert few.kernel_info["engine"] == 1 and few.kernels_per_execute == 3
    with pytest.raises(RuntimeError):
        _plan(100, "leg2cheb", batch=8, device=dev, engine=2)  # L = 0: no hierarchy to stream


def test_tile_engine_back_to_back_and_zero_vectors():
    dev = _dev()
    n, V = 2000, 20
    p = _plan(n, "leg2cheb", batch=V, device=dev, engine=2)
    x1 = batch("normal", n, V, seed=8).to(dev)
    x2 = torch.zeros_like(x1)
    z1a = p.execute(x1)
    z2 = p.execute(x2)
    z1b = p.execute(x1)
    assert torch.equal(z1a, z1b)
    assert torch.count_nonzero(z2) == 0
    np.testing.assert_array_equal(z1a.cpu().numpy()[3], p.execute(x1).cpu().numpy()[3])


# engine 3: up kernel (8-vector tiles) + the per-range pass; ranges split the leaves of each tile
# (n = 100000 -> L = 10 with 8 levels of c in the global scratch)
@pytest.mark.parametrize("direction", ["leg2cheb", "cheb2leg"])
@pytest.mark.parametrize("n,V", [(161, 8), (1000, 9), (4096, 8), (20000, 5), (39836, 9), (100000, 16)])
def test_range_engine_vs_oracle(direction, n, V):
    dev = _dev()
    x = batch("normal_exp1000", n, V, seed=12)
    p = _plan(n, direction, batch=V, device=dev, engine=3)
    assert p.kernel_info["engine"] == 3 and p.kernels_per_execute == 2
    z = p.execute(x.to(dev)).cpu().numpy()
    vs = range(V) if n <= 20000 else (0, V - 1)
    for v in vs:
        e = oracle.einf(z[v], oracle.transform_rows(direction, x[v].numpy()))
        assert e <= GATE, (n, V, v, direction, e, p.desc)


def test_range_engine_matches_level_pipeline():
    dev = _dev()
    n, V = 100000, 24
    x = batch("normal_exp1000", n, V, seed=13).to(dev)
    for direction in ("leg2cheb", "cheb2leg"):
        p1 = _plan(n, direction, batch=V, device=dev, engine=1)
        p3 = _plan(n, direction, batch=V, device=dev, engine=3)
        z1 = torch.full_like(x, float("nan"))
        z3 = torch.full_like(x, float("nan"))
        p1.execute(x, out=z1)
        p3.execute(x, out=z3)
        torch.cuda.synchronize()
        e = (z1 - z3).abs().max().item() / z1.abs().max().item()
        assert e <= 1e-13, (direction, e)


def test_range_engine_automatic_choice():
    # engine 3 from ~1.6e6 coefficients in batches of >= 8 vectors (tools/engine_cross_all.py)
    dev = _dev()
    p = _plan(1000000, "leg2cheb", batch=16, device=dev)  # L = 13, 2 tiles: engine 3
    assert p.kernel_info["engine"] == 3 and p.kernel_info["range_len"] >= 8
    r = _plan(65536, "leg2cheb", batch=16, device=dev)  # 1.05e6 coefficients: level-pipelined kernels
    assert r.kernel_info["engine"] == 1
    q = _plan(100000, "leg2cheb", batch=1, device=dev)  # single vector: level-pipelined kernels
    assert q.kernel_info["engine"] == 1
    with pytest.raises(RuntimeError):
        _plan(100000, "leg2cheb", batch=8, device=dev, engine=4)


def test_range_engine_staging_paths_and_continuation():
    # n = 300000: L = 12, s = 19 (general band path), chunk roots on level 2 -> cross-chunk continuation
    # of the persistent up pass; V = 9: a ragged second tile; an odd ld_in forces the 8-byte staging path,
    # the batch layout the strided one: all three must agree bit for bit
    dev = _dev()
    n, V = 300000, 9
    x = batch("normal_exp1000", n, V, seed=14)
    rows = np.unique(np.concatenate([np.arange(48), n - 1 - np.arange(48), np.random.default_rng(3).integers(0, n, 96)]))
    for direction in ("leg2cheb", "cheb2leg"):
        p = _plan(n, direction, batch=V, device=dev, engine=3)
        assert p.kernel_info["engine"] == 3
        z = p.execute(x.to(dev))
        xin = torch.zeros(V, n + 1, dtype=torch.float64)
        xin[:, :n] = x
        po = _plan(n, direction, batch=V, device=dev, engine=3, ld_in=n + 1)
        zo = po.execute(xin.to(dev))
        pb = _plan(n, direction, batch=V, device=dev, engine=3, layout="batch")
        zb = pb.execute(x.t().contiguous().to(dev))
        assert torch.equal(z, zo)
        assert torch.equal(z, zb.t().contiguous())
        zc = z.cpu().numpy()
        for v in (0, V - 1):
            e = oracle.einf(zc[v][rows], oracle.transform_rows(direction, x[v].numpy(), rows))
            assert e <= GATE, (direction, v, e)


def test_execute_checks_extents():
    # input / output tensors must cover the extent the kernels address ((rows - 1) ld + cols elements)
    dev = _dev()
    n, V = 1000, 9
    p = _plan(n, "leg2cheb", batch=V, device=dev, engine=2, ld_out=n + 5)
    x = batch("normal", n, V, seed=15).to(dev)
    with pytest.raises(ValueError):
        p.execute(x[:, : n - 1].contiguous())
    with pytest.raises(ValueError):
        p.execute(x, out=torch.empty(V, n, dtype=torch.float64, device=dev))  # ld_out = n + 5
    z = p.execute(x)  # default output allocated with ld_out
    assert z.shape == (V, n + 5)
    assert torch.equal(z[:, :n], _plan(n, "leg2cheb", batch=V, device=dev, engine=2).execute(x))


@pytest.mark.parametrize("V", [24, 40, 48, 72])
def test_range_engine_units_fit_one_wave(V):
    # (tile, range) units <= CTAs: a tile count that does not divide the slot count must not leave a
    # straggler round (was 30-40% slower, tools/range_batches.py)
    dev = _dev()
    p = _plan(2000000, "leg2cheb", batch=V, device=dev, engine=3)
    ki = p.kernel_info
    assert ki["engine"] == 3
    assert ((V + 7) // 8) * ki["ranges"] <= ki["tile_grid"]
