"""GPU parity at BASELINE.json's full sizes (cfg2-cfg5), in the launch configuration bench.py uses,
on sampled outputs the oracle computes row by row."""
import numpy as np
import pytest
import torch

import oracle
from lc_inputs import CONFIGS, config_batch, vector

pytestmark = pytest.mark.gpu


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


def _rows(n, seed=1, s=32):
    """C-4: 2048 uniform rows, the first and last 256, and both sides of random 2s-tile boundaries."""
    rng = np.random.default_rng(seed)
    r = set(rng.choice(n, size=min(n, 2048), replace=False).tolist())
    r |= set(range(min(n, 256))) | set(range(max(0, n - 256), n))
    for u in rng.integers(1, max(2, n // (2 * s)), size=256):
        r |= {int(2 * s * u - 1), int(2 * s * u)}
    return np.array(sorted(x for x in r if 0 <= x < n), dtype=np.int64)


@pytest.mark.parametrize("cfg", ["cfg2", "cfg2b"])
def test_cfg2_single_vector_full_size(cfg):
    from paper_2411_00033_b200 import Plan
    dev = _dev()
    c = CONFIGS[cfg]
    n = c["n"]
    x = config_batch(cfg)
    xd = x.to(dev)
    pl, pc = Plan(n, "leg2cheb", device=dev), Plan(n, "cheb2leg", device=dev)
    z = pl.execute(xd)
    y = pc.execute(z)
    rows = _rows(n)
    f = x[0].numpy()
    for d, out, inp in (("leg2cheb", z, f), ("cheb2leg", y, z.cpu().numpy()[0])):
        ref = oracle.transform_rows(d, inp, rows)
        assert oracle.einf(out.cpu().numpy()[0][rows], ref) <= 1e-12, d
    assert oracle.einf(y.cpu().numpy()[0], f) <= 1e-12  # round trip (exact result: the input)


def test_cfg3_batched_full_size():
    from paper_2411_00033_b200 import Plan
    dev = _dev()
    n, V = CONFIGS["cfg3"]["n"], CONFIGS["cfg3"]["batch"]
    x = config_batch("cfg3")
    xd = x.to(dev)
    pl, pc = Plan(n, "leg2cheb", batch=V, device=dev), Plan(n, "cheb2leg", batch=V, device=dev)
    z = pl.execute(xd)
    y = pc.execute(z)
    zh, yh = z.cpu().numpy(), y.cpu().numpy()
    rng = np.random.default_rng(1)
    vs = sorted({0, V - 1} | set(rng.choice(V, 30, replace=False).tolist()))  # 32 full vectors
    for v in vs:
        assert oracle.einf(zh[v], oracle.l2c(x[v].numpy())) <= 1e-12, v
        assert oracle.einf(yh[v], oracle.c2l(zh[v])) <= 1e-12, v
        assert oracle.einf(yh[v], x[v].numpy()) <= 1e-12, v


@pytest.mark.slow
def test_cfg4_large_round_trip_sampled():
    from paper_2411_00033_b200 import Plan
    dev = _dev()
    n, V = CONFIGS["cfg4"]["n"], CONFIGS["cfg4"]["batch"]
    x = config_batch("cfg4", pin=True)
    xd = x.to(dev, non_blocking=True)
    pl, pc = Plan(n, "leg2cheb", batch=V, device=dev), Plan(n, "cheb2leg", batch=V, device=dev)
    z = pl.execute(xd)
    y = pc.execute(z)
    torch.cuda.synchronize()
    rng = np.random.default_rng(1)
    rows = np.array(sorted(set(rng.choice(n, 24, replace=False).tolist()) | {0, 1, 2, 39, 40, n - 2, n - 1}))
    for v in (0, 17, V - 1):
        zv = z[v].cpu().numpy()
        assert oracle.einf(zv[rows], oracle.l2c_rows(x[v].numpy(), rows)) <= 1e-11, v
        assert oracle.einf(y[v].cpu().numpy()[rows], oracle.c2l_rows(zv, rows)) <= 1e-11, v
        assert oracle.einf(y[v].cpu().numpy(), x[v].numpy()) <= 1e-11, v  # round trip, all entries
    del xd, z, y


def test_cfg5_tensor_product_2d_single_gpu():
    from paper_2411_00033_b200.dist import tensor_product_2d
    dev = _dev()
    n = CONFIGS["cfg5"]["n"]
    F = torch.stack([torch.from_numpy(vector("normal_over_ij", n, seed=0, v=i)) for i in range(n)])
    Z = tensor_product_2d(F.to(dev)).cpu().numpy()  # L2C along axis 1, then along axis 0
    rng = np.random.default_rng(1)
    js = sorted(rng.choice(n, 8, replace=False).tolist()) + [0, n - 1]
    is_ = np.array(sorted(set(rng.choice(n, 64, replace=False).tolist()) | {0, 1, n - 1}))
    Fn = F.numpy()
    for j in js:
        # g_k = (row transform of row k) at output j, for all k; then Z_ij = column transform of g at i
        g = np.array([float(oracle.l2c_rows(Fn[k], [j])[0]) for k in range(n)])
        ref = oracle.l2c_rows(g, is_)
        assert oracle.einf(Z[is_, j], ref) <= 1e-12, j
