"""GPU parity at BASELINE.json's full sizes (cfg2-cfg5), in the launch configuration bench.py uses,
on sampled outputs the oracle computes row by row."""
import numpy as np
import pytest
import torch

import oracle
from lc_inputs import CONFIGS, config_batch, vector
from parity_util import c4_rows, check_round_trip, check_rows

pytestmark = pytest.mark.gpu


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


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
    rows = c4_rows(n, pl.desc["s"])  # tile boundaries at the plan's own s (31 at 1e6, 32 at 2^20)
    f = x[0].numpy()
    zh = z.cpu().numpy()[0]
    check_rows("leg2cheb", f, zh, rows, cfg)
    check_rows("cheb2leg", zh, y.cpu().numpy()[0], rows, cfg)
    check_round_trip(f, y.cpu().numpy()[0], pl.desc["s"], cfg)


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
    allrows = np.arange(n)
    for v in vs:
        check_rows("leg2cheb", x[v].numpy(), zh[v], allrows, f"cfg3 v={v}")
        check_rows("cheb2leg", zh[v], yh[v], allrows, f"cfg3 v={v}")
        check_round_trip(x[v].numpy(), yh[v], pl.desc["s"], f"cfg3 v={v}")


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
    assert pl.kernel_info["engine"] == 3
    sp = pl.desc["s"]
    rows = c4_rows(n, sp, uniform=1024, tiles=128)  # >= 1000 rows per vector, boundaries at s = 20
    rng = np.random.default_rng(1)
    vs = sorted({0, V - 1} | set(rng.choice(np.arange(1, V - 1), 2, replace=False).tolist()))
    for v in vs:  # 4 vectors
        zv = z[v].cpu().numpy()
        check_rows("leg2cheb", x[v].numpy(), zv, rows, f"cfg4 v={v}")
        check_rows("cheb2leg", zv, y[v].cpu().numpy(), rows, f"cfg4 v={v}")
    yh = y.cpu().numpy()
    for v in range(V):  # every vector, every entry
        check_round_trip(x[v].numpy(), yh[v], sp, f"cfg4 v={v}")
    del xd, z, y


def test_cfg5_tensor_product_2d_single_gpu():
    from paper_2411_00033_b200.dist import tensor_product_2d
    dev = _dev()
    n = CONFIGS["cfg5"]["n"]
    F = torch.stack([torch.from_numpy(vector("normal_over_ij", n, seed=0, v=i)) for i in range(n)])
    Z = tensor_product_2d(F.to(dev)).cpu().numpy()  # L2C along axis 1, then along axis 0
    rng = np.random.default_rng(1)
    js = np.array(sorted(set(rng.choice(n, 62, replace=False).tolist()) | {0, n - 1}))  # 64 columns
    is_ = np.array(sorted(set(rng.choice(n, 64, replace=False).tolist()) | {0, 1, n - 1}))
    Fn = F.numpy()
    # g[k, c] = (row transform of row k) at output column js[c], for all k (one oracle call per row)
    g = np.stack([oracle.l2c_rows(Fn[k], js) for k in range(n)])
    for c, j in enumerate(js):
        ref, ab = oracle.l2c_rows(g[:, c], is_, with_abs=True)
        e = oracle.einf(Z[is_, j], ref)
        assert e <= 1e-12, (j, e)
