"""Seeded sweep over (n, batch, engine, direction, layout): every engine against the oracle on
sampled rows (all rows up to n = 4096), and the engines against each other element by element.

The sizes are drawn so that the sweep crosses level counts L = 1 .. 11, odd and even s, ragged
batches (not multiples of the 8-vector tile), and both layouts; the gate is the north-star 1e-12.
"""
import numpy as np
import pytest
import torch

import oracle
from lc_inputs import batch

pytestmark = pytest.mark.gpu

GATE = 1e-12


def _cases(count=14, seed=2024):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        n = int(np.exp(rng.uniform(np.log(130), np.log(150000))))
        V = int(rng.integers(1, 40))
        direction = "leg2cheb" if rng.integers(0, 2) == 0 else "cheb2leg"
        layout = "vec" if rng.integers(0, 3) else "batch"
        out.append((n, V, direction, layout))
    return out


@pytest.mark.parametrize("n,V,direction,layout", _cases())
def test_engines_agree_with_oracle(n, V, direction, layout):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2411_00033_b200 import Plan
    dev = torch.device("cuda", 0)
    x = batch("normal_exp1000", n, V, seed=n % 997)
    xin = (x if layout == "vec" else x.t().contiguous()).to(dev)
    rng = np.random.default_rng(n)
    rows = None if n <= 4096 else np.unique(np.concatenate([np.arange(64), n - 1 - np.arange(64),
                                                           rng.integers(0, n, 192)]))
    ref = [oracle.transform_rows(direction, x[v].numpy(), rows) for v in (0, V - 1)]
    results = {}
    for engine in (1, 2, 3):
        try:
            p = Plan(n, direction, batch=V, device=dev, layout=layout, engine=engine)
        except RuntimeError:
            continue  # engine not applicable (L = 0 or s > 32)
        z = p.execute(xin)
        z = (z if layout == "vec" else z.t()).cpu().numpy()
        for i, v in enumerate((0, V - 1)):
            zv = z[v] if rows is None else z[v][rows]
            e = oracle.einf(zv, ref[i])
            assert e <= GATE, (n, V, direction, layout, engine, v, e)
        results[engine] = z
    engines = sorted(results)
    for e in engines[1:]:
        d = np.max(np.abs(results[e] - results[engines[0]])) / np.max(np.abs(results[engines[0]]))
        assert d <= 1e-13, (n, V, direction, layout, engines[0], e, d)
