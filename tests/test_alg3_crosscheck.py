"""NEXT-3: the O(N log N) modal FMM of Alg. 2/3 with its own A_hat
(tests/alg3_model.py: mpmath Lambda, scipy DCT-II; nothing from the CUDA path) as an independent
cross-check of the planner and of step 3.

* CPU (`-m "not gpu"`): the model reproduces the oracle's plain definitions -- this validates the
  model's A_hat, hierarchy and band independently of the library.
* GPU: the library's A_hat arena (built on the device) equals the model's block by
  block, and the library's fast O(N) transform (Alg. 4) agrees with the model's Alg. 3 result.
"""
import functools

import numpy as np
import pytest
import torch

import oracle
from alg3_model import Alg3
from lc_inputs import vector

M = 18


@functools.lru_cache(maxsize=None)
def _model(n, direction):
    return Alg3(n, direction)


@pytest.mark.parametrize("direction", ["leg2cheb", "cheb2leg"])
@pytest.mark.parametrize("n,kind", [(1000, "normal"), (4096, "uniform_r0"), (3900, "normal")])
def test_alg3_model_matches_oracle(n, kind, direction):
    m = _model(n, direction)
    f = vector(kind, n, seed=23)
    z = m(f)
    ref = oracle.transform_rows(direction, f)
    # Table 1: the modal FMM is within ~1e-15 (L2C) of the 32-digit result
    assert oracle.einf(z, ref) < (2e-15 if direction == "leg2cheb" else 5e-15)


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


@pytest.mark.gpu
@pytest.mark.parametrize("direction", ["leg2cheb", "cheb2leg"])
@pytest.mark.parametrize("n", [4096, 3900])
def test_gpu_plan_ahat_equals_model(n, direction):
    from paper_2411_00033_b200 import Plan
    dev = _dev()
    m = _model(n, direction)
    p = Plan(n, direction, device=dev)
    d = p.desc
    assert (d["L"], d["s"], d["N"]) == (m.L, m.s, m.N)
    A = p.export("ahat").reshape(-1, M, M)
    worst = 0.0
    q = 0
    for g in range(m.L):  # level-major (g, b, r) arena order (eq:cfrompq), DESIGN.md section 5
        for b in range((2 << g) - 1):
            for r in range(3):
                ref = m.A[(g, b, r)]
                err = np.max(np.abs(A[q] - ref)) / np.max(np.abs(ref))
                worst = max(worst, err)
                assert err < 1e-14, (direction, n, g, b, r, err)
                q += 1
    assert q == d["nc"]


@pytest.mark.gpu
@pytest.mark.parametrize("engine", [1, 2, 3])
@pytest.mark.parametrize("direction", ["leg2cheb", "cheb2leg"])
def test_gpu_transform_equals_alg3(direction, engine):
    from paper_2411_00033_b200 import Plan
    dev = _dev()
    n, V = 4096, 8
    m = _model(n, direction)
    x = torch.stack([torch.from_numpy(vector("normal", n, seed=300 + v)) for v in range(V)])
    p = Plan(n, direction, batch=V, device=dev, engine=engine)
    z = p.execute(x.to(dev)).cpu().numpy()
    for v in range(V):
        zm = m(x[v].numpy())
        assert np.max(np.abs(z[v] - zm)) / np.max(np.abs(zm)) < 2e-15, (engine, v)
