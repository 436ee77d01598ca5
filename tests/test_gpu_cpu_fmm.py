"""The CPU O(N) baseline (cpu_fmm/, a reported baseline of bench.py) against the oracle.  It needs a
GPU plan for its tables (lc_plan_export), hence the gpu mark."""
import numpy as np
import pytest
import torch

import oracle
from lc_inputs import vector

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("direction", ["leg2cheb", "cheb2leg"])
@pytest.mark.parametrize("n", [100, 1000, 4096, 20000])
def test_cpu_fmm_vs_oracle(direction, n):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from cpu_fmm import CpuFmm
    from paper_2411_00033_b200 import Plan
    p = Plan(n, direction, device=torch.device("cuda", 0))
    f = vector("uniform_r0.5", n, seed=3)
    z = CpuFmm(p)(f)
    e = oracle.einf(z, oracle.transform_rows(direction, f))
    assert e <= 1e-12, (n, direction, e)
    zg = p.execute(torch.from_numpy(f).reshape(1, -1).cuda()).cpu().numpy()[0]
    assert np.max(np.abs(zg - z)) <= 1e-12 * np.max(np.abs(z))
