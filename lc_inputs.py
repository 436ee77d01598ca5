"""Seeded synthetic coefficient generators shared by tests/, bench.py and smoke().

This module holds NO arithmetic of the method (no Lambda, no connection
matrix, no FMM): only the input recipes of BASELINE.json's configs and of the
paper's own accuracy workloads.  Both the oracle side and
the CUDA side consume the same host buffers produced here.

Every vector is generated independently from (seed, vector index) with a
torch CPU Philox/MT generator, so a single vector of a huge batch can be
regenerated for the oracle without materialising the batch.
"""
from __future__ import annotations

import numpy as np
import torch

# BASELINE.json configs (names used throughout tests/ and bench.py)
CONFIGS = {
    # cfg1: one vector, n=1024, f_j = xi_j/(j+1), xi ~ N(0,1), seed 0
    "cfg1": dict(n=1024, batch=1, kind="normal_over_j1"),
    # cfg2: one vector, n=1e6, f_j = s_j/(j+1), s_j = +-1 seeded
    "cfg2": dict(n=1_000_000, batch=1, kind="sign_over_j1"),
    "cfg2b": dict(n=1 << 20, batch=1, kind="sign_over_j1"),
    # cfg3: 4096 vectors of n=4096, N(0,1) exp(-j/1000)
    "cfg3": dict(n=4096, batch=4096, kind="normal_exp1000"),
    # cfg4: 64 vectors of n=1e7, N(0,1)/(j+1)^1.5
    "cfg4": dict(n=10_000_000, batch=64, kind="normal_over_j15"),
    # cfg5: 8192 x 8192 array, N(0,1)/((i+1)(j+1))
    "cfg5": dict(n=8192, batch=8192, kind="normal_over_ij"),
}


def _gen(seed: int, v: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed) * 1_000_003 + int(v))
    return g


def vector(kind: str, n: int, seed: int = 0, v: int = 0, row: int | None = None) -> np.ndarray:
    """One fp64 coefficient vector of length n (vector index v of a batch)."""
    g = _gen(seed, v)
    j = torch.arange(n, dtype=torch.float64)
    if kind == "normal_over_j1":
        x = torch.randn(n, generator=g, dtype=torch.float64) / (j + 1)
    elif kind == "sign_over_j1":
        s = torch.randint(0, 2, (n,), generator=g, dtype=torch.int64).to(torch.float64) * 2 - 1
        x = s / (j + 1)
    elif kind == "normal_exp1000":
        x = torch.randn(n, generator=g, dtype=torch.float64) * torch.exp(-j / 1000.0)
    elif kind == "normal_over_j15":
        x = torch.randn(n, generator=g, dtype=torch.float64) / (j + 1) ** 1.5
    elif kind == "normal_over_ij":
        i = v if row is None else row
        x = torch.randn(n, generator=g, dtype=torch.float64) / ((j + 1) * (i + 1))
    elif kind == "normal":
        x = torch.randn(n, generator=g, dtype=torch.float64)
    elif kind.startswith("uniform_r"):
        # paper workload: u_k/(k+1)^r, u ~ U[0,1]
        r = float(kind[len("uniform_r"):])
        x = torch.rand(n, generator=g, dtype=torch.float64) / (j + 1) ** r
    else:
        raise ValueError(kind)
    return x.numpy()


def batch(kind: str, n: int, nvec: int, seed: int = 0, v0: int = 0, out: torch.Tensor | None = None) -> torch.Tensor:
    """[nvec][n] row-major fp64 host tensor (vectors v0..v0+nvec-1)."""
    if out is None:
        out = torch.empty((nvec, n), dtype=torch.float64)
    for k in range(nvec):
        out[k] = torch.from_numpy(vector(kind, n, seed, v0 + k))
    return out


def config_batch(name: str, nvec: int | None = None, seed: int = 0, v0: int = 0, pin: bool = False) -> torch.Tensor:
    c = CONFIGS[name]
    nv = c["batch"] if nvec is None else nvec
    out = torch.empty((nv, c["n"]), dtype=torch.float64, pin_memory=pin)
    return batch(c["kind"], c["n"], nv, seed, v0, out)
