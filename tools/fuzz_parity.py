"""Seeded fuzz of the three engines with NON-decaying inputs (`normal`, `uniform_r0.5`): random n, batch,
direction, layout and s_hat; vectors 0 and V-1 against the oracle on C-4 rows at the plan's own s (E_inf gate
and the per-row diagnostic of tests/parity_util.py), and the engines against each other per 2s-block (each
block relative to its own max, so a wrong tail block cannot hide behind a large head).
Test infrastructure (it calls oracle/ through tests/parity_util.py); prints one line per case.
usage: python tools/fuzz_parity.py [count] [seed] [nmax]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import parity_util as pu  # noqa: E402
from lc_inputs import batch  # noqa: E402
from paper_2411_00033_b200 import Plan  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 60
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 7
nmax = int(sys.argv[3]) if len(sys.argv) > 3 else 400000
rng = np.random.default_rng(seed)
dev = torch.device("cuda", 0)
bad = 0
worst_e = worst_d = worst_x = 0.0
t0 = time.time()
for case in range(count):
    n = int(np.exp(rng.uniform(np.log(130), np.log(nmax))))
    V = int(rng.integers(1, 40))
    direction = "leg2cheb" if rng.integers(0, 2) == 0 else "cheb2leg"
    layout = "vec" if rng.integers(0, 3) else "batch"
    kind = "normal" if rng.integers(0, 3) else "uniform_r0.5"
    s_hat = int(rng.choice([0, 0, 0, 16, 24, 32, 48, 64]))
    x = batch(kind, n, V, seed=1000 + case)
    xin = (x if layout == "vec" else x.t().contiguous()).to(dev)
    results, line = {}, []
    for engine in (1, 2, 3):
        try:
            p = Plan(n, direction, batch=V, device=dev, layout=layout, engine=engine, s_hat=s_hat)
        except RuntimeError:
            continue  # engine not applicable (L = 0, s > 40 on engines 2/3)
        z = p.execute(xin)
        z = (z if layout == "vec" else z.t()).cpu().numpy()
        s = int(p.desc["s"])
        rows = np.arange(n) if n <= 4096 else pu.c4_rows(n, s, seed=case, uniform=192, tiles=24, tail_tiles=2)
        for v in sorted({0, V - 1}):
            try:
                e, d = pu.check_rows(direction, x[v].numpy(), z[v], rows, tag=f"fuzz{case} e{engine} v{v}")
                worst_e, worst_d = max(worst_e, e), max(worst_d, d)
            except AssertionError as err:
                bad += 1
                line.append(f"FAIL {err}")
        results[engine] = (z, s)
    engines = sorted(results)
    z0, s0 = results[engines[0]]
    for e in engines[1:]:
        for v in range(V):
            b = pu.blockwise_einf(results[e][0][v], z0[v], 2 * s0)
            worst_x = max(worst_x, b)
            if b > pu.BLOCK_RT:  # engines differ by summation order only (all-positive inputs: cancellation in C2L)
                bad += 1
                line.append(f"FAIL engines {engines[0]} vs {e} vector {v}: per-block diff {b:.2e}")
    print(f"case {case:3d} n={n:7d} V={V:2d} {direction} {layout:5s} {kind:12s} s_hat={s_hat:2d} s={s0:2d} "
          f"engines {engines} {'ok' if not line else '; '.join(line)}", flush=True)
print(f"{count} cases (seed {seed}) in {time.time() - t0:.0f} s: failures {bad}; max E_inf {worst_e:.2e}, "
      f"max per-row diagnostic {worst_d:.2e}, max per-block engine difference {worst_x:.2e}")
sys.exit(1 if bad else 0)
