"""Engine 1 vs engine 3 time per transform over (n, batch) (CUDA events).  usage: python tools/engine_cross3.py"""
import sys

import torch

sys.path.insert(0, '.')
from paper_2411_00033_b200 import Plan  # noqa: E402

dev = torch.device("cuda", 0)
for n in (100000, 1000000, 10000000):
    for V in (8, 16, 32, 64):
        if n * V > 64 * 10 ** 7:
            continue
        x = torch.randn(V, n, dtype=torch.float64, device=dev)
        res = []
        for e in (1, 3):
            p = Plan(n, "leg2cheb", batch=V, device=dev, engine=e)
            y = torch.empty_like(x)
            for _ in range(2):
                p.execute(x, out=y)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            reps = 10 if n * V <= 10 ** 8 else 3
            e0.record()
            for _ in range(reps):
                p.execute(x, out=y)
            e1.record()
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1) / reps * 1e3)
            del p
        print(f"n={n:9d} V={V:3d}  engine1 {res[0]:10.1f} us  engine3 {res[1]:10.1f} us  ratio {res[0] / res[1]:5.2f}",
              flush=True)
