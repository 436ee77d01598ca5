"""Engine 1 vs engine 2 time per transform over (n, batch) (CUDA events, graph-free).
usage: python tools/engine_cross.py"""
import sys

import torch

sys.path.insert(0, '.')
from lc_inputs import batch as mk  # noqa: E402
from paper_2411_00033_b200 import Plan  # noqa: E402

dev = torch.device("cuda", 0)
for n in (1024, 4096, 16384, 65536):
    for V in (8, 32, 128, 512, 2048):
        if n * V > 2 ** 26:
            continue
        x = mk("normal", n, V, seed=1).to(dev)
        res = []
        for e in (1, 2):
            try:
                p = Plan(n, "leg2cheb", batch=V, device=dev, engine=e)
            except Exception as ex:  # noqa: BLE001
                res.append(None)
                continue
            y = torch.empty_like(x)
            for _ in range(3):
                p.execute(x, out=y)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(20):
                p.execute(x, out=y)
            e1.record()
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1) / 20 * 1e3)
        print(f"n={n:6d} V={V:5d} tiles={(V + 7) // 8:4d}  engine1 {res[0]:9.1f} us  engine2 "
              f"{res[1] if res[1] is None else round(res[1], 1)} us", flush=True)
