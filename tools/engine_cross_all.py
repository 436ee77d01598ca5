"""Time per transform of engines 1, 2, 3 (and the automatic choice) over (n, batch), CUDA events.
usage: python tools/engine_cross_all.py [engines, e.g. 0,1,3] [n,n,...] [V,V,...]"""
import sys

import torch

sys.path.insert(0, '.')
from paper_2411_00033_b200 import Plan  # noqa: E402
from paper_2411_00033_b200._lib import LegChebError  # noqa: E402

dev = torch.device("cuda", 0)
ENG = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 1, 2, 3]
NS = [int(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else [20000, 65536, 150000, 300000, 1000000, 3000000]
VS = [int(a) for a in sys.argv[3].split(",")] if len(sys.argv) > 3 else [4, 8, 16, 32, 64, 128]
for n in NS:
    for V in VS:
        if n * V > 2 * 10 ** 8:
            continue
        x = torch.randn(V, n, dtype=torch.float64, device=dev)
        res = {}
        for e in ENG:
            try:
                p = Plan(n, "leg2cheb", batch=V, device=dev, engine=e)
            except (LegChebError, RuntimeError):
                continue
            y = torch.empty_like(x)
            for _ in range(2):
                p.execute(x, out=y)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            reps = 10
            e0.record()
            for _ in range(reps):
                p.execute(x, out=y)
            e1.record()
            torch.cuda.synchronize()
            res[e if e else "auto=%d" % p.kernel_info["engine"]] = e0.elapsed_time(e1) / reps * 1e3
            p.close()
        print(f"n={n} V={V} s={p.desc['s']} L={p.desc['L']}: " + "  ".join(f"{k}: {v:.1f} us" for k, v in res.items()),
              flush=True)
