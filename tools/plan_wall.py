"""Wall time of lc_plan_create (through Plan) per call: the first call of a process pays the CUDA module load,
the kernel attribute configuration and the first pool allocation; later calls show the steady cost.
usage: python tools/plan_wall.py n [batch] [reps]"""
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_2411_00033_b200 import Plan  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
V = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 8
dev = torch.device("cuda", 0)
torch.zeros(1, device=dev)
torch.cuda.synchronize()
for d in ("leg2cheb", "cheb2leg"):
    walls, devs = [], []
    keep = None
    for r in range(reps):
        t = time.perf_counter()
        p = Plan(n, d, batch=V, device=dev)
        torch.cuda.synchronize()
        walls.append((time.perf_counter() - t) * 1e3)
        devs.append(p.desc.get("plan_device_ms", float("nan")))
        if r % 2 == 0:
            keep = p  # alternate: destroy-before-create and create-while-alive
        else:
            del p
    print(f"n={n} V={V} {d}: wall ms per create {[round(w, 3) for w in walls]}  device ms {[round(x, 3) for x in devs]}")
