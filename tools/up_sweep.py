"""Engine-3 up-kernel subtree depth sweep at the cfg4 shape (64 x 1e7): per-kernel times (CUDA events).
usage: python tools/up_sweep.py"""
import sys

import torch

sys.path.insert(0, '.')
from paper_2411_00033_b200 import Plan  # noqa: E402

dev = torch.device("cuda", 0)
n, V = 10 ** 7, 64
x = torch.randn(V, n, dtype=torch.float64, device=dev)
y = torch.empty_like(x)
for k in (2, 3, 4, 5):
    try:
        p = Plan(n, "leg2cheb", batch=V, device=dev, engine=3, up_subtree=k)
    except Exception as e:  # noqa: BLE001
        print("kup", k, "unavailable", e)
        continue
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for _ in range(2):
        p.execute_timed(x, y, ev)
    torch.cuda.synchronize()
    t = [0.0, 0.0]
    for _ in range(3):
        p.execute_timed(x, y, ev)
        torch.cuda.synchronize()
        t[0] += ev[0].elapsed_time(ev[1]) / 3
        t[1] += ev[1].elapsed_time(ev[2]) / 3
    ki = p.kernel_info
    print(f"kup {k}: up {t[0]:.2f} ms  range {t[1]:.2f} ms  smem_up {ki['smem_up']}  up_grid {ki['up_grid']}", flush=True)
    del p
