"""Engine-3 time per transform over batch sizes whose tile count does not divide the slot count
(the range count must keep every (tile, range) unit in one wave).  usage: python tools/range_batches.py n"""
import sys

import torch

sys.path.insert(0, '.')
from paper_2411_00033_b200 import Plan  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000000
dev = torch.device("cuda", 0)
for V in (24, 40, 48, 56, 64, 72, 88):
    x = torch.randn(V, n, dtype=torch.float64, device=dev)
    p = Plan(n, "leg2cheb", batch=V, device=dev, engine=3)
    y = torch.empty_like(x)
    for _ in range(3):
        p.execute(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        p.execute(x, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    ki = p.kernel_info
    print(f"V={V:3d} tiles={(V + 7) // 8} grid={ki['tile_grid']} ranges={ki['ranges']} {ms:8.3f} ms  {n * V / ms / 1e6:7.2f} Gcoef/s")
    p.close()
    del x, y
