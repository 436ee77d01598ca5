"""Small driver for ncu captures: a few executes of one config (no timing).
usage: python tools/prof_cfg.py n batch [reps] [direction] [vt]"""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2411_00033_b200 import Plan  # noqa: E402
from lc_inputs import vector  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
d = sys.argv[4] if len(sys.argv) > 4 else "leg2cheb"
vt = int(sys.argv[5]) if len(sys.argv) > 5 else 0
dev = torch.device("cuda", 0)
x = torch.from_numpy(np.stack([vector("sign_over_j1", n, 0, v) for v in range(batch)])).to(dev)
p = Plan(n, d, batch=batch, device=dev, vt=vt)
for _ in range(reps):
    y = p.execute(x)
torch.cuda.synchronize()
print("ok", p.kernel_info)
