"""One engine-2 execute (ncu driver): python tools/prof_tile1.py n batch"""
import sys

import torch

sys.path.insert(0, '.')
from lc_inputs import batch as mk  # noqa: E402
from paper_2411_00033_b200 import Plan  # noqa: E402

n, V = int(sys.argv[1]), int(sys.argv[2])
x = mk("normal", n, V, seed=1).cuda()
p = Plan(n, "leg2cheb", batch=V, device=torch.device("cuda", 0), engine=2)
for _ in range(2):
    y = p.execute(x)
torch.cuda.synchronize()
print("ok")
