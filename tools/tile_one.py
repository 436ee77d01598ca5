"""One small engine-2 execute checked against the oracle (debug helper).
usage: python tools/tile_one.py n V [direction]"""
import sys

import torch

sys.path.insert(0, '.')
import oracle  # noqa: E402
from lc_inputs import batch  # noqa: E402
from paper_2411_00033_b200 import Plan  # noqa: E402

n, V = int(sys.argv[1]), int(sys.argv[2])
d = sys.argv[3] if len(sys.argv) > 3 else "leg2cheb"
x = batch("normal_exp1000", n, V, seed=11)
p = Plan(n, d, batch=V, device=torch.device("cuda", 0), engine=2)
z = p.execute(x.cuda()).cpu().numpy()
torch.cuda.synchronize()
print(n, V, d, "max err", max(oracle.einf(z[v], oracle.transform_rows(d, x[v].numpy())) for v in range(V)), flush=True)
