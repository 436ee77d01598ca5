"""engine 1 vs engine 2 vs oracle per vector (debug helper). usage: python tools/tile_dbg.py n V [seed]"""
import sys

import torch

sys.path.insert(0, '.')
import oracle  # noqa: E402
from lc_inputs import batch  # noqa: E402
from paper_2411_00033_b200 import Plan  # noqa: E402

n, V = int(sys.argv[1]), int(sys.argv[2])
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 6
dev = torch.device("cuda", 0)
x = batch("normal_exp1000", n, V, seed=seed)
z1 = Plan(n, "leg2cheb", batch=V, device=dev, engine=1).execute(x.to(dev)).cpu().numpy()
z2 = Plan(n, "leg2cheb", batch=V, device=dev, engine=2).execute(x.to(dev)).cpu().numpy()
for v in range(V):
    ref = oracle.transform_rows("leg2cheb", x[v].numpy())
    e1, e2 = oracle.einf(z1[v], ref), oracle.einf(z2[v], ref)
    bad = abs(z2[v] - ref).argmax()
    print(v, f"e1 {e1:.2e} e2 {e2:.2e} worst row {bad}")
