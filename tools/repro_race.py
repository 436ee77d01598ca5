import sys, torch, numpy as np
sys.path.insert(0, '.')
import oracle
from lc_inputs import vector
from paper_2411_00033_b200 import Plan
dev = torch.device('cuda', 0)
for n, d in [(65659, 'cheb2leg'), (65659, 'leg2cheb'), (20000, 'cheb2leg'), (1 << 20, 'cheb2leg')]:
    f = vector("uniform_r0", n, seed=1)
    p = Plan(n, d, device=dev)
    x = torch.from_numpy(f).reshape(1, -1).to(dev)
    zs = oracle.transform_rows(d, f) if n < 100000 else None
    outs = []
    bad = 0
    for it in range(200):
        z = p.execute(x)
        outs.append(z.clone())
    torch.cuda.synchronize()
    ref = outs[0]
    ndiff = sum(int(not torch.equal(o, ref)) for o in outs)
    e = oracle.einf(ref.cpu().numpy()[0], zs) if zs is not None else -1
    worst = max(oracle.einf(o.cpu().numpy()[0], zs) for o in outs) if zs is not None else -1
    print(n, d, p.desc['L'], 'ndiff', ndiff, 'einf0 %.2e worst %.2e' % (e, worst), flush=True)
