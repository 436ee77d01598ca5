"""Time one transform per plan over s_hat (engine 2 / 3 / 1) with CUDA events.
usage: python tools/s_sweep.py n batch engine s_hat..."""
import sys

import torch

sys.path.insert(0, '.')
from paper_2411_00033_b200 import Plan  # noqa: E402
from lc_inputs import batch as mkbatch  # noqa: E402

n, V, eng = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dev = torch.device("cuda", 0)
x = mkbatch("normal", n, V, seed=1).to(dev)
ref = None
for sh in [int(a) for a in sys.argv[4:]]:
    p = Plan(n, "leg2cheb", batch=V, device=dev, s_hat=sh, engine=eng)
    y = p.execute(x)
    for _ in range(3):
        p.execute(x, out=y)
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); p.execute(x, out=y); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    err = 0.0 if ref is None else float((y - ref).abs().max() / ref.abs().max())
    ref = y.clone() if ref is None else ref
    d = p.desc
    print(f"n={n} V={V} engine={eng} s_hat={sh} s={d['s']} L={d['L']} median {ts[5]:.4f} ms min {ts[0]:.4f} ms  diff {err:.1e}")
