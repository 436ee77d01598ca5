"""Time one transform per batch size (CUDA events, median of 10).
usage: python tools/v_sweep.py n engine V..."""
import sys

import torch

sys.path.insert(0, '.')
import os  # noqa: E402
from paper_2411_00033_b200 import _lib  # noqa: E402
if os.environ.get("LC_LIB"):  # A/B builds: LC_LIB=liblegcheb_x.so
    _lib.LIB_PATH = _lib.LIB_PATH.replace("liblegcheb.so", os.environ["LC_LIB"])
from paper_2411_00033_b200 import Plan  # noqa: E402
from lc_inputs import batch as mkbatch  # noqa: E402

n, eng = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda", 0)
for V in [int(a) for a in sys.argv[3:]]:
    x = mkbatch("normal", n, V, seed=1).to(dev)
    p = Plan(n, "leg2cheb", batch=V, device=dev, engine=eng)
    y = p.execute(x)
    for _ in range(3):
        p.execute(x, out=y)
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); p.execute(x, out=y); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    ki = p.kernel_info
    print(f"n={n} V={V} engine={eng} median {ts[5]:.4f} ms min {ts[0]:.4f} ms  {ki}")
