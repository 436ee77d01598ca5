"""Round-trip time (leg2cheb then cheb2leg) of one batch, CUDA-graph replays timed per replay with
events (median / min over `reps`), as bench.py times its step.  A/B builds: LC_LIB=liblegcheb_x.so.
usage: [LC_S_HAT=..] [LC_ENGINE=..] python tools/rt_time.py n [batch] [reps]"""
import os
import sys

import torch

sys.path.insert(0, '.')
from paper_2411_00033_b200 import _lib  # noqa: E402
if os.environ.get("LC_LIB"):
    _lib.LIB_PATH = _lib.LIB_PATH.replace("liblegcheb.so", os.environ["LC_LIB"])
from paper_2411_00033_b200 import Plan  # noqa: E402
from lc_inputs import batch as mkbatch  # noqa: E402

n = int(sys.argv[1])
V = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 200
dev = torch.device("cuda", 0)
x = mkbatch("normal", n, V, seed=1).to(dev)
kw = {}
if os.environ.get("LC_S_HAT"):
    kw["s_hat"] = int(os.environ["LC_S_HAT"])
if os.environ.get("LC_ENGINE"):
    kw["engine"] = int(os.environ["LC_ENGINE"])
pl, pc = Plan(n, "leg2cheb", batch=V, device=dev, **kw), Plan(n, "cheb2leg", batch=V, device=dev, **kw)
tmp, y = torch.empty_like(x), torch.empty_like(x)
s = torch.cuda.Stream(dev)
with torch.cuda.stream(s):
    for _ in range(3):
        pl.execute(x, tmp); pc.execute(tmp, y)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    pl.execute(x, tmp); pc.execute(tmp, y)
for _ in range(10):
    g.replay()
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
for a, b in ev:
    a.record(); g.replay(); b.record()
torch.cuda.synchronize()
ts = sorted(a.elapsed_time(b) for a, b in ev)
err = float((y - x).abs().max() / x.abs().max())
print(f"{os.environ.get('LC_LIB', 'liblegcheb.so')} n={n} V={V} s={pl.desc['s']} L={pl.desc['L']} engine={pl.kernel_info.get('engine')}: round trip median {1e3 * ts[reps // 2]:.1f} us "
      f"min {1e3 * ts[0]:.1f} us  (per transform {1e3 * ts[reps // 2] / 2:.1f} us)  rt err {err:.1e}")
