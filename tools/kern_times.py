"""Per-kernel times (lc_execute_timed: events between kernels, so no PDL overlap) and the graph-replayed
transform time of one plan; A/B builds via LC_LIB=liblegcheb_x.so.
usage: [LC_LIB=..] python tools/kern_times.py n batch [s_hat] [engine] [reps]"""
import os
import sys

import torch

sys.path.insert(0, '.')
from paper_2411_00033_b200 import _lib  # noqa: E402
if os.environ.get("LC_LIB"):
    _lib.LIB_PATH = _lib.LIB_PATH.replace("liblegcheb.so", os.environ["LC_LIB"])
from paper_2411_00033_b200 import Plan  # noqa: E402
from lc_inputs import batch as mkbatch  # noqa: E402

n, V = int(sys.argv[1]), int(sys.argv[2])
s_hat = int(sys.argv[3]) if len(sys.argv) > 3 else 0
engine = int(sys.argv[4]) if len(sys.argv) > 4 else 0
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
dev = torch.device("cuda", 0)
x = mkbatch("normal", n, V, seed=1).to(dev)
for direction in ("leg2cheb", "cheb2leg"):
    p = Plan(n, direction, batch=V, device=dev, s_hat=s_hat, engine=engine)
    y = torch.empty_like(x)
    k = p.kernels_per_execute
    ts = [[] for _ in range(k)]
    for r in range(reps + 2):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(k + 1)]
        p.execute_timed(x, y, ev)
        torch.cuda.synchronize()
        if r >= 2:
            for i in range(k):
                ts[i].append(ev[i].elapsed_time(ev[i + 1]))
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        p.execute(x, y)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        p.execute(x, y)
    g.replay()
    torch.cuda.synchronize()
    tt = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        tt.append(a.elapsed_time(b))
    ki = p.kernel_info
    med = lambda a: sorted(a)[len(a) // 2]
    print(f"{os.environ.get('LC_LIB', 'liblegcheb.so')} {direction} n={n} V={V} s={p.desc['s']} L={p.desc['L']} "
          f"engine={ki.get('engine')} kernels(ms)=" + " ".join(f"{med(t):.4f}" for t in ts) +
          f"  graph {med(tt):.4f} ms")
    p.close()
