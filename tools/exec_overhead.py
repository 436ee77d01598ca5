"""Host cost of lc_execute outside a CUDA graph: wall time per call of back-to-back asynchronous executes
(Python ctypes call included) against the device time per transform of a graph replay.
usage: python tools/exec_overhead.py n [batch] [calls]"""
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_2411_00033_b200 import Plan  # noqa: E402
from lc_inputs import batch as mkbatch  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
V = int(sys.argv[2]) if len(sys.argv) > 2 else 1
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
dev = torch.device("cuda", 0)
x = mkbatch("normal", n, V, seed=1).to(dev)
p = Plan(n, "leg2cheb", batch=V, device=dev)
y = torch.empty_like(x)
for _ in range(20):
    p.execute(x, y)
torch.cuda.synchronize()
# (a) enqueue only: the host returns before the device finishes
t = time.perf_counter()
for _ in range(calls):
    p.execute(x, y)
t_enq = (time.perf_counter() - t) / calls * 1e6
torch.cuda.synchronize()
t_all = (time.perf_counter() - t) / calls * 1e6
# (b) graph replay of one execute
s = torch.cuda.Stream(dev)
with torch.cuda.stream(s):
    p.execute(x, y)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    p.execute(x, y)
for _ in range(20):
    g.replay()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(calls):
    g.replay()
torch.cuda.synchronize()
t_graph = (time.perf_counter() - t) / calls * 1e6
print(f"n={n} V={V}: lc_execute enqueue {t_enq:.1f} us per call (host), {t_all:.1f} us per call until the device is done; "
      f"graph replay {t_graph:.1f} us per call")
