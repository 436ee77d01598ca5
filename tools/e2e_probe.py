"""End-to-end host pipeline probe: per-step time of lc_execute_host_chain([leg2cheb, cheb2leg]) calls
round-robin over k streams (huge-page host buffers), several trials per k, to study the copy/compute
overlap.  usage: python tools/e2e_probe.py n [batch] [steps]"""
import sys

import torch

sys.path.insert(0, '.')
from paper_2411_00033_b200 import Plan, execute_host_chain, host_empty, new_chain_stage  # noqa: E402
from lc_inputs import batch as mkbatch  # noqa: E402

n = int(sys.argv[1])
V = int(sys.argv[2]) if len(sys.argv) > 2 else 1
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 300
dev = torch.device("cuda", 0)
pl, pc = Plan(n, "leg2cheb", batch=V, device=dev), Plan(n, "cheb2leg", batch=V, device=dev)
xh = host_empty((V, n))
xh.copy_(mkbatch("normal", n, V, seed=1))
for k in (1, 2, 3, 4, 6):
    streams = [torch.cuda.Stream(dev) for _ in range(k)]
    hy = [host_empty((V, n)) for _ in range(k)]
    st = [new_chain_stage([pl, pc]) for _ in range(k)]
    ws = [[pl.new_workspace(streams[b]), pc.new_workspace(streams[b])] for b in range(k)]
    torch.cuda.synchronize()
    res = []
    for trial in range(4):
        for i in range(k):
            execute_host_chain([pl, pc], xh, hy[i], st[i], stream=streams[i], workspaces=ws[i])
        torch.cuda.synchronize()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        h0.record(cur)
        for s in streams:
            s.wait_event(h0)
        for i in range(steps):
            b = i % k
            execute_host_chain([pl, pc], xh, hy[b], st[b], stream=streams[b], workspaces=ws[b])
        for s in streams:
            e = torch.cuda.Event()
            e.record(s)
            cur.wait_event(e)
        h1.record(cur)
        torch.cuda.synchronize()
        res.append(h0.elapsed_time(h1) / steps * 1e3)
    print(f"n={n} V={V} streams {k}: us per step " + " ".join(f"{r:6.1f}" for r in res) +
          f"   (coef/s best {2 * n * V / min(res) * 1e6:.3e})")

# the copy engines alone in the same pattern (H2D then D2H per step, round-robin over k streams)
d_bufs = [torch.empty((V, n), dtype=torch.float64, device=dev) for _ in range(6)]
for k in (2, 3, 4):
    streams = [torch.cuda.Stream(dev) for _ in range(k)]
    hy = [host_empty((V, n)) for _ in range(k)]
    torch.cuda.synchronize()
    res = []
    for trial in range(3):
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        h0.record(cur)
        for s in streams:
            s.wait_event(h0)
        for i in range(steps):
            b = i % k
            with torch.cuda.stream(streams[b]):
                d_bufs[b].copy_(xh, non_blocking=True)
                hy[b].copy_(d_bufs[b], non_blocking=True)
        for s in streams:
            e = torch.cuda.Event()
            e.record(s)
            cur.wait_event(e)
        h1.record(cur)
        torch.cuda.synchronize()
        res.append(h0.elapsed_time(h1) / steps * 1e3)
    print(f"copies only, streams {k}: us per step " + " ".join(f"{r:6.1f}" for r in res))
