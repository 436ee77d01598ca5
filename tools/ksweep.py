"""Sweep execution-kernel configurations for one workload; per-kernel CUDA-event times (no graph)."""
import itertools, json, sys
import torch


def gpu_warmup(seconds=1.0):
    """Run dense work for `seconds` so the SM clock ramps up from idle before timing."""
    import time
    a = torch.randn(4096, 4096, device="cuda")
    t = time.time()
    while time.time() - t < seconds:
        a = a @ a
        a /= a.norm()
    torch.cuda.synchronize()
sys.path.insert(0, '.')
from lc_inputs import vector
from paper_2411_00033_b200 import Plan

def run(n, d, V=1, reps=30, **opts):
    dev = torch.device('cuda', 0)
    x = torch.stack([torch.from_numpy(vector("sign_over_j1", n, 0, v)) for v in range(V)]).to(dev)
    y = torch.empty_like(x)
    p = Plan(n, d, batch=V, device=dev, **opts)
    kpe = p.kernels_per_execute
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(kpe + 1)]
    for _ in range(200):
        p.execute(x, y)
    acc = [0.0] * kpe
    for _ in range(reps):
        p.execute_timed(x, y, ev)
        torch.cuda.synchronize()
        for i in range(kpe):
            acc[i] += ev[i].elapsed_time(ev[i + 1]) * 1e3 / reps
    # plain (PDL-chained) execution time
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(reps):
        p.execute(x, y)
    s1.record(); torch.cuda.synchronize()
    tot = s0.elapsed_time(s1) * 1e3 / reps
    cfg = {k: p.desc[k] for k in ('vt', 'subtree', 'stage_blocks', 'stages')}
    print(json.dumps({"n": n, "dir": d, "V": V, "opts": opts, "cfg": cfg, "kernels_us": [round(a, 1) for a in acc],
                      "chained_us": round(tot, 1)}), flush=True)
    p.close()

if __name__ == "__main__":
    gpu_warmup(1.5)
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
    import itertools
    for kup in (4, 5, 6):
        run(n, "leg2cheb", up_subtree=kup)
    for k in (3, 4, 5):
        run(n, "leg2cheb", subtree=k)
    for cb, nst in ((3, 2), (3, 3), (3, 4), (2, 6), (4, 3), (6, 2)):
        run(n, "leg2cheb", stage_blocks=cb, stages=nst)
