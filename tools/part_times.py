"""NEXT-2 evidence on one GPU: device time of each part of a partitioned single-vector transform
(lc_plan_opts.part_index / part_count), parts run alone one after another.  On G GPUs the parts run
concurrently, so the slowest part plus the all-gather of the rows bounds one transform.
usage: python tools/part_times.py n [parts ...] [--up]   (--up: partitioned upward pass, phases 0 + 1 per part;
the exchange between them is an all-gather of a few hundred KB, not timed here)"""
import json
import sys

import torch

sys.path.insert(0, ".")
from lc_inputs import vector  # noqa: E402
from paper_2411_00033_b200 import Plan  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
up = "--up" in sys.argv
parts_list = [int(a) for a in sys.argv[2:] if a != "--up"] or [1, 2, 4, 8]
dev = torch.device("cuda", 0)
x = torch.from_numpy(vector("sign_over_j1", n, seed=0)).reshape(1, -1).to(dev)
out = torch.empty_like(x)
res = {"n": n, "part_up": up}
for G in parts_list:
    times = []
    for p in range(G):
        plan = Plan(n, "leg2cheb", device=dev, part_index=p, part_count=G, part_up=int(up)) if G > 1 \
            else Plan(n, "leg2cheb", device=dev)
        ws = plan.new_workspace()
        pu = G > 1 and up

        def run():
            if pu:
                plan.execute_part(0, x, out, ws)
                plan.execute_part(1, x, out, ws)
            else:
                plan.execute(x, out)
        for _ in range(20):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 200
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / reps * 1e3)
        plan.close()
    res[f"G={G}"] = {"part_us": [round(t, 1) for t in times], "max_part_us": round(max(times), 1)}
    print(G, [round(t, 1) for t in times], flush=True)
print(json.dumps(res))
