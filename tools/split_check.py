"""Functional check of dist.SingleVectorTransform across processes (torchrun, gloo, ranks may share a GPU):
every step's round trip against the whole (unpartitioned) plans.  usage: torchrun --nproc-per-node 2 tools/split_check.py"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from lc_inputs import vector  # noqa: E402
from paper_2411_00033_b200 import Plan  # noqa: E402
from paper_2411_00033_b200.dist import SingleVectorTransform  # noqa: E402

dist.init_process_group(os.environ.get("LC_DIST_BACKEND", "gloo"))
rank = dist.get_rank()
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
dev = torch.device("cuda", torch.cuda.current_device())
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
x = torch.from_numpy(vector("sign_over_j1", n, seed=0)).to(dev)
pl, pc = Plan(n, "leg2cheb", device=dev), Plan(n, "cheb2leg", device=dev)
zref = pl.execute(x.reshape(1, -1)).reshape(-1)
yref = pc.execute(zref.reshape(1, -1)).reshape(-1)
up = len(sys.argv) > 2 and sys.argv[2] == "up"  # partitioned upward pass with the root / halo exchange
sl = SingleVectorTransform(n, "leg2cheb", device=dev, part_up=up)
sc = SingleVectorTransform(n, "cheb2leg", device=dev, part_up=up)
for it in range(5):
    z = sl(x)
    ez = float((z - zref).abs().max() / zref.abs().max())
    y = sc(z)
    ey = float((y - yref).abs().max() / yref.abs().max())
    ez_part = float((z[sl.row_lo:sl.row_hi] - zref[sl.row_lo:sl.row_hi]).abs().max())
    print(f"rank {rank} it {it}: z err {ez:.3e} (own rows abs {ez_part:.3e}) y err {ey:.3e}", flush=True)
dist.destroy_process_group()
