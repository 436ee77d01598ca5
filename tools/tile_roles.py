"""Per-warp cycle accounting of the per-tile kernel (debug build liblegcheb_dbg.so): role work,
M2L jobs, end-of-step wait, averaged over CTAs, per leaf step (engine 2, or 3 for the range kernel).
usage: python tools/tile_roles.py n batch [engine]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2411_00033_b200 import _lib  # noqa: E402
_lib.LIB_PATH = _lib.LIB_PATH.replace("liblegcheb.so", "liblegcheb_dbg.so")
from paper_2411_00033_b200 import Plan  # noqa: E402
from lc_inputs import batch as mkbatch  # noqa: E402

n, V = int(sys.argv[1]), int(sys.argv[2])
engine = int(sys.argv[3]) if len(sys.argv) > 3 else 2
dev = torch.device("cuda", 0)
x = mkbatch("normal", n, V, seed=1).to(dev)
p = Plan(n, "leg2cheb", batch=V, device=dev, engine=engine)
lib = _lib.load()
lib.lc_debug_timestamps.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_longlong]
for _ in range(3):
    p.execute(x)
torch.cuda.synchronize()
lib.lc_debug_clear()
p.execute(x)
torch.cuda.synchronize()
buf = np.zeros(1 << 20, dtype=np.uint64)
lib.lc_debug_timestamps(0, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), buf.size)
grid = p.kernel_info["tile_grid"]
a = buf[: grid * 64].reshape(grid, 8, 8).astype(np.float64)
steps = a[:, :, 4].sum(axis=0)
print(f"n={n} batch={V} grid={grid}; cycles per leaf step, mean over CTAs")
for w in range(8):
    st = max(steps[w], 1)
    print(f"warp {w}: stage {a[:, w, 5].sum() / st:6.0f}  role-a {a[:, w, 0].sum() / st:7.0f}  role-b {a[:, w, 1].sum() / st:7.0f}  "
          f"m2l {a[:, w, 2].sum() / st:7.0f}  end {a[:, w, 3].sum() / st:7.0f}")
