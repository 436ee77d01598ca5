"""Per-CTA band-unit phase sums of the debug build (slots 3..6 of the streaming kernel)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2411_00033_b200 import _lib  # noqa: E402
_lib.LIB_PATH = _lib.LIB_PATH.replace("liblegcheb.so", "liblegcheb_dbg.so")
from paper_2411_00033_b200 import Plan  # noqa: E402
from lc_inputs import vector  # noqa: E402

n, batch, vt = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dev = torch.device("cuda", 0)
x = torch.from_numpy(np.stack([vector("sign_over_j1", n, 0, v) for v in range(batch)])).to(dev)
p = Plan(n, "leg2cheb", batch=batch, device=dev, vt=vt)
lib = _lib.load()
lib.lc_debug_timestamps.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_longlong]
for _ in range(3):
    p.execute(x)
torch.cuda.synchronize()
lib.lc_debug_clear()
p.execute(x)
torch.cuda.synchronize()
buf = np.zeros(1 << 20, dtype=np.uint64)
lib.lc_debug_timestamps(1, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), buf.size)
a = buf.reshape(-1, 8).astype(np.int64)[: p.kernel_info["stream_grid"]]
units = a[:, 6]
print("CTAs", len(a), "band units per CTA mean", units.mean())
for k, name in ((3, "load wait"), (4, "compute"), (5, "store")):
    print(f"{name:10s} total per CTA mean {a[:, k].mean() / 1e3:8.2f} us, per unit {a[:, k].sum() / max(units.sum(), 1) / 1e3:7.3f} us")
print("kernel span (slot1-slot0) mean", ((a[:, 1] - a[:, 0]) / 1e3).mean(), "us")
