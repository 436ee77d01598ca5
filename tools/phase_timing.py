"""Per-CTA phase timestamps (%globaltimer) of the instrumented build liblegcheb_dbg.so."""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2411_00033_b200 import _lib
_lib.LIB_PATH = _lib.LIB_PATH.replace("liblegcheb.so", "liblegcheb_dbg.so")
from paper_2411_00033_b200 import Plan
from lc_inputs import vector

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
d = sys.argv[2] if len(sys.argv) > 2 else "leg2cheb"
opts = dict(a.split("=") for a in sys.argv[3:])
opts = {k: int(v) for k, v in opts.items()}
dev = torch.device("cuda", 0)
x = torch.from_numpy(vector("sign_over_j1", n, 0, 0)).reshape(1, -1).to(dev)
p = Plan(n, d, device=dev, **opts)
lib = _lib.load()
lib.lc_debug_timestamps.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_longlong]
for _ in range(3):
    y = p.execute(x)
torch.cuda.synchronize()
# clear, run once
ts = {}
buf = np.zeros(1 << 20, dtype=np.uint64)
lib.lc_debug_timestamps  # noqa
zero = np.zeros(1 << 20, dtype=np.uint64)
y = p.execute(x)
torch.cuda.synchronize()
t0 = None
for kern, name in enumerate(["up", "m2l", "down"]):
    lib.lc_debug_timestamps(kern, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), buf.size)
    a = buf.reshape(-1, 8).astype(np.int64).copy()
    a = a[a[:, 0] > 0]
    ts[name] = a
t0 = min(ts[k][:, 0].min() for k in ts)
print("config", p.desc["vt"], p.desc["subtree"], p.desc["stage_blocks"], p.desc["stages"])
for name, a in ts.items():
    start = (a[:, 0] - t0) / 1e3
    print(f"{name}: CTAs {len(a)}  first start {start.min():.1f} us  last start {start.max():.1f} us")
    for ph in range(1, 8):
        m = a[:, ph] > 0
        if m.sum() == 0:
            continue
        dt = (a[m, ph] - a[m, 0]) / 1e3
        end = (a[m, ph] - t0) / 1e3
        print(f"   phase {ph}: n={m.sum():5d} since-CTA-start med {np.median(dt):7.2f} max {dt.max():7.2f} us;"
              f" abs end max {end.max():7.2f} us")
