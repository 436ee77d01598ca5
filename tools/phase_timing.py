"""Per-CTA phase timestamps (%globaltimer) of the instrumented build liblegcheb_dbg.so."""
import ctypes, sys
import numpy as np
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
gpu_warmup(1.5)
for _ in range(200):
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
for kern, name in enumerate(["up", "fmm", "down"]):
    lib.lc_debug_timestamps(kern, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), buf.size)
    a = buf.reshape(-1, 8).astype(np.int64).copy()
    a = a[a[:, 0] > 0]
    if len(a):
        ts[name] = a
t0 = min(ts[k][:, 0].min() for k in ts if k != "up")
print("config", p.desc["vt"], p.desc["subtree"], p.desc["stage_blocks"], p.desc["stages"])
if "up" in ts:  # up-role task 0: slots 0 (input ready) 1 (step 1) 2 (merges) 3 (writes) 4 (fence)
    a = ts.pop("up")
    d = np.diff(a[:, :5], axis=1) / 1e3
    print("up task0 phase durations med (us): step1 %.2f merges %.2f write %.2f fence %.2f; input ready at %.2f us"
          % tuple(list(np.median(d, axis=0)) + [np.median((a[:, 0] - t0) / 1e3)]))
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
