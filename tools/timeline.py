"""Per-CTA phase timeline (%globaltimer, ns) of one execute, from the instrumented build
liblegcheb_dbg.so (`make debug`).  Slots (see LC_TS in lc_exec.cu):
  up:     0 start 1 staged 2 step1 3 subtree-M2M 4 written 5 continuation 6 cont-done 7 exit
  stream: 0 start 1 end 2 first-M2L-wait 3 first-slot-full 4 fine-w-flag 5 coarse-w-flag
  down:   0 start 1 after-griddep-wait 2 loaded 3 chain 4 subtree 5 end
usage: python tools/timeline.py n direction [opt=val ...]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2411_00033_b200 import _lib  # noqa: E402
_lib.LIB_PATH = _lib.LIB_PATH.replace("liblegcheb.so", "liblegcheb_dbg.so")
from paper_2411_00033_b200 import Plan  # noqa: E402
from lc_inputs import vector  # noqa: E402


def gpu_warmup(seconds=1.0):
    import time
    a = torch.randn(4096, 4096, device="cuda")
    t = time.time()
    while time.time() - t < seconds:
        a = a @ a
        a /= a.norm()
    torch.cuda.synchronize()


n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
d = sys.argv[2] if len(sys.argv) > 2 else "leg2cheb"
opts = {k: int(v) for k, v in (a.split("=") for a in sys.argv[3:])}
batch = opts.pop("batch", 1)
dev = torch.device("cuda", 0)
x = torch.from_numpy(np.stack([vector("sign_over_j1", n, 0, v) for v in range(batch)])).to(dev)
p = Plan(n, d, batch=batch, device=dev, **opts)
lib = _lib.load()
lib.lc_debug_timestamps.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_longlong]
gpu_warmup(1.5)
for _ in range(300 if n * batch < 10**7 else 5):
    y = p.execute(x)
torch.cuda.synchronize()
NAMES = {"up": ["start", "staged", "step1", "subtreeM2M", "written", "cont", "contdone", "exit"],
         "upb": ["start", "lvlL-2", "lvlL-3", "merge0", "merge0done", "cont", "contdone", "end"],
         "stream": ["start", "end", "banddone", "-", "-", "-", "-", "m2ldone"],
         "down": ["start", "gdwait", "loaded", "chain", "subtree", "end", "lvl1-3", "lvlsdone"]}
for rep in range(2):
    lib.lc_debug_clear()
    torch.cuda.synchronize()
    y = p.execute(x)
    torch.cuda.synchronize()
    buf = np.zeros(1 << 20, dtype=np.uint64)
    ts = {}
    for kern, name in enumerate(n for n in NAMES if n != "upb"):
        lib.lc_debug_timestamps(kern, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), buf.size)
        a = buf.reshape(-1, 8).astype(np.int64).copy()
        if name == "up":  # lc_upb_kernel (split up pass) writes rows 100000 + CTA of the up table
            ub = a[100000:]
            ts["upb"] = ub[ub[:, 0] > 0]
            a = a[:100000]
        ts[name] = a[a[:, 0] > 0]
    t0 = ts["up"][:, 0].min() if len(ts["up"]) else ts["stream"][:, 0].min()
    ts = {k: ts[k] for k in ("up", "upb", "stream", "down") if k in ts}
    allv = np.concatenate([a[a > 0] for a in ts.values()])
    diffs = np.diff(np.unique(allv))
    print(f"=== rep {rep}: n={n} {d} batch={batch} desc vt={p.desc['vt']} subtree={p.desc['subtree']}"
          f" stage_blocks={p.desc['stage_blocks']} stages={p.desc['stages']}; timer granularity ~{np.min(diffs) if len(diffs) else 0} ns")
    for name, a in ts.items():
        if not len(a):
            continue
        st = (a[:, 0] - t0) / 1e3
        print(f"{name:6s}: CTAs {len(a):5d}  start min {st.min():7.2f} med {np.median(st):7.2f} max {st.max():7.2f} us")
        for ph in range(1, 8):
            if NAMES[name][ph] == "-":
                continue
            m = a[:, ph] > 0
            if m.sum() == 0:
                continue
            dt = (a[m, ph] - a[m, 0]) / 1e3
            end = (a[m, ph] - t0) / 1e3
            print(f"   {ph} {NAMES[name][ph]:11s} n={m.sum():5d}  since start med {np.median(dt):7.2f} max {dt.max():7.2f}"
                  f"  | abs min {end.min():7.2f} med {np.median(end):7.2f} max {end.max():7.2f} us")
