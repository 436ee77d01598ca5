"""Pinned host -> device copy throughput by size and by host allocation: cudaHostAlloc (torch
pin_memory) vs an mmap'ed buffer with transparent huge pages (madvise) registered with
cudaHostRegister.  usage: python tools/h2d_sizes.py"""
import ctypes
import mmap

import numpy as np
import torch

dev = torch.device("cuda", 0)
libc = ctypes.CDLL("libc.so.6")
MADV_HUGEPAGE = 14


def thp_pinned(nbytes):
    """A 2 MB-aligned anonymous mapping advised for huge pages, touched, then page-locked."""
    al = 1 << 21
    m = mmap.mmap(-1, nbytes + al, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    base = ctypes.addressof(ctypes.c_char.from_buffer(m))
    off = (-base) % al
    addr = base + off
    rc = libc.madvise(ctypes.c_void_p(addr), ctypes.c_size_t(nbytes), MADV_HUGEPAGE)
    arr = np.frombuffer(m, dtype=np.uint8, count=nbytes, offset=off)
    arr[:] = 1  # touch
    t = torch.from_numpy(arr).view(torch.float64)
    err = torch.cuda.cudart().cudaHostRegister(addr, nbytes, 0)
    return t, m, rc, int(err)


def bw(h, d, reps=50):
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


try:
    print("THP:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
except OSError as e:
    print("THP: n/a", e)
keep = []
for mb in [2, 8, 16, 64]:
    n = int(mb * (1 << 20))
    d = torch.empty(n // 8, dtype=torch.float64, device=dev)
    h = torch.empty(n // 8, dtype=torch.float64).pin_memory()
    t1 = bw(h, d)
    th, m, rc, err = thp_pinned(n)
    keep.append(m)
    t2 = bw(th, d)
    t3 = bw(d, th) if False else None
    print(f"{mb:3d} MiB  cudaHostAlloc h2d {n / t1 / 1e6:5.1f} GB/s   THP+register h2d {n / t2 / 1e6:5.1f} GB/s "
          f"(madvise rc {rc}, register err {err}, pinned {th.is_pinned()})")
