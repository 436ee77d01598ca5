"""CPU baseline of the same O(N) algorithm (cpu_fmm.c): a REPORTED baseline for bench.py, not the
oracle and not part of the product.  The plan tables come from a GPU plan (lc_plan_export)."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "cpu_fmm.c")
LIB = os.path.join(HERE, "libcpufmm.so")
_lib = None


def build(force: bool = False) -> None:
    if force or not os.path.exists(LIB) or os.path.getmtime(SRC) > os.path.getmtime(LIB):
        subprocess.run(["gcc", "-O3", "-fopenmp", "-shared", "-fPIC", SRC, "-o", LIB, "-lm"], check=True)


def load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(LIB)
        d = ctypes.POINTER(ctypes.c_double)
        lib.cpu_fmm_execute.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                        d, d, d, d, d, d, d]
        lib.cpu_fmm_execute.restype = ctypes.c_int
        lib.cpu_fmm_threads.restype = ctypes.c_int
        lib.cpu_fmm_set_threads.argtypes = [ctypes.c_int]
        lib.cpu_fmm_set_threads.restype = None
        _lib = lib
    return _lib


def threads() -> int:
    return int(load().cpu_fmm_threads())


def set_threads(t: int) -> None:
    load().cpu_fmm_set_threads(int(t))


class CpuFmm:
    """The execution stage on the host, with the tables of a GPU plan (paper_2411_00033_b200.Plan)."""

    def __init__(self, plan):
        d = plan.desc
        self.n, self.N, self.L, self.s = int(d["n"]), int(d["N"]), int(d["L"]), int(d["s"])
        self.dir = int(d["direction"])
        self.tabB = np.ascontiguousarray(plan.export("tabB"))
        self.tabA = np.ascontiguousarray(plan.export("tabA"))
        self.A = np.ascontiguousarray(plan.export("ahat")) if self.L > 0 else np.zeros(1)
        self.B = np.ascontiguousarray(plan.export("B"))
        self.T = np.ascontiguousarray(plan.export("T"))

    def __call__(self, f: np.ndarray) -> np.ndarray:
        lib = load()
        f = np.ascontiguousarray(f, dtype=np.float64)
        z = np.empty(self.n, dtype=np.float64)
        p = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
        rc = lib.cpu_fmm_execute(self.dir, self.n, self.N, self.L, self.s, p(self.A), p(self.tabA), p(self.tabB),
                                 p(self.T), p(self.B), p(f), p(z))
        if rc != 0:
            raise MemoryError("cpu_fmm_execute: allocation failed")
        return z
