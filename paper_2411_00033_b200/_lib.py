"""ctypes binding of the C ABI in include/legcheb.h (argument marshalling only).

Every arithmetic step of the transform runs in the sm_100a kernels of
liblegcheb.so; this module only loads the library and declares signatures.
There is no CPU fallback: if the extension is missing the import fails.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblegcheb.so")

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_vp = ctypes.c_void_p
c_dp = ctypes.POINTER(ctypes.c_double)


class PlanOpts(ctypes.Structure):
    _fields_ = [("s_hat", c_i64), ("M", c_i32), ("layout", c_i32), ("ld_in", c_i64), ("ld_out", c_i64),
                ("device", c_i32), ("vt", c_i32), ("subtree", c_i32), ("stage_blocks", c_i32), ("stages", c_i32),
                ("up_subtree", c_i32), ("engine", c_i32), ("part_index", c_i32), ("part_count", c_i32),
                ("part_up", c_i32), ("out_block", c_i64)]


class PlanDesc(ctypes.Structure):
    _fields_ = [("n", c_i64), ("N", c_i64), ("L", c_i64), ("s", c_i64), ("M", c_i64), ("batch", c_i64),
                ("nc", c_i64), ("direction", c_i64), ("band_nnz", c_i64), ("plan_bytes", ctypes.c_size_t),
                ("workspace_bytes", ctypes.c_size_t), ("flops_alg", ctypes.c_double), ("bytes_alg", ctypes.c_double),
                ("vt", c_i32), ("subtree", c_i32), ("stage_blocks", c_i32), ("stages", c_i32),
                ("kernels_per_execute", c_i32), ("plan_device_ms", ctypes.c_double), ("row_lo", c_i64),
                ("row_hi", c_i64)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


# name -> (restype, argtypes); must match include/legcheb.h (checked by tests/test_host.py)
SIGNATURES = {
    "lc_geometry": (c_i32, [c_i64, c_i64, ctypes.POINTER(PlanDesc)]),
    "lc_partition": (c_i32, [c_i64, c_i64, c_i32, c_i32, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
    "lc_plan_create": (c_i32, [ctypes.POINTER(c_vp), c_i64, c_i32, c_i64, ctypes.POINTER(PlanOpts)]),
    "lc_plan_describe": (c_i32, [c_vp, ctypes.POINTER(PlanDesc)]),
    "lc_workspace_bytes": (ctypes.c_size_t, [c_vp]),
    "lc_workspace_init": (c_i32, [c_vp, c_vp, c_vp]),
    "lc_execute": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "lc_execute_part": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "lc_execute_timed": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.POINTER(c_vp), c_i32]),
    "lc_host_stage_bytes": (ctypes.c_size_t, [c_vp]),
    "lc_execute_host": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "lc_host_chain_stage_bytes": (ctypes.c_size_t, [ctypes.POINTER(c_vp), c_i32]),
    "lc_execute_host_chain": (c_i32, [ctypes.POINTER(c_vp), c_i32, c_vp, c_vp, c_vp, ctypes.POINTER(c_vp), c_vp]),
    "lc_host_alloc": (c_i32, [ctypes.c_size_t, ctypes.POINTER(c_vp)]),
    "lc_host_free": (c_i32, [c_vp]),
    "lc_plan_export": (c_i32, [c_vp, c_i32, c_dp, c_i64]),
    "lc_plan_kernel_info": (c_i32, [c_vp, ctypes.POINTER(c_i64), c_i32, ctypes.POINTER(c_i32)]),
    "lc_plan_destroy": (c_i32, [c_vp]),
    "lc_status_string": (ctypes.c_char_p, [c_i32]),
    "lc_version": (ctypes.c_char_p, []),
    "lc_last_error": (ctypes.c_char_p, []),
}

_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "or `make` (there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class LegChebError(RuntimeError):
    def __init__(self, fn: str, status: int):
        msg = load().lc_status_string(status).decode()
        if status in (3, 4):
            msg += " [" + load().lc_last_error().decode() + "]"
        super().__init__(f"{fn} failed: {msg} (status {status})")
        self.status = status


def check(fn: str, status: int) -> None:
    if status != 0:
        raise LegChebError(fn, status)
