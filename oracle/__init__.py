"""CPU oracle for the Legendre<->Chebyshev connection transform (arXiv 2411.00033).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  The product path (``paper_2411_00033_b200``) never imports it, and it
never imports the product path.

The arithmetic lives in ``oracle.c`` (x87 long double, Neumaier-compensated
sums, O(n^2) direct definitions); this module is ctypes marshalling plus the
relative max-norm of PAPER.md:525-529 (eq:Einf).

Functions
---------
lam(n)                     lambda_k = Lambda(k), k < n
l2c_rows(f, rows)          rows of C^{-1} A f                 PAPER.md:24-46, Alg. 1
c2l_rows(f, rows)          rows of A^{-1} C f (eq:Lxymod rows) PAPER.md:31, 509-514
c2l_backsub(f)             A^{-1} C f by back-substitution
l2c_rows_q, c2l_rows_q     the same rows in __float128 with plain sums (cross-check tier of the
                           compensated long-double sums)
l2c(f), c2l(f)             all rows
einf(z, zstar)             ||z - z*||_inf / ||z*||_inf        PAPER.md:527 (eq:Einf)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

LD = np.longdouble
_ldp = ctypes.POINTER(ctypes.c_longdouble)
_lp = ctypes.POINTER(ctypes.c_long)


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC",
               _SRC, "-o", _LIB, "-lquadmath", "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


def _get():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.orc_lambda.argtypes = [ctypes.c_long, _ldp]
        lib.orc_lambda.restype = None
        for name in ("orc_l2c_rows", "orc_c2l_rows"):
            fn = getattr(lib, name)
            fn.argtypes = [_ldp, ctypes.c_long, _lp, ctypes.c_long, _ldp, _ldp]
            fn.restype = ctypes.c_int
        for name in ("orc_l2c_rows_q", "orc_c2l_rows_q"):
            fn = getattr(lib, name)
            fn.argtypes = [_ldp, ctypes.c_long, _lp, ctypes.c_long, _ldp, ctypes.c_int]
            fn.restype = ctypes.c_int
        lib.orc_c2l_backsub.argtypes = [_ldp, ctypes.c_long, _ldp]
        lib.orc_c2l_backsub.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ld(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=LD))


def lam(n: int) -> np.ndarray:
    out = np.empty(int(n), dtype=LD)
    _get().orc_lambda(int(n), out.ctypes.data_as(_ldp))
    return out


def _rows(fn, f, rows, with_abs):
    f = _ld(f)
    n = f.shape[0]
    if rows is None:
        rows = np.arange(n, dtype=np.int64)
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    if rows.size and (rows.min() < 0 or rows.max() >= n):
        raise IndexError("row out of range")
    out = np.empty(rows.shape[0], dtype=LD)
    ab = np.empty(rows.shape[0], dtype=LD)
    rc = fn(f.ctypes.data_as(_ldp), n, rows.ctypes.data_as(_lp), rows.shape[0],
            out.ctypes.data_as(_ldp), ab.ctypes.data_as(_ldp))
    if rc:
        raise RuntimeError(f"oracle failed rc={rc}")
    return (out, ab) if with_abs else out


def l2c_rows(f, rows=None, with_abs: bool = False):
    return _rows(_get().orc_l2c_rows, f, rows, with_abs)


def c2l_rows(f, rows=None, with_abs: bool = False):
    return _rows(_get().orc_c2l_rows, f, rows, with_abs)


def _rows_q(fn, f, rows, lam_ld):
    f = _ld(f)
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    if rows.size and (rows.min() < 0 or rows.max() >= f.shape[0]):
        raise IndexError("row out of range")
    out = np.empty(rows.shape[0], dtype=LD)
    rc = fn(f.ctypes.data_as(_ldp), f.shape[0], rows.ctypes.data_as(_lp), rows.shape[0], out.ctypes.data_as(_ldp),
            int(bool(lam_ld)))
    if rc:
        raise RuntimeError(f"oracle failed rc={rc}")
    return out


def l2c_rows_q(f, rows, lam_ld: bool = False):
    """L2C rows in __float128 (plain sums): the cross-check tier of l2c_rows.  lam_ld: use the
    long-double lambda (isolates the summation) instead of the quad recurrence."""
    return _rows_q(_get().orc_l2c_rows_q, f, rows, lam_ld)


def c2l_rows_q(f, rows, lam_ld: bool = False):
    """C2L rows (eq:Lxymod) in __float128 (plain sums): the cross-check tier of c2l_rows."""
    return _rows_q(_get().orc_c2l_rows_q, f, rows, lam_ld)


def c2l_backsub(f) -> np.ndarray:
    f = _ld(f)
    out = np.empty_like(f)
    rc = _get().orc_c2l_backsub(f.ctypes.data_as(_ldp), f.shape[0], out.ctypes.data_as(_ldp))
    if rc:
        raise RuntimeError(f"oracle failed rc={rc}")
    return out


def l2c(f):
    return l2c_rows(f)


def c2l(f):
    return c2l_rows(f)


def transform_rows(direction: str, f, rows=None, with_abs: bool = False):
    if direction in ("l2c", "leg2cheb", 0):
        return l2c_rows(f, rows, with_abs)
    if direction in ("c2l", "cheb2leg", 1):
        return c2l_rows(f, rows, with_abs)
    raise ValueError(direction)


def einf(z, zstar) -> float:
    """Relative max norm E_inf = ||z - z*||_inf / ||z*||_inf."""
    z = np.asarray(z, dtype=LD)
    zs = np.asarray(zstar, dtype=LD)
    den = np.max(np.abs(zs))
    if den == 0:
        raise ZeroDivisionError("zero reference norm")
    return float(np.max(np.abs(z - zs)) / den)
