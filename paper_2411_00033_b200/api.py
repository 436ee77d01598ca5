"""Python API over the C ABI: plans and transforms on torch CUDA tensors.

    plan = Plan(n, "leg2cheb", batch=V)          # lc_plan_create
    z = plan.execute(x)                          # lc_execute on torch's current stream
    leg2cheb(x), cheb2leg(x)                     # cached-plan conveniences

PyTorch provides device memory and streams only; the transform itself is the
sm_100a kernels of liblegcheb.so (Alg. 4, alg:fastercomplete).
"""
from __future__ import annotations

import ctypes
import threading

import numpy as np
import torch

from . import _lib

DIRECTIONS = {"leg2cheb": 0, "l2c": 0, 0: 0, "cheb2leg": 1, "c2l": 1, 1: 1}
LAYOUTS = {"vec": 0, "batch": 1, 0: 0, 1: 1}
EXPORTS = {"tabB": 0, "tabA": 1, "ahat": 2, "B": 3, "T": 4}


def geometry(n: int, s_hat: int = 0) -> dict:
    """Host-only decomposition (eq:numlevels, eq:Ntot, eq:total_blocks_and_mats) and work model."""
    d = _lib.PlanDesc()
    _lib.check("lc_geometry", _lib.load().lc_geometry(int(n), int(s_hat), ctypes.byref(d)))
    return d.as_dict()


def partition(n: int, part_index: int, part_count: int, s_hat: int = 0) -> tuple[int, int]:
    """Output rows [lo, hi) of part part_index of part_count (lc_partition; host only): contiguous runs of
    whole groups of leaf segments, for one long transform split over several GPUs (NEXT-2)."""
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    _lib.check("lc_partition", _lib.load().lc_partition(int(n), int(s_hat), int(part_index), int(part_count),
                                                        ctypes.byref(lo), ctypes.byref(hi)))
    return int(lo.value), int(hi.value)


class _HostBuffer:
    """Owner of one lc_host_alloc buffer: released (lc_host_free) when the last view of it is gone."""

    def __init__(self, nbytes: int):
        ptr = ctypes.c_void_p()
        _lib.check("lc_host_alloc", _lib.load().lc_host_alloc(int(nbytes), ctypes.byref(ptr)))
        self.ptr = ptr.value

    def __del__(self):
        if self.ptr:
            _lib.load().lc_host_free(ctypes.c_void_p(self.ptr))
            self.ptr = None


def host_empty(shape, dtype=torch.float64) -> torch.Tensor:
    """A zero-filled CPU tensor in page-locked host memory on huge pages (lc_host_alloc), for
    Plan.execute_host / host<->device copies: on this pool's B200 boxes 8-16 MiB host-to-device copies
    from such memory run at ~55 GB/s against 12-15 GB/s from torch.empty(..., pin_memory=True).
    The memory is freed when the tensor (and every view of it) is gone."""
    shape = tuple(int(d) for d in (shape if isinstance(shape, (tuple, list, torch.Size)) else (shape,)))
    itemsize = torch.empty((), dtype=dtype).element_size()
    nbytes = max(1, int(np.prod(shape, dtype=np.int64)) * itemsize)
    owner = _HostBuffer(nbytes)
    raw = (ctypes.c_char * nbytes).from_address(owner.ptr)
    raw.owner = owner  # the numpy array -> raw -> owner chain keeps the mapping alive
    arr = np.frombuffer(raw, dtype=np.uint8, count=nbytes)
    return torch.from_numpy(arr)[: nbytes - nbytes % itemsize].view(dtype).reshape(shape)


def _stream_handle(stream, device=None) -> int:
    """cudaStream_t of `stream`; None -> torch's current stream of `device` (the plan's device)."""
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


class Plan:
    """A transform plan (immutable) for `batch` vectors of length n on one device."""

    def __init__(self, n: int, direction="leg2cheb", batch: int = 1, device=None, s_hat: int = 0,
                 layout="vec", ld_in: int = 0, ld_out: int = 0, vt: int = 0, subtree: int = 0,
                 stage_blocks: int = 0, stages: int = 0, up_subtree: int = 0,
                 engine: int = 0, part_index: int = 0, part_count: int = 0, part_up: int = 0,
                 out_block: int = 0):
        lib = _lib.load()
        if device is None:
            device = torch.cuda.current_device()
        device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.device = device
        self.n, self.batch = int(n), int(batch)
        self.direction = DIRECTIONS[direction]
        self.layout = LAYOUTS[layout]
        opts = _lib.PlanOpts(s_hat=s_hat, M=18, layout=self.layout, ld_in=ld_in, ld_out=ld_out,
                             device=device.index if device.index is not None else -1, vt=vt, subtree=subtree,
                             stage_blocks=stage_blocks, stages=stages, up_subtree=up_subtree,
                             engine=engine, part_index=part_index, part_count=part_count, part_up=part_up,
                             out_block=out_block)
        h = ctypes.c_void_p()
        with torch.cuda.device(device):
            _lib.check("lc_plan_create", lib.lc_plan_create(ctypes.byref(h), self.n, self.direction, self.batch,
                                                            ctypes.byref(opts)))
        self._h = h
        self._lib = lib
        d = _lib.PlanDesc()
        _lib.check("lc_plan_describe", lib.lc_plan_describe(h, ctypes.byref(d)))
        self.desc = d.as_dict()
        self.ld_in = ld_in or (self.n if self.layout == 0 else self.batch)
        self.ld_out = ld_out or (self.n if self.layout == 0 else self.batch)
        self.out_block = int(out_block)
        self._ws_lock = threading.Lock()
        self._ws_by_stream: dict = {}

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.lc_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    @property
    def workspace_bytes(self) -> int:
        return int(self._lib.lc_workspace_bytes(self._h))

    @property
    def kernel_info(self) -> dict:
        """Kernel configuration of the plan (lc_plan_kernel_info)."""
        buf = (ctypes.c_int64 * 32)()
        nw = ctypes.c_int32(0)
        _lib.check("lc_plan_kernel_info", self._lib.lc_plan_kernel_info(self._h, buf, 32, ctypes.byref(nw)))
        names = ["stream_grid", "smem_stream", "smem_up", "kup", "grup", "kb", "cb", "nst", "vt", "stream_occ",
                 "m2l_units", "band_units", "up_grid", "kd", "smem_down", "engine", "tile_grid", "smem_tile",
                 "ranges", "range_len", "up_ksub", "part_lo", "part_hi", "part_up"]
        return {k: int(buf[i]) for i, k in enumerate(names[:nw.value])}

    @property
    def kernels_per_execute(self) -> int:
        return int(self.desc["kernels_per_execute"])

    def _shape(self, ld=None, output=False):
        if output and self.out_block:  # column-blocked: [n / B][batch][B]
            B = self.out_block
            return ((self.n + B - 1) // B, self.batch, B)
        ld = self.ld_in if ld is None else ld
        return (self.batch, ld) if self.layout == 0 else (self.n, ld)

    def _check(self, x: torch.Tensor, what: str):
        if x.device != self.device or x.dtype != torch.float64 or not x.is_contiguous():
            raise ValueError(f"{what}: need a contiguous float64 tensor on {self.device}")
        ld = self.ld_in if what == "input" else self.ld_out
        rows, cols = (self.batch, self.n) if self.layout == 0 else (self.n, self.batch)
        need = (rows - 1) * ld + cols  # the extent the kernels address (rows of stride ld)
        if what == "output" and self.out_block:
            need = -(-self.n // self.out_block) * self.batch * self.out_block
        if x.numel() < need:
            raise ValueError(f"{what}: {x.numel()} elements, the plan addresses {need}")

    @property
    def plan_device_ms(self) -> float:
        """Device time of the planning kernels measured at create (CUDA events)."""
        return float(self.desc["plan_device_ms"])

    @property
    def host_stage_bytes(self) -> int:
        return int(self._lib.lc_host_stage_bytes(self._h))

    def new_workspace(self, stream=None) -> torch.Tensor:
        ws = torch.empty(max(1, self.workspace_bytes), dtype=torch.uint8, device=self.device)
        _lib.check("lc_workspace_init", self._lib.lc_workspace_init(
            self._h, ctypes.c_void_p(ws.data_ptr()), ctypes.c_void_p(_stream_handle(stream, self.device))))
        return ws

    @property
    def in_extent(self) -> int:
        """Elements spanned by the input array (layout and leading dimension)."""
        rows, cols = (self.batch, self.n) if self.layout == 0 else (self.n, self.batch)
        return (rows - 1) * self.ld_in + cols

    @property
    def out_extent(self) -> int:
        """Elements spanned by the output array (layout, leading dimension, column blocking)."""
        if self.out_block:
            return -(-self.n // self.out_block) * self.batch * self.out_block
        rows, cols = (self.batch, self.n) if self.layout == 0 else (self.n, self.batch)
        return (rows - 1) * self.ld_out + cols

    def new_host_stage(self) -> torch.Tensor:
        """Caller-owned device staging for execute_host (lc_host_stage_bytes)."""
        return torch.empty(max(1, self.host_stage_bytes), dtype=torch.uint8, device=self.device)

    def workspace_for(self, stream=None) -> torch.Tensor:
        """A workspace owned by this Plan object for one stream (created on first use), so that calls
        on different streams never share the counters and flags a workspace holds (legcheb.h)."""
        h = _stream_handle(stream, self.device)
        with self._ws_lock:
            ws = self._ws_by_stream.get(h)
            if ws is None:
                ws = self.new_workspace(stream)
                self._ws_by_stream[h] = ws
            return ws

    # -- execution
    def execute(self, x: torch.Tensor, out: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
                stream=None) -> torch.Tensor:
        """out = transform(x) on the device; x is [batch, n] (vec layout) or [n, batch] (batch layout)."""
        self._check(x, "input")
        if out is None:
            out = torch.empty(self._shape(self.ld_out, output=True), dtype=torch.float64, device=self.device)
        self._check(out, "output")
        ws = ctypes.c_void_p(workspace.data_ptr()) if workspace is not None else ctypes.c_void_p()
        _lib.check("lc_execute", self._lib.lc_execute(self._h, ctypes.c_void_p(x.data_ptr()),
                                                      ctypes.c_void_p(out.data_ptr()), ws,
                                                      ctypes.c_void_p(_stream_handle(stream, self.device))))
        return out

    def execute_part(self, phase: int, x: torch.Tensor, out: torch.Tensor, workspace: torch.Tensor,
                     stream=None) -> torch.Tensor:
        """lc_execute_part: phase 0 (upward pass of the part's subtrees) or 1 (the rest), for plans with
        part_up = 1; the caller exchanges the w roots / halo in `workspace` in between (dist.py)."""
        self._check(x, "input")
        self._check(out, "output")
        _lib.check("lc_execute_part", self._lib.lc_execute_part(
            self._h, int(phase), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()),
            ctypes.c_void_p(workspace.data_ptr()), ctypes.c_void_p(_stream_handle(stream, self.device))))
        return out

    def execute_timed(self, x: torch.Tensor, out: torch.Tensor, events, stream=None) -> None:
        """lc_execute that records CUDA events around each kernel (events: list of torch.cuda.Event)."""
        for e in events:  # torch creates the underlying cudaEvent_t lazily, on first record
            if not e.cuda_event:
                e.record(torch.cuda.current_stream(self.device) if stream is None else stream)
        arr = (ctypes.c_void_p * len(events))(*[ctypes.c_void_p(e.cuda_event) for e in events])
        _lib.check("lc_execute_timed", self._lib.lc_execute_timed(
            self._h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(),
            ctypes.c_void_p(_stream_handle(stream, self.device)), arr, len(events)))

    def execute_host(self, h_in: torch.Tensor, h_out: torch.Tensor, stream=None, stage: torch.Tensor | None = None,
                     workspace: torch.Tensor | None = None) -> None:
        """End-to-end call with HOST buffers (lc_execute_host: H2D, transform, D2H enqueued on stream; no
        sync).  stage / workspace: caller-owned device buffers (new_host_stage / new_workspace), or None
        for the plan-owned ones (then calls must be serialised on one stream)."""
        _check_host(h_in, self.in_extent)
        _check_host(h_out, self.out_extent)
        if stage is not None and (stage.device != self.device or stage.numel() * stage.element_size() <
                                  self.host_stage_bytes):
            raise ValueError(f"stage: need {self.host_stage_bytes} bytes on {self.device}")
        _lib.check("lc_execute_host", self._lib.lc_execute_host(
            self._h, ctypes.c_void_p(h_in.data_ptr()), ctypes.c_void_p(h_out.data_ptr()),
            ctypes.c_void_p(stage.data_ptr() if stage is not None else None),
            ctypes.c_void_p(workspace.data_ptr() if workspace is not None else None),
            ctypes.c_void_p(_stream_handle(stream, self.device))))

    def export(self, what: str) -> np.ndarray:
        """Copy plan data to the host: tabB, tabA, ahat, B, T (tests/diagnostics)."""
        lens = {"tabB": self.desc["N"], "tabA": 2 * self.desc["s"], "ahat": self.desc["nc"] * 324, "B": 324,
                "T": 2 * self.desc["s"] * 18}
        out = np.zeros(max(1, lens[what]), dtype=np.float64)
        _lib.check("lc_plan_export", self._lib.lc_plan_export(
            self._h, EXPORTS[what], out.ctypes.data_as(_lib.c_dp), out.size))
        return out[: lens[what]]


def _check_host(t: torch.Tensor, extent: int) -> None:
    if t.device.type != "cpu" or t.dtype != torch.float64 or not t.is_contiguous():
        raise ValueError("host buffers must be contiguous float64 CPU tensors")
    if t.numel() < extent:
        raise ValueError(f"host buffer of {t.numel()} elements, the plan addresses {extent}")


def chain_stage_bytes(plans) -> int:
    """lc_host_chain_stage_bytes: device staging of execute_host_chain for these plans."""
    arr = (ctypes.c_void_p * len(plans))(*[p._h for p in plans])
    return int(_lib.load().lc_host_chain_stage_bytes(arr, len(plans)))


def new_chain_stage(plans) -> torch.Tensor:
    """Caller-owned device staging for execute_host_chain (on the plans' device)."""
    return torch.empty(max(1, chain_stage_bytes(plans)), dtype=torch.uint8, device=plans[0].device)


def execute_host_chain(plans, h_in: torch.Tensor, h_out: torch.Tensor, stage: torch.Tensor, stream=None,
                       workspaces=None) -> None:
    """lc_execute_host_chain: h_in -> device, plans[0], ..., plans[-1] one after another on the device,
    result -> h_out; enqueued on stream (no sync).  E.g. a round trip [leg2cheb plan, cheb2leg plan] or
    the two passes of a 2-D transform.  stage: new_chain_stage(plans); workspaces: None (the plans' own;
    calls serialised on one stream) or one per plan."""
    plans = list(plans)
    if not plans:
        raise ValueError("execute_host_chain needs at least one plan")
    _check_host(h_in, plans[0].in_extent)
    _check_host(h_out, plans[-1].out_extent)
    need = chain_stage_bytes(plans)
    if stage.device != plans[0].device or stage.numel() * stage.element_size() < need:
        raise ValueError(f"stage: need {need} bytes on {plans[0].device}")
    arr = (ctypes.c_void_p * len(plans))(*[p._h for p in plans])
    ws = None
    if workspaces is not None:
        if len(workspaces) != len(plans):
            raise ValueError("one workspace per plan")
        ws = (ctypes.c_void_p * len(plans))(*[w.data_ptr() for w in workspaces])
    _lib.check("lc_execute_host_chain", _lib.load().lc_execute_host_chain(
        arr, len(plans), ctypes.c_void_p(h_in.data_ptr()), ctypes.c_void_p(h_out.data_ptr()),
        ctypes.c_void_p(stage.data_ptr()), ws, ctypes.c_void_p(_stream_handle(stream, plans[0].device))))


_cache: dict = {}
_cache_lock = threading.Lock()


def _cached(n, direction, batch, device) -> Plan:
    key = (n, DIRECTIONS[direction], batch, str(device))
    with _cache_lock:
        p = _cache.get(key)
        if p is None:
            p = Plan(n, direction, batch, device)
            _cache[key] = p
        return p


def _run(x: torch.Tensor, direction) -> torch.Tensor:
    squeeze = x.dim() == 1
    x2 = x.reshape(1, -1) if squeeze else x
    if x2.dim() != 2:
        raise ValueError("expected [n] or [batch, n]")
    x2 = x2.contiguous()
    p = _cached(x2.shape[1], direction, x2.shape[0], x2.device)
    out = p.execute(x2, workspace=p.workspace_for())  # one workspace per stream: safe across streams/threads
    return out.reshape(-1) if squeeze else out


def leg2cheb(x: torch.Tensor) -> torch.Tensor:
    """Chebyshev coefficients of the Legendre series x (last axis), f_cheb = C^{-1} A f_leg."""
    return _run(x, "leg2cheb")


def cheb2leg(x: torch.Tensor) -> torch.Tensor:
    """Legendre coefficients of the Chebyshev series x (last axis), f_leg = A^{-1} C f_cheb."""
    return _run(x, "cheb2leg")
