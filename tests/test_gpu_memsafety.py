"""Memory-safety and race checks of our own (compute-sanitizer is closed on this GPU pool: runs under it
left GPUs needing a reset).  Three checks per engine, both directions, both layouts:

* write canaries: out and the caller-owned workspace sit inside larger buffers whose margins (and,
  with a padded leading dimension, the gaps between rows) hold a NaN bit pattern that must survive
  the execution bit for bit -- any out-of-range store would overwrite it;
* read poison: the input's margins and row gaps hold NaN; the zero padding n -> N is virtual
  (SURVEY R0), so a kernel that reads beyond a row's n entries or outside the input's extent would
  carry a NaN into the output, which must instead match the oracle;
* race stress: 40 executions of one plan enqueued back to back on one stream, alternating two
  inputs, must reproduce the first result of each input bit for bit (the kernels hand data between
  CTAs and kernels through release/acquire flags, counters and mbarrier rings; a missing fence or a
  flag re-armed too early shows up as a nondeterministic result).
"""
import ctypes

import numpy as np
import pytest
import torch

import oracle
from lc_inputs import batch

pytestmark = pytest.mark.gpu

NAN_BITS = 0x7FF8DEADBEEF0001  # a quiet NaN payload no arithmetic produces
MARGIN = 4096  # doubles of canary on each side


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


def _plan(*a, **k):
    from paper_2411_00033_b200 import Plan
    return Plan(*a, **k)


def _poisoned(rows, ld, dev):
    """A [MARGIN + rows*ld + MARGIN] fp64 buffer filled with the NaN pattern; returns (buffer, view)."""
    buf = torch.full((2 * MARGIN + rows * ld,), 0, dtype=torch.int64, device=dev)
    buf.fill_(NAN_BITS)
    buf = buf.view(torch.float64)
    return buf, buf[MARGIN:MARGIN + rows * ld].view(rows, ld)


CASES = [(1, 3000, 3), (1, 70001, 1), (2, 3000, 16), (2, 1500, 9), (3, 40000, 8), (3, 9000, 11)]


@pytest.mark.parametrize("layout", ["vec", "batch"])
@pytest.mark.parametrize("direction", ["leg2cheb", "cheb2leg"])
@pytest.mark.parametrize("engine,n,V", CASES)
def test_canaries_and_poison(engine, n, V, direction, layout):
    dev = _dev()
    x = batch("normal", n, V, seed=n + V)
    if layout == "vec":
        ld_in, ld_out = n + 5, n + 3
        rows_in, cols = V, n
    else:
        ld_in, ld_out = V + 3, V + 1
        rows_in, cols = n, V
    p = _plan(n, direction, batch=V, device=dev, engine=engine, layout=layout, ld_in=ld_in, ld_out=ld_out)
    bin_, xin = _poisoned(rows_in, ld_in, dev)
    xin[:, :cols] = (x if layout == "vec" else x.t()).to(dev)
    bout, zout = _poisoned(rows_in, ld_out, dev)
    ws_bytes = (max(8, p.workspace_bytes) + 255) // 256 * 256
    wbuf = torch.empty(2 * MARGIN * 8 + ws_bytes, dtype=torch.uint8, device=dev)
    wbuf.view(torch.int64).fill_(NAN_BITS)
    ws = wbuf[MARGIN * 8: MARGIN * 8 + ws_bytes]
    from paper_2411_00033_b200 import _lib
    _lib.check("lc_workspace_init", p._lib.lc_workspace_init(p.handle, ctypes.c_void_p(ws.data_ptr()), None))
    in_before = bin_.clone()
    wb_before = wbuf.clone()
    for _ in range(2):
        p.execute(xin, zout, workspace=ws)
    torch.cuda.synchronize()
    # input unmodified (legcheb.h), its margins and gaps included
    assert torch.equal(bin_.view(torch.int64), in_before.view(torch.int64))
    # output: margins and row gaps still hold the NaN pattern, bit for bit
    ob = bout.view(torch.int64)
    assert bool((ob[:MARGIN] == NAN_BITS).all()) and bool((ob[-MARGIN:] == NAN_BITS).all())
    gaps = ob[MARGIN:MARGIN + rows_in * ld_out].view(rows_in, ld_out)[:, cols:]
    assert bool((gaps == NAN_BITS).all())
    # workspace margins untouched
    assert torch.equal(wbuf[: MARGIN * 8], wb_before[: MARGIN * 8])
    assert torch.equal(wbuf[MARGIN * 8 + ws_bytes:], wb_before[MARGIN * 8 + ws_bytes:])
    # results finite and equal to the oracle (no NaN read from the poisoned gaps / margins)
    z = zout[:, :cols].cpu().numpy()
    z = z if layout == "vec" else z.T
    assert np.isfinite(z).all()
    rows = np.unique(np.r_[0:min(n, 128), np.linspace(0, n - 1, 128).astype(np.int64)])
    for v in (0, V - 1):
        ref = oracle.transform_rows(direction, x[v].numpy(), rows)
        assert oracle.einf(z[v][rows], ref) <= 1e-12, (engine, n, V, v)


@pytest.mark.parametrize("engine,n,V", [(1, 1_000_000, 1), (1, 70001, 3), (2, 4096, 64), (3, 300000, 16)])
def test_back_to_back_bitwise_reproducible(engine, n, V):
    dev = _dev()
    xs = [batch("normal", n, V, seed=900 + k).to(dev) for k in range(2)]
    for direction in ("leg2cheb", "cheb2leg"):
        p = _plan(n, direction, batch=V, device=dev, engine=engine)
        outs = [p.execute(xs[i % 2]) for i in range(40)]
        torch.cuda.synchronize()
        for i in range(2, 40):
            assert torch.equal(outs[i], outs[i % 2]), (engine, n, V, direction, i)
