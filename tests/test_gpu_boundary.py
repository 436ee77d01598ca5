"""The C-ABI contract of include/legcheb.h on the GPU: host-buffer execution (lc_execute_host), its
thread safety with caller-owned staging and workspaces, the aliasing error, stream-ordered plan
destruction, and per-stream workspaces of the Python conveniences (leg2cheb / cheb2leg).

Every result is checked against the CPU oracle (the plain definitions of PAPER.md:29-32, eq:directmv).
"""
import threading
import time

import numpy as np
import pytest
import torch

import oracle
from lc_inputs import batch, vector

pytestmark = pytest.mark.gpu

GATE = 1e-12


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


def _plan(*a, **k):
    from paper_2411_00033_b200 import Plan
    return Plan(*a, **k)


def _rows(n, count=300, seed=3):
    rng = np.random.default_rng(seed)
    return np.unique(np.r_[0:min(n, 64), rng.integers(0, n, count), n - 1])


@pytest.mark.parametrize("direction", ["leg2cheb", "cheb2leg"])
@pytest.mark.parametrize("n,V,engine", [(5000, 1, 0), (3000, 24, 2), (300000, 8, 3), (100000, 3, 1)])
def test_execute_host_vs_oracle(direction, n, V, engine):
    dev = _dev()
    x = batch("uniform_r0", n, V, seed=7).pin_memory()
    out = torch.empty_like(x).pin_memory()
    p = _plan(n, direction, batch=V, device=dev, engine=engine)
    p.execute_host(x, out)  # plan-owned staging and workspace
    torch.cuda.synchronize()
    rows = _rows(n)
    for v in sorted({0, V - 1}):
        ref = oracle.transform_rows(direction, x[v].numpy(), rows)
        assert oracle.einf(out[v].numpy()[rows], ref) <= GATE, (v, engine)
    # identical to the device-buffer call (same kernels, same arithmetic)
    zd = p.execute(x.to(dev)).cpu()
    assert torch.equal(zd, out)


def test_execute_host_two_threads_two_streams_one_plan():
    """Two host threads drive one plan on two streams with their own staging and workspaces."""
    dev = _dev()
    n, V = 200000, 2
    p = _plan(n, "leg2cheb", batch=V, device=dev)
    xs = [batch("uniform_r0.5", n, V, seed=50 + t).pin_memory() for t in range(2)]
    outs = [torch.empty_like(xs[t]).pin_memory() for t in range(2)]
    stages = [p.new_host_stage() for _ in range(2)]
    wss = [p.new_workspace() for _ in range(2)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(2)]
    torch.cuda.synchronize()
    errors = []

    def work(t):
        try:
            torch.cuda.set_device(dev)
            for _ in range(5):
                p.execute_host(xs[t], outs[t], stream=streams[t], stage=stages[t], workspace=wss[t])
            streams[t].synchronize()
        except Exception as e:  # surfaced below
            errors.append(e)

    th = [threading.Thread(target=work, args=(t,)) for t in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    rows = _rows(n)
    for t in range(2):
        for v in range(V):
            ref = oracle.l2c_rows(xs[t][v].numpy(), rows)
            assert oracle.einf(outs[t][v].numpy()[rows], ref) <= GATE, (t, v)


def test_aliasing_is_rejected():
    from paper_2411_00033_b200._lib import LegChebError
    dev = _dev()
    n = 4096
    p = _plan(n, "leg2cheb", device=dev)
    buf = torch.zeros(2 * n, dtype=torch.float64, device=dev)
    with pytest.raises(LegChebError) as ei:
        p.execute(buf[:n].view(1, n), buf[:n].view(1, n))  # in == out
    assert ei.value.status == 5  # LC_ERR_ALIASING
    with pytest.raises(LegChebError) as ei:
        p.execute(buf[:n].view(1, n), buf[n // 2:n // 2 + n].view(1, n))  # partial overlap
    assert ei.value.status == 5
    p.execute(buf[:n].view(1, n), buf[n:].view(1, n))  # adjacent, disjoint: accepted
    torch.cuda.synchronize()


def test_destroy_waits_for_own_work_only():
    """lc_plan_destroy orders its frees after the plan's own executions but does not wait for an
    unrelated stream (no cudaDeviceSynchronize / cudaFree device-wide sync)."""
    dev = _dev()
    other = torch.cuda.Stream(device=dev)
    mine = torch.cuda.Stream(device=dev)
    n = 100000
    x = torch.from_numpy(vector("uniform_r0.5", n, seed=61)).reshape(1, -1).to(dev)
    p = _plan(n, "leg2cheb", device=dev)
    torch.cuda.synchronize()
    with torch.cuda.stream(other):
        torch.cuda._sleep(3_000_000_000)  # ~1.5 s of GPU clock cycles on an unrelated stream
    with torch.cuda.stream(mine):
        z = p.execute(x, stream=mine)
    t0 = time.perf_counter()
    p.close()  # lc_plan_destroy
    dt = time.perf_counter() - t0
    busy = not other.query()
    torch.cuda.synchronize()
    ref = oracle.l2c_rows(x.cpu().numpy()[0], _rows(n))
    assert oracle.einf(z.cpu().numpy()[0][_rows(n)], ref) <= GATE
    assert busy and dt < 0.75, (dt, busy)


def test_convenience_functions_on_two_streams():
    """leg2cheb() from two streams at once: each stream gets its own workspace."""
    from paper_2411_00033_b200 import leg2cheb
    dev = _dev()
    n = 150000
    xs = [torch.from_numpy(vector("uniform_r0.5", n, seed=70 + t)).to(dev) for t in range(2)]
    st = [torch.cuda.Stream(device=dev) for _ in range(2)]
    torch.cuda.synchronize()
    outs = [[], []]
    for _ in range(4):
        for t in range(2):
            with torch.cuda.stream(st[t]):
                outs[t].append(leg2cheb(xs[t]))
    torch.cuda.synchronize()
    rows = _rows(n)
    for t in range(2):
        ref = oracle.l2c_rows(xs[t].cpu().numpy(), rows)
        for z in outs[t]:
            assert oracle.einf(z.cpu().numpy()[rows], ref) <= GATE, t


@pytest.mark.parametrize("direction", ["leg2cheb", "cheb2leg"])
@pytest.mark.parametrize("n,V,B,engine", [(8192, 24, 2048, 0), (8192, 16, 1024, 2), (5000, 9, 1250, 0),
                                          (5000, 9, 1024, 0), (300000, 8, 37500, 3)])
def test_column_blocked_output(direction, n, V, B, engine):
    """lc_plan_opts.out_block (the 2-D pass-1 epilogue writing rows packed by destination rank): the
    output [ceil(n/B)][V][B] holds exactly the vector-contiguous result, re-blocked, bit for bit."""
    dev = _dev()
    x = batch("normal", n, V, seed=n + B).to(dev)
    pb = _plan(n, direction, batch=V, device=dev, engine=engine, out_block=B)
    assert pb.kernel_info["engine"] in (2, 3)  # engine 1 (automatic for few tiles) hands over to engine 2
    ref = _plan(n, direction, batch=V, device=dev, engine=pb.kernel_info["engine"]).execute(x)
    nb = -(-n // B)
    out = torch.full((nb, V, B), float("nan"), dtype=torch.float64, device=dev)
    pb.execute(x, out)
    torch.cuda.synchronize()
    for k in range(nb):
        w = min(B, n - k * B)
        assert torch.equal(out[k, :, :w], ref[:, k * B:k * B + w]), k
        assert bool(torch.isnan(out[k, :, w:]).all())  # past n: untouched


def test_host_alloc_buffers():
    """lc_host_alloc / lc_host_free (legcheb.h): page-locked, zero-filled, usable by lc_execute_host with
    the same result as the device call; bad arguments are rejected; the memory is released with the
    last view."""
    import ctypes
    import gc

    from paper_2411_00033_b200 import _lib, host_empty
    dev = _dev()
    lib = _lib.load()
    n, V = 100003, 3
    x = host_empty((V, n))
    assert x.is_pinned() and x.dtype == torch.float64 and x.shape == (V, n) and not bool(x.any())
    x.copy_(batch("normal", n, V, seed=91))
    out = host_empty((V, n))
    p = _plan(n, "cheb2leg", batch=V, device=dev)
    p.execute_host(x, out)
    torch.cuda.synchronize()
    assert torch.equal(out, p.execute(x.to(dev)).cpu())
    # odd sizes and 1-D shapes; a view outlives its base tensor
    y = host_empty(7)[2:5]
    gc.collect()
    y.fill_(1.0)
    assert y.sum().item() == 3.0
    # errors
    ptr = ctypes.c_void_p()
    assert lib.lc_host_alloc(0, ctypes.byref(ptr)) == 1  # LC_ERR_INVALID_ARG
    assert lib.lc_host_free(ctypes.c_void_p(12345)) == 1
    assert lib.lc_host_alloc(1 << 20, ctypes.byref(ptr)) == 0
    assert lib.lc_host_free(ptr) == 0
    assert lib.lc_host_free(ptr) == 1  # double free is rejected, not a crash


def test_execute_host_column_blocked():
    """lc_execute_host of an out_block plan copies back the whole blocked output (its extent is
    ceil(n/B) V B, more than n V when B does not divide n)."""
    from paper_2411_00033_b200 import host_empty
    dev = _dev()
    n, V, B = 5000, 9, 1024
    x = host_empty((V, n))
    x.copy_(batch("normal", n, V, seed=5))
    pb = _plan(n, "leg2cheb", batch=V, device=dev, out_block=B)
    nb = -(-n // B)
    out = host_empty((nb, V, B))
    out.fill_(float("nan"))
    pb.execute_host(x, out)
    torch.cuda.synchronize()
    ref = pb.execute(x.to(dev)).cpu()
    for k in range(nb):
        w = min(B, n - k * B)
        assert torch.equal(out[k, :, :w], ref[k, :, :w]), k


@pytest.mark.parametrize("n,V", [(1000000, 1), (4096, 64), (70001, 3)])
def test_execute_host_chain_round_trip(n, V):
    """lc_execute_host_chain of [leg2cheb, cheb2leg]: one copy each way, the same bits as the two device
    calls, on two streams with their own staging and workspaces; bad arguments are rejected."""
    import ctypes

    from paper_2411_00033_b200 import _lib, execute_host_chain, host_empty, new_chain_stage
    dev = _dev()
    pl = _plan(n, "leg2cheb", batch=V, device=dev)
    pc = _plan(n, "cheb2leg", batch=V, device=dev)
    x = host_empty((V, n))
    x.copy_(batch("uniform_r0.5", n, V, seed=21))
    xd = x.to(dev)
    ref = pc.execute(pl.execute(xd)).cpu()
    streams = [torch.cuda.Stream(device=dev) for _ in range(2)]
    outs = [host_empty((V, n)) for _ in range(2)]
    # (the staging and workspaces stay referenced until the streams are done: torch's caching allocator
    # would hand memory freed on the current stream to the next allocation while the side stream runs)
    stages = [new_chain_stage([pl, pc]) for _ in range(2)]
    wss = [[pl.new_workspace(streams[k]), pc.new_workspace(streams[k])] for k in range(2)]
    for k in range(2):
        execute_host_chain([pl, pc], x, outs[k], stages[k], stream=streams[k], workspaces=wss[k])
    torch.cuda.synchronize()
    for k in range(2):
        assert torch.equal(outs[k], ref), k
    assert float((outs[0] - x).abs().max() / x.abs().max()) <= GATE
    # errors: no staging; a chain whose next plan reads more than the previous one wrote
    lib = _lib.load()
    arr = (ctypes.c_void_p * 2)(pl._h, pc._h)
    assert lib.lc_execute_host_chain(arr, 2, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(outs[0].data_ptr()),
                                     None, None, None) == 1
    big = _plan(n + 1, "cheb2leg", batch=V, device=dev)
    arr2 = (ctypes.c_void_p * 2)(pl._h, big._h)
    st = new_chain_stage([pl, big])
    assert lib.lc_execute_host_chain(arr2, 2, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(outs[0].data_ptr()),
                                     ctypes.c_void_p(st.data_ptr()), None, None) == 1
    assert lib.lc_host_chain_stage_bytes(arr, 0) == 0


def test_execute_host_chain_2d():
    """The two passes of the 2-D tensor-product transform (rows on a vector-layout plan, then columns on
    a batch-layout plan of the same array) as one host chain equal the two device passes."""
    from paper_2411_00033_b200 import execute_host_chain, host_empty, new_chain_stage
    dev = _dev()
    n = 2048
    x = host_empty((n, n))
    x.copy_(batch("normal", n, n, seed=4))
    pr = _plan(n, "leg2cheb", batch=n, device=dev)
    pcol = _plan(n, "leg2cheb", batch=n, device=dev, layout="batch")
    ref = pcol.execute(pr.execute(x.to(dev))).cpu()
    out = host_empty((n, n))
    execute_host_chain([pr, pcol], x, out, new_chain_stage([pr, pcol]))
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
