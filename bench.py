#!/usr/bin/env python
"""Benchmark of the B200 Legendre<->Chebyshev execution stage (one JSON line on rank 0).

Default workload (BASELINE.json configs[1], "cfg2"): one fp64 vector of
n = 1e6 Legendre coefficients f_j = s_j/(j+1), s_j = +-1; a *step* is one
leg2cheb followed by one cheb2leg (the round trip), i.e. one pass of the whole
hot path in both directions.  Metric: coefficients/s = 2 n V / step time
(n unpadded, V vectors, 2 transforms), summed over ranks.

After the headline record, the batched half of the metric is measured the
same way and attached as "batched" (default cfg3: 4096 vectors of n = 4096,
sharded over the ranks; --batched cfg4/cfg5/none).

Multi-GPU (one process per GPU, NCCL; `--gpus N` launches torchrun itself when
WORLD_SIZE is unset): cfg2 does not shard (one vector couples all leaves
through the coarse levels), so N GPUs run N independent replicas (weak
scaling); cfg3/cfg4 shard the batch and cfg5 partitions rows with an
all-to-all between the passes (strong scaling).  Timing: CUDA events on the
launching stream inside a barrier + synchronize bracket, max over ranks;
per-step events give the median and minimum step.

--impl reference runs the CPU oracle (oracle/, long-double direct O(n^2)
rows) on a bounded row sample of the same workload, on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASELINE["metric"]
UNIT = "coefficients/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


FP64_PEAK_TFLOPS = 34.2  # profiles/r1_fp64_peak.txt: DFMA microbenchmark on this pool's B200 at 1965 MHz
DMMA_PEAK_TFLOPS = 37.0  # profiles/r1_dmma_peak.txt: fp64 tensor-core MMA (m8n8k4) microbenchmark


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        time.sleep(0.15)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                power.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(nm)
        loaded = [c for c in sm if c > 600] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(power) if power else None}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        # LC_DIST_BACKEND=gloo with more ranks than GPUs: a functional check of the multi-rank code path on
        # a one-GPU box (ranks share the device; the timings of such a run mean nothing)
        backend = os.environ.get("LC_DIST_BACKEND", backend)
        if torch.cuda.is_available():
            local = local % torch.cuda.device_count() if backend == "gloo" else local
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------------------- workloads
def workload(config: str, world: int, rank: int):
    """(n, V_local, kind, vector index offset, scaling) for this rank."""
    from lc_inputs import CONFIGS
    c = CONFIGS[config]
    n, V = c["n"], c["batch"]
    if V == 1:
        return n, 1, c["kind"], rank, "weak"          # replicas, one vector per rank
    base, rem = divmod(V, world)
    vloc = base + (1 if rank < rem else 0)
    v0 = rank * base + min(rank, rem)
    return n, vloc, c["kind"], v0, "strong"


def make_input(kind, n, V, v0, pin):
    from lc_inputs import batch
    if pin:  # page-locked host memory on huge pages (lc_host_alloc): full PCIe rate for the e2e copies
        from paper_2411_00033_b200 import host_empty
        out = host_empty((V, n))
    else:
        out = torch.empty((V, n), dtype=torch.float64)
    return batch(kind, n, V, seed=0, v0=v0, out=out)


# --------------------------------------------------------------------------- our arm
def kernel_names(pl):
    kpe = pl.kernels_per_execute
    engine = pl.kernel_info.get("engine", 1)
    if engine == 3:
        return ["lc_up3_kernel", "lc_range_kernel"], engine
    if kpe == 1:
        return ["lc_tile_kernel"], engine
    return (["lc_up_kernel"] if kpe == 3 else []) + ["lc_stream_kernel", "lc_down_kernel"], engine


def make_plans(config, n, V, dev, world, opts):
    """The plans one step uses, with their creation times (wall, and device time of the planner)."""
    from paper_2411_00033_b200 import Plan
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if config == "cfg5":
        C = n // world
        # N > 1: pass 1 writes its rows packed by destination rank from the kernel epilogue (out_block)
        pl = Plan(n, "leg2cheb", batch=V, device=dev, out_block=C if world > 1 else 0, **opts)
        pc = Plan(n, "leg2cheb", batch=C, device=dev, layout="batch", **opts)
    else:
        pl = Plan(n, "leg2cheb", batch=V, device=dev, **opts)
        pc = Plan(n, "cheb2leg", batch=V, device=dev, **opts)
    wall = (time.perf_counter() - t0) * 1e3
    # one more leg2cheb plan, created and destroyed: the steady cost of lc_plan_create (the first creation of
    # a process also pays the CUDA module load and the kernel attribute configuration)
    t1 = time.perf_counter()
    extra = Plan(n, "leg2cheb", batch=V, device=dev, **opts)
    torch.cuda.synchronize()
    steady = (time.perf_counter() - t1) * 1e3
    extra.close()
    plan = {"wall_ms_both": wall, "wall_ms_steady_one": steady, "device_ms": [pl.plan_device_ms, pc.plan_device_ms],
            "plan_bytes": [int(pl.desc["plan_bytes"]), int(pc.desc["plan_bytes"])],
            "note": "plan creation (lambda, A_hat, tables) is outside the timed region, as in the paper"}
    return pl, pc, plan


def timed_replays(fn, steps, stream):
    """fn() `steps` times with a CUDA event after each step (same stream); returns the total and the
    per-step durations in ms."""
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record(stream)
    for i in range(steps):
        fn()
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    return ev[0].elapsed_time(ev[steps]), per


def measure(config, args, world, rank, local, headline=True):
    """One JSON record (bench contract keys) for `config` on this rank set."""
    from paper_2411_00033_b200 import Plan, execute_host_chain, host_empty, new_chain_stage
    from paper_2411_00033_b200.api import chain_stage_bytes
    from paper_2411_00033_b200.dist import tensor_product_2d
    dev = torch.device("cuda", local)
    n, V, kind, v0, scaling = workload(config, world, rank)
    two_d = config == "cfg5"
    if args.split_vector and V == 1 and world > 1 and not two_d:
        v0 = 0  # one vector split over the ranks: every rank holds the same input
    if two_d:
        scaling = "strong"
    xh = make_input(kind, n, V, v0, pin=True)
    x = xh.to(dev)
    tmp = torch.empty_like(x)
    y = torch.empty_like(x)
    opts = dict(vt=args.vt, subtree=args.subtree, stage_blocks=args.stage_blocks, stages=args.stages,
                engine=args.engine, up_subtree=args.up_subtree)
    stream = torch.cuda.current_stream(dev)
    pl, pc, plan_info = make_plans(config, n, V, dev, world, opts)
    C = n // world
    chunks = args.chunks if (two_d and world > 1 and V % max(1, args.chunks) == 0) else 1
    split = args.split_vector and V == 1 and world > 1 and not two_d  # NEXT-2: one vector over the ranks
    if split:
        from paper_2411_00033_b200.dist import SingleVectorTransform
        scaling = "strong"
        sl = SingleVectorTransform(n, "leg2cheb", device=dev, part_up=True)
        sc = SingleVectorTransform(n, "cheb2leg", device=dev, part_up=True)
    if two_d:
        # rows [v0, v0+V) of the n x n array on this rank; pass 1 along axis 1 (V row vectors), all-to-all,
        # pass 2 along axis 0 (n/world column vectors, batch-contiguous); with chunks > 1 pass 1 runs in
        # row chunks whose all-to-all overlaps the next chunk (dist._chunked_exchange)
        ycol = torch.empty((n, C), dtype=torch.float64, device=dev)
        from paper_2411_00033_b200 import Plan as _Plan
        pk = _Plan(n, "leg2cheb", batch=V // chunks, device=dev, out_block=C, **opts) if chunks > 1 else pl
        packed = world > 1
        tmpk = torch.empty((V // chunks, n), dtype=torch.float64, device=dev)

        def step():
            if chunks > 1:
                tensor_product_2d(x, row_fn=lambda a: pk.execute(a, tmpk), col_fn=lambda a: pc.execute(a, ycol),
                                  chunks=chunks, row_packed=packed)
            else:
                tensor_product_2d(x, row_fn=lambda a: pl.execute(a, tmp), col_fn=lambda a: pc.execute(a, ycol),
                                  row_packed=packed)
    elif split:
        xf = x.reshape(-1)

        def step():  # every rank: its rows of leg2cheb, all-gather, its rows of cheb2leg, all-gather
            y.copy_(sc(sl(xf)).reshape(1, -1))
    else:
        def step():
            pl.execute(x, tmp)
            pc.execute(tmp, y)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    graph = None
    if not args.no_graph:
        try:
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream(dev)
            s.wait_stream(stream)
            with torch.cuda.stream(s):
                step()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                step()
            torch.cuda.synchronize()
            graph = g
            for _ in range(3):
                graph.replay()
            torch.cuda.synchronize()
        except Exception as e:  # graph capture unavailable: eager launches
            graph = None
            print(f"[bench] graph capture failed ({e}); eager launches", file=sys.stderr)
    run = graph.replay if graph is not None else step

    clocks = ClockSampler(local)
    barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    barrier(world)
    torch.cuda.synchronize()
    ms_local, per_step = timed_replays(run, args.steps, stream)
    barrier(world)
    clk = clocks.stop()
    ms = allreduce_max(ms_local, world)
    coeffs = 2.0 * n * V  # per rank per step (2 transforms or 2 passes)
    total_coeffs = allreduce_sum(coeffs, world) if not split else coeffs  # split: one vector in total
    value = total_coeffs * args.steps / (ms / 1e3)
    med_ms = allreduce_max(statistics.median(per_step), world)
    min_ms = allreduce_max(min(per_step), world)

    # correctness of what was timed: round trip back to the input (gate 1e-12 for n <= 1e6)
    rt = None if two_d else float((y - x).abs().max() / x.abs().max())

    # ---- the 2-D passes and the all-to-all timed separately
    passes = None
    if two_d:
        tm = {}
        acc = {"pass1_ms": 0.0, "alltoall_ms": 0.0, "pass2_ms": 0.0}
        reps = max(3, min(args.steps, 50))
        for _ in range(reps):
            tensor_product_2d(x, row_fn=lambda a: pl.execute(a, tmp), col_fn=lambda a: pc.execute(a, ycol),
                              timing=tm, row_packed=packed)
            for k in acc:
                acc[k] += tm[k] / reps
        passes = {k: allreduce_max(v, world) for k, v in acc.items()}
        passes["alltoall_bytes_sent_per_rank"] = 8 * V * C * (world - 1)
        if chunks > 1:
            ov = 0.0
            for _ in range(reps):
                tensor_product_2d(x, row_fn=lambda a: pk.execute(a, tmpk), col_fn=lambda a: pc.execute(a, ycol),
                                  chunks=chunks, timing=tm, row_packed=packed)
                ov += tm["pass1_and_alltoall_overlapped_ms"] / reps
            passes["pass1_and_alltoall_overlapped_ms"] = allreduce_max(ov, world)
            passes["chunks"] = chunks

    # ---- per-kernel durations (events around each kernel, same stream) for the roofline
    kpe = pl.kernels_per_execute
    names, engine = kernel_names(pl)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(kpe + 1)]
    evc = [torch.cuda.Event(enable_timing=True) for _ in range(pc.kernels_per_execute + 1)]
    ksteps = max(3, min(args.steps, 200))
    per_kernel = [[0.0] * kpe, [0.0] * kpe]
    for _ in range(ksteps):
        pl.execute_timed(x, tmp, evs)
        if two_d:
            pl.execute_timed(x, tmp, evc)
        else:
            pc.execute_timed(tmp, y, evc)
        torch.cuda.synchronize()
        for d, ev in enumerate((evs, evc)):
            for i in range(kpe):
                per_kernel[d][i] += ev[i].elapsed_time(ev[i + 1]) / ksteps
    hbm, hbm_src = peaks()
    dl = pl.desc
    # algorithmic bytes per launch (f in, z out, A_hat once, lambda once; work arrays excluded):
    # the up kernel reads f, the streaming kernel reads A_hat and lambda (and f again for the band),
    # the down kernel writes z
    alg = {"lc_up_kernel": 8.0 * n * V, "lc_up3_kernel": 8.0 * n * V,
           "lc_stream_kernel": 8.0 * 324 * dl["nc"] + 8.0 * dl["N"], "lc_down_kernel": 8.0 * n * V}
    if kpe == 2 and engine == 1:  # L = 0: no up kernel, the streaming kernel reads f
        alg["lc_stream_kernel"] += 8.0 * n * V
    # the per-tile kernel (engine 2) is the whole transform: f in, z out, A_hat and lambda once
    alg["lc_tile_kernel"] = 16.0 * n * V + 8.0 * 324 * dl["nc"] + 8.0 * dl["N"]
    alg["lc_range_kernel"] = 8.0 * n * V + 8.0 * 324 * dl["nc"] + 8.0 * dl["N"]  # f in (band), z out, A_hat, lambda
    avg_ms = {nm: 0.5 * (per_kernel[0][i] + per_kernel[1][i]) for i, nm in enumerate(names)}
    dom = "lc_tile_kernel" if kpe == 1 else ("lc_range_kernel" if engine == 3 else "lc_stream_kernel")
    dom_ms = avg_ms[dom]
    dom_bytes = alg[dom]
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = load_traffic(config, dom)
    fp64_peak = max(FP64_PEAK_TFLOPS, DMMA_PEAK_TFLOPS)
    if kpe == 1 or engine == 3:
        # fp64 tensor-core bound: algorithmic flops of one transform over the kernel time, against the
        # measured DMMA peak (the higher of the two fp64 peaks, so the fraction is conservative)
        fk = dl["flops_alg"]
        if engine == 3:  # the range kernel does steps 3-7: drop step 1 and the M2M half of F_alg
            Lq, sq, Mq = dl["L"], dl["s"], 18
            fk -= 8.0 * ((2 ** Lq) - 1) * sq * Mq + 4.0 * (Mq * Mq + 2 * Mq) * ((2 ** Lq) - Lq - 1)
        tf = fk * V / (dom_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "kernel": dom, "achieved": tf, "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": tf / DMMA_PEAK_TFLOPS, "traffic": traffic, "algorithmic_flops_per_launch": fk * V,
                "algorithmic_bytes_per_launch": dom_bytes, "achieved_hbm_gbs": achieved, "avg_launch_ms": dom_ms,
                "peak_source": "measured fp64 DMMA m8n8k4 (profiles/r1_dmma_peak.txt); fp64 has no tcgen05 kind"}
    else:
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm,
                "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                "algorithmic_bytes_per_launch": dom_bytes, "avg_launch_ms": dom_ms,
                "peak_source": hbm_src}
    # transform-level roofline (slower of fp64 flops at the fp64 peak -- the DMMA pipe, 37.0 TF -- and
    # bytes at the HBM peak), per transform, against the median step
    t_roof = max(dl["flops_alg"] * V / (fp64_peak * 1e12), dl["bytes_alg"] / (hbm * 1e9))
    t_meas = ms_local / args.steps / 2 * 1e-3
    t_med = med_ms / 2 * 1e-3

    # ---- e2e through the C ABI with HOST buffers, pipelined over streams (the call is thread- and
    # stream-safe with distinct staging and workspaces, legcheb.h)
    e2e_steps = max(3, min(args.steps, args.e2e_steps))
    # one C-ABI call per step (lc_execute_host_chain): the step's input H2D, leg2cheb then cheb2leg (2-D:
    # the row pass then the column pass) on the device, the result D2H; --e2e-streams buffer sets (chain
    # staging + a workspace per plan, per stream) when they fit, else fewer
    # large batches (cfg4: 5 GB per step) go in sub-batches of their own plans, so that one sub-batch's
    # copies overlap another's transforms (the device-timed value above keeps the whole-batch plans)
    ech = 1
    if not two_d and V >= 16 and 8 * n * V >= (1 << 30):
        ech = next(c for c in (8, 4, 2, 1) if V % c == 0)
    Vc = V // ech
    if ech > 1:
        pl_e = Plan(n, "leg2cheb", batch=Vc, device=dev, engine=args.engine)
        pc_e = Plan(n, "cheb2leg", batch=Vc, device=dev, engine=args.engine)
    else:
        pl_e, pc_e = pl, pc
    chain = [pl_e, pc_e]
    per_set = chain_stage_bytes(chain) + pl_e.workspace_bytes + pc_e.workspace_bytes
    free_b = torch.cuda.mem_get_info(dev)[0]
    nbuf = max(1, args.e2e_streams)
    while nbuf > 1 and nbuf * per_set >= 0.6 * free_b:
        nbuf -= 1
    streams = [torch.cuda.Stream(dev) for _ in range(nbuf)]
    hy = [host_empty((n, C) if two_d else (Vc, n)) for _ in range(nbuf)]
    if two_d and world > 1:
        ycols = [torch.empty((n, C), dtype=torch.float64, device=dev) for _ in range(nbuf)]
        tmps = [torch.empty_like(x) for _ in range(nbuf)]
        stages = [None] * nbuf
    else:
        stages = [new_chain_stage(chain) for _ in range(nbuf)]
    ws_l = [pl_e.new_workspace(streams[b]) for b in range(nbuf)]
    ws_c = [pc_e.new_workspace(streams[b]) for b in range(nbuf)]
    torch.cuda.synchronize()

    def host_steps(k0, k):
        for i in range(k0, k0 + k):
            if two_d and world > 1:
                b = i % nbuf
                sb = streams[b]
                with torch.cuda.stream(sb):
                    xd = xh.to(dev, non_blocking=True)
                    zc = tensor_product_2d(xd, row_fn=lambda a: pl.execute(a, tmps[b], workspace=ws_l[b], stream=sb),
                                           col_fn=lambda a: pc.execute(a, ycols[b], workspace=ws_c[b], stream=sb),
                                           row_packed=True)
                    hy[b].copy_(zc, non_blocking=True)
                continue
            for c in range(ech):  # one chain call per sub-batch (one per step without sub-batches)
                b = (i * ech + c) % nbuf
                execute_host_chain(chain, xh[c * Vc:(c + 1) * Vc], hy[b], stages[b], stream=streams[b],
                                   workspaces=[ws_l[b], ws_c[b]])

    host_steps(0, max(1, nbuf // ech))
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    h0 = torch.cuda.Event(enable_timing=True)
    h1 = torch.cuda.Event(enable_timing=True)
    h0.record(stream)
    for sb in streams:
        sb.wait_event(h0)
    host_steps(nbuf, e2e_steps)
    for sb in streams:
        e = torch.cuda.Event()
        e.record(sb)
        stream.wait_event(e)
    h1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    e2e_ms = allreduce_max(h0.elapsed_time(h1), world)
    e2e_val = total_coeffs * e2e_steps / (e2e_ms / 1e3)
    qlast = (nbuf + e2e_steps) * ech - 1  # the last chain call: its buffer and sub-batch
    rt_host = None if two_d else float((hy[qlast % nbuf] - xh[(qlast % ech) * Vc:(qlast % ech + 1) * Vc]).abs().max() /
                                       xh.abs().max())
    bytes_vec = 8 * n * V
    h2d, d2h = bytes_vec, 8 * n * C if two_d else bytes_vec

    cpu = None
    cfmm = None
    if headline and rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(config, n, kind, budget_s=args.cpu_seconds)
        try:
            cfmm = cpu_fmm_baseline(n, kind, dev, budget_s=args.cpu_seconds)
        except Exception as e:  # reported baseline only: never fail the GPU line for it
            cfmm = {"unavailable": f"{type(e).__name__}: {e}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json recipe)",
        "config": {"workload": (f"{config}: leg2cheb then cheb2leg (round trip) of one fp64 vector of n={n} "
                                f"split over {world} GPUs by output rows (NEXT-2, rows all-gathered)") if split else
                               (f"{config}: leg2cheb then cheb2leg (round trip) of {V} fp64 vector(s) "
                                f"of n={n} per GPU") if not two_d else
                               (f"cfg5: 2-D leg2cheb of an {n}x{n} fp64 array (axis 1, all-to-all, axis 0), "
                                f"{V} rows per GPU"), "n": n, "vectors_per_gpu": V, "N_padded": dl["N"],
                   "L": dl["L"], "s": dl["s"], "M": 18, "s_hat": 40, "transforms_per_step": 2,
                   "input_kind": kind,
                   "l2": f"no flush: per-step working set {2 * 8 * 324 * dl['nc'] / 1e6:.0f} MB of A_hat + "
                         f"{3 * bytes_vec / 1e6:.0f} MB of vectors vs 126 MB L2" if dl["nc"] > 0 and
                         2 * 8 * 324 * dl['nc'] + 3 * bytes_vec > 126e6 else
                         ("no flush: per-step vectors " f"{3 * bytes_vec / 1e6:.0f} MB vs 126 MB L2"),
                   "graph": graph is not None, "kernel_cfg": {**{k: dl[k] for k in ("vt", "subtree", "stage_blocks",
                                                                                    "stages")}, "engine": engine}},
        "step_ms": {"median": med_ms, "min": min_ms, "mean": ms / args.steps,
                    "note": "per-step CUDA events between graph replays; max over ranks"},
        "roofline": roof,
        "roofline_transform": {"t_roof_us": t_roof * 1e6, "t_measured_us": t_meas * 1e6,
                               "t_median_us": t_med * 1e6, "frac": t_roof / t_meas, "frac_median": t_roof / t_med,
                               "fp64_peak_tflops": fp64_peak, "hbm_gbs": hbm,
                               "flops_alg_per_vector": dl["flops_alg"], "bytes_alg": dl["bytes_alg"]},
        "kernel_ms": {"leg2cheb": per_kernel[0], "cheb2leg": per_kernel[1], "names": names,
                      "algorithmic_bytes": [alg[nm] for nm in names],
                      "achieved_gbs": [alg[nm] / (avg_ms[nm] * 1e-3) / 1e9 for nm in names],
                      "note": "lc_execute_timed puts an event between kernels, so they run without their PDL "
                              "overlap: per-kernel times sum to more than the graph-replayed step"},
        "plan": plan_info,
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": e2e_steps, "ms_per_step": e2e_ms / e2e_steps,
                "path": ("lc_execute_host_chain (C ABI, one call per step or sub-batch: the input H2D from page-locked huge-page "
                         "host memory (lc_host_alloc), " + ("the row pass then the column pass" if two_d else
                                                            "leg2cheb then cheb2leg") +
                         f" on the device, the result D2H); {nbuf} stream(s), caller-owned staging and workspaces" +
                         (f"; {ech} sub-batches of {Vc} vectors per step, each its own call" if ech > 1 else ""))
                        if not (two_d and world > 1) else
                        f"H2D + tensor_product_2d (NCCL all-to-all) + D2H, {nbuf} stream(s)"},
        "gpu_launches": (kpe + pc.kernels_per_execute) * args.steps,
        "clocks": clk,
        "round_trip_einf": {"device": rt, "host_path": rt_host},
    }
    if passes is not None:
        line["passes_ms"] = passes
    if headline:
        line["cpu_baseline"] = cpu
        line["cpu_fmm_baseline"] = cfmm
    for p in (pl, pc):
        p.close()
    return line


def run_gpu(args, world, rank, local):
    line = measure(args.config, args, world, rank, local, headline=True)
    if args.batched != "none" and args.batched != args.config:
        # the batched half of the metric ("at N=1e6 & batched"): cfg3 by default, sharded over the ranks
        sub = measure(args.batched, args, world, rank, local, headline=False)
        line["batched"] = {k: sub[k] for k in ("metric", "value", "unit", "n_gpus", "ms_per_step", "scaling",
                                                "config", "step_ms", "roofline", "roofline_transform", "kernel_ms",
                                                "plan", "e2e", "gpu_launches", "clocks", "round_trip_einf")
                           if k in sub}
        if "passes_ms" in sub:
            line["batched"]["passes_ms"] = sub["passes_ms"]
    return line


def allreduce_sum(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
    return float(t.item())


def load_traffic(config, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from the committed
    ncu --set full capture (profiles/ncu_traffic.json, written from the .ncu-rep), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    try:
        d = json.load(open(p))
        return d.get(config, {}).get(kernel)
    except Exception:
        return None


# --------------------------------------------------------------------------- CPU oracle
def _oracle_rows_rate(n, kind, v, rows):
    import oracle
    from lc_inputs import vector
    f = vector(kind, n, seed=0, v=v)
    t0 = time.perf_counter()
    oracle.l2c_rows(f, rows)
    oracle.c2l_rows(f, rows)
    dt = time.perf_counter() - t0
    return 2 * len(rows), dt


def cpu_baseline(config, n, kind, budget_s=15.0):
    """The oracle (long-double direct rows, OpenMP over rows) on a bounded row sample of the workload."""
    rng = np.random.default_rng(1)
    cores = len(os.sched_getaffinity(0))
    r = 64
    done, dt = _oracle_rows_rate(n, kind, 0, np.sort(rng.choice(n, size=min(r, n), replace=False)))
    per = dt / done
    r2 = int(min(n, max(r, budget_s / per / 2)))
    rows = np.sort(rng.choice(n, size=r2, replace=False))
    done, dt = _oracle_rows_rate(n, kind, 0, rows)
    return {"value": done / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{r2} uniformly sampled output rows (seed 1) of leg2cheb and of cheb2leg of vector 0 at n={n}; "
                      f"long-double compensated O(n) per row, OpenMP over rows; {dt:.1f} s",
            "seconds": dt, "full_transform_extrapolated_s": dt / done * 2 * n}


def cpu_fmm_baseline(n, kind, dev, budget_s=10.0):
    """The same O(N) algorithm on the host (cpu_fmm/, C + OpenMP over the blocks of each step, plan tables
    exported from the GPU plans): leg2cheb then cheb2leg of vector 0, on ONE core (the paper's setting,
    PAPER.md:563: ~20 ms per 1e6 transform single-threaded on an M3) and on all host cores;
    fastest and median of the repetitions that fit the budget (the paper reports the fastest)."""
    import cpu_fmm
    from lc_inputs import vector
    from paper_2411_00033_b200 import Plan
    pa, pb = Plan(n, "leg2cheb", device=dev), Plan(n, "cheb2leg", device=dev)
    a, b = cpu_fmm.CpuFmm(pa), cpu_fmm.CpuFmm(pb)
    pa.close()
    pb.close()
    f = vector(kind, n, seed=0, v=0)
    cores = len(os.sched_getaffinity(0))
    out = {"unit": UNIT, "kind": "cpu O(N) FMM: the same algorithm in C + OpenMP (plan tables from the GPU plan)"}
    for label, t in (("one_core", 1), ("all_cores", cores)):
        cpu_fmm.set_threads(t)
        b(a(f))  # warm-up
        times, t0 = [], time.perf_counter()
        while True:
            t1 = time.perf_counter()
            b(a(f))
            times.append(time.perf_counter() - t1)
            if time.perf_counter() - t0 > budget_s / 4 or len(times) >= 50:
                break
        out[label] = {"value": 2 * n / min(times), "value_median": 2 * n / statistics.median(times), "cores": t,
                      "reps": len(times), "ms_per_transform_min": min(times) / 2 * 1e3,
                      "ms_per_transform_median": statistics.median(times) / 2 * 1e3}
    cpu_fmm.set_threads(cores)
    out.update(value=out["all_cores"]["value"], cores=cores,
               sample=f"round trips (leg2cheb then cheb2leg) of vector 0 at n={n}; fastest of the repetitions")
    return out


def run_reference(args, world, rank):
    if rank != 0:
        return None
    from lc_inputs import CONFIGS
    c = CONFIGS[args.config]
    n, kind = c["n"], c["kind"]
    rng = np.random.default_rng(1)
    cores = len(os.sched_getaffinity(0))
    # size each step so that warmup + steps fit in ~budget seconds
    _, dt = _oracle_rows_rate(n, kind, 0, np.sort(rng.choice(n, size=min(32, n), replace=False)))
    per_row = dt / (2 * min(32, n))
    total_budget = args.ref_seconds
    rows_per_step = int(max(2, min(n, total_budget / max(1, args.steps + args.warmup) / per_row / 2)))
    rows = np.sort(rng.choice(n, size=rows_per_step, replace=False))
    for _ in range(args.warmup):
        _oracle_rows_rate(n, kind, 0, rows)
    t0 = time.perf_counter()
    done = 0
    for _ in range(args.steps):
        d, _ = _oracle_rows_rate(n, kind, 0, rows)
        done += d
    dt = time.perf_counter() - t0
    val = done / dt
    return {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f80 (x87 long double)",
        "data": "synthetic (seeded, BASELINE.json recipe)",
        "config": {"workload": f"{args.config}: leg2cheb and cheb2leg rows of n={n} (oracle, bounded row sample)",
                   "n": n, "rows_per_step_per_direction": rows_per_step},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{rows_per_step} sampled rows per direction per step (seed 1), vector 0"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=["cfg1", "cfg2", "cfg2b", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--vt", type=int, default=0)
    ap.add_argument("--engine", type=int, default=0,
                    help="0 automatic, 1 level-pipelined kernels, 2 per-tile kernel, 3 up kernel + per-range pass")
    ap.add_argument("--subtree", type=int, default=0)
    ap.add_argument("--up-subtree", type=int, default=0)
    ap.add_argument("--stage-blocks", type=int, default=0)
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=60.0)
    ap.add_argument("--e2e-steps", type=int, default=200)
    ap.add_argument("--e2e-streams", type=int, default=3,
                    help="streams (with their own staging and workspaces) the host-buffer e2e pipeline uses")
    ap.add_argument("--split-vector", action="store_true",
                    help="cfg2/cfg2b at N > 1: one vector split over the ranks by output rows (NEXT-2) "
                         "instead of one replica per rank")
    ap.add_argument("--chunks", type=int, default=4,
                    help="cfg5 at N > 1: pass-1 row chunks whose all-to-all overlaps the next chunk (1: no overlap)")
    ap.add_argument("--batched", default="cfg3", choices=["cfg3", "cfg4", "cfg5", "none"],
                    help="batched sub-record measured after the headline config (the metric's 'batched' half)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # not launched by torchrun: launch one process per GPU ourselves (same flags)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        os.execv(sys.executable, cmd)
    if args.impl == "reference":
        # CPU oracle arm: rank 0 alone runs it; other ranks exit 0 without work (no process group needed)
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        line = run_reference(args, world, rank)
        if rank == 0 and line is not None:
            print(json.dumps(line), flush=True)
        return
    world, rank, local = dist_setup()
    if world != args.gpus and rank == 0:
        print(f"[bench] --gpus {args.gpus} but WORLD_SIZE={world}: measuring {world} rank(s)", file=sys.stderr)
    line = run_gpu(args, world, rank, local)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
