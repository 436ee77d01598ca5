#!/usr/bin/env python
"""Benchmark of the B200 Legendre<->Chebyshev execution stage (one JSON line on rank 0).

Default workload (BASELINE.json configs[1], "cfg2"): one fp64 vector of
n = 1e6 Legendre coefficients f_j = s_j/(j+1), s_j = +-1; a *step* is one
leg2cheb followed by one cheb2leg (the round trip), i.e. one pass of the whole
hot path in both directions.  Metric: coefficients/s = 2 n V / step time
(n unpadded, V vectors, 2 transforms), summed over ranks.

Multi-GPU (torchrun, one process per GPU, NCCL): cfg2 does not shard (one
vector couples all leaves through the coarse levels), so N GPUs run N
independent replicas (weak scaling).  --config cfg3/cfg4 shard the batch
(strong scaling).  Timing: CUDA events on the launching stream inside a
barrier + synchronize bracket, max over ranks.

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
        if torch.cuda.is_available():
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
    out = torch.empty((V, n), dtype=torch.float64, pin_memory=pin)
    return batch(kind, n, V, seed=0, v0=v0, out=out)


# --------------------------------------------------------------------------- our arm
def run_gpu(args, world, rank, local):
    from paper_2411_00033_b200 import Plan
    from paper_2411_00033_b200.dist import tensor_product_2d
    dev = torch.device("cuda", local)
    n, V, kind, v0, scaling = workload(args.config, world, rank)
    xh = make_input(kind, n, V, v0, pin=True)
    x = xh.to(dev)
    tmp = torch.empty_like(x)
    y = torch.empty_like(x)
    opts = dict(vt=args.vt, subtree=args.subtree, stage_blocks=args.stage_blocks, stages=args.stages,
                engine=args.engine, up_subtree=args.up_subtree)
    stream = torch.cuda.current_stream(dev)
    two_d = args.config == "cfg5"
    if two_d:
        # rows [v0, v0+V) of the n x n array on this rank; pass 1 along axis 1 (V row vectors), all-to-all,
        # pass 2 along axis 0 (n/world column vectors, batch-contiguous)
        scaling = "strong"
        C = n // world
        pl = Plan(n, "leg2cheb", batch=V, device=dev, **opts)
        pc = Plan(n, "leg2cheb", batch=C, device=dev, layout="batch", **opts)
        ycol = torch.empty((n, C), dtype=torch.float64, device=dev)

        def step():
            tensor_product_2d(x, row_fn=lambda a: pl.execute(a, tmp), col_fn=lambda a: pc.execute(a, ycol))
    else:
        pl = Plan(n, "leg2cheb", batch=V, device=dev, **opts)
        pc = Plan(n, "cheb2leg", batch=V, device=dev, **opts)

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

    clocks = ClockSampler(local)
    barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clk = clocks.stop()
    ms_local = e0.elapsed_time(e1)
    ms = allreduce_max(ms_local, world)
    coeffs = 2.0 * n * V  # per rank per step
    total_coeffs = allreduce_sum(coeffs, world)
    value = total_coeffs * args.steps / (ms / 1e3)

    # correctness of what was timed: round trip back to the input (gate 1e-12 for n <= 1e6)
    rt = None if two_d else float((y - x).abs().max() / x.abs().max())

    # ---- per-kernel durations (events around each kernel, same stream) for the roofline
    kpe = pl.kernels_per_execute
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(kpe + 1)]
    evc = [torch.cuda.Event(enable_timing=True) for _ in range(kpe + 1)]
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
    engine = pl.kernel_info.get("engine", 1)
    if engine == 3:
        names = ["lc_up3_kernel", "lc_range_kernel"]
    else:
        names = ["lc_tile_kernel"] if kpe == 1 else (["lc_up_kernel"] if kpe == 3 else []) + ["lc_stream_kernel",
                                                                                             "lc_down_kernel"]
    # algorithmic bytes per launch (f in, z out, A_hat once, lambda once; work arrays excluded):
    # the up kernel reads f, the streaming kernel reads A_hat and lambda (and f again for the band),
    # the down kernel writes z
    alg = {"lc_up_kernel": 8.0 * n * V, "lc_up3_kernel": 8.0 * n * V, "lc_stream_kernel": 8.0 * 324 * dl["nc"] + 8.0 * dl["N"],
           "lc_down_kernel": 8.0 * n * V}
    if kpe == 2:
        alg["lc_stream_kernel"] += 8.0 * n * V
    # the per-tile kernel (engine 2) is the whole transform: f in, z out, A_hat and lambda once
    alg["lc_tile_kernel"] = 16.0 * n * V + 8.0 * 324 * dl["nc"] + 8.0 * dl["N"]
    alg["lc_range_kernel"] = 8.0 * n * V + 8.0 * 324 * dl["nc"] + 8.0 * dl["N"]  # f in (band), z out, A_hat, lambda
    avg_ms = {nm: 0.5 * (per_kernel[0][i] + per_kernel[1][i]) for i, nm in enumerate(names)}
    dom = "lc_tile_kernel" if kpe == 1 else ("lc_range_kernel" if engine == 3 else "lc_stream_kernel")
    down_ms = avg_ms[dom]
    down_bytes = alg[dom]
    achieved = down_bytes / (down_ms * 1e-3) / 1e9
    traffic = load_traffic(args.config, dom)
    if kpe == 1 or engine == 3:
        # fp64 tensor-core bound: algorithmic flops of one transform over the kernel time, against the
        # measured DMMA peak (the higher of the two fp64 peaks, so the fraction is conservative)
        fk = dl["flops_alg"]
        if engine == 3:  # the range kernel does steps 3-7: drop step 1 and the M2M half of F_alg
            Lq, sq, Mq = dl["L"], dl["s"], 18
            fk -= 8.0 * ((2 ** Lq) - 1) * sq * Mq + 4.0 * (Mq * Mq + 2 * Mq) * ((2 ** Lq) - Lq - 1)
        tf = fk * V / (down_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "kernel": dom, "achieved": tf, "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": tf / DMMA_PEAK_TFLOPS, "traffic": traffic, "algorithmic_flops_per_launch": fk * V,
                "algorithmic_bytes_per_launch": down_bytes, "achieved_hbm_gbs": achieved, "avg_launch_ms": down_ms,
                "peak_source": "measured fp64 DMMA m8n8k4 (profiles/r1_dmma_peak.txt)"}
    else:
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm,
                "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                "algorithmic_bytes_per_launch": down_bytes, "avg_launch_ms": down_ms,
                "peak_source": hbm_src}
    # transform-level roofline (slower of fp64 flops at the measured DFMA peak and bytes at HBM peak)
    t_roof = max(dl["flops_alg"] * V / (FP64_PEAK_TFLOPS * 1e12), dl["bytes_alg"] / (hbm * 1e9))
    t_meas = ms_local / args.steps / 2 * 1e-3

    # ---- e2e through the C ABI with HOST buffers (lc_execute_host: H2D, kernels, D2H per transform)
    hz = torch.empty_like(xh).pin_memory()
    hy = torch.empty_like(xh).pin_memory() if not two_d else torch.empty((n, n // world), dtype=torch.float64).pin_memory()
    e2e_steps = max(3, min(args.steps, args.e2e_steps))

    def host_step():
        if two_d and world == 1:
            pl.execute_host(xh, hz)
            pc.execute_host(hz.view(n, n), hy)
        elif two_d:
            xd = xh.to(dev, non_blocking=True)
            zc = tensor_product_2d(xd, row_fn=lambda a: pl.execute(a, tmp), col_fn=lambda a: pc.execute(a, ycol))
            hy.copy_(zc, non_blocking=True)
        else:
            pl.execute_host(xh, hz)
            pc.execute_host(hz, hy)

    # 1-D configs: the round trip of a host vector, pipelined over three streams (the H2D of step i+1
    # and the D2H of step i-1 overlap the two transforms of step i; double-buffered on the device)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    if not two_d:
        xb = [torch.empty_like(x) for _ in range(2)]
        tb = [torch.empty_like(x) for _ in range(2)]
        yb = [torch.empty_like(x) for _ in range(2)]
        hyb = [torch.empty_like(xh).pin_memory() for _ in range(2)]
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_comp = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        for b in range(2):  # mark every buffer free
            ev_comp[b].record(stream)
            ev_out[b].record(stream)

    def pipelined(steps, h0=None, h1=None):
        if h0 is not None:
            h0.record(s_in)
        for i in range(steps):
            b = i & 1
            s_in.wait_event(ev_comp[b])  # xb[b] consumed by step i-2
            with torch.cuda.stream(s_in):
                xb[b].copy_(xh, non_blocking=True)
            ev_in[b].record(s_in)
            stream.wait_event(ev_in[b])
            stream.wait_event(ev_out[b])  # yb[b] read back by step i-2
            with torch.cuda.stream(stream):
                pl.execute(xb[b], tb[b])
                pc.execute(tb[b], yb[b])
            ev_comp[b].record(stream)
            s_out.wait_event(ev_comp[b])
            with torch.cuda.stream(s_out):
                hyb[b].copy_(yb[b], non_blocking=True)
            ev_out[b].record(s_out)
        if h1 is not None:
            h1.record(s_out)

    h0 = torch.cuda.Event(enable_timing=True)
    h1 = torch.cuda.Event(enable_timing=True)
    if two_d:
        for _ in range(2):
            host_step()
        torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        h0.record(stream)
        for _ in range(e2e_steps):
            host_step()
        h1.record(stream)
    else:
        pipelined(2)
        torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        pipelined(e2e_steps, h0, h1)
    torch.cuda.synchronize()
    barrier(world)
    e2e_ms = allreduce_max(h0.elapsed_time(h1), world)
    e2e_val = total_coeffs * e2e_steps / (e2e_ms / 1e3)
    rt_host = None if two_d else float((hyb[(e2e_steps - 1) & 1] - xh).abs().max() / xh.abs().max())
    bytes_vec = 8 * n * V
    h2d = bytes_vec * (1 if (two_d and world > 1) else 2)
    d2h = 8 * hy.numel() if two_d else 2 * bytes_vec
    if two_d and world == 1:
        h2d, d2h = 2 * bytes_vec, 2 * bytes_vec
    if not two_d:
        h2d, d2h = bytes_vec, bytes_vec

    cpu = None
    cfmm = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, n, kind, budget_s=args.cpu_seconds)
        try:
            cfmm = cpu_fmm_baseline(n, kind, dev, budget_s=args.cpu_seconds)
        except Exception as e:  # reported baseline only: never fail the GPU line for it
            cfmm = {"unavailable": f"{type(e).__name__}: {e}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json recipe)",
        "config": {"workload": (f"{args.config}: leg2cheb then cheb2leg (round trip) of {V} fp64 vector(s) "
                                f"of n={n} per GPU") if not two_d else
                               (f"cfg5: 2-D leg2cheb of an {n}x{n} fp64 array (axis 1, all-to-all, axis 0), "
                                f"{V} rows per GPU"), "n": n, "vectors_per_gpu": V, "N_padded": dl["N"],
                   "L": dl["L"], "s": dl["s"], "M": 18, "s_hat": 32, "transforms_per_step": 2,
                   "input_kind": kind,
                   "l2": f"no flush: per-step working set {2 * 8 * 324 * dl['nc'] / 1e6:.0f} MB of A_hat + "
                         f"{3 * bytes_vec / 1e6:.0f} MB of vectors vs 126 MB L2" if dl["nc"] > 0 else "small",
                   "graph": graph is not None, "kernel_cfg": {**{k: dl[k] for k in ("vt", "subtree", "stage_blocks",
                                                                                    "stages")},
                                                                 "engine": pl.kernel_info.get("engine", 1)}},
        "roofline": roof,
        "roofline_transform": {"t_roof_us": t_roof * 1e6, "t_measured_us": t_meas * 1e6,
                               "frac": t_roof / t_meas, "fp64_peak_tflops": FP64_PEAK_TFLOPS,
                               "flops_alg_per_vector": dl["flops_alg"], "bytes_alg": dl["bytes_alg"]},
        "kernel_ms": {"leg2cheb": per_kernel[0], "cheb2leg": per_kernel[1], "names": names,
                      "algorithmic_bytes": [alg[nm] for nm in names],
                      "achieved_gbs": [alg[nm] / (avg_ms[nm] * 1e-3) / 1e9 for nm in names]},
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": e2e_steps, "ms_per_step": e2e_ms / e2e_steps,
                "path": ("pinned host vector -> H2D -> leg2cheb -> cheb2leg (lc_execute) -> D2H, pipelined over "
                         "three streams with double-buffered device arrays") if not two_d else
                        ("lc_execute_host (C ABI, pinned host buffers) x2 per step" if world == 1
                         else "H2D + tensor_product_2d (NCCL all-to-all) + D2H")},
        "gpu_launches": kpe * 2 * args.steps,
        "clocks": clk,
        "round_trip_einf": {"device": rt, "host_path": rt_host},
        "cpu_baseline": cpu,
        "cpu_fmm_baseline": cfmm,
    }
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
    """The same O(N) algorithm on the host cores (cpu_fmm/, C + OpenMP, plan tables exported from the
    GPU plans): leg2cheb then cheb2leg of vector 0, repeated within the time budget (at least once)."""
    import cpu_fmm
    from lc_inputs import vector
    from paper_2411_00033_b200 import Plan
    a = cpu_fmm.CpuFmm(Plan(n, "leg2cheb", device=dev))
    b = cpu_fmm.CpuFmm(Plan(n, "cheb2leg", device=dev))
    f = vector(kind, n, seed=0, v=0)
    reps, t0 = 0, time.perf_counter()
    while True:
        b(a(f))
        reps += 1
        dt = time.perf_counter() - t0
        if dt > budget_s / 2 or reps >= 50:
            break
    return {"value": 2 * n * reps / dt, "unit": UNIT, "cores": cpu_fmm.threads(),
            "kind": "cpu O(N) FMM: the same algorithm in C + OpenMP (plan tables from the GPU plan)",
            "sample": f"{reps} round trip(s) (leg2cheb then cheb2leg) of vector 0 at n={n}; {dt:.2f} s",
            "seconds": dt}


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
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        # CPU oracle arm: rank 0 alone runs it; other ranks exit 0 without work (no process group needed)
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        line = run_reference(args, world, rank)
        if rank == 0 and line is not None:
            print(json.dumps(line), flush=True)
        return
    world, rank, local = dist_setup()
    line = run_gpu(args, world, rank, local)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
