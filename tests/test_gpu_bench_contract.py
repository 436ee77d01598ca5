"""bench.py keeps the driver's JSON-line contract (one line on rank 0 with the required keys), for our
arm on a small config and for the reference arm (the CPU oracle)."""
import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"]


def _run(args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                         cwd=ROOT, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_line_ours():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run(["--config", "cfg1", "--batched", "cfg3", "--steps", "5", "--warmup", "3", "--no-cpu-baseline",
              "--e2e-steps", "3"])
    for k in REQUIRED:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["value"] > 0
    assert "workload" in d["config"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    for k in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert k in d["clocks"], k
    assert d["gpu_launches"] > 0
    assert d["round_trip_einf"]["device"] <= 1e-12 and d["round_trip_einf"]["host_path"] <= 1e-12
    b = d["batched"]  # the batched half of the metric
    assert b["value"] > 0 and b["roofline"]["bound"] == "tensor" and b["round_trip_einf"]["device"] <= 1e-12


def test_bench_line_reference():
    # runs on the host cores only (the oracle arm): part of the CPU suite
    d = _run(["--impl", "reference", "--config", "cfg1", "--steps", "2", "--warmup", "1", "--ref-seconds", "3"])
    assert d["impl"] == "reference" and d["value"] > 0
    for k in ("metric", "unit", "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["cores"] >= 1
