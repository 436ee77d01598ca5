"""Seeded fuzz of the three engines with non-decaying inputs (tools/fuzz_parity.py): random n, batch, direction,
layout and s_hat; the oracle on C-4 rows at the plan's own s with the per-row diagnostic, and the engines against
each other per 2s-block.  The test runs 32 cases; 3360 cases (seeds 7, 11, 23 and 101, n up to 3e6) are recorded in
profiles/r2_fuzz_parity.txt."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fuzz_three_engines_nondecaying():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_parity.py"), "32", "3", "300000"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "32 cases (seed 3)" in r.stdout and "failures 0" in r.stdout
