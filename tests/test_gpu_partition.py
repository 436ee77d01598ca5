"""NEXT-2 on one GPU: a long transform split into parts by output rows (lc_plan_opts.part_index /
part_count).  Each part's plan computes its rows with the same arithmetic as the whole plan (bit for
bit), writes nothing outside them, and the parts together equal the oracle (PAPER.md:179-198 for the
vector views the split follows).  The parts run one after another here (one GPU); on several GPUs
paper_2411_00033_b200.dist.SingleVectorTransform runs one part per rank and all-gathers the rows."""
import numpy as np
import pytest
import torch

from lc_inputs import vector
from parity_util import c4_rows, check_rows

pytestmark = pytest.mark.gpu

NAN_BITS = 0x7FF8DEADBEEF0001


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


@pytest.mark.parametrize("direction", ["leg2cheb", "cheb2leg"])
@pytest.mark.parametrize("n,parts", [(70001, 2), (1_000_000, 3), (1_000_000, 8), (4_000_017, 5), (10_000_000, 8)])
def test_parts_equal_whole_plan(n, parts, direction):
    from paper_2411_00033_b200 import Plan, partition
    dev = _dev()
    f = vector("normal", n, seed=77)
    x = torch.from_numpy(f).reshape(1, -1).to(dev)
    whole = Plan(n, direction, device=dev).execute(x)
    combined = torch.empty_like(whole)
    covered = 0
    for p in range(parts):
        lo, hi = partition(n, p, parts)
        plan = Plan(n, direction, device=dev, part_index=p, part_count=parts)
        assert (plan.desc["row_lo"], plan.desc["row_hi"]) == (lo, hi) and plan.kernel_info["engine"] == 1
        out = torch.full((1, n), 0, dtype=torch.int64, device=dev)
        out.fill_(NAN_BITS)
        out = out.view(torch.float64)
        plan.execute(x, out)
        torch.cuda.synchronize()
        ob = out.view(torch.int64)[0]
        assert bool((ob[:lo] == NAN_BITS).all()) and bool((ob[hi:] == NAN_BITS).all())  # nothing outside
        assert torch.equal(out[0, lo:hi], whole[0, lo:hi]), (p, lo, hi)  # same arithmetic, bit for bit
        combined[0, lo:hi] = out[0, lo:hi]
        covered += hi - lo
    assert covered == n
    rows = c4_rows(n, Plan(n, direction, device=dev).desc["s"], uniform=1024, tiles=128)
    check_rows(direction, f, combined.cpu().numpy()[0], rows, f"partitioned n={n} parts={parts}")


def test_partition_geometry():
    from paper_2411_00033_b200 import partition
    for n in (129, 5000, 70001, 1_000_000, 10_000_000):
        for parts in (1, 2, 3, 7, 8):
            spans = [partition(n, p, parts) for p in range(parts)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(parts - 1))
