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


@pytest.mark.parametrize("direction", ["leg2cheb", "cheb2leg"])
@pytest.mark.parametrize("n,parts", [(70001, 2), (1_000_000, 3), (1_000_000, 8), (4_000_017, 5), (10_000_000, 8),
                                     (300_000, 7)])
def test_partitioned_up_pass_equals_whole_plan(n, parts, direction):
    """part_up = 1: each part runs the upward pass of its own subtrees only (lc_execute_part phase 0);
    the subtree roots of all parts and each part's w halo are exchanged (dist.PartExchange, here as
    local copies between the parts' workspaces in place of the all-gather); phase 1 merges the coarse
    levels and finishes the part's rows -- equal to the whole plan bit for bit."""
    from paper_2411_00033_b200 import Plan, partition
    from paper_2411_00033_b200.dist import PartExchange
    dev = _dev()
    f = vector("normal", n, seed=78)
    x = torch.from_numpy(f).reshape(1, -1).to(dev)
    whole = Plan(n, direction, device=dev).execute(x)
    plans = [Plan(n, direction, device=dev, part_index=p, part_count=parts, part_up=1) for p in range(parts)]
    assert all(pl.kernel_info["part_up"] == 1 for pl in plans)
    infos = [dict(pl.kernel_info, L=pl.desc["L"]) for pl in plans]
    wss = [pl.new_workspace() for pl in plans]
    outs = []
    for pl, ws in zip(plans, wss):
        o = torch.full((1, n), 0, dtype=torch.int64, device=dev)
        o.fill_(NAN_BITS)
        outs.append(o.view(torch.float64))
        pl.execute_part(0, x, outs[-1], ws)
    units = [ws.view(torch.float64)[: ws.numel() // 8 // 18 * 18].view(-1, 18) for ws in wss]
    xs = [PartExchange(n, parts, infos, p) for p in range(parts)]
    gathered = torch.cat([units[p][torch.tensor(xs[p].send_index, device=dev)] for p in range(parts)])
    for p in range(parts):
        src = torch.tensor(xs[p].recv_src, dtype=torch.int64, device=dev)
        dst = torch.tensor(xs[p].recv_dst, dtype=torch.int64, device=dev)
        units[p][dst] = gathered[src]
    for pl, ws, o in zip(plans, wss, outs):
        pl.execute_part(1, x, o, ws)
    torch.cuda.synchronize()
    for p in range(parts):
        lo, hi = partition(n, p, parts)
        ob = outs[p].view(torch.int64)[0]
        assert bool((ob[:lo] == NAN_BITS).all()) and bool((ob[hi:] == NAN_BITS).all())
        assert torch.equal(outs[p][0, lo:hi], whole[0, lo:hi]), (p, lo, hi)
    # lc_execute refuses a part_up plan (it needs the exchange between its phases)
    from paper_2411_00033_b200._lib import LegChebError
    with pytest.raises(LegChebError):
        plans[0].execute(x)


@pytest.mark.parametrize("direction", ["leg2cheb", "cheb2leg"])
def test_parts_of_a_batch(direction):
    """Partitioned plans of several vectors (vector tiles of 2 and 4): each part's rows of every vector
    equal the whole plan's bit for bit; a partitioned upward pass needs one vector."""
    from paper_2411_00033_b200 import Plan, partition
    from paper_2411_00033_b200._lib import LegChebError
    dev = _dev()
    for n, V, parts in ((200000, 3, 3), (1_000_000, 5, 4)):
        x = torch.stack([torch.from_numpy(vector("normal", n, seed=90 + v)) for v in range(V)]).to(dev)
        whole = Plan(n, direction, batch=V, device=dev, engine=1).execute(x)
        for p in range(parts):
            lo, hi = partition(n, p, parts)
            z = Plan(n, direction, batch=V, device=dev, part_index=p, part_count=parts).execute(x)
            assert torch.equal(z[:, lo:hi], whole[:, lo:hi]), (n, V, p)
        with pytest.raises(LegChebError):
            Plan(n, direction, batch=V, device=dev, part_index=0, part_count=parts, part_up=1)
