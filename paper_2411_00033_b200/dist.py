"""Multi-GPU drivers over torch.distributed (one process per GPU; NCCL over NVLink).

Three partitionings:

* batch sharding (cfg3, cfg4): independent vectors are split contiguously over the ranks; every rank
  holds the full plan (replicated) and transforms its own slice -- there is no collective on the data
  path (`shard_range`, `BatchedTransform`).
* 2-D tensor-product transform (cfg5): an n0 x n1 array partitioned by rows.  Pass 1 transforms along
  axis 1 (each local row is one vector); an all-to-all transposes the row slabs into column slabs;
  pass 2 transforms along axis 0 with the batch-contiguous layout (LC_BATCH_CONTIGUOUS), so no local
  transpose is needed after the exchange (`tensor_product_2d`).
* one long vector (NEXT-2): output rows split over the ranks (`SingleVectorTransform`), the input
  replicated, the slices all-gathered.

The per-pass transform is injectable (`row_fn`, `col_fn`) so that the index algebra can be tested on
CPU ranks with gloo; the default is the sm_100a library through `Plan`.
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, stop) of `total` items owned by `rank` (the first total % world ranks get one more)."""
    base, rem = divmod(total, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


class BatchedTransform:
    """Transform of this rank's contiguous slice of a batch of vectors (no communication).

    `transform` replaces the sm_100a plan by another callable on [rows, n] (tests use a CPU stand-in);
    the product path always builds a `Plan`."""

    def __init__(self, n: int, direction: str, total_batch: int, group=None, device=None,
                 transform: Optional[Callable] = None, **opts):
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.start, self.stop = shard_range(total_batch, self.world, self.rank)
        self.n = n
        self.plan = None
        self.transform = transform
        if transform is None and self.stop > self.start:
            # a rank that owns no vectors (total_batch < world) has no plan and returns empty outputs
            from .api import Plan
            self.plan = Plan(n, direction, batch=self.stop - self.start, device=device, **opts)

    def __call__(self, x_local: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        if x_local.shape[0] != self.stop - self.start:
            raise ValueError(f"rank {self.rank} owns vectors [{self.start}, {self.stop})")
        if self.stop == self.start:
            return x_local.new_empty((0, self.n)) if out is None else out
        if self.transform is not None:
            y = self.transform(x_local)
            return y if out is None else out.copy_(y)
        return self.plan.execute(x_local, out)


class PartExchange:
    """Index maps of the workspace exchange between the parts of a partitioned single-vector plan whose
    upward pass is partitioned too (lc_plan_opts.part_up, lc_execute_part).

    After phase 0 every part holds w of its own subtrees.  Phase 1 needs, per part, every subtree root
    (level grup, whole vector: the coarse levels are merged from them on each part) and, on each fine
    level g >= grup, the two segments that follow the part (the columns u+2, u+3 of its last rows,
    eq:globalij).  Each part publishes its roots and its first two segments of every fine level; the
    receiving side scatters what it lacks.  `send_index` (w units to pack) is the same layout on every
    part; `recv_src` / `recv_dst` map rows of the stacked [parts, K] gather to w units of this part.
    w unit = VM = 18 doubles of one (level, sigma, segment), tile 0 (batch 1)."""

    def __init__(self, n: int, parts: int, plan_info: list[dict], me: int):
        self.parts, self.me = parts, me
        L = plan_info[me]["L"]
        kup, gr = plan_info[me]["kup"], plan_info[me]["grup"]
        self.L, self.gr = L, gr
        unit = lambda g, sg, t: 2 * ((4 << g) - 4) + sg * (4 << g) + t  # noqa: E731
        nseg = lambda g: 4 << g  # noqa: E731
        spans = [(pi["part_lo"], pi["part_hi"]) for pi in plan_info]  # leaf segments
        roots = [(lo >> kup, hi >> kup) for lo, hi in spans]
        self.maxroots = max(b - a for a, b in roots)
        nfine = L - gr
        self.K = 2 * self.maxroots + nfine * 2 * 2

        def send_units(r):
            lo, hi = spans[r]
            a, b = roots[r]
            idx = []
            for sg in range(2):
                idx += [unit(gr, sg, t) for t in range(a, b)] + [0] * (self.maxroots - (b - a))
            for g in range(gr, L):
                lo_g = lo >> (L - 1 - g)
                for sg in range(2):
                    for i in range(2):
                        t = lo_g + i
                        idx.append(unit(g, sg, t) if (hi > lo and t < nseg(g)) else 0)
            return idx

        self.send_index = send_units(me)
        src, dst = [], []
        lo_me, hi_me = spans[me]
        for r in range(parts):  # the roots of every other part
            if r == me:
                continue
            a, b = roots[r]
            for sg in range(2):
                for k, t in enumerate(range(a, b)):
                    src.append(r * self.K + sg * self.maxroots + k)
                    dst.append(unit(gr, sg, t))
        if hi_me > lo_me:  # the halo: 2 segments after the part on every fine level, from their owners
            for g in range(gr, L):
                sh = L - 1 - g
                hi_g = (hi_me - 1 >> sh) + 1
                for t in range(hi_g, min(hi_g + 2, nseg(g))):
                    owner = next((r for r in range(parts) if spans[r][1] > spans[r][0]
                                  and (spans[r][0] >> sh) <= t <= ((spans[r][1] - 1) >> sh)), None)
                    if owner is None:  # zero padding past the last part: w stays 0 (never written)
                        continue
                    i = t - (spans[owner][0] >> sh)
                    assert i in (0, 1), "halo segment beyond the owner's first two"
                    for sg in range(2):
                        src.append(owner * self.K + 2 * self.maxroots + ((g - gr) * 2 + sg) * 2 + i)
                        dst.append(unit(g, sg, t))
        self.recv_src, self.recv_dst = src, dst

    def tensors(self, device):
        t = lambda a: torch.tensor(a, dtype=torch.int64, device=device)  # noqa: E731
        return t(self.send_index), t(self.recv_src), t(self.recv_dst)


class SingleVectorTransform:
    """One long transform split over the ranks by output rows (NEXT-2).

    Every rank holds the whole input vector (replicated; `broadcast` it first if it lives on one rank)
    and runs a partitioned plan (lc_plan_opts.part_index / part_count): the upward pass whole, then the
    M2L of its own rows and their ancestor segments, the band of its rows and the downward pass of its
    subtrees -- so the A_hat stream and the band, the bulk of the work, are divided by the rank count.
    Rank r's rows are [row_lo, row_hi) (`partition`); `gather=True` all-gathers the slices into the
    full result on every rank (NCCL over NVLink).  `transform` replaces the plan by a callable
    (x_full, lo, hi) -> rows lo..hi (tests use a CPU stand-in); the product path builds a `Plan`."""

    def __init__(self, n: int, direction: str, group=None, device=None, transform: Optional[Callable] = None,
                 part_up: bool = False, **opts):
        from .api import partition
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.n = n
        self.spans = [partition(n, r, self.world) for r in range(self.world)]
        self.row_lo, self.row_hi = self.spans[self.rank]
        self.transform = transform
        self.plan = None
        self.part_up = bool(part_up) and self.world > 1 and transform is None
        if transform is None:
            from .api import Plan
            self.plan = Plan(n, direction, batch=1, device=device, part_index=self.rank, part_count=self.world,
                             part_up=int(self.part_up), **opts)
            assert (self.plan.desc["row_lo"], self.plan.desc["row_hi"]) == (self.row_lo, self.row_hi)
            self.part_up = self.part_up and bool(self.plan.kernel_info["part_up"])
            if self.part_up:
                # every part's geometry (identical plans but for the range) for the exchange maps
                info = dict(self.plan.kernel_info, L=self.plan.desc["L"])
                infos = [None] * self.world
                dist.all_gather_object(infos, {k: info[k] for k in ("L", "kup", "grup", "part_lo", "part_hi")},
                                       group=group)
                self.xch = PartExchange(n, self.world, infos, self.rank)
                self.ws = self.plan.new_workspace()
                self.w_units = self.ws.view(torch.float64)[: self.ws.numel() // 8 // 18 * 18].view(-1, 18)
                self.send_idx, self.recv_src, self.recv_dst = self.xch.tensors(self.ws.device)
                self.out = torch.empty((1, n), dtype=torch.float64, device=self.ws.device)

    def __call__(self, x_full: torch.Tensor, gather: bool = True) -> torch.Tensor:
        """x_full: the whole [n] input on this rank.  Returns the full [n] result (gather) or this
        rank's rows [row_lo, row_hi)."""
        if x_full.numel() != self.n:
            raise ValueError(f"need the whole vector of {self.n} coefficients on every rank")
        lo, hi = self.row_lo, self.row_hi
        if self.transform is not None:
            mine = self.transform(x_full, lo, hi)
        elif self.part_up:
            x2 = x_full.reshape(1, -1)
            self.plan.execute_part(0, x2, self.out, self.ws)  # upward pass of this part's subtrees
            send = self.w_units[self.send_idx]  # roots + first two segments of every fine level
            recv = send.new_empty((self.world * send.shape[0], 18))
            dist.all_gather_into_tensor(recv, send, group=self.group)
            self.w_units[self.recv_dst] = recv[self.recv_src]  # every root, the halo of the next part
            self.plan.execute_part(1, x2, self.out, self.ws)
            mine = self.out.reshape(-1)[lo:hi]
        else:
            z = self.plan.execute(x_full.reshape(1, -1))  # rows outside [lo, hi) are not written
            mine = z.reshape(-1)[lo:hi]
        if not gather or self.world == 1:
            return mine.clone() if gather else mine
        width = max(b - a for a, b in self.spans)
        send = x_full.new_zeros(width)
        send[: hi - lo] = mine
        recv = x_full.new_empty(self.world * width)
        dist.all_gather_into_tensor(recv, send, group=self.group)
        return torch.cat([recv[r * width: r * width + (b - a)] for r, (a, b) in enumerate(self.spans)])


def pack_for_transpose(y_rows: torch.Tensor, world: int) -> torch.Tensor:
    """[R, n1] row slab -> [world, R, C] with block d = columns [d C, (d+1) C) (C = n1 / world)."""
    R, n1 = y_rows.shape
    C = n1 // world
    return y_rows.reshape(R, world, C).permute(1, 0, 2).contiguous()


def transpose_rows_to_cols(y_rows: torch.Tensor, group=None) -> torch.Tensor:
    """All-to-all: row slab [R, n1] of every rank -> column slab [n0, C] (row-major, C = n1 / world).

    Rank r sends block (its rows) x (columns of rank d) to rank d; stacking the received blocks over
    the source ranks gives rows in global order, i.e. the column slab in the batch-contiguous layout."""
    world = dist.get_world_size(group)
    R, n1 = y_rows.shape
    if n1 % world:
        raise ValueError("n1 must be divisible by the number of ranks")
    send = pack_for_transpose(y_rows, world)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv.view(-1), send.view(-1), group=group)
    return recv.reshape(world * R, n1 // world)


def transpose_cols_to_rows(z_cols: torch.Tensor, group=None) -> torch.Tensor:
    """Inverse exchange: column slab [n0, C] -> row slab [R, n1] (R = n0 / world)."""
    world = dist.get_world_size(group)
    n0, C = z_cols.shape
    send = z_cols.reshape(world, n0 // world, C).contiguous()
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv.view(-1), send.view(-1), group=group)
    return recv.permute(1, 0, 2).reshape(n0 // world, world * C)


def _chunked_exchange(x_rows: torch.Tensor, row_fn: Callable, chunks: int, group=None,
                      timing: Optional[dict] = None, row_packed: bool = False) -> torch.Tensor:
    """Pass 1 in `chunks` row chunks with the all-to-all of chunk k overlapping pass 1 of chunk k+1.

    Chunk k's output [Rk, n1] is packed by destination ([world, Rk, C]) and exchanged with
    all_to_all_single on a communication stream while the next chunk transforms; the received
    [chunks][world][Rk][C] blocks are rows s R + k Rk + r of the column slab, which one local permute
    puts in the batch-contiguous [n0, C] order pass 2 reads."""
    world = dist.get_world_size(group)
    R, n1 = x_rows.shape
    Rk, C = R // chunks, n1 // world
    recv = x_rows.new_empty((chunks, world, Rk, C))
    cuda = x_rows.is_cuda
    main = torch.cuda.current_stream(x_rows.device) if cuda else None
    comm = torch.cuda.Stream(x_rows.device) if cuda else None
    sends = []
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)] if (cuda and timing is not None) else None
    if ev:
        ev[0].record(main)
    for k in range(chunks):
        yk = row_fn(x_rows[k * Rk:(k + 1) * Rk])
        send = yk.reshape(world, Rk, C) if row_packed else pack_for_transpose(yk, world)
        sends.append(send)  # kept alive until the exchange completes
        if cuda:
            done = torch.cuda.Event()
            done.record(main)
            with torch.cuda.stream(comm):
                comm.wait_event(done)
                dist.all_to_all_single(recv[k].view(-1), send.view(-1), group=group)
        else:
            dist.all_to_all_single(recv[k].view(-1), send.view(-1), group=group)
    if cuda:
        main.wait_stream(comm)
        if ev:
            ev[1].record(main)
            torch.cuda.synchronize()
            timing.update(pass1_and_alltoall_overlapped_ms=ev[0].elapsed_time(ev[1]))
    return recv.permute(1, 0, 2, 3).reshape(world * R, C)


def tensor_product_2d(x_rows: torch.Tensor, group=None, row_fn: Optional[Callable] = None,
                      col_fn: Optional[Callable] = None, direction: str = "leg2cheb",
                      restore_rows: bool = False, timing: Optional[dict] = None, chunks: int = 1,
                      row_packed: bool = False) -> torch.Tensor:
    """2-D transform of an n0 x n1 array partitioned by rows (this rank: [n0/world, n1]).

    Pass 1 along axis 1 on the row slab, all-to-all, pass 2 along axis 0 on the column slab
    ([n0, n1/world], batch-contiguous).  Returns the column slab, or the row slab if restore_rows.
    chunks > 1 (world > 1): pass 1 in row chunks, each chunk's all-to-all overlapping the next
    chunk's transform (SURVEY 8(e) "chunk pass 1 by destination ... on a comm stream").
    row_packed: row_fn already returns its rows packed by destination ([world, rows, n1/world], a plan
    with out_block = n1/world writes them so from its kernel epilogue); the default plan does that."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    R, n1 = x_rows.shape
    n0 = R * world
    C = n1 // world
    if chunks < 1 or R % chunks:
        raise ValueError("chunks must divide the rows of the slab")
    if row_fn is None or col_fn is None:
        from .api import Plan
        if row_fn is None:
            # world > 1: the pass-1 epilogue writes the rows packed by destination (lc_plan_opts.out_block)
            prow = Plan(n1, direction, batch=R // chunks if world > 1 else R, device=x_rows.device,
                        out_block=C if world > 1 else 0)
            row_fn = prow.execute
            row_packed = world > 1
        if col_fn is None:
            pcol = Plan(n0, direction, batch=C, device=x_rows.device, layout="batch")
            col_fn = pcol.execute
    if world > 1 and chunks > 1:
        yc = _chunked_exchange(x_rows, row_fn, chunks, group, timing, row_packed)
        z = col_fn(yc)
        return transpose_cols_to_rows(z, group) if restore_rows else z
    ev = None
    if timing is not None and x_rows.is_cuda:
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
    y = row_fn(x_rows)
    if ev:
        ev[1].record()
    # one rank: the row-major [n0, n1] result already is the batch-contiguous column layout
    if world > 1 and row_packed:
        recv = torch.empty_like(y)
        dist.all_to_all_single(recv.view(-1), y.reshape(-1), group=group)
        yc = recv.reshape(world * R, C)
    else:
        yc = transpose_rows_to_cols(y, group) if world > 1 else y
    if ev:
        ev[2].record()
    z = col_fn(yc)
    if ev:
        ev[3].record()
        torch.cuda.synchronize()
        timing.update(pass1_ms=ev[0].elapsed_time(ev[1]), alltoall_ms=ev[1].elapsed_time(ev[2]),
                      pass2_ms=ev[2].elapsed_time(ev[3]))
    return transpose_cols_to_rows(z, group) if (restore_rows and world > 1) else z
