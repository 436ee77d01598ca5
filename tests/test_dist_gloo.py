"""World-size-2 (and 3) gloo tests of the multi-GPU host logic on CPU ranks: batch sharding index maps
and the 2-D tensor-product transform with its all-to-all transposes.  The per-pass transform is the
CPU oracle (a test stand-in; the product path never imports it)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_00033_b200.dist import (pack_for_transpose, shard_range, tensor_product_2d,
                                        transpose_cols_to_rows, transpose_rows_to_cols)


def test_shard_range_covers_exactly():
    for total in (1, 7, 64, 4096, 4097):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_pack_for_transpose_blocks():
    y = torch.arange(4 * 6, dtype=torch.float64).reshape(4, 6)
    p = pack_for_transpose(y, 3)
    for d in range(3):
        assert torch.equal(p[d], y[:, 2 * d:2 * d + 2])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_rows(x):  # transform each row (a vector) with the oracle: stand-in for the GPU plan
    import oracle
    return torch.from_numpy(np.stack([oracle.l2c(r.numpy()).astype(np.float64) for r in x]))


def _oracle_cols_batch_layout(x):  # x: [n0, C] batch-contiguous columns
    import oracle
    cols = [oracle.l2c(x[:, j].numpy()).astype(np.float64) for j in range(x.shape[1])]
    return torch.from_numpy(np.stack(cols, axis=1))


def _worker(rank, world, port, n0, n1, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(5)
        full = torch.randn(n0, n1, generator=g, dtype=torch.float64)
        full /= torch.outer(torch.arange(1, n0 + 1, dtype=torch.float64), torch.arange(1, n1 + 1, dtype=torch.float64))
        R = n0 // world
        mine = full[rank * R:(rank + 1) * R].contiguous()
        # the exchange alone round-trips
        back = transpose_cols_to_rows(transpose_rows_to_cols(mine), None)
        ok_roundtrip = torch.equal(back, mine)
        # the column slab after the exchange holds columns [rank C, (rank+1) C) of the full array
        C = n1 // world
        cols = transpose_rows_to_cols(mine)
        ok_cols = torch.equal(cols, full[:, rank * C:(rank + 1) * C])
        z = tensor_product_2d(mine, None, row_fn=_oracle_rows, col_fn=_oracle_cols_batch_layout)
        zr = tensor_product_2d(mine, None, row_fn=_oracle_rows, col_fn=_oracle_cols_batch_layout,
                               restore_rows=True)
        # pass 1 in chunks, each chunk's all-to-all overlapping the next chunk (same result, bit for bit)
        zc = tensor_product_2d(mine, None, row_fn=_oracle_rows, col_fn=_oracle_cols_batch_layout,
                               chunks=R if R % 2 else 2) if R > 1 else z
        # pass 1 writing its rows packed by destination (what a plan with out_block = n1/world does)
        C = n1 // world

        def rows_packed(a):
            return _oracle_rows(a).reshape(a.shape[0], world, C).permute(1, 0, 2).contiguous()

        zp = tensor_product_2d(mine, None, row_fn=rows_packed, col_fn=_oracle_cols_batch_layout, row_packed=True)
        zpc = tensor_product_2d(mine, None, row_fn=rows_packed, col_fn=_oracle_cols_batch_layout, row_packed=True,
                                chunks=R if R % 2 else 2) if R > 1 else zp
        assert torch.equal(zp, z) and torch.equal(zpc, z)
        results[rank] = (ok_roundtrip, ok_cols, z.numpy().copy(), zr.numpy().copy(), zc.numpy().copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n0,n1", [(2, 40, 24), (3, 33, 27)])
def test_tensor_product_2d_gloo(world, n0, n1):
    import oracle
    mgr = mp.Manager()
    results = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, n0, n1, results), nprocs=world, join=True)
    g = torch.Generator().manual_seed(5)
    full = torch.randn(n0, n1, generator=g, dtype=torch.float64)
    full /= torch.outer(torch.arange(1, n0 + 1, dtype=torch.float64), torch.arange(1, n1 + 1, dtype=torch.float64))
    # reference: L2C along axis 1 then axis 0 (separable 2-D transform, SURVEY C-4 for cfg5)
    ref = np.stack([oracle.l2c(r).astype(np.float64) for r in full.numpy()])
    ref = np.stack([oracle.l2c(ref[:, j]).astype(np.float64) for j in range(n1)], axis=1)
    C = n1 // world
    R = n0 // world
    for r in range(world):
        ok_rt, ok_cols, z, zr, zc = results[r]
        assert ok_rt and ok_cols
        assert np.array_equal(zc, z)
        assert np.max(np.abs(z - ref[:, r * C:(r + 1) * C])) <= 1e-15 * np.max(np.abs(ref))
        assert np.max(np.abs(zr - ref[r * R:(r + 1) * R])) <= 1e-15 * np.max(np.abs(ref))


def _batch_worker(rank, world, port, total, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = shard_range(total, world, rank)
        t = torch.tensor([b - a], dtype=torch.int64)
        dist.all_reduce(t)
        mx = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)  # bench.py's max-over-ranks timing reduction
        results[rank] = (a, b, int(t.item()), float(mx.item()))
    finally:
        dist.destroy_process_group()


def test_batch_sharding_gloo():
    world, total = 2, 4097
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_batch_worker, args=(world, _free_port(), total, results), nprocs=world, join=True)
    assert results[0][:2] == (0, 2049) and results[1][:2] == (2049, 4097)
    assert all(results[r][2] == total and results[r][3] == float(world) for r in range(world))


def _batched_worker(rank, world, port, n, total, results):
    from paper_2411_00033_b200.dist import BatchedTransform
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(9)
        full = torch.randn(total, n, generator=g, dtype=torch.float64)
        bt = BatchedTransform(n, "leg2cheb", total, transform=_oracle_rows)  # CPU stand-in for the plan
        mine = full[bt.start:bt.stop].contiguous()
        z = bt(mine)
        # gather every rank's slice to rank 0 in rank order (sizes differ by at most one)
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([z.shape[0]]))
        mx = int(max(t.item() for t in sizes))
        pad = torch.zeros(mx, n, dtype=torch.float64)
        pad[: z.shape[0]] = z
        parts = [torch.zeros(mx, n, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, pad)
        if rank == 0:
            results[0] = torch.cat([p[: int(sz.item())] for p, sz in zip(parts, sizes)]).numpy()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,total", [(2, 7), (3, 2)])
def test_batched_transform_end_to_end_gloo(world, total):
    """BatchedTransform end to end on CPU ranks (oracle as the per-rank transform): every vector is
    transformed exactly once, by the rank that owns it, including ranks that own none (total < world)."""
    import oracle
    n = 50
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_batched_worker, args=(world, _free_port(), n, total, results), nprocs=world, join=True)
    g = torch.Generator().manual_seed(9)
    full = torch.randn(total, n, generator=g, dtype=torch.float64)
    ref = np.stack([oracle.l2c(r.numpy()).astype(np.float64) for r in full])
    assert np.array_equal(results[0], ref)


def _single_vector_worker(rank, world, port, n, results):
    from paper_2411_00033_b200.dist import SingleVectorTransform
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(13)
        x = torch.randn(n, generator=g, dtype=torch.float64)  # the whole vector on every rank

        def rows(xf, lo, hi):  # CPU stand-in for the partitioned plan: the oracle's rows lo..hi
            return torch.from_numpy(oracle.l2c_rows(xf.numpy(), np.arange(lo, hi)).astype(np.float64))

        t = SingleVectorTransform(n, "leg2cheb", transform=rows)
        results[rank] = (t.row_lo, t.row_hi, t(x).numpy().copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 3000), (3, 5000)])
def test_single_vector_split_gloo(world, n):
    """NEXT-2 host logic on CPU ranks: the row partition covers [0, n) once (some parts may be empty)
    and the all-gathered slices are the whole transform on every rank."""
    import oracle
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_single_vector_worker, args=(world, _free_port(), n, results), nprocs=world, join=True)
    g = torch.Generator().manual_seed(13)
    ref = oracle.l2c(torch.randn(n, generator=g, dtype=torch.float64).numpy()).astype(np.float64)
    spans = sorted((results[r][0], results[r][1]) for r in range(world))
    assert spans[0][0] == 0 and spans[-1][1] == n
    for r in range(world):
        assert np.array_equal(results[r][2], ref)


def test_part_exchange_maps_cover_what_phase_1_reads():
    """Host logic of the partitioned upward pass (NEXT-2): after the exchange every part holds all
    subtree roots and, on every fine level, the two segments after its range, each taken from the part
    that owns it (checked against a synthetic w where every unit holds its own index)."""
    from paper_2411_00033_b200.dist import PartExchange
    for L, kup, nparts_spans in ((13, 6, [(0, 192), (192, 448), (448, 16384)]),
                                 (10, 6, [(0, 64), (64, 128), (128, 192), (192, 2048)]),
                                 (8, 6, [(0, 0), (0, 64), (64, 512)]),
                                 (10, 6, [(0, 640), (640, 1920)])):  # padding groups past the last part
        gr = L - 1 - kup
        parts = len(nparts_spans)
        infos = [dict(L=L, kup=kup, grup=gr, part_lo=a, part_hi=b) for a, b in nparts_spans]
        nunits = 2 * ((4 << L) - 4)
        unit = lambda g, sg, t: 2 * ((4 << g) - 4) + sg * (4 << g) + t  # noqa: E731
        xs = [PartExchange(0, parts, infos, p) for p in range(parts)]
        # w of each part after phase 0: only its own subtrees' units are valid (value = unit index)
        ws = []
        for p, (a, b) in enumerate(nparts_spans):
            w = np.full(nunits, -1.0)
            for g in range(gr, L):
                sh = L - 1 - g
                for sg in range(2):
                    for t in range(a >> sh, (b >> sh) if b > a else a >> sh):
                        w[unit(g, sg, t)] = unit(g, sg, t)
            ws.append(w)
        gathered = np.concatenate([ws[p][xs[p].send_index] for p in range(parts)])
        for p, (a, b) in enumerate(nparts_spans):
            w = ws[p].copy()
            w[xs[p].recv_dst] = gathered[xs[p].recv_src]
            last = max(bb for _, bb in nparts_spans)
            for sg in range(2):  # every root (past the last part: zero padding, owned by no part)
                for t in range(4 << gr):
                    assert w[unit(gr, sg, t)] == (unit(gr, sg, t) if t < (last >> kup) else -1.0)
            if b > a:  # the halo (up to the last part's end: past it w is zero padding, never written)
                for g in range(gr, L):
                    sh = L - 1 - g
                    hi_g = ((b - 1) >> sh) + 1
                    for t in range(hi_g, min(hi_g + 2, 4 << g, ((last - 1) >> sh) + 1)):
                        for sg in range(2):
                            assert w[unit(g, sg, t)] == unit(g, sg, t), (L, p, g, t)
