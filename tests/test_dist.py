"""Multi-process (world_size 2 and 3, gloo, CPU) tests of the sharding logic of
paper_2103_10765_b200/dist.py: partitions (plain and tile-aligned), slab halos, the
point-to-point gather of row blocks into rank 0's full tables, and the chunked gather that
overlaps the matching (uneven blocks, ragged last tile).  The CUDA kernels are exercised by the GPU tests
(tests/test_gpu_parity.py::test_row_ranges_concatenate_to_full emulates the shards on one GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_10765_b200 import dist as gd


def test_row_partition_covers_and_balances():
    for Ry in (1, 7, 64, 681):
        for world in (1, 2, 3, 4, 8):
            parts = gd.row_partition(Ry, world)
            assert parts[0][0] == 0 and parts[-1][1] == Ry
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))


def test_row_partition_tile_aligned():
    """align = 16 (the matcher's tile height): every block but the last is whole tiles, tile
    counts differ by at most one, the blocks tile [0, Ry)."""
    for Ry in (1, 15, 16, 17, 64, 83, 681):
        for world in (1, 2, 3, 4, 8):
            parts = gd.row_partition(Ry, world, 16)
            assert parts[0][0] == 0 and parts[-1][1] == Ry
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            tiles = [-(-(b - a) // 16) for a, b in parts]
            assert max(tiles) - min(tiles) <= 1
            assert all((b - a) % 16 == 0 for a, b in parts if b < Ry)
    # c3 at 8 GPUs: 43 tiles -> 6,6,6,5,5,5,5,5 (the last one 9 rows short)
    assert [b - a for a, b in gd.row_partition(681, 8, 16)] == [96, 96, 96, 80, 80, 80, 80, 73]


def test_chunk_rows():
    for k0, k1, n in [(0, 96, 3), (608, 681, 3), (0, 5, 4), (16, 16, 2), (32, 200, 1), (0, 681, 7)]:
        ch = gd.chunk_rows(k0, k1, n)
        if k1 <= k0:
            assert ch == []
            continue
        assert ch[0][0] == k0 and ch[-1][1] == k1 and len(ch) <= max(1, n)
        assert all(ch[i][1] == ch[i + 1][0] for i in range(len(ch) - 1))
        assert all((b - a) % 16 == 0 for a, b in ch[:-1])


def test_slab_bounds_contain_every_window():
    """Every candidate row of every reference in [k0, k1) lies in the slab (clamped window)."""
    for H, P, S, r in [(2048, 8, 3, 19), (201, 8, 3, 19), (512, 12, 4, 19), (50, 8, 3, 40)]:
        Ry = gd.grid_counts(H, P, S)[1]
        for world in (2, 4, 8):
            for k0, k1 in gd.row_partition(Ry, world):
                if k1 <= k0:
                    continue
                y0, y1 = gd.slab_bounds(H, P, S, r, k0, k1)
                for k in range(k0, k1):
                    ry = gd.ref_row_y(k, H, P, S)
                    lo, hi = max(0, ry - r), min(H - P, ry + r) + P
                    assert y0 <= lo and hi <= y1
    # at 8 GPUs the c3 slabs are at most ~300 rows
    Ry = gd.grid_counts(2048, 8, 3)[1]
    assert max(np.diff(gd.slab_bounds(2048, 8, 3, 19, a, b))[0]
               for a, b in gd.row_partition(Ry, 8)) <= 300


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Ry, Rx, K = 23, 5, 4
        ranges = gd.row_partition(Ry, world)
        a, b = ranges[rank]
        # a fake table whose values encode the global row: what rank 0 must reassemble
        idx = (torch.arange(a, b).view(-1, 1, 1) * 1000 + torch.arange(Rx * K).view(1, Rx, K)).int()
        dst = -idx
        nv = torch.arange(a, b).view(-1, 1).expand(-1, Rx).contiguous().int()
        full = None
        if rank == 0:
            full = (torch.zeros((Ry, Rx, K), dtype=torch.int32),
                    torch.zeros((Ry, Rx, K), dtype=torch.int32),
                    torch.zeros((Ry, Rx), dtype=torch.int32))
        gd.gather_rows((idx, dst, nv), full, ranges, rank, world)
        if rank == 0:
            exp = (torch.arange(Ry).view(-1, 1, 1) * 1000 + torch.arange(Rx * K).view(1, Rx, K)).int()
            ok = (torch.equal(full[0], exp) and torch.equal(full[1], -exp)
                  and torch.equal(full[2], torch.arange(Ry).view(-1, 1).expand(-1, Rx).int()))
            q.put(ok)
    finally:
        dist.destroy_process_group()


def _expected(Ry, Rx, K):
    idx = (torch.arange(Ry).view(-1, 1, 1) * 1000 + torch.arange(Rx * K).view(1, Rx, K)).int()
    return idx, -idx, torch.arange(Ry).view(-1, 1).expand(-1, Rx).contiguous().int()


def _worker_chunked(rank, world, port, q, Ry, nchunk):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Rx, K = 5, 4
        ranges = gd.row_partition(Ry, world, 16)
        a, b = ranges[rank]
        parts = (torch.full((b - a, Rx, K), -9, dtype=torch.int32),
                 torch.full((b - a, Rx, K), -9, dtype=torch.int32),
                 torch.full((b - a, Rx), -9, dtype=torch.int32))
        full = None
        if rank == 0:
            full = (torch.zeros((Ry, Rx, K), dtype=torch.int32),
                    torch.zeros((Ry, Rx, K), dtype=torch.int32),
                    torch.zeros((Ry, Rx), dtype=torch.int32))
        calls = []

        def compute(r0, r1, outs):  # stands in for gbm3d_block_match_rows on rows [r0, r1)
            calls.append((r0, r1))
            exp = _expected(Ry, Rx, K)
            for o, e in zip(outs, exp):
                o.copy_(e[r0:r1])

        gd.gather_rows_chunked(compute, parts, full, ranges, rank, world, nchunk)
        ok = calls == gd.chunk_rows(a, b, nchunk)
        if rank == 0:
            ok = ok and all(torch.equal(f, e) for f, e in zip(full, _expected(Ry, Rx, K)))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    return q


@pytest.mark.parametrize("world", [2, 3])
def test_gather_rows_gloo(world):
    q = _spawn(_worker, world)
    assert q.get(timeout=10) is True


@pytest.mark.parametrize("world,Ry,nchunk", [(2, 83, 3), (3, 681, 3), (3, 40, 4), (2, 9, 2)])
def test_gather_rows_chunked_gloo(world, Ry, nchunk):
    """Each rank computes its tile-aligned rows in chunks; rank 0 ends with the whole table
    (its own rows written in place, the others' chunks received as they finish)."""
    q = _spawn(_worker_chunked, world, Ry, nchunk)
    res = dict(q.get(timeout=10) for _ in range(world))
    assert all(res[r] for r in range(world)), res
