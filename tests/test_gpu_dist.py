"""The row-sharded pipeline's CUDA path on one GPU (-m gpu): a 1-rank NCCL group runs
dist.gather_rows_chunked with its two compute streams + comm stream (tile chunks matched with
gbm3d_block_match_rows into the full tables) and must equal one whole-image call bit for bit.
(Multi-rank transfers are covered by the gloo tests in test_dist.py; this pool has one GPU.)"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_chunked_sharded_pipeline_single_rank():
    import torch.distributed as dist

    import paper_2103_10765_b200 as g
    from paper_2103_10765_b200 import dist as gd
    from synth import CONFIGS, config_images
    cfg = CONFIGS["c3"]
    call = cfg.calls[0]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        dev = torch.device("cuda", 0)
        img = torch.from_numpy(config_images(cfg)[0]).to(dev)
        Ry, Rx = g.grid_dims(cfg.H, cfg.W, call.patch, call.stride)
        ranges = gd.row_partition(Ry, 1, gd.TILE_ROWS)
        full = (torch.full((Ry, Rx, call.K), -7, dtype=torch.int32, device=dev),
                torch.full((Ry, Rx, call.K), -7, dtype=torch.int32, device=dev),
                torch.full((Ry, Rx), -7, dtype=torch.int32, device=dev))
        streams = tuple(torch.cuda.Stream(device=dev) for _ in range(3))
        gd._sharded_step(g, cfg, call, img, 0, ranges, 0, 1, None, full, streams, nchunk=5)
        torch.cuda.synchronize()
        ref = g.block_match(img, call.patch, call.stride, call.radius, call.K, call.tau)
        torch.cuda.synchronize()
        for a, b in zip(full, ref):
            assert torch.equal(a, b)
    finally:
        dist.destroy_process_group()


def test_peer_store_tables_single_rank():
    """The fused gather: PeerTables allocates the tables in torch symmetric memory, the matcher
    writes its rows through the views of rank 0's buffer (here the rank itself), and after the
    device barrier the tables equal one whole-image call bit for bit (two steps, the second
    over stale contents)."""
    import torch.distributed as dist

    import paper_2103_10765_b200 as g
    from paper_2103_10765_b200 import dist as gd
    from synth import CONFIGS, config_images
    cfg = CONFIGS["c3"]
    call = cfg.calls[0]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        img = torch.from_numpy(config_images(cfg)[0]).to(dev)
        Ry, Rx = g.grid_dims(cfg.H, cfg.W, call.patch, call.stride)
        ranges = gd.row_partition(Ry, 1, gd.TILE_ROWS)
        peer = gd.PeerTables(Ry, Rx, call.K, dev)
        peer.buf.fill_(-7)
        ref = g.block_match(img, call.patch, call.stride, call.radius, call.K, call.tau)
        for _ in range(2):
            gd._peer_step(g, cfg, call, img, 0, ranges, 0, peer)
            torch.cuda.synchronize()
            for a, b in zip(peer.tables, ref):
                assert torch.equal(a, b)
            peer.buf.fill_(-7)
    finally:
        dist.destroy_process_group()
