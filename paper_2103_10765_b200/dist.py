"""Multi-GPU partitioning of the block-matching stage.

One process per GPU (torchrun), torch.distributed for the plumbing:

* row sharding (one large image, c3): the reference grid rows are split into contiguous blocks
  (sizes differ by <= 1).  Rank g copies only the image rows its references read -- a slab with
  a (radius)-row halo above and (radius + patch)-row halo below, the overlapping-support
  decomposition the paper uses for large images -- computes its rows with
  ``gbm3d_block_match_rows`` (global raster indices), and the tables are gathered to rank 0 with
  point-to-point NCCL transfers straight into the final [Ry, Rx, K] buffers.  The only exchange
  step of the path is that gather.
* batch split (many images, c4): images are split across ranks; no collective.

Concatenating row ranges is byte-identical to one call (reading R16), so the gathered
table equals the single-GPU table bit for bit.  The partition helpers are pure functions and
the gather works on any backend (gloo on CPU in tests, NCCL over NVLink on the box).
"""
from __future__ import annotations

import os
import statistics
import time
from typing import List, Sequence, Tuple

import torch
import torch.distributed as dist


def grid_counts(L: int, P: int, S: int) -> Tuple[int, int]:
    """(regular count, full count) of reference positions along one axis (reading R3)."""
    reg = (L - P) // S + 1
    return reg, reg + (1 if (L - P) % S else 0)


def ref_row_y(k: int, H: int, P: int, S: int) -> int:
    reg, _ = grid_counts(H, P, S)
    return k * S if k < reg else H - P


def row_partition(Ry: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous reference-row blocks, sizes differing by at most one."""
    base, extra = divmod(Ry, world)
    out, a = [], 0
    for g in range(world):
        b = a + base + (1 if g < extra else 0)
        out.append((a, b))
        a = b
    return out


def slab_bounds(H: int, P: int, S: int, r: int, k0: int, k1: int) -> Tuple[int, int]:
    """Image rows [y0, y1) read by reference rows [k0, k1): the references' own rows plus a
    radius-row halo on each side (the window is clamped to the image, reading R2)."""
    if k1 <= k0:
        return 0, 0
    y_first = ref_row_y(k0, H, P, S)
    y_last = ref_row_y(k1 - 1, H, P, S)
    return max(0, y_first - r), min(H, y_last + r + P)


def batch_partition(B: int, world: int) -> List[Tuple[int, int]]:
    return row_partition(B, world)


def gather_rows(parts: Sequence[torch.Tensor], full: torch.Tensor | None, ranges, rank: int,
                world: int, dst: int = 0):
    """Gather row blocks of one or more tables to ``dst``.  ``parts`` are this rank's local
    tables (first dim = its reference rows); on ``dst``, ``full`` is a list of full tables that
    receive every block in place.  Point-to-point ops, batched; works with gloo and NCCL."""
    ops = []
    if rank == dst:
        for t, f in zip(parts, full):
            a, b = ranges[dst]
            f[a:b].copy_(t)
        for g in range(world):
            if g == dst:
                continue
            a, b = ranges[g]
            for f in full:
                if b > a:
                    ops.append(dist.P2POp(dist.irecv, f[a:b], g))
    else:
        a, b = ranges[rank]
        if b > a:
            for t in parts:
                ops.append(dist.P2POp(dist.isend, t.contiguous(), dst))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def block_match_rowsharded(img_rows: torch.Tensor, slab_y0: int, H: int, W: int, patch: int,
                           stride: int, radius: int, K: int, tau, rank: int, world: int,
                           gather: bool = True):
    """Row-sharded matching of one H x W image.  ``img_rows`` holds image rows
    [slab_y0, slab_y0 + rows) and must contain this rank's slab.  Returns the full tables on
    rank 0 (None elsewhere) when ``gather``, else this rank's block and its row range."""
    import paper_2103_10765_b200 as g
    Ry, Rx = g.grid_dims(H, W, patch, stride)
    ranges = row_partition(Ry, world)
    k0, k1 = ranges[rank]
    y0, y1 = slab_bounds(H, patch, stride, radius, k0, k1)
    slab = img_rows[y0 - slab_y0:y1 - slab_y0].contiguous()
    local = g.block_match_rows(slab, y0, H, W, patch, stride, radius, K, tau, k0, k1)
    if not gather:
        return local, (k0, k1)
    full = None
    if rank == 0:
        full = (torch.empty((Ry, Rx, K), dtype=torch.int32, device=local[0].device),
                torch.empty((Ry, Rx, K), dtype=torch.int32, device=local[0].device),
                torch.empty((Ry, Rx), dtype=torch.int32, device=local[0].device))
    gather_rows(local, full, ranges, rank, world)
    return full


# ------------------------------------------------------------------------------ bench (N > 1)
def _init():
    if not dist.is_initialized():
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend)
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    return rank, world, local


def _e2e_bytes(cfg, call, Ry, Rx, world):
    """Bytes per step over all ranks: the slabs (with their halo rows) or images in, the tables
    out (idx, dist int32 [.., K] and n_valid int32)."""
    if cfg.B == 1:
        ranges = row_partition(Ry, world)
        rows_in = 0
        for k0, k1 in ranges:
            y0, y1 = slab_bounds(cfg.H, call.patch, call.stride, call.radius, k0, k1)
            rows_in += y1 - y0
        h2d = rows_in * cfg.W * 2
    else:
        h2d = cfg.B * cfg.H * cfg.W * 2
    d2h = cfg.B * Ry * Rx * (2 * call.K + 1) * 4
    return {"h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}


def _e2e_multi(args, cfg, call, g, dev, rank, world, sharded):
    """Per-step wall time (ms, max over ranks) of host input -> match -> host tables."""
    from synth import config_images
    Ry, Rx = g.grid_dims(cfg.H, cfg.W, call.patch, call.stride)
    if sharded:
        img = torch.from_numpy(config_images(cfg)[0])
        k0, k1 = row_partition(Ry, world)[rank]
        y0, y1 = slab_bounds(cfg.H, call.patch, call.stride, call.radius, k0, k1)
        h_in = img[y0:y1].contiguous().pin_memory()
        n_img, rows = 1, k1 - k0
    else:
        b0, b1 = batch_partition(cfg.B, world)[rank]
        h_in = torch.from_numpy(config_images(cfg)[b0:b1]).pin_memory()
        n_img, rows = b1 - b0, Ry
    shape = (n_img, rows, Rx) if not sharded else (rows, Rx)
    h_out = (torch.empty(shape + (call.K,), dtype=torch.int32, pin_memory=True),
             torch.empty(shape + (call.K,), dtype=torch.int32, pin_memory=True),
             torch.empty(shape, dtype=torch.int32, pin_memory=True))
    d_out = tuple(torch.empty_like(t, device=dev) for t in h_out)
    ws = None
    if not sharded:
        ws = torch.empty(g.host_workspace_bytes(n_img, cfg.H, cfg.W, call.patch, call.stride,
                                                call.K), dtype=torch.uint8, device=dev)

    d_in = torch.empty(h_in.shape, dtype=h_in.dtype, device=dev)
    copy_stream = torch.cuda.Stream(device=dev)
    # row chunks of the rank's range (multiples of 16 rows): the copy of chunk c's tables
    # overlaps the matching of chunk c + 1
    nck = max(1, min(6, rows // 32))
    stepr = ((rows + nck - 1) // nck + 15) // 16 * 16
    chunks = [(a, min(rows, a + stepr)) for a in range(0, rows, stepr)]

    def step():
        if sharded:
            comp = torch.cuda.current_stream(dev)
            with torch.cuda.stream(copy_stream):
                d_in.copy_(h_in, non_blocking=True)
            comp.wait_stream(copy_stream)
            for a, b in chunks:
                dv = tuple(t[a:b] for t in d_out)
                g.block_match_rows(d_in, y0, cfg.H, cfg.W, call.patch, call.stride, call.radius,
                                   call.K, call.tau, k0 + a, k0 + b, out=dv)
                copy_stream.wait_stream(comp)
                with torch.cuda.stream(copy_stream):
                    for h, d in zip(h_out, dv):
                        h[a:b].copy_(d, non_blocking=True)
            copy_stream.synchronize()
        else:
            # the pipelined host-buffer entry (copies overlapped with the matching)
            g.block_match_host(h_in, call.patch, call.stride, call.radius, call.K, call.tau,
                               workspace=ws, out=h_out)

    for _ in range(max(1, args.warmup)):
        step()
    dist.barrier()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        ts.append(time.perf_counter() - t0)
    t = torch.tensor([1e3 * sum(ts) / len(ts)], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def bench_multi(args, cfg, call, sampler=None):
    """N-GPU measurement: c3 row-sharded + NCCL gather to rank 0 (timed), c4 batch split
    (no collective).  Max over ranks of the per-rank device time.  `sampler` (optional, with
    start() / stop() / summary()) samples this rank's GPU clocks around the timed region; rank
    0 reports the lowest median clock and the union of throttle reasons over the ranks.  The
    end-to-end leg times, per step and on every rank, the pinned-host copy of the rank's input
    (slab or images), the match and the copy of the rank's tables back to pinned host memory
    (wall clock, max over ranks)."""
    import paper_2103_10765_b200 as g
    from synth import config_images

    rank, world, local = _init()
    dev = torch.device("cuda", local)
    sharded = cfg.B == 1
    flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)
    Ry, Rx = g.grid_dims(cfg.H, cfg.W, call.patch, call.stride)
    if sharded:
        img = torch.from_numpy(config_images(cfg)[0])
        ranges = row_partition(Ry, world)
        k0, k1 = ranges[rank]
        y0, y1 = slab_bounds(cfg.H, call.patch, call.stride, call.radius, k0, k1)
        slab = img[y0:y1].contiguous().to(dev)
        local_out = (torch.empty((k1 - k0, Rx, call.K), dtype=torch.int32, device=dev),
                     torch.empty((k1 - k0, Rx, call.K), dtype=torch.int32, device=dev),
                     torch.empty((k1 - k0, Rx), dtype=torch.int32, device=dev))
        full = None
        if rank == 0:
            full = (torch.empty((Ry, Rx, call.K), dtype=torch.int32, device=dev),
                    torch.empty((Ry, Rx, call.K), dtype=torch.int32, device=dev),
                    torch.empty((Ry, Rx), dtype=torch.int32, device=dev))

        def step():
            g.block_match_rows(slab, y0, cfg.H, cfg.W, call.patch, call.stride, call.radius,
                               call.K, call.tau, k0, k1, out=local_out)
            gather_rows(local_out, full, ranges, rank, world)
        my_refs = (k1 - k0) * Rx
    else:
        ranges = batch_partition(cfg.B, world)
        b0, b1 = ranges[rank]
        imgs = torch.from_numpy(config_images(cfg)[b0:b1]).to(dev)
        outs = (torch.empty((b1 - b0, Ry, Rx, call.K), dtype=torch.int32, device=dev),
                torch.empty((b1 - b0, Ry, Rx, call.K), dtype=torch.int32, device=dev),
                torch.empty((b1 - b0, Ry, Rx), dtype=torch.int32, device=dev))

        def step():
            g.block_match(imgs, call.patch, call.stride, call.radius, call.K, call.tau,
                          check=False, out=outs)
        my_refs = (b1 - b0) * Ry * Rx

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    if sampler is not None:
        sampler.start()
        t_end = time.time() + 1.0  # clock soak inside the sampled window
        while time.time() < t_end:
            step()
            torch.cuda.synchronize()
        dist.barrier()
    stream = torch.cuda.current_stream()
    times = []
    for _ in range(args.steps):
        flush.zero_()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record(stream)
        step()
        e.record(stream)
        times.append((s, e))
    torch.cuda.synchronize()
    dist.barrier()
    clocks = None
    if sampler is not None:
        sampler.stop()
        clocks = sampler.summary()
    ms = torch.tensor([sum(s.elapsed_time(e) for s, e in times) / args.steps], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    launches = g.last_launch_count()
    e2e_ms = _e2e_multi(args, cfg, call, g, dev, rank, world, sharded)
    all_clocks = [None] * world
    dist.all_gather_object(all_clocks, clocks)
    total_refs = Ry * Rx * cfg.B
    line = None
    if rank == 0:
        t = float(ms.item())
        line = {"metric": "ref patches matched/sec", "value": total_refs / (t * 1e-3),
                "unit": "refs/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": t, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f16+i32", "data": "synthetic",
                "config": {"workload": f"{cfg.name}: {cfg.note}", "H": cfg.H, "W": cfg.W,
                           "B": cfg.B, "patch": call.patch, "stride": call.stride,
                           "radius": call.radius, "K": call.K, "tau": call.tau,
                           "parallelism": ("rows+nccl-gather" if sharded else "batch") +
                           f"x{world}", "l2": "256 MiB write between timed steps"},
                "gpu_launches": launches * args.steps,
                "rank0_refs": my_refs}
        if e2e_ms is not None:
            line["e2e"] = {"value": total_refs / (e2e_ms * 1e-3), "unit": "refs/s",
                           "ms_per_step": e2e_ms, **_e2e_bytes(cfg, call, Ry, Rx, world),
                           "note": "per rank: pinned H2D of its input, match, D2H of its "
                                   "tables; wall clock, max over ranks"}
        cl = [c for c in all_clocks if c]
        if cl:
            mhz = [c["sm_mhz"] for c in cl if c.get("sm_mhz")]
            line["clocks"] = {"sm_mhz": min(mhz) if mhz else None,
                              "sm_max_mhz": max((c.get("sm_max_mhz") or 0) for c in cl) or None,
                              "reasons": sorted({r for c in cl for r in c.get("reasons", [])}),
                              "per_rank_sm_mhz": [c.get("sm_mhz") for c in all_clocks if c]}
    dist.destroy_process_group()
    return line
