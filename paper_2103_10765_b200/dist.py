"""Multi-GPU partitioning of the block-matching stage.

One process per GPU (torchrun), torch.distributed for the plumbing:

* row sharding (one large image, c3): the reference grid rows are split into contiguous blocks
  of whole 16-row tiles of the tensor-core kernel (balanced in tiles; only the last block is
  ragged).  Rank g copies only the image rows its references read -- a slab with a (radius)-row
  halo above and (radius + patch)-row halo below, the overlapping-support decomposition the
  paper uses for large images -- and computes its rows with
  ``gbm3d_block_match_rows`` (global raster indices) in chunks of whole tiles on two alternating
  compute streams.  Each chunk's tables go to rank 0 with point-to-point NCCL transfers on a
  communication stream as soon as the chunk is done, so the gather overlaps the matching of the
  next chunk; rank 0 computes its own rows straight into the final [Ry, Rx, K] buffers and
  receives the others' chunks into them.  The only exchange step of the path is that gather.
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


TILE_ROWS = 16  # reference rows of one tensor-core tile (match_tc16.cuh TY)


def row_partition(Ry: int, world: int, align: int = 1) -> List[Tuple[int, int]]:
    """Contiguous reference-row blocks covering [0, Ry).  ``align`` = 1: sizes differ by at most
    one.  ``align`` > 1 (the matcher's tile height): blocks are whole multiples of ``align`` rows
    (only the last block may be ragged) with tile counts differing by at most one, so no rank
    pays for partial tiles in the middle of the image."""
    if align <= 1:
        base, extra = divmod(Ry, world)
        sizes = [base + (1 if g < extra else 0) for g in range(world)]
    else:
        nt = -(-Ry // align)
        base, extra = divmod(nt, world)
        sizes = [(base + (1 if g < extra else 0)) * align for g in range(world)]
    out, a = [], 0
    for sz in sizes:
        b = min(Ry, a + sz)
        out.append((a, b))
        a = b
    return out


def chunk_rows(k0: int, k1: int, nchunk: int, align: int = TILE_ROWS) -> List[Tuple[int, int]]:
    """Split [k0, k1) into at most ``nchunk`` pieces of whole ``align``-row tiles (the last one
    may be ragged): the granules of the overlapped gather."""
    n = k1 - k0
    if n <= 0:
        return []
    per = -(-n // max(1, nchunk))             # ceil(n / nchunk) rows per chunk
    step = -(-per // align) * align           # rounded up to whole tiles
    return [(a, min(k1, a + step)) for a in range(k0, k1, step)]


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


def gather_rows_chunked(compute, parts, full, ranges, rank: int, world: int, nchunk: int,
                        dst: int = 0, streams=None, host=None):
    """Compute this rank's reference rows chunk by chunk and gather them to ``dst`` while the
    next chunk is being computed.

    ``compute(a, b, outs)`` fills global rows [a, b) of every table into the views ``outs``.
    On ``dst`` the views are slices of the full tables ``full`` (its own rows land in place);
    elsewhere they are slices of the local tables ``parts`` (first dim = the rank's rows), and
    each finished chunk is sent to ``dst``, which receives every other rank's chunks straight
    into ``full``.  Chunks are whole tiles (``chunk_rows``) and deterministic on every rank, so
    the point-to-point ops pair up in order.  With CUDA ``streams`` = (compute0, compute1, comm)
    chunks alternate between the two compute streams (consecutive chunk kernels overlap on the
    SMs) and the transfers run on the comm stream after an event per chunk: the gather overlaps
    the matching (NCCL over NVLink).  Without streams (gloo / CPU) every step is synchronous.
    ``host`` (dst only, with streams): pinned host tables shaped like ``full``; every chunk is
    copied out as soon as it is complete there (own chunks after their kernel, received chunks
    after their transfer), so the copy to the host overlaps the rest of the step."""
    my = ranges[rank]
    mine = chunk_rows(my[0], my[1], nchunk)
    reqs = []

    def views(a, b):
        if rank == dst:
            return tuple(f[a:b] for f in full)
        return tuple(t[a - my[0]:b - my[0]] for t in parts)

    if rank == dst:
        recv_plan = {g: chunk_rows(ranges[g][0], ranges[g][1], nchunk) for g in range(world)
                     if g != dst}
        nmax = max([len(mine)] + [len(v) for v in recv_plan.values()])
    else:
        nmax = len(mine)
    cur = torch.cuda.current_stream() if streams else None
    if streams:
        for st in streams[:2]:
            st.wait_stream(cur)  # the inputs are ready on the caller's stream
    for c in range(nmax):
        ev = None
        if c < len(mine):
            a, b = mine[c]
            outs = views(a, b)
            if streams:
                with torch.cuda.stream(streams[c & 1]):
                    compute(a, b, outs)
                    if host is not None and rank == dst:
                        for h, o in zip(host, outs):
                            h[a:b].copy_(o, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(streams[c & 1])
            else:
                compute(a, b, outs)
        ops = []
        if rank == dst:
            for g, plan in recv_plan.items():
                if c < len(plan):
                    a, b = plan[c]
                    ops += [dist.P2POp(dist.irecv, f[a:b], g) for f in full]
        elif ev is not None or (not streams and c < len(mine)):
            a, b = mine[c]
            ops += [dist.P2POp(dist.isend, v, dst) for v in views(a, b)]
        if ops:
            if streams:
                if ev is not None:
                    streams[2].wait_event(ev)
                with torch.cuda.stream(streams[2]):
                    got = dist.batch_isend_irecv(ops)
                    reqs += got
                    if host is not None and rank == dst:
                        for r in got:
                            r.wait()  # the comm stream now follows the received chunk
                        for g, plan in recv_plan.items():
                            if c < len(plan):
                                a, b = plan[c]
                                for h, f in zip(host, full):
                                    h[a:b].copy_(f[a:b], non_blocking=True)
            else:
                for r in dist.batch_isend_irecv(ops):
                    r.wait()
    if streams:
        with torch.cuda.stream(streams[2]):
            for r in reqs:
                r.wait()
        for st in streams:
            cur.wait_stream(st)


def block_match_rowsharded(img_rows: torch.Tensor, slab_y0: int, H: int, W: int, patch: int,
                           stride: int, radius: int, K: int, tau, rank: int, world: int,
                           gather: bool = True):
    """Row-sharded matching of one H x W image.  ``img_rows`` holds image rows
    [slab_y0, slab_y0 + rows) and must contain this rank's slab.  Returns the full tables on
    rank 0 (None elsewhere) when ``gather``, else this rank's block and its row range."""
    import paper_2103_10765_b200 as g
    Ry, Rx = g.grid_dims(H, W, patch, stride)
    ranges = row_partition(Ry, world, TILE_ROWS)
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


# --------------------------------------------------------------- peer stores (symmetric memory)
class PeerTables:
    """Row-sharded output tables in symmetric memory: the gather fused into the matcher.

    Every rank allocates the same buffer (idx, dist [Ry, Rx, K] and n_valid [Ry, Rx], one int32
    allocation) with torch's symmetric memory and rendezvouses; ``dst_views`` are views of rank
    ``dst``'s buffer mapped into this rank's address space (NVLink peer memory on the box).  Each
    rank's matching kernel is handed those views as its output pointers, so its 16-byte result
    stores travel straight to rank ``dst`` tile by tile while the next tiles are matched -- no
    separate gather, no staging copy.  ``finish`` is the stream-ordered device barrier of the
    symmetric-memory handle: after it, rank ``dst`` sees every rank's rows.  ``tables`` on rank
    ``dst`` are the full tables."""

    def __init__(self, Ry: int, Rx: int, K: int, dev, dst: int = 0, group=None):
        import torch.distributed._symmetric_memory as symm
        grp = group if group is not None else dist.group.WORLD
        n = Ry * Rx * (2 * K + 1)
        self.buf = symm.empty(n, dtype=torch.int32, device=dev)
        try:
            self.hdl = symm.rendezvous(self.buf, grp)
        except RuntimeError:
            symm.enable_symm_mem_for_group(grp.group_name)
            self.hdl = symm.rendezvous(self.buf, grp)
        peer = self.hdl.get_buffer(dst, (n,), torch.int32)
        t = Ry * Rx * K
        self.dst_views = (peer[:t].view(Ry, Rx, K), peer[t:2 * t].view(Ry, Rx, K),
                          peer[2 * t:].view(Ry, Rx))
        self.tables = (self.buf[:t].view(Ry, Rx, K), self.buf[t:2 * t].view(Ry, Rx, K),
                       self.buf[2 * t:].view(Ry, Rx))

    def rows(self, a: int, b: int):
        """Output views of global reference rows [a, b) in rank ``dst``'s tables."""
        return tuple(v[a:b] for v in self.dst_views)

    def finish(self):
        self.hdl.barrier(channel=0)


def _peer_step(g, cfg, call, slab, y0, ranges, rank, peer: PeerTables):
    """One row-sharded step with the gather fused into the matcher: this rank's rows are matched
    straight into rank 0's tables (peer stores), then the device barrier."""
    k0, k1 = ranges[rank]
    if k1 > k0:
        g.block_match_rows(slab, y0, cfg.H, cfg.W, call.patch, call.stride, call.radius, call.K,
                           call.tau, k0, k1, out=peer.rows(k0, k1))
    peer.finish()


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
    out (idx, dist int32 [.., K] and n_valid int32; for c3 the full table, on rank 0)."""
    if cfg.B == 1:
        rows_in = 0
        for k0, k1 in row_partition(Ry, world, TILE_ROWS):
            y0, y1 = slab_bounds(cfg.H, call.patch, call.stride, call.radius, k0, k1)
            rows_in += y1 - y0
        h2d = rows_in * cfg.W * 2
    else:
        h2d = cfg.B * cfg.H * cfg.W * 2
    d2h = cfg.B * Ry * Rx * (2 * call.K + 1) * 4
    return {"h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}


def _sharded_step(g, cfg, call, slab, y0, ranges, rank, world, local_out, full, streams,
                  nchunk=3, host=None):
    """One row-sharded matching step: this rank's rows in tile chunks, each gathered to rank 0
    while the next is matched (gather_rows_chunked); with ``host``, rank 0 also copies every
    completed chunk to those pinned host tables."""
    def compute(a, b, outs):
        g.block_match_rows(slab, y0, cfg.H, cfg.W, call.patch, call.stride, call.radius, call.K,
                           call.tau, a, b, out=outs)
    gather_rows_chunked(compute, local_out, full, ranges, rank, world, nchunk, streams=streams,
                        host=host)


def _e2e_multi(args, cfg, call, g, dev, rank, world, sharded):
    """Per-step wall time (ms, max over ranks) of host input -> match -> host tables.  c3: every
    rank copies its pinned slab in, matches its rows with the chunked gather, and rank 0 copies
    the FULL table back to pinned host memory; c4: every rank runs the pipelined host entry on
    its images (its tables come back to its host)."""
    from synth import config_images
    Ry, Rx = g.grid_dims(cfg.H, cfg.W, call.patch, call.stride)
    if sharded:
        img = torch.from_numpy(config_images(cfg)[0])
        ranges = row_partition(Ry, world, TILE_ROWS)
        k0, k1 = ranges[rank]
        y0, y1 = slab_bounds(cfg.H, call.patch, call.stride, call.radius, k0, k1)
        h_in = img[y0:y1].contiguous().pin_memory()
        d_in = torch.empty(h_in.shape, dtype=h_in.dtype, device=dev)
        local_out = (torch.empty((k1 - k0, Rx, call.K), dtype=torch.int32, device=dev),
                     torch.empty((k1 - k0, Rx, call.K), dtype=torch.int32, device=dev),
                     torch.empty((k1 - k0, Rx), dtype=torch.int32, device=dev))
        full = h_out = None
        if rank == 0:
            full = (torch.empty((Ry, Rx, call.K), dtype=torch.int32, device=dev),
                    torch.empty((Ry, Rx, call.K), dtype=torch.int32, device=dev),
                    torch.empty((Ry, Rx), dtype=torch.int32, device=dev))
            h_out = tuple(torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in full)
        streams = tuple(torch.cuda.Stream(device=dev) for _ in range(3))
    else:
        b0, b1 = batch_partition(cfg.B, world)[rank]
        h_in = torch.from_numpy(config_images(cfg)[b0:b1]).pin_memory()
        n_img = b1 - b0
        shape = (n_img, Ry, Rx)
        h_out = (torch.empty(shape + (call.K,), dtype=torch.int32, pin_memory=True),
                 torch.empty(shape + (call.K,), dtype=torch.int32, pin_memory=True),
                 torch.empty(shape, dtype=torch.int32, pin_memory=True))
        ws = torch.empty(g.host_workspace_bytes(n_img, cfg.H, cfg.W, call.patch, call.stride,
                                                call.K), dtype=torch.uint8, device=dev)

    def step():
        if sharded:
            d_in.copy_(h_in, non_blocking=True)
            _sharded_step(g, cfg, call, d_in, y0, ranges, rank, world, local_out, full, streams,
                          nchunk=6, host=h_out)
            torch.cuda.current_stream(dev).synchronize()
        else:
            # the pipelined host-buffer entry (copies overlapped with the matching)
            g.block_match_host(h_in, call.patch, call.stride, call.radius, call.K, call.tau,
                               workspace=ws, out=h_out, device=dev)

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
    """N-GPU measurement: c3 row-sharded with the tables gathered on rank 0 (timed; by default
    the matcher stores its rows straight into rank 0's symmetric-memory tables, `PeerTables`;
    `--gather nccl` = the chunked NCCL gather), c4 batch split (no collective).  Max over ranks of the per-rank device time.  `sampler` (optional, with
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
        ranges = row_partition(Ry, world, TILE_ROWS)
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
        streams = tuple(torch.cuda.Stream(device=dev) for _ in range(3))
        # the gather: fused into the matcher as peer stores to rank 0's symmetric-memory tables
        # (default), else the chunked NCCL point-to-point gather overlapped with the matching
        peer = None
        gather_mode = getattr(args, "gather", "peer")
        if gather_mode == "peer":
            try:
                peer = PeerTables(Ry, Rx, call.K, dev)
            except Exception as e:  # no symmetric memory on this stack: the NCCL gather
                gather_mode = f"nccl (peer stores unavailable: {type(e).__name__})"

        def step():
            if peer is not None:
                _peer_step(g, cfg, call, slab, y0, ranges, rank, peer)
            else:
                _sharded_step(g, cfg, call, slab, y0, ranges, rank, world, local_out, full,
                              streams)
        my_refs = (k1 - k0) * Rx
    else:
        gather_mode = None
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
                           "parallelism": ("rows+" + ("peer-store-gather" if peer is not None
                                                      else "nccl-gather")
                                           if sharded else "batch") + f"x{world}",
                           "l2": "256 MiB write between timed steps"},
                "table_gather": gather_mode,
                "gpu_launches": launches * args.steps,
                "rank0_refs": my_refs}
        if e2e_ms is not None:
            line["e2e"] = {"value": total_refs / (e2e_ms * 1e-3), "unit": "refs/s",
                           "ms_per_step": e2e_ms, **_e2e_bytes(cfg, call, Ry, Rx, world),
                           "note": ("c3: pinned H2D of every rank's slab, chunked match + "
                                    "gather, D2H of the full table on rank 0" if sharded else
                                    "per rank: the pipelined host entry on its images") +
                                   "; wall clock, max over ranks"}
        cl = [c for c in all_clocks if c]
        if cl:
            mhz = [c["sm_mhz"] for c in cl if c.get("sm_mhz")]
            line["clocks"] = {"sm_mhz": min(mhz) if mhz else None,
                              "sm_max_mhz": max((c.get("sm_max_mhz") or 0) for c in cl) or None,
                              "reasons": sorted({r for c in cl for r in c.get("reasons", [])}),
                              "per_rank_sm_mhz": [c.get("sm_mhz") for c in all_clocks if c]}
    dist.destroy_process_group()
    return line
