#!/usr/bin/env python
"""Bench for the B200 block-matching library (G-BM3D hot path, arXiv 2103.10765).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3|c4] [--impl ours|reference]

One "step" = one pass of the whole hot path (grid, per-displacement SSD box
sums, top-K selection, table write) over the configured synthetic workload.  Default workload:
c3 (2048^2, P8 s3 r19 K32 -- BASELINE.json configs[3]); c4 (64 x 512^2, K16) is measured
beside it at N=1 and reported under "also".  Rank 0 prints ONE JSON line.  For N > 1 run
under torchrun: c3 is row-sharded with halos and the tables gathered to rank 0 over NCCL;
c4 is batch-split (no collective).  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2
N_SMS = 148


def a_eval(stride: int) -> int:
    """Algorithmic int32 ops per candidate evaluation of the SSD form:
    per pixel-displacement 1 ISUB + 1 IMUL + 1 IADD3 (vertical running sum), 1/s IADD3
    (horizontal), 1/s^2 compare -> 3 s^2 + s + 1 per evaluation."""
    return 3 * stride * stride + stride + 1


def total_evals(H, W, P, s, r):
    def axis(L):
        pos = list(range(0, L - P + 1, s))
        if (L - P) % s:
            pos.append(L - P)
        return [min(L - P, p + r) - max(0, p - r) + 1 for p in pos]
    wy, wx = axis(H), axis(W)
    return sum(a * b - 1 for a in wy for b in wx), len(wy) * len(wx)


class ClockSampler:
    """nvidia-smi sampler of SM clocks and throttle reasons (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return self
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        def num(v):
            try:
                return float(v)
            except ValueError:
                return None
        sm = [num(r[0]) for r in self.rows if num(r[0]) is not None]
        mx = [num(r[1]) for r in self.rows if num(r[1]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[4:8]) if v == "Active"})
        top = max(sm) if sm else 0
        load = [v for v in sm if v >= 0.5 * top] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows),
                "power_w_max": max((num(r[2]) or 0.0) for r in self.rows)}


def _events_ms(fn, stream, torch):
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record(stream)
    fn()
    e.record(stream)
    return s, e


def measure_device(step, K, W, flush, torch, dist_barrier=None, soak_s=1.0):
    """W warm-up steps, a clock soak, then exactly K timed steps (per-step CUDA events on the
    launching stream; the L2 flush between steps is outside the events)."""
    stream = torch.cuda.current_stream()
    for _ in range(W):
        step()
    torch.cuda.synchronize()
    t_end = time.time() + soak_s  # clock sampling window before the timed region
    while time.time() < t_end:
        step()
        torch.cuda.synchronize()
    if dist_barrier:
        dist_barrier()
    torch.cuda.synchronize()
    evs = []
    for _ in range(K):
        flush()
        evs.append(_events_ms(step, stream, torch))
    torch.cuda.synchronize()
    if dist_barrier:
        dist_barrier()
    return [s.elapsed_time(e) for s, e in evs]


def oracle_sample_rate(cfg, call, target_s, seed=0, threads=0):
    """Time the oracle (as it stands) on a random sample of the workload's references, sized to
    ~target_s seconds.  Returns (refs/s, evals/s, n_refs, seconds, threads)."""
    import numpy as np

    import oracle
    from synth import make_image
    img = make_image(cfg.H, cfg.W, cfg.n_rect, cfg.n_tex, cfg.sigma, cfg.seeds[0])
    gy = oracle.grid(cfg.H, call.patch, call.stride)
    gx = oracle.grid(cfg.W, call.patch, call.stride)
    rng = np.random.default_rng(seed)

    def run(n):
        py = rng.integers(0, len(gy), n)
        px = rng.integers(0, len(gx), n)
        t0 = time.perf_counter()
        oracle.block_match_refs(img, call.patch, call.stride, call.radius, call.K, call.tau, py,
                                px, threads=threads)
        return time.perf_counter() - t0

    n0 = 2000
    t0 = run(n0)
    n = max(n0, int(n0 * target_s / max(t0, 1e-3)))
    t = run(n)
    evals_total, refs_total = total_evals(cfg.H, cfg.W, call.patch, call.stride, call.radius)
    ev_per_ref = evals_total / refs_total
    return n / t, n * ev_per_ref / t, n, t, threads or oracle.max_threads()


def bench_reference(args, cfg, call, rank):
    """--impl reference: the oracle as it stands on the host cores; each step one bounded
    sample of the workload (~3 s)."""
    if rank != 0:
        return
    import oracle
    threads = oracle.max_threads()
    rates = []
    per = None
    for i in range(args.warmup + args.steps):
        rate, evr, n, t, thr = oracle_sample_rate(cfg, call, 3.0, seed=i)
        if i >= args.warmup:
            rates.append(rate)
            per = (n, t)
    value = statistics.mean(rates)
    line = {
        "impl": "reference", "metric": "ref patches matched/sec", "value": value,
        "unit": "refs/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * per[1], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "i64", "data": "synthetic",
        "config": workload_config(cfg, call, args),
        "cpu_baseline": {"value": value, "unit": "refs/s", "cores": threads, "kind": "oracle",
                         "sample": f"{per[0]} random references of {cfg.name} per step"},
        "e2e": {"value": value, "unit": "refs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(cfg, call, args):
    return {"workload": f"{cfg.name}: {cfg.note}", "H": cfg.H, "W": cfg.W, "B": cfg.B,
            "patch": call.patch, "stride": call.stride, "radius": call.radius, "K": call.K,
            "tau": call.tau, "parallelism": ("rows" if cfg.name == "c3" else "batch") +
            f"x{args.gpus}", "l2": "256 MiB write between timed steps (outside the events)"}


def measured_peak(key, default):
    """Driver-written MEASURED_PEAKS.json (this pool's B200s), else the recipe's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            v = json.load(f).get(key)
            return (float(v), "MEASURED_PEAKS.json") if v else (default, "B200_PROFILING.md")
    except (OSError, ValueError):
        return default, "B200_PROFILING.md"


def build_id(g):
    """Source hash the loaded libgbm3d.so was built from (gbm3d_version: "... src <id>")."""
    v = g.version()
    return v.split("src ")[-1].strip() if "src " in v else None


def load_ncu(name, bid):
    """ncu counters of the step's dominant kernel for workload `name` from the committed capture
    profiles/ncu_counters.json, only if that capture was taken of this very build (same source
    id); the DRAM read + write bytes of that capture are the roofline's `traffic`."""
    path = os.path.join(ROOT, "profiles", "ncu_counters.json")
    try:
        with open(path) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None, {"note": "no profiles/ncu_counters.json"}
    c = d.get(name)
    if c is None:
        return None, {"note": f"no capture for {name}"}
    if d.get("build") != bid:
        return None, {"note": f"capture of build {d.get('build')}, not of this build {bid}",
                      "stale": c}
    out = dict(c)
    out["build"] = bid
    out["source"] = d.get("source", "")
    return c.get("dram_bytes"), out


def measure_int_peaks(g):
    """integer instruction throughput measured in this run (the library's
    microkernels on every SM): lane-instructions per second for the ALU pipe alone, the FMA
    pipe alone, IMNMX, and IMAD + IADD3 mixed (the issue bound)."""
    return {k: g.int_peak(k) / 1e12 for k in ("alu", "fma", "minmax", "mixed")}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def tensor_roofline(evals, patch, ms):
    """Secondary: the Eq. (2) inner products <f_p, f_q> (2 P^2 flops per evaluation) run on
    tcgen05 kind::f16; fp16 dense peak = the measured bf16 burst peak (same rate)."""
    peak, src = measured_peak("bf16_tflops", 2250.0)
    ach = evals * 2 * patch * patch / (ms * 1e-3) / 1e12
    return {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
            "frac": ach / peak, "peak_source": src,
            "note": "algorithmic inner-product flops only; not the binding resource"}


def run_ours_single(args, cfg, call, torch, g, want_e2e=True, want_cpu=True):
    """N = 1 measurement of one workload; returns the JSON dict."""
    from synth import config_images
    dev = torch.device("cuda", 0)
    imgs = torch.from_numpy(config_images(cfg)).to(dev)
    img = imgs if cfg.B > 1 else imgs[0].contiguous()
    assert g.check_range(img, call.patch), "synthetic image outside the int32 domain"
    Ry, Rx = g.grid_dims(cfg.H, cfg.W, call.patch, call.stride)
    shape = ((cfg.B,) if cfg.B > 1 else ()) + (Ry, Rx, call.K)
    outs = (torch.empty(shape, dtype=torch.int32, device=dev),
            torch.empty(shape, dtype=torch.int32, device=dev),
            torch.empty(shape[:-1], dtype=torch.int32, device=dev))
    flush_buf = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)

    def step():
        g.block_match(img, call.patch, call.stride, call.radius, call.K, call.tau, check=False,
                      method=args.method, out=outs)

    step()
    launches_per_step = g.last_launch_count()
    # profiling runs (--step-only) list the step's kernels alone: no microkernels there
    peaks = measure_int_peaks(g) if not args.step_only else {k: float("nan") for k in
                                                             ("alu", "fma", "minmax", "mixed")}
    sampler = ClockSampler(0).start()
    times = measure_device(step, args.steps, args.warmup, flush_buf.zero_, torch)
    sampler.stop()
    clocks = sampler.summary()
    ms = statistics.mean(times)
    evals1, refs1 = total_evals(cfg.H, cfg.W, call.patch, call.stride, call.radius)
    evals, refs = evals1 * cfg.B, refs1 * cfg.B
    value = refs / (ms * 1e-3)
    A = a_eval(call.stride)
    achieved = evals * A / (ms * 1e-3) / 1e12
    peak = peaks["mixed"]
    bid = build_id(g)
    traffic, ncu = load_ncu(cfg.name, bid)
    line = {
        "metric": "ref patches matched/sec", "value": value, "unit": "refs/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f16+i32", "data": "synthetic",
        "config": workload_config(cfg, call, args),
        "gevals_per_s": evals / (ms * 1e-3) / 1e9,
        "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "ops_per_eval": A, "evals_per_launch": evals,
                     "peak_basis": "measured in this run: IMAD + IADD3 microkernel on all SMs "
                                   "(integer issue bound, SURVEY 8(d) P_int = best measured)",
                     "alu_pipe_peak": peaks["alu"], "frac_of_alu_pipe": achieved / peaks["alu"],
                     "model": "SURVEY 8(d) SSD-form work A_eval = 3s^2+s+1 int32 ops per "
                              "candidate evaluation (closed-form count, self excluded); the "
                              "product-form kernel moves the inner products to tcgen05, so this "
                              "is the method's ALU-roofline time bound, not an issue count",
                     "timed": "whole step (persistent tc16 kernel + marked-tile scan)"},
        "int_peaks_tops": peaks,
        "ncu": ncu,
        "build": bid,
        "roofline_tensor": tensor_roofline(evals, call.patch, ms),
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
        "kernel_ms": {"mean": ms, "min": min(times), "max": max(times)},
    }
    if args.step_only:   # profiling runs: the timed step's kernels alone
        return line
    line["gather"] = run_gather(args, cfg, call, torch, g, img, outs[0], flush_buf)
    line["wiener"] = run_wiener(args, cfg, call, torch, g, img, outs, flush_buf)
    line["stage1"] = run_stage1(args, cfg, call, torch, g, img, flush_buf)
    line["denoiser"] = run_denoiser(args, cfg, torch, img, flush_buf)
    if want_cpu:
        line["small_configs"] = run_small_configs(torch, g)
    if want_e2e:
        line["e2e"] = run_e2e(args, cfg, call, torch, g)
    if want_cpu:
        rate, evr, n, t, thr = oracle_sample_rate(cfg, call, args.cpu_seconds)
        rate1, evr1, n1, t1, _ = oracle_sample_rate(cfg, call, args.cpu_seconds / 2, seed=1,
                                                    threads=1)
        line["cpu_baseline"] = {"value": rate, "unit": "refs/s", "cores": thr, "kind": "oracle",
                                "sample": f"{n} random references of {cfg.name} "
                                          f"({n * evals1 / refs1:.3g} evals) in {t:.1f} s",
                                "gevals_per_s": evr / 1e9, "cpu_model": cpu_model(),
                                "single_thread": {"value": rate1, "unit": "refs/s",
                                                  "gevals_per_s": evr1 / 1e9,
                                                  "sample": f"{n1} random references in "
                                                            f"{t1:.1f} s, 1 thread"}}
    del imgs, outs, flush_buf
    return line


def run_gather(args, cfg, call, torch, g, img, idx, flush_buf):
    """the matched-block groups (5D tensor of PAPER.md:217) from this step's table,
    timed like the step (events, L2 flushed between launches).  HBM-write bound: roofline
    bytes = groups written + table read + image read, against MEASURED_PEAKS hbm_gbs."""
    grp = torch.empty(tuple(idx.shape) + (call.patch, call.patch), dtype=torch.int16,
                      device=idx.device)

    def step():
        g.gather_groups(img, idx, call.patch, out=grp)

    times = measure_device(step, args.steps, args.warmup, flush_buf.zero_, torch, soak_s=0.2)
    ms = statistics.mean(times)
    nbytes = grp.numel() * 2 + idx.numel() * 4 + img.numel() * 2
    peak, src = measured_peak("hbm_gbs", 7672.0)
    ach = nbytes / (ms * 1e-3) / 1e9
    del grp
    return {"what": "gbm3d_gather_groups: [.., K, P, P] int16 blocks of the step's table",
            "ms": ms, "blocks_per_s": idx.numel() / (ms * 1e-3),
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                         "frac": ach / peak, "bytes_per_launch": nbytes, "peak_source": src}}


FP32_FMA_LANES_PER_SM = 128  # FFMA with an immediate operand: 32 lanes/clk/SMSP (the
                             # 3-register form issues at half that rate; B300_MICROARCH)


def run_wiener(args, cfg, call, torch, g, img, outs, flush_buf):
    """stage-2 collaborative Wiener filtering + aggregation of every group, the
    noise-free synthetic image standing in for the basic estimate (DESIGN.md W-readings) and the
    groups matched on it (the step's configuration).  Roofline: fp32 FMA pipe; algorithmic
    flops per block = three separable 8x8 DCTs
    (2 x 512 FMA each) + three Haar cascades (64 x log2 K butterflies of 2 flops) + shrinkage."""
    from synth import make_image
    if call.patch != 8 or call.K & (call.K - 1):
        return None
    B = cfg.B
    seeds = list(cfg.seeds)[:B]
    clean = [make_image(cfg.H, cfg.W, cfg.n_rect, cfg.n_tex, cfg.sigma, sd, return_clean=True)
             for sd in seeds]
    basic = torch.from_numpy(np.stack([c[1] for c in clean]).astype(np.float32)).to(img.device)
    sig = [c[2] for c in clean]
    # stage 2 groups the blocks by matching on the basic estimate: the
    # step's tables come from the noisy image, so match once more on the stand-in (untimed)
    est = torch.from_numpy(np.stack([c[1] for c in clean]).astype(np.int16)).to(img.device)
    if B == 1:
        basic = basic[0].contiguous()
        est = est[0].contiguous()
    outs = g.block_match(est, call.patch, call.stride, call.radius, call.K, call.tau, check=False)
    out = torch.empty(basic.shape, dtype=torch.float32, device=img.device)
    ws = torch.empty(g.load_library().gbm3d_wiener_workspace_bytes(B, cfg.H, cfg.W),
                     dtype=torch.uint8, device=img.device)
    idx, _, nv = outs

    def step():
        g.wiener_stage2(img, basic, idx, nv, call.patch, sig, out=out, workspace=ws)

    times = measure_device(step, args.steps, args.warmup, flush_buf.zero_, torch, soak_s=0.2)
    ms = statistics.mean(times)
    blocks = idx.numel()
    lg = int(math.log2(call.K))
    # per block: three 2D DCTs as 16 even/odd 8-point transforms (8 adds + 32 FMA = 72 flops),
    # three Haar cascades (64 coefficients x log2 K levels x 2 flops, counted for every lane),
    # shrinkage and product (64 x 6), weighted numerator (64 x 2)
    flops_blk = 3 * 16 * 72 + 3 * 64 * lg * 2 + 64 * 6 + 64 * 2
    ach = blocks * flops_blk / (ms * 1e-3) / 1e12
    sm_max = 1965.0
    peak = FP32_FMA_LANES_PER_SM * 2 * N_SMS * sm_max * 1e6 / 1e12
    del basic, out, ws
    return {"what": "gbm3d_wiener_stage2: DCT2 x Haar Wiener shrinkage of every group + weighted "
                    "aggregation (basic estimate = the noise-free synthetic image)",
            "ms": ms, "groups_per_s": idx[..., 0].numel() / (ms * 1e-3),
            "roofline": {"bound": "fp32", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                         "frac": ach / peak, "flops_per_block": flops_blk,
                         "peak_basis": "128 FFMA lanes/clk/SM (immediate-operand form; the "
                                       "3-register form issues at half rate) x 2 x 148 SMs x "
                                       "1965 MHz"}}


def run_stage1(args, cfg, call, torch, g, img, flush_buf):
    """stage-1 global volume hard thresholding of the workload's image(s) with
    tiling references (stride = patch = 8, K = 16, the paper's K), matching included in the
    tables but not in the timing.  HBM roofline on ALGORITHMIC bytes: the call's inputs (image,
    tables) and output (fp32 image), read / written once.  The method's volume of matched blocks
    (K x H x W) does not fit on chip, so the implementation's own traffic is far larger
    (`impl_traffic_model`: ~14.5 fp32 volume passes); both are reported."""
    N, K, levels = 8, 16, 3
    if cfg.H % 16 or cfg.W % 16:
        return None
    idx, dist, nv = g.block_match(img, N, N, call.radius, K, None, check=False)
    sig = list(cfg_sigmas(cfg))
    out = torch.empty(img.shape, dtype=torch.float32, device=img.device)
    ws = torch.empty(g.load_library().gbm3d_stage1_workspace_bytes(cfg.B, cfg.H, cfg.W, N, K),
                     dtype=torch.uint8, device=img.device)

    def step():
        g.stage1_denoise(img, idx, nv, N, sig, levels, out=out, workspace=ws)

    times = measure_device(step, args.steps, args.warmup, flush_buf.zero_, torch, soak_s=0.2)
    ms = statistics.mean(times)
    vol = cfg.B * K * cfg.H * cfg.W * 4
    # per spin (fused 2D passes): level-1 analysis writes the 4 subbands (1 vol; the volume is
    # gathered from the image), levels l >= 2 read + write the band (2 vol / 4^(l-1)), the z
    # pass reads + writes (2), synthesis mirrors the analysis with level 1 reading the
    # coefficients and storing U (spin 0: 2) or adding into it (spin 1: 3); then TV + the
    # aggregation read U once (1)
    band = sum(2 / 4 ** (l - 1) for l in range(2, levels + 1))
    passes = (1 + band + 2 + band + 2) + (1 + band + 2 + band + 3) + 1
    impl_bytes = passes * vol
    nbytes = img.numel() * 2 + idx.numel() * 4 + nv.numel() * 4 + out.numel() * 4
    peak, src = measured_peak("hbm_gbs", 7672.0)
    ach = nbytes / (ms * 1e-3) / 1e9
    del out, ws
    return {"what": "gbm3d_stage1_denoise: bior1.5 x Haar global volume hard thresholding, 2 cycle "
                    "spins, 1/TV weights, aggregation (tiling refs N=8, K=16)",
            "ms": ms, "pixels_per_s": cfg.B * cfg.H * cfg.W / (ms * 1e-3),
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                         "frac": ach / peak, "bytes_per_call": nbytes, "peak_source": src,
                         "basis": "algorithmic bytes: image + tables in, fp32 image out"},
            "impl_traffic_model": {"bytes_per_call": impl_bytes,
                                   "gbs": impl_bytes / (ms * 1e-3) / 1e9,
                                   "frac_of_hbm": impl_bytes / (ms * 1e-3) / 1e9 / peak,
                                   "note": "~14.5 fp32 volume passes of the fused schedule "
                                           "(DESIGN.md 7.7)"}}


def run_denoiser(args, cfg, torch, img, flush_buf):
    """The whole two-stage G-BM3D (paper_2103_10765_b200.denoise: stage 1 with 3 translation
    trials of tiling matching + global volume thresholding, stage 2 matching on the basic
    estimate + Wiener filtering) on the workload's image, single images only.  Context: the
    paper's Table II times G-BM3D2 on a 2048^2 image at 20.58 s (MATLAB, Titan Xp)."""
    from paper_2103_10765_b200.denoise import denoise
    from synth import make_image
    if cfg.B != 1 or cfg.H % 16 or cfg.W % 16:
        return None
    _, clean, sig = make_image(cfg.H, cfg.W, cfg.n_rect, cfg.n_tex, cfg.sigma, cfg.seeds[0],
                               return_clean=True)
    out = {}

    def step():
        out["y"] = denoise(img, sig)

    times = measure_device(step, max(3, args.steps // 4), args.warmup, flush_buf.zero_, torch,
                           soak_s=0.2)
    ms = statistics.mean(times)
    y = out["y"].double().cpu().numpy()
    noisy = img.double().cpu().numpy()
    psnr = lambda a: float(10 * np.log10(255.0 ** 2 / np.mean((a - clean) ** 2)))
    return {"what": "denoise(): G-BM3D2 = stage 1 (3 trials: P16 s16 K16 r16 matching + global "
                    "volume thresholding) + stage 2 (P8 s3 K32 r16 matching on the basic "
                    "estimate + Wiener), synthetic image",
            "ms": ms, "psnr_noisy_db": psnr(noisy), "psnr_out_db": psnr(y),
            "paper_context": {"G-BM3D2_2048_s": 20.58, "source": "P:324 Table II, MATLAB on a "
                              "Titan Xp, other images; context only"}}


def run_small_configs(torch, g):
    """the latency of the small configs c0-c2 (parity cases) at 1 GPU: device
    time per call (CUDA events around 50 back-to-back calls, after warm-up), and the same call
    replayed from a captured CUDA graph (launch overhead removed)."""
    from synth import CONFIGS, config_images
    res = {}
    for name in ("c0", "c1", "c2"):
        cfg = CONFIGS[name]
        img = torch.from_numpy(config_images(cfg)[0]).cuda()
        for ci, call in enumerate(cfg.calls):
            Ry, Rx = g.grid_dims(cfg.H, cfg.W, call.patch, call.stride)
            outs = (torch.empty((Ry, Rx, call.K), dtype=torch.int32, device="cuda"),
                    torch.empty((Ry, Rx, call.K), dtype=torch.int32, device="cuda"),
                    torch.empty((Ry, Rx), dtype=torch.int32, device="cuda"))

            def step():
                g.block_match(img, call.patch, call.stride, call.radius, call.K, call.tau,
                              check=False, out=outs)

            for _ in range(10):
                step()
            torch.cuda.synchronize()
            reps = 50
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(reps):
                step()
            e.record()
            torch.cuda.synchronize()
            us = 1e3 * s.elapsed_time(e) / reps
            launches = g.last_launch_count()
            graph_us = None
            try:
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr):
                    step()
                for _ in range(5):
                    gr.replay()
                torch.cuda.synchronize()
                s.record()
                for _ in range(reps):
                    gr.replay()
                e.record()
                torch.cuda.synchronize()
                graph_us = 1e3 * s.elapsed_time(e) / reps
            except Exception as exc:  # capture unsupported: report it, keep the eager number
                graph_us = f"capture failed: {type(exc).__name__}"
            res[f"{name}.call{ci}"] = {"us_per_call": us, "graph_us_per_call": graph_us,
                                       "refs": Ry * Rx, "refs_per_s": Ry * Rx / (us * 1e-6),
                                       "launches": launches, "P": call.patch, "s": call.stride,
                                       "K": call.K, "tau": call.tau}
    return res


def cfg_sigmas(cfg):
    from synth import make_image
    if cfg.sigma is not None:
        return [cfg.sigma] * cfg.B
    # per-image sigma of the recipe (drawn by the generator)
    return [make_image(cfg.H, cfg.W, cfg.n_rect, cfg.n_tex, None, s, return_clean=True)[2]
            for s in list(cfg.seeds)[:cfg.B]]


def run_e2e(args, cfg, call, torch, g):
    """Same metric through the host-buffer C-ABI entry: pinned H2D of the images, the match,
    D2H of idx/dist/n_valid, all inside each timed step."""
    from synth import config_images
    h = torch.from_numpy(config_images(cfg)).pin_memory()
    Ry, Rx = g.grid_dims(cfg.H, cfg.W, call.patch, call.stride)
    B = cfg.B
    ws = torch.empty(g.host_workspace_bytes(B, cfg.H, cfg.W, call.patch, call.stride, call.K),
                     dtype=torch.uint8, device="cuda")
    out = (torch.empty((B, Ry, Rx, call.K), dtype=torch.int32, pin_memory=True),
           torch.empty((B, Ry, Rx, call.K), dtype=torch.int32, pin_memory=True),
           torch.empty((B, Ry, Rx), dtype=torch.int32, pin_memory=True))

    def step():
        g.block_match_host(h, call.patch, call.stride, call.radius, call.K, call.tau,
                           workspace=ws, out=out)

    for _ in range(max(1, args.warmup)):
        step()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        ts.append(time.perf_counter() - t0)
    t = statistics.mean(ts)
    _, refs1 = total_evals(cfg.H, cfg.W, call.patch, call.stride, call.radius)
    return {"value": refs1 * B / t, "unit": "refs/s", "ms_per_step": 1e3 * t,
            "h2d_bytes_per_step": int(h.numel() * 2),
            "d2h_bytes_per_step": int(sum(o.numel() * 4 for o in out))}


def add_multi_roofline(line, cfg, call, g):
    """The N-GPU line's ALU roofline, per GPU: the closed-form evaluations over all ranks / N
    against rank 0's measured integer issue peak, at the max-over-ranks step time (which
    includes the c3 gather)."""
    n = line["n_gpus"]
    ms = line["ms_per_step"]
    evals1, _ = total_evals(cfg.H, cfg.W, call.patch, call.stride, call.radius)
    evals = evals1 * cfg.B
    A = a_eval(call.stride)
    peaks = measure_int_peaks(g)
    peak = peaks["mixed"]
    achieved = evals / n * A / (ms * 1e-3) / 1e12
    line["gevals_per_s"] = evals / (ms * 1e-3) / 1e9
    line["int_peaks_tops"] = peaks
    line["roofline"] = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TOP/s",
                        "frac": achieved / peak, "traffic": None, "ops_per_eval": A,
                        "peak_basis": "measured on rank 0's GPU in this run (IMAD + IADD3)",
                        "per": "GPU (evaluations / N over the max-over-ranks step time)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=["c0", "c1", "c2", "c3", "c4"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--method", default="auto", choices=["auto", "ssd", "product", "direct"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-also", action="store_true", help="skip the secondary c4 line")
    ap.add_argument("--gather", default="peer", choices=["peer", "nccl"],
                    help="N > 1, c3: tables to rank 0 by peer stores from the matcher into "
                         "symmetric memory (default) or by the chunked NCCL gather")
    ap.add_argument("--step-only", action="store_true",
                    help="only the timed matching step (no gather / stage legs, e2e, CPU "
                         "baseline): for ncu launch lists of the step")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    from synth import CONFIGS
    cfg = CONFIGS[args.config]
    call = cfg.calls[0]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))

    if args.impl == "reference":
        bench_reference(args, cfg, call, rank)
        return

    import torch
    import paper_2103_10765_b200 as g
    if world > 1 or args.gpus > 1:
        from paper_2103_10765_b200 import dist as gdist
        local = int(os.environ.get("LOCAL_RANK", "0"))
        line = gdist.bench_multi(args, cfg, call, sampler=ClockSampler(local))
        if line is not None and rank == 0:
            add_multi_roofline(line, cfg, call, g)
            # the same config object as the N = 1 line and the reference arm
            line["config"] = workload_config(cfg, call, args)
            print(json.dumps(line), flush=True)
        return
    torch.cuda.set_device(0)
    line = run_ours_single(args, cfg, call, torch, g)
    if not args.no_also and args.config != "c4":
        c4 = CONFIGS["c4"]
        also = run_ours_single(args, c4, c4.calls[0], torch, g, want_e2e=True, want_cpu=False)
        line["also"] = {"c4": {k: also[k] for k in ("value", "unit", "ms_per_step",
                                                    "gevals_per_s", "roofline",
                                                    "roofline_tensor", "e2e", "config",
                                                    "clocks", "gpu_launches", "ncu", "gather",
                                                    "wiener", "stage1")}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
