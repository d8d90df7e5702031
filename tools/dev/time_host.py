"""Dev: end-to-end time of block_match_host (pinned host buffers) on a config, and the raw
pinned D2H / H2D bandwidth of the same byte counts."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2103_10765_b200 as g
from synth import CONFIGS, config_images
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]; call = cfg.calls[0]
h = torch.from_numpy(config_images(cfg)).pin_memory()
Ry, Rx = g.grid_dims(cfg.H, cfg.W, call.patch, call.stride)
B = cfg.B
ws = torch.empty(g.host_workspace_bytes(B, cfg.H, cfg.W, call.patch, call.stride, call.K), dtype=torch.uint8, device="cuda")
out = (torch.empty((B, Ry, Rx, call.K), dtype=torch.int32, pin_memory=True),
       torch.empty((B, Ry, Rx, call.K), dtype=torch.int32, pin_memory=True),
       torch.empty((B, Ry, Rx), dtype=torch.int32, pin_memory=True))
step = lambda: g.block_match_host(h, call.patch, call.stride, call.radius, call.K, call.tau, workspace=ws, out=out)
for _ in range(5): step()
ts = []
for _ in range(30):
    t0 = time.perf_counter(); step(); ts.append(time.perf_counter() - t0)
nb = sum(o.numel() * 4 for o in out)
d = torch.empty(nb // 4, dtype=torch.int32, device="cuda"); hp = torch.empty(nb // 4, dtype=torch.int32, pin_memory=True)
for _ in range(3): hp.copy_(d); torch.cuda.synchronize()
t2 = []
for _ in range(10):
    t0 = time.perf_counter(); hp.copy_(d); torch.cuda.synchronize(); t2.append(time.perf_counter() - t0)
print(f"host e2e {cfg.name}: mean {1e3*statistics.mean(ts):.3f} ms  median {1e3*statistics.median(ts):.3f} ms; "
      f"raw D2H {nb/1e6:.1f} MB: {1e3*statistics.median(t2):.3f} ms = {nb/statistics.median(t2)/1e9:.1f} GB/s")
