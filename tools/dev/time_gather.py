"""Dev: device time of the group gather on a config's table (CUDA events, L2 flushed)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2103_10765_b200 as g
from synth import CONFIGS, config_images
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]; c = cfg.calls[0]
imgs = torch.from_numpy(config_images(cfg)).cuda()
img = imgs if cfg.B > 1 else imgs[0].contiguous()
idx, dist, nv = g.block_match(img, c.patch, c.stride, c.radius, c.K, c.tau, check=False)
out = g.gather_groups(img, idx, c.patch)
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
ts = []
for _ in range(10):
    flush.zero_(); s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); g.gather_groups(img, idx, c.patch, out=out); e.record(); torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
print(f"gather {cfg.name}: {np.median(ts):.3f} ms  {out.numel() * 2 / np.median(ts) / 1e6:.0f} GB/s (writes)")
