"""Quick device timing of one config (CUDA events, L2 flushed between reps).  Dev tool, not the
bench; parity checks live in tests/."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_10765_b200 as g  # noqa: E402
from synth import CONFIGS, config_images  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--method", default="auto")
a = ap.parse_args()
cfg = CONFIGS[a.config]
c = cfg.calls[0]
imgs_np = config_images(cfg)
imgs = torch.from_numpy(imgs_np).cuda()
img = imgs if cfg.B > 1 else imgs[0].contiguous()
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
for _ in range(3):
    out = g.block_match(img, c.patch, c.stride, c.radius, c.K, c.tau, check=False, method=a.method)
torch.cuda.synchronize()
ts = []
for _ in range(a.reps):
    flush.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    out = g.block_match(img, c.patch, c.stride, c.radius, c.K, c.tau, check=False, method=a.method)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
print(f"{a.config} {os.environ.get('GBM3D_STRIP_SOLO', '0')} median {np.median(ts):.3f} ms  min {min(ts):.3f}")
