"""Run one block-matching call of a config (for ncu / compute-sanitizer captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2103_10765_b200 as g  # noqa: E402
from synth import CONFIGS, config_images  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--call", type=int, default=0)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--images", type=int, default=0)
ap.add_argument("--method", default="auto")
a = ap.parse_args()
cfg = CONFIGS[a.config]
c = cfg.calls[a.call]
imgs = torch.from_numpy(config_images(cfg, a.images or None)).cuda()
img = imgs if imgs.shape[0] > 1 else imgs[0].contiguous()
for _ in range(a.reps):
    out = g.block_match(img, c.patch, c.stride, c.radius, c.K, c.tau, check=False, method=a.method)
torch.cuda.synchronize()
print("ok", [tuple(t.shape) for t in out])
