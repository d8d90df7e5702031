"""Dev: one call of each small config (c0, c1 both calls, c2) for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2103_10765_b200 as g
from synth import CONFIGS, config_images
for name in ("c0", "c1", "c2"):
    cfg = CONFIGS[name]
    img = torch.from_numpy(config_images(cfg)[0]).cuda()
    for call in cfg.calls:
        g.block_match(img, call.patch, call.stride, call.radius, call.K, call.tau, check=False)
torch.cuda.synchronize()
print("ok")
