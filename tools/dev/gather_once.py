"""Dev: one c3 match + gather (for ncu captures of the gather kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2103_10765_b200 as g
from synth import CONFIGS, config_images
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]; c = cfg.calls[0]
imgs = torch.from_numpy(config_images(cfg)).cuda()
img = imgs if cfg.B > 1 else imgs[0].contiguous()
idx, dist, nv = g.block_match(img, c.patch, c.stride, c.radius, c.K, c.tau, check=False)
for _ in range(2):
    grp = g.gather_groups(img, idx, c.patch)
torch.cuda.synchronize()
print("ok", tuple(grp.shape))
