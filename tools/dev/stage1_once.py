"""Dev: one c3-sized stage-1 call (tiling refs N=8, K=16) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2103_10765_b200 as g
from synth import CONFIGS, make_image
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
noisy, clean, sig = make_image(cfg.H, cfg.W, cfg.n_rect, cfg.n_tex, cfg.sigma, cfg.seeds[0], return_clean=True)
z = torch.from_numpy(noisy).cuda()
idx, dist, nv = g.block_match(z, 8, 8, 19, 16, None, check=False)
for _ in range(2):
    out = g.stage1_denoise(z, idx, nv, 8, sig)
torch.cuda.synchronize()
print("ok", float(out.mean()))
