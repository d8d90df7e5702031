"""Dev: one block_match call of a shape on a config's image (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2103_10765_b200 as g
from synth import CONFIGS, make_image
name, P, S, r, K = sys.argv[1].split(":")
cfg = CONFIGS[name]
z = torch.from_numpy(make_image(cfg.H, cfg.W, cfg.n_rect, cfg.n_tex, cfg.sigma, cfg.seeds[0])).cuda()
g.block_match(z, int(P), int(S), int(r), int(K), None, check=False)
torch.cuda.synchronize()
print("ok")
