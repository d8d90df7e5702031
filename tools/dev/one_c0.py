"""Dev: one c0 matching call vs the oracle (quick GPU check of a build)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2103_10765_b200 as g
import oracle
from synth import config_images
cfg = sys.argv[1] if len(sys.argv) > 1 else "c0"
img = config_images(cfg)[0]
t = torch.from_numpy(img).cuda()
idx, dist, nv = g.block_match(t, 8, 3, 19, 16, None, check=False)
torch.cuda.synchronize()
e = oracle.block_match(img, 8, 3, 19, 16, None)
print("idx", np.array_equal(idx.cpu().numpy(), e[0]), "dist", np.array_equal(dist.cpu().numpy(), e[1]),
      "nv", np.array_equal(nv.cpu().numpy(), e[2]))
