"""Dev: tiny matcher + gather + Wiener calls (for compute-sanitizer memcheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2103_10765_b200 as g
from synth import make_image
noisy, clean, sig = make_image(64, 72, 6, 1, 25.0, 0, return_clean=True)
z = torch.from_numpy(noisy).cuda()
for K in (16, 32):
    idx, dist, nv = g.block_match(z, 8, 3, 19, K, None)
    grp = g.gather_groups(z, idx, 8)
    out = g.wiener_stage2(z, torch.from_numpy(clean.astype(np.float32)).cuda(), idx, nv, 8, sig)
idx, dist, nv = g.block_match(z[:64, :64].contiguous(), 8, 8, 11, 8, None)
vol = g.gather_volume(z[:64, :64].contiguous(), idx, 8)
torch.cuda.synchronize()
print("ok")
