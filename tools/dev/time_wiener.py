"""Dev: device time of the stage-2 Wiener call on a config (CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2103_10765_b200 as g
from synth import CONFIGS, make_image
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]; c = cfg.calls[0]
noisy, clean, sig = make_image(cfg.H, cfg.W, cfg.n_rect, cfg.n_tex, cfg.sigma, cfg.seeds[0], return_clean=True)
z = torch.from_numpy(noisy).cuda(); bsc = torch.from_numpy(clean.astype(np.float32)).cuda()
idx, dist, nv = g.block_match(torch.from_numpy(clean).cuda(), c.patch, c.stride, c.radius, c.K, c.tau, check=False)
out = g.wiener_stage2(z, bsc, idx, nv, 8, sig)
ts = []
for _ in range(5):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); g.wiener_stage2(z, bsc, idx, nv, 8, sig, out=out); e.record(); torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
print(f"wiener {cfg.name}: {np.median(ts):.3f} ms")
