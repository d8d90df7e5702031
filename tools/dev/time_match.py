"""Dev: device time of one block_match call (CUDA events) on a config's image with explicit
(patch, stride, radius, K); saves the tables for cross-variant comparison."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2103_10765_b200 as g
from synth import CONFIGS, make_image
cfg = CONFIGS[sys.argv[1]]
P, S, r, K = (int(v) for v in sys.argv[2:6])
noisy = make_image(cfg.H, cfg.W, cfg.n_rect, cfg.n_tex, cfg.sigma, cfg.seeds[0])
z = torch.from_numpy(noisy).cuda()
idx, dist, nv = g.block_match(z, P, S, r, K, None, check=False)
ts = []
for _ in range(7):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); g.block_match(z, P, S, r, K, None, check=False); e.record(); torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
print(f"match {cfg.name} P{P} s{S} r{r} K{K}: {np.median(ts):.3f} ms  launches {g.load_library().gbm3d_last_launch_count()}")
tag = os.environ.get("TAG", "x")
np.save(f"gpurun_out/m_{tag}_idx.npy", idx.cpu().numpy()); np.save(f"gpurun_out/m_{tag}_dist.npy", dist.cpu().numpy())
