"""Dev: device time of block_match for several (config, P, s, r, K) shapes (events, median)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2103_10765_b200 as g
from synth import CONFIGS, make_image
for spec in sys.argv[1:]:
    parts = spec.split(":")
    name, P, S, r, K = parts[:5]
    method = parts[5] if len(parts) > 5 else "auto"
    P, S, r, K = int(P), int(S), int(r), int(K)
    cfg = CONFIGS[name]
    z = torch.from_numpy(make_image(cfg.H, cfg.W, cfg.n_rect, cfg.n_tex, cfg.sigma, cfg.seeds[0])).cuda()
    for _ in range(3):
        g.block_match(z, P, S, r, K, None, check=False, method=method)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); g.block_match(z, P, S, r, K, None, check=False, method=method); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    print(f"{name} P{P} s{S} r{r} K{K} {method}: {np.median(ts)*1e3:.1f} us  launches {g.last_launch_count()}")
