"""Dev: device time of one config image under arbitrary (K, tau, method) to separate the
selection cost from the rest of the pipeline.  Usage: time_params.py c3 K:tau:method ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2103_10765_b200 as g
from synth import CONFIGS, config_images
cfg = CONFIGS[sys.argv[1]]; c = cfg.calls[0]
imgs = torch.from_numpy(config_images(cfg)).cuda()
img = imgs if cfg.B > 1 else imgs[0].contiguous()
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
for spec in sys.argv[2:]:
    K, tau, method = spec.split(":")
    K = int(K); tau = None if tau == "none" else int(tau)
    f = lambda: g.block_match(img, c.patch, c.stride, c.radius, K, tau, check=False, method=method)
    for _ in range(3): f()
    torch.cuda.synchronize(); ts = []
    for _ in range(10):
        flush.zero_(); s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); f(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    print(f"{sys.argv[1]} K={K} tau={tau} {method}: median {np.median(ts):.3f} ms min {min(ts):.3f}", flush=True)
