"""Dev: device time of gbm3d_wiener_stage2 on c3 (the bench's Wiener leg setup, shortened)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2103_10765_b200 as g
from synth import CONFIGS, config_images, make_image
cfg = CONFIGS["c3"]; call = cfg.calls[0]
img = torch.from_numpy(config_images(cfg)[0]).cuda()
_, clean, sig = make_image(cfg.H, cfg.W, cfg.n_rect, cfg.n_tex, cfg.sigma, cfg.seeds[0], return_clean=True)
basic = torch.from_numpy(clean.astype(np.float32)).cuda()
est = torch.from_numpy(clean.astype(np.int16)).cuda()
idx, _, nv = g.block_match(est, call.patch, call.stride, call.radius, call.K, call.tau, check=False)
out = torch.empty(basic.shape, dtype=torch.float32, device="cuda")
ws = torch.empty(g.load_library().gbm3d_wiener_workspace_bytes(1, cfg.H, cfg.W), dtype=torch.uint8, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
for _ in range(3):
    g.wiener_stage2(img, basic, idx, nv, call.patch, [sig], out=out, workspace=ws)
ts = []
for _ in range(10):
    flush.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); g.wiener_stage2(img, basic, idx, nv, call.patch, [sig], out=out, workspace=ws); e.record()
    torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
print("wiener c3 median %.3f ms" % np.median(ts))
