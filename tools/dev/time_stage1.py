"""Dev: device time of the stage-1 call on a config (CUDA events), plus the output's mean and
a checksum so variants can be compared."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2103_10765_b200 as g
from synth import CONFIGS, make_image
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
noisy, clean, sig = make_image(cfg.H, cfg.W, cfg.n_rect, cfg.n_tex, cfg.sigma, cfg.seeds[0], return_clean=True)
z = torch.from_numpy(noisy).cuda()
idx, dist, nv = g.block_match(z, 8, 8, 19, 16, None, check=False)
out = g.stage1_denoise(z, idx, nv, 8, sig)
ws = torch.empty(g.load_library().gbm3d_stage1_workspace_bytes(1, cfg.H, cfg.W, 8, 16), dtype=torch.uint8, device="cuda")
ts = []
for _ in range(5):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); g.stage1_denoise(z, idx, nv, 8, sig, out=out, workspace=ws); e.record(); torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
o = out.cpu().numpy().astype(np.float64)
mse = np.mean((o - clean) ** 2)
print(f"stage1 {cfg.name}: {np.median(ts):.3f} ms  mse {mse:.4f} (noisy {np.mean((noisy - clean.astype(np.float64)) ** 2):.2f})")
np.save(os.path.join("gpurun_out", f"s1_{os.environ.get('TAG', 'x')}.npy"), o.astype(np.float32))
