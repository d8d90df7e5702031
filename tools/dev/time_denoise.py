"""Dev: device time of the whole two-stage denoise() on a config image (CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2103_10765_b200.denoise import denoise
from synth import CONFIGS, make_image
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
noisy, clean, sig = make_image(cfg.H, cfg.W, cfg.n_rect, cfg.n_tex, cfg.sigma, cfg.seeds[0], return_clean=True)
z = torch.from_numpy(noisy).cuda()
y = denoise(z, sig)
ts = []
for _ in range(5):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); y = denoise(z, sig); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
psnr = 10 * np.log10(255 ** 2 / np.mean((y.cpu().numpy().astype(np.float64) - clean) ** 2))
print(f"denoise {cfg.name}: {np.median(ts):.3f} ms  psnr {psnr:.2f} dB")
