"""Dev: stage-1 block size 8 vs 16 (the paper's N) in denoise(): time and PSNR."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2103_10765_b200 import denoise as dn
from synth import CONFIGS, make_image
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
noisy, clean, sig = make_image(cfg.H, cfg.W, cfg.n_rect, cfg.n_tex, cfg.sigma, cfg.seeds[0], return_clean=True)
z = torch.from_numpy(noisy).cuda()
psnr = lambda y: 10 * np.log10(255 ** 2 / np.mean((y.cpu().numpy().astype(np.float64) - clean) ** 2))
for N in (8, 16):
    for two in (False, True):
        def run():
            b = dn.stage1(z, sig, patch=N)
            return dn.stage2(z, b, sig) if two else b
        y = run()
        ts = []
        for _ in range(5):
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record(); y = run(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
        print(f"N={N} {'G-BM3D2' if two else 'G-BM3D1'}: {np.median(ts):.2f} ms  psnr {psnr(y):.2f} dB")
