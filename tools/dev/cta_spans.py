"""Dev: per-CTA start/end (%globaltimer) of one c3 run with a GBM3D_TC_TRACE build: CTA
durations, gaps between consecutive CTAs on an SM, and the kernel span."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2103_10765_b200 as g
from synth import CONFIGS, config_images
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]; c = cfg.calls[0]
imgs = torch.from_numpy(config_images(cfg)).cuda()
img = imgs if cfg.B > 1 else imgs[0].contiguous()
for _ in range(3):
    g.block_match(img, c.patch, c.stride, c.radius, c.K, c.tau, check=False)
torch.cuda.synchronize()
lib = g.load_library()
n = 65536
buf = (ctypes.c_longlong * (3 * n))()
lib.gbm3d_dev_cta_spans(buf, n)
a = np.array(buf, dtype=np.int64).reshape(n, 3)
Ry, Rx = g.grid_dims(cfg.H, cfg.W, c.patch, c.stride)
nct = ((Rx + 7) // 8) * ((Ry + 15) // 16) * cfg.B
a = a[:nct]
t0 = a[:, 0].min()
dur = a[:, 1] - a[:, 0]
print(f"CTAs {nct}, kernel span {(a[:,1].max()-t0)/1e3:.1f} us, CTA duration mean {dur.mean()/1e3:.2f} us "
      f"min {dur.min()/1e3:.2f} max {dur.max()/1e3:.2f}")
gaps = []
for s in np.unique(a[:, 2]):
    r = a[a[:, 2] == s]
    r = r[np.argsort(r[:, 0])]
    gaps += list(r[1:, 0] - r[:-1, 1])
    if s == 0:
        print("SM0 CTAs:", len(r), "first start", (r[0,0]-t0)/1e3, "us, last end", (r[-1,1]-t0)/1e3, "us")
gaps = np.array(gaps)
print(f"gap between consecutive CTAs on an SM: mean {gaps.mean()/1e3:.2f} us, median {np.median(gaps)/1e3:.2f} us")
busy = dur.sum() / (len(np.unique(a[:, 2])) * (a[:, 1].max() - t0))
print(f"SM busy fraction {busy:.3f}")
