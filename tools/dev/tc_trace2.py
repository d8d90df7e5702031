"""Dev: timeline of persistent CTA 10 of the tc16 kernel (GBM3D_TC_TRACE build)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2103_10765_b200 as g
from synth import CONFIGS, config_images
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]; c = cfg.calls[0]
imgs = torch.from_numpy(config_images(cfg)).cuda()
img = imgs if cfg.B > 1 else imgs[0].contiguous()
for _ in range(2):
    g.block_match(img, c.patch, c.stride, c.radius, c.K, c.tau, check=False, method="product")
torch.cuda.synchronize()
lib = g.load_library()
buf = (ctypes.c_longlong * 8192)()
lib.gbm3d_dev_tc_trace(buf, 8192)
t = np.array(buf, dtype=np.int64)
t0 = t[2000]
rel = lambda x: int(x - t0) if x else -1
print("tile | prod: start raw info centred mmadone xa epidone nc | mma: start end | epi w0: start first end | sel w0..3 start/first/rows/out")
for it in range(12):
    pr = [rel(t[2000 + it * 8 + k]) for k in range(8)]
    mm = [rel(t[3000 + it * 4 + k]) for k in range(2)]
    ep = [rel(t[4000 + it * 16 + k]) for k in (0, 1, 2)] + ["init", rel(t[4400 + it * 8]), "tfull", rel(t[4000 + it * 16 + 3]), "sempty", rel(t[4700 + it * 8])]
    se = [[rel(t[5000 + it * 16 + w * 4 + k]) for k in range(4)] for w in range(4)]
    print(it, pr, mm, ep, se)
print("tile 5 w0 per row: sel wait-start, sfull got, end, R | epi: start, tfull got, sempty got, staged")
for k in range(48):
    print(k, rel(t[6200 + k]), rel(t[6300 + k]), rel(t[6000 + k]), int(t[6100 + k]), "|",
          rel(t[6400 + k]), rel(t[6500 + k]), rel(t[6600 + k]), "gate", rel(t[6800 + k]), "ld", rel(t[6900 + k]),
          "cmp", rel(t[7000 + k]), rel(t[6700 + k]))
