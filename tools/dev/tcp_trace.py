"""dev: per-CTA phase times of the patch-12 tensor-core kernel (trace build, GBM3D_TCP_TRACE=1)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2103_10765_b200 as g
from synth import config_images
img = torch.from_numpy(config_images("c2")[0]).cuda()
lib = ctypes.CDLL(os.environ["GBM3D_LIB"])
for _ in range(3):
    lib.gbm3d_dev_tcp_cnt_reset()
    g.block_match(img, 12, 4, 19, 16, 720000, check=False)
torch.cuda.synchronize()
n = 128
buf = np.zeros((n, 12), np.int64)
lib.gbm3d_dev_tcp_trace(buf.ctypes.data_as(ctypes.c_void_p), n)
t0 = buf[:, 0].min()
b = (buf - t0) / 1000.0
print("start   spread (us)", b[:, 0].min(), b[:, 0].max())
print("raw     (us) median", np.median(b[:, 1] - b[:, 0]), "max", (b[:, 1] - b[:, 0]).max())
print("hs      (us) median", np.median(b[:, 8] - b[:, 0]))
print("nq      (us) median", np.median(b[:, 9] - b[:, 0]))
print("prolog  (us) median", np.median(b[:, 2] - b[:, 0]), "max", (b[:, 2] - b[:, 0]).max())
for w in range(4):
    print(f"warp {w} main (us) median", np.median(b[:, 3 + w] - b[:, 2]), "max", (b[:, 3 + w] - b[:, 2]).max())
print("end     (us) median", np.median(b[:, 7] - b[:, 0]), "max", b[:, 7].max())
cnt = np.zeros((n, 4, 6), np.int64)
lib.gbm3d_dev_tcp_cnt(cnt.ctypes.data_as(ctypes.c_void_p), n)
tot = cnt.sum(axis=(0, 1))
print("per warp averages over CTAs: wait cyc %.0f scan cyc %.0f round cyc %.0f rounds %.1f rows %.1f dense rows %.1f"
      % tuple(cnt.mean(axis=(0, 1))))
print("cycles per round %.1f, scan cycles per row %.1f" % (tot[2] / max(1, tot[3]), tot[1] / max(1, tot[4])))
w = cnt[:, :, 0] + cnt[:, :, 1] + cnt[:, :, 2]
i = np.unravel_index(np.argmax(w), w.shape)
print("slowest warp", i, cnt[i])
