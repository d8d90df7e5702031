"""Dev: run c3 once with a GBM3D_TC_TRACE build and print the timeline of CTA (10,10)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2103_10765_b200 as g
from synth import CONFIGS, config_images
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]; c = cfg.calls[0]
K = int(sys.argv[2]) if len(sys.argv) > 2 else c.K
tau = (None if sys.argv[3] == "none" else int(sys.argv[3])) if len(sys.argv) > 3 else c.tau
img = torch.from_numpy(config_images(cfg)[0]).cuda()
for _ in range(2):
    g.block_match(img, c.patch, c.stride, c.radius, K, tau, check=False, method="product")
torch.cuda.synchronize()
lib = g.load_library()
buf = (ctypes.c_longlong * 8192)()
lib.gbm3d_dev_tc_trace(buf, 8192)
t = np.array(buf, dtype=np.int64)
t0 = t[0]
print("kernel start -> prologue end:", t0 - t[2], " prologue end -> kernel end:", t[1] - t0)
print("prologue marks from start (raw, plane, nc, loop):", [int(t[i] - t[2]) for i in (3, 4, 5, 0)])
print("output marks from loop start (out start, staged, stored, end):", [int(t[i] - t0) for i in (7, 8, 9, 1)])
mma = t[16:16 + 84] - t0
print("mma commit issue times:", mma.tolist())
for w in range(4):
    tf = t[1000 + 200 * w:1000 + 200 * w + 84] - t0
    st = t[2000 + 200 * w:2000 + 200 * w + 84]
    st = np.where(st > 0, st - t0, -1)
    sel = t[3000 + 200 * w:3000 + 200 * w + 60]
    sel = np.where(sel > 0, sel - t0, -1)
    rr = t[4000 + 200 * w:4000 + 200 * w + 60]
    print(f"w{w} tfull:", tf.tolist())
    print(f"w{w} staged:", st.tolist())
    print(f"w{w} selector batches (end time):", sel.tolist())
    print(f"w{w} selector R:", rr.tolist())

print("selector phases per row (w0): wait-start, ready, R-known, end")
for u in range(48):
    a, b, c_, e = t[5000 + u] - t0, t[6000 + u] - t0, t[7000 + u] - t0, t[3000 + u] - t0
    print(u, a, b - a, c_ - b, e - c_, "R", t[4000 + u])
