"""Dev study (CPU, oracle only): how tight would per-reference gate seeds from neighbouring
references be?  Pass fraction of the window under the seed and the fraction of references whose
true (K-1)-th distance exceeds it (where the c3 time goes)."""
import numpy as np, sys, time
sys.path.insert(0, '/root/repo')
import oracle
from synth import CONFIGS, config_images
cfg = CONFIGS['c3']; c = cfg.calls[0]
img = config_images(cfg)[0]
H, W = img.shape; P, S, r, K = c.patch, c.stride, c.radius, c.K
# crop a region to keep it cheap
img = img[:600, :600].copy(); H, W = img.shape
t0 = time.time()
idx, dist, nv = oracle.block_match(img, P, S, r, K, None)
print('oracle', time.time() - t0, dist.shape)
D = dist[..., K - 1].astype(np.float64)   # (K-1)th neighbour distance per ref
Ry, Rx = D.shape
# tiles of 16 x 8 refs; checkerboard A/B
TY, TX = 16, 8
ty = np.arange(Ry) // TY; tx = np.arange(Rx) // TX
A = ((ty[:, None] + tx[None, :]) % 2) == 0
# seed for B refs: max of D over A refs within a (2*TY x 2*TX) neighbourhood
from scipy.ndimage import maximum_filter
DA = np.where(A, D, 0)
rng = np.random.default_rng(0)
img64 = img.astype(np.int64)
def all_d(y, x):
    ys, xs = y * S, x * S
    ys = min(ys, H - P); xs = min(xs, W - P)
    ref = img64[ys:ys+P, xs:xs+P]
    out = []
    for cy in range(max(0, ys - r), min(H - P, ys + r) + 1):
        for cx in range(max(0, xs - r), min(W - P, xs + r) + 1):
            if cy == ys and cx == xs: continue
            out.append(((img64[cy:cy+P, cx:cx+P] - ref) ** 2).sum())
    return np.array(out)
for win, alpha in [((2*TY+1, 2*TX+1), 1.0), ((2*TY+1, 2*TX+1), 1.25), ((TY+1, TX+1), 1.25), ((9, 9), 1.25), ((9, 9), 1.5), ((33, 17), 1.5)]:
    seed = alpha * maximum_filter(DA, size=win)
    Bm = ~A
    fail = (D > seed) & Bm
    # pass fraction on a sample of B refs
    ys, xs = np.nonzero(Bm)
    sel = rng.choice(len(ys), 150, replace=False)
    pf = []; pf_inc = []
    for i in sel:
        d = all_d(ys[i], xs[i])
        pf.append(np.mean(d < seed[ys[i], xs[i]]))
    print(f"win {win} alpha {alpha}: fail {fail.sum() / Bm.sum():.4f}  pass frac {np.mean(pf):.4f}")
