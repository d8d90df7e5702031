"""GPU parity (-m gpu): the CUDA path through the C ABI vs the CPU oracle, bit-exact on
idx, dist and n_valid (integer work: every output is unique under the (d, idx) order,
DESIGN.md reading R5, so array_equal is the bar)."""
import numpy as np
import pytest

import oracle
from synth import CONFIGS, config_images, special_image

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _gbm3d():
    import paper_2103_10765_b200 as g
    return g


def _gpu(img, P, s, r, K, tau, method="auto"):
    g = _gbm3d()
    t = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    idx, dist, nv = g.block_match(t, P, s, r, K, tau, method=method)
    torch.cuda.synchronize()
    return idx.cpu().numpy(), dist.cpu().numpy(), nv.cpu().numpy()


def _assert_same(got, exp, what=""):
    names = ("idx", "dist", "n_valid")
    for g_, e_, n in zip(got, exp, names):
        if not np.array_equal(g_, e_):
            bad = np.argwhere(g_ != e_)
            pytest.fail(f"{what} {n} differs at {len(bad)} positions, first {bad[:5].tolist()}: "
                        f"got {g_[tuple(bad[0])]} expected {e_[tuple(bad[0])]}")


import functools


@functools.lru_cache(maxsize=None)
def _oracle_config(name, ci):
    cfg = CONFIGS[name]
    c = cfg.calls[ci]
    imgs = config_images(cfg)
    if cfg.B > 1:
        return oracle.block_match_batched(imgs, c.patch, c.stride, c.radius, c.K, c.tau)
    return oracle.block_match(imgs[0], c.patch, c.stride, c.radius, c.K, c.tau)


def _product_supported(P, s, r, K, tau=None, method="product"):
    """Shapes the tensor-core product kernels take (include/gbm3d.h, GBM3D_METHOD_PRODUCT):
    P8 s3 r<=21 (fp16 and int8 kernels); P12 s4 r<=21 with tau - 1 within the 32-bit key's
    d range (fp16 kernel only)."""
    if P == 8 and s == 3:
        return 7 * s + 2 * r + 1 <= 64 and 2 <= K <= 32
    if P == 12 and s == 4 and method == "product":
        return r <= 21 and 2 <= K <= 32
    return False


# ----------------------------------------------------------------- the five BASELINE configs
@pytest.mark.parametrize("name,ci", [("c0", 0), ("c1", 0), ("c1", 1), ("c2", 0)])
def test_config_parity_small(name, ci):
    cfg = CONFIGS[name]
    c = cfg.calls[ci]
    img = config_images(cfg)[0]
    _assert_same(_gpu(img, c.patch, c.stride, c.radius, c.K, c.tau),
                 oracle.block_match(img, c.patch, c.stride, c.radius, c.K, c.tau), name)


@pytest.mark.parametrize("method", ["auto", "ssd", "product", "product_i8"])
def test_config_parity_c3_full(method):
    """2048^2, K=32: whole table bit-exact (auto = the bench's launch configuration)."""
    cfg = CONFIGS["c3"]
    c = cfg.calls[0]
    img = config_images(cfg)[0]
    _assert_same(_gpu(img, c.patch, c.stride, c.radius, c.K, c.tau, method=method),
                 _oracle_config("c3", 0), f"c3 {method}")


@pytest.mark.parametrize("method", ["auto", "ssd", "product", "product_i8"])
def test_config_parity_c4_all_images(method):
    """Batch of 64 512^2 images in ONE batched launch (auto = the bench's configuration)."""
    cfg = CONFIGS["c4"]
    c = cfg.calls[0]
    imgs = config_images(cfg)
    got = _gpu(imgs, c.patch, c.stride, c.radius, c.K, c.tau, method=method)
    _assert_same(got, _oracle_config("c4", 0), f"c4 {method}")


@pytest.mark.parametrize("method", ["ssd", "product", "product_i8"])
@pytest.mark.parametrize("name,ci", [("c0", 0), ("c1", 0), ("c1", 1)])
def test_config_parity_small_methods(name, ci, method):
    cfg = CONFIGS[name]
    c = cfg.calls[ci]
    img = config_images(cfg)[0]
    _assert_same(_gpu(img, c.patch, c.stride, c.radius, c.K, c.tau, method=method),
                 _oracle_config(name, ci), f"{name}/{ci} {method}")


# ----------------------------------------------------------------- shapes and edge cases
EDGE = [
    # (H, W, P, s, r, K, tau, kind)
    (8, 8, 8, 3, 19, 16, None, "uniform"),      # H = W = P: a single reference, window of one
    (8, 40, 8, 3, 19, 16, None, "uniform"),     # H = P
    (40, 8, 8, 3, 5, 16, None, "uniform"),      # W = P
    (37, 53, 8, 3, 0, 16, None, "uniform"),     # r = 0
    (30, 31, 8, 3, 32, 64, None, "uniform"),    # r >= H: global search, K > window count
    (45, 61, 8, 3, 19, 1, None, "uniform"),     # K = 1
    (45, 61, 8, 3, 19, 16, 0, "uniform"),       # tau = 0
    (45, 61, 8, 3, 19, 16, 90000, "uniform"),   # tau active
    (65, 33, 8, 3, 19, 32, None, "uniform"),    # odd W, ragged tiles
    (70, 29, 8, 3, 7, 16, None, "uniform"),     # W < 32 reference columns
    (200, 300, 8, 3, 19, 32, None, "uniform"),  # several CTAs x warps, ragged tail
    (60, 70, 8, 9, 19, 16, None, "uniform"),    # stride > patch (direct kernel)
    (60, 70, 8, 8, 19, 16, None, "uniform"),    # stride = patch (paper tiling, strip s8)
    (256, 200, 8, 8, 16, 16, None, "uniform"),  # stage-1 tiling, several strips, ragged
    (104, 96, 8, 8, 19, 32, 200000, "uniform"), # tiling with tau, K32
    (72, 88, 8, 8, 16, 16, None, "constant"),   # tiling, pure tie order
    (61, 59, 12, 4, 19, 16, 720000, "uniform"),
    (81, 97, 8, 2, 11, 16, None, "uniform"),
    (81, 97, 8, 4, 19, 24, None, "uniform"),
    (50, 50, 5, 2, 6, 10, None, "uniform"),     # no fast kernel: direct
    (64, 64, 16, 16, 32, 64, None, "uniform"),  # maximum patch, radius, K
    (70, 90, 8, 3, 19, 16, None, "constant"),   # all-zero distances: pure tie order
    (70, 90, 8, 3, 19, 32, None, "periodic"),
    (70, 90, 8, 3, 19, 16, None, "checker"),
]


@pytest.mark.parametrize("H,W,P,s,r,K,tau,kind", EDGE)
def test_edge_cases(H, W, P, s, r, K, tau, kind):
    img = special_image(kind, H, W, seed=H * 1000 + W, lo=-250, hi=500, value=77)
    _assert_same(_gpu(img, P, s, r, K, tau), oracle.block_match(img, P, s, r, K, tau),
                 f"{kind} {H}x{W} P{P} s{s} r{r} K{K} tau{tau}")


@pytest.mark.parametrize("method,H,W,P,s,r,K,tau,kind",
                         [(m,) + e for m in ("product", "product_i8") for e in EDGE
                          if _product_supported(e[2], e[3], e[4], e[5], e[6], m)])
def test_edge_cases_product(H, W, P, s, r, K, tau, kind, method):
    img = special_image(kind, H, W, seed=H * 1000 + W, lo=-250, hi=500, value=77)
    _assert_same(_gpu(img, P, s, r, K, tau, method=method), oracle.block_match(img, P, s, r, K, tau),
                 f"{method} {kind} {H}x{W} P{P} s{s} r{r} K{K} tau{tau}")


def test_product_mixed_range_tiles():
    """fp16 tiles next to tiles whose pixel range exceeds the fp16 exactness bound (marked and
    recomputed by the int8 kernel in the same call)."""
    rng = np.random.default_rng(7)
    img = rng.integers(-100, 356, size=(150, 170)).astype(np.int16)
    img[60:110, 20:90] = rng.choice(np.array([-900, 900], np.int16), size=(50, 70))
    for K in (16, 32):
        _assert_same(_gpu(img, 8, 3, 19, K, None, method="product"),
                     oracle.block_match(img, 8, 3, 19, K, None), f"mixed tiles K{K}")


def test_product_unsupported_shape_reports():
    g = _gbm3d()
    img = torch.from_numpy(config_images("c2")[0]).cuda()
    with pytest.raises(g.GBM3DError):   # no int8 kernel for P12
        g.block_match(img, 12, 4, 19, 16, 720000, method="product_i8")
    with pytest.raises(g.GBM3DError):   # radius above the P12 shared-memory bound
        g.block_match(img, 12, 4, 22, 16, 720000, method="product")


P12_CASES = [
    # H, W, r, K, tau, kind: ragged tiles, windows clipped at every border, K and tau extremes
    (61, 59, 19, 16, 720000, "uniform"),
    (130, 75, 19, 32, 720000, "uniform"),
    (100, 140, 21, 16, 500000, "uniform"),
    (90, 90, 5, 2, 1000000, "uniform"),
    (70, 66, 0, 16, 100, "uniform"),        # r = 0: only the reference
    (80, 80, 19, 16, 0, "uniform"),         # tau = 0: nothing passes
    (76, 92, 19, 16, 2097152, "uniform"),   # tau - 1 = dsat exactly
    (70, 90, 19, 16, 720000, "constant"),   # all-zero distances: pure tie order
    (70, 90, 19, 32, 720000, "periodic"),
    (70, 90, 19, 16, 720000, "checker"),
    (12, 12, 19, 16, 5000, "uniform"),      # one reference
]


@pytest.mark.parametrize("H,W,r,K,tau,kind", P12_CASES)
def test_p12_product_edge_cases(H, W, r, K, tau, kind):
    """The patch-12 tensor-core kernel (AUTO for c2's shape) on ragged, clipped and degenerate
    inputs, bit-exact against the oracle."""
    img = special_image(kind, H, W, seed=H * 1000 + W, lo=-150, hi=400, value=77)
    exp = oracle.block_match(img, 12, 4, r, K, tau)
    _assert_same(_gpu(img, 12, 4, r, K, tau, method="product"), exp, f"P12 {kind} {H}x{W} r{r} K{K}")
    _assert_same(_gpu(img, 12, 4, r, K, tau), exp, f"P12 auto {kind} {H}x{W} r{r} K{K}")


@pytest.mark.parametrize("tau", [None, 1 << 33, 2097153])
def test_p12_product_above_key_range(tau):
    """tau - 1 above the 32-bit key's d range (2^21 - 1 at r <= 22): references whose lists end
    short (high-contrast tiles where fewer than K - 1 candidates have d <= 2^21 - 1) are
    recomputed exactly with 64-bit keys, in the fp16 path and in the exact int32 path."""
    rng = np.random.default_rng(11)
    img = rng.integers(-60, 300, size=(120, 140)).astype(np.int16)      # d ~ 144 * 2 * 10^4 > 2^21
    img[40:80, 30:100] = rng.integers(0, 12, size=(40, 70)).astype(np.int16)  # lists that fill
    exp = oracle.block_match(img, 12, 4, 19, 16, tau)
    _assert_same(_gpu(img, 12, 4, 19, 16, tau, method="product"), exp, f"P12 tau {tau}")
    _assert_same(_gpu(img, 12, 4, 19, 16, tau), exp, f"P12 auto tau {tau}")


@pytest.mark.parametrize("H,W,r,K,tau,sigma,seed", [
    (140, 130, 19, 16, 720000, 50.0, 1),
    (97, 151, 19, 32, 400000, 25.0, 2),
    (120, 100, 21, 16, 2000000, 10.0, 3),
    (64, 200, 13, 8, 90000, 5.0, 4),
])
def test_p12_product_natural(H, W, r, K, tau, sigma, seed):
    """Natural-looking images (filled lists, ties between flat-region candidates) through the
    patch-12 tensor-core kernel, bit-exact against the oracle, single and batched."""
    from synth import make_image
    img = make_image(H, W, 12, 3, sigma, seed)
    exp = oracle.block_match(img, 12, 4, r, K, tau)
    _assert_same(_gpu(img, 12, 4, r, K, tau, method="product"), exp, f"P12 natural {H}x{W}")
    imgs = np.stack([img, make_image(H, W, 6, 2, sigma, seed + 50)])
    g = _gbm3d()
    i, d, n = g.block_match(torch.from_numpy(imgs).cuda(), 12, 4, r, K, tau, method="product")
    eb = oracle.block_match_batched(imgs, 12, 4, r, K, tau)
    _assert_same((i.cpu().numpy(), d.cpu().numpy(), n.cpu().numpy()), eb, "P12 natural batched")


def test_p12_product_exact_int_path(monkeypatch):
    """Tiles above the fp16 exactness bound take the kernel's exact int32 path: with the bound
    forced to 0 (dev switch GBM3D_TCP_MMAX, read once per process -> a subprocess) every tile
    does, and the c2 table plus a mixed-range image still match the oracle."""
    import subprocess, sys, os, json
    code = r'''
import numpy as np, torch, json, sys
import paper_2103_10765_b200 as g
from synth import config_images
img = config_images("c2")[0][:200, :180].copy()
rng = np.random.default_rng(3)
img2 = rng.integers(-100, 356, size=(150, 170)).astype(np.int16)
img2[60:110, 20:90] = rng.choice(np.array([-900, 900], np.int16), size=(50, 70))
out = []
for im, tau in ((img, 720000), (img2, 2000000), (img2, None)):
    i, d, n = g.block_match(torch.from_numpy(im).cuda(), 12, 4, 19, 16, tau, method="product")
    out.append([i.cpu().numpy().tolist(), d.cpu().numpy().tolist(), n.cpu().numpy().tolist()])
json.dump(out, sys.stdout)
'''
    rng = np.random.default_rng(3)
    img2 = rng.integers(-100, 356, size=(150, 170)).astype(np.int16)
    img2[60:110, 20:90] = rng.choice(np.array([-900, 900], np.int16), size=(50, 70))
    cases = ((config_images("c2")[0][:200, :180].copy(), 720000), (img2, 2000000), (img2, None))
    for mmax in ("0", None):
        env = dict(os.environ)
        if mmax is not None:
            env["GBM3D_TCP_MMAX"] = mmax
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                           cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        assert r.returncode == 0, r.stderr[-2000:]
        got = json.loads(r.stdout)
        for (im, tau), gg in zip(cases, got):
            exp = oracle.block_match(im, 12, 4, 19, 16, tau)
            _assert_same(tuple(np.array(x, dtype=np.int32) for x in gg), exp,
                         f"P12 exact path mmax={mmax} tau={tau}")


@pytest.mark.parametrize("seed", range(12))
def test_fuzz(seed):
    rng = np.random.default_rng(100 + seed)
    P, s = [(8, 3), (12, 4), (8, 2), (8, 4), (6, 3), (3, 1)][seed % 6]
    H = int(rng.integers(P, 140))
    W = int(rng.integers(P, 140))
    r = int(rng.integers(0, 25))
    K = int(rng.integers(1, 65))
    tau = [None, int(rng.integers(0, 300000))][seed % 2]
    img = special_image("uniform", H, W, seed=seed, lo=-200, hi=455)
    _assert_same(_gpu(img, P, s, r, K, tau), oracle.block_match(img, P, s, r, K, tau),
                 f"fuzz {seed}: {H}x{W} P{P} s{s} r{r} K{K} tau{tau}")


@pytest.mark.parametrize("method", ["auto", "ssd", "product_i8"])
def test_large_distances_exact_fallback(method):
    """Distances above the 32-bit key's d range (2^21-1 at r=19) with no tau: lists fill
    with saturated-range candidates and the in-kernel exact path must take over."""
    img = special_image("uniform", 60, 70, seed=9, lo=-1400, hi=1400)  # E[d] ~ 8e7 >> 2^21
    _assert_same(_gpu(img, 8, 3, 19, 16, None, method=method),
                 oracle.block_match(img, 8, 3, 19, 16, None), f"large distances {method}")


@pytest.mark.parametrize("method", ["auto", "ssd", "product_i8"])
def test_int16_extremes_within_precondition(method):
    rng = np.random.default_rng(3)
    img = rng.choice(np.array([-2896, 2896, 0, 1000], np.int16), size=(50, 60))  # 8^2*5792^2 < 2^31
    _assert_same(_gpu(img, 8, 3, 19, 16, None, method=method),
                 oracle.block_match(img, 8, 3, 19, 16, None), f"extremes {method}")


def test_direct_method_agrees():
    img = config_images("c0")[0]
    _assert_same(_gpu(img, 8, 3, 19, 16, None, method="direct"),
                 oracle.block_match(img, 8, 3, 19, 16, None), "direct")


# ----------------------------------------------------------------- variants (reading R16)
def test_batched_equals_single_calls():
    imgs = config_images("c4", n_images=3)[:, :200, :180].copy()
    g = _gbm3d()
    tb = torch.from_numpy(imgs).cuda()
    bi, bd, bn = g.block_match(tb, 8, 3, 19, 16)
    for i in range(3):
        si, sd, sn = g.block_match(tb[i].contiguous(), 8, 3, 19, 16)
        assert torch.equal(bi[i], si) and torch.equal(bd[i], sd) and torch.equal(bn[i], sn)


@pytest.mark.parametrize("cuts", [[7, 30], [1, 2, 64, 65], [33], [65]])
def test_row_ranges_concatenate_to_full(cuts):
    """Emulated sharding on one GPU: slabs with halo rows, global indices."""
    g = _gbm3d()
    img = config_images("c1")[0][:201, :].copy()   # 201 x 256 -> Ry = 66 (appended last row)
    H, W, P, s, r, K = 201, 256, 8, 3, 19, 32
    Ry, Rx = g.grid_dims(H, W, P, s)
    assert Ry == 66
    splits = [0] + cuts + [Ry]
    full = [t.cpu() for t in g.block_match(torch.from_numpy(img).cuda(), P, s, r, K)]
    parts = []
    for a, b in zip(splits[:-1], splits[1:]):
        y0 = min(a * s, H - P)
        y1 = min(b - 1, Ry - 1)
        ylast = min(y1 * s, H - P)
        lo, hi = max(0, y0 - r), min(H, ylast + r + P)
        slab = torch.from_numpy(img[lo:hi].copy()).cuda()
        parts.append([t.cpu() for t in g.block_match_rows(slab, lo, H, W, P, s, r, K, None, a, b)])
    for i in range(3):
        assert torch.equal(torch.cat([p[i] for p in parts]), full[i])


@pytest.mark.parametrize("cuts", [[17], [5, 40, 41]])
def test_row_ranges_p12_product(cuts):
    """Row-range calls (emulated shards with halo slabs) through the patch-12 tensor-core kernel:
    tiles start at the call's first row and read only the slab; the concatenation equals the
    oracle's full table."""
    g = _gbm3d()
    img = config_images("c2")[0][:230, :150].copy()
    H, W, P, s, r, K, tau = 230, 150, 12, 4, 19, 16, 720000
    Ry, Rx = g.grid_dims(H, W, P, s)
    splits = [0] + cuts + [Ry]
    parts = []
    for a, b in zip(splits[:-1], splits[1:]):
        y0 = min(a * s, H - P)
        ylast = min(min(b - 1, Ry - 1) * s, H - P)
        lo, hi = max(0, y0 - r), min(H, ylast + r + P)
        slab = torch.from_numpy(img[lo:hi].copy()).cuda()
        parts.append([t.cpu().numpy() for t in g.block_match_rows(slab, lo, H, W, P, s, r, K, tau, a, b)])
    got = tuple(np.concatenate([p[i] for p in parts]) for i in range(3))
    _assert_same(got, oracle.block_match(img, P, s, r, K, tau), f"P12 rows {cuts}")


def test_rows_rejects_short_slab():
    g = _gbm3d()
    img = torch.zeros((100, 64), dtype=torch.int16, device="cuda")
    with pytest.raises(g.GBM3DError):
        g.block_match_rows(img[10:50].contiguous(), 10, 200, 64, 8, 3, 19, 16, None, 10, 20)


def test_host_entry_matches_device_entry():
    g = _gbm3d()
    imgs = config_images("c4", n_images=2)
    h = torch.from_numpy(imgs).pin_memory()
    hi, hd, hn = g.block_match_host(h, 8, 3, 19, 16)
    di, dd, dn = g.block_match(torch.from_numpy(imgs).cuda(), 8, 3, 19, 16)
    assert torch.equal(hi, di.cpu()) and torch.equal(hd, dd.cpu()) and torch.equal(hn, dn.cpu())


@pytest.mark.parametrize("P,s,r,K", [(8, 3, 19, 32), (8, 8, 16, 16), (12, 4, 19, 16)])
def test_host_entry_single_image_row_chunks(P, s, r, K):
    """One large image: the host entry copies the pixels in row bands and matches row chunks
    (a short first chunk, then equal ones) on two streams; the tables must equal the device
    entry's on the c3 image, and the oracle's on sampled references."""
    g = _gbm3d()
    img = config_images("c3")[0]
    hi, hd, hn = g.block_match_host(torch.from_numpy(img).pin_memory(), P, s, r, K)
    di, dd, dn = g.block_match(torch.from_numpy(img).cuda(), P, s, r, K)
    for a, b in ((hi, di), (hd, dd), (hn, dn)):
        assert torch.equal(a.reshape(b.shape), b.cpu())
    # sampled references against the oracle (first and last reference rows, chunk borders)
    Ry, Rx = di.shape[:2]
    rng = np.random.default_rng(P * 100 + s)
    rows = [0, 31, 32, 33, Ry - 1] + list(rng.integers(0, Ry, 3))
    refs = [(int(y), int(x)) for y in rows for x in (0, Rx - 1, int(rng.integers(0, Rx)))]
    py, px = np.array(refs).T
    ei, ed, en = oracle.block_match_refs(img, P, s, r, K, None, py, px)
    assert np.array_equal(di.cpu().numpy()[py, px], ei)
    assert np.array_equal(dd.cpu().numpy()[py, px], ed)
    assert np.array_equal(dn.cpu().numpy()[py, px], en)


def test_check_range_and_error_codes():
    g = _gbm3d()
    ok = torch.from_numpy(config_images("c0")[0]).cuda()
    assert g.check_range(ok, 8)
    bad = torch.tensor([[-20000, 20000], [0, 1]], dtype=torch.int16, device="cuda")
    assert not g.check_range(bad, 2)
    with pytest.raises(g.GBM3DError):
        g.block_match(bad, 2, 1, 1, 2)            # check=True refuses out-of-domain images
    with pytest.raises(g.GBM3DError):
        g.block_match(ok, 17, 3, 19, 16)          # patch > 16 -> UNSUPPORTED


def test_check_range_cache_follows_modifications():
    """A passed range check is remembered per tensor object and version counter: an in-place
    write that breaks the bound is caught again, a larger patch is re-checked."""
    g = _gbm3d()
    img = torch.zeros((16, 16), dtype=torch.int16, device="cuda")
    img[0, 0] = 5000
    assert g.check_range(img, 8)                  # 64 * 5000^2 < 2^31
    assert g._range_cached(img, 8) and g._range_cached(img, 4)
    assert not g._range_cached(img, 12)           # a larger patch is checked again
    assert not g.check_range(img, 12)             # 144 * 5000^2 > 2^31
    img[1, 1] = -5000                             # in place: version counter bumps
    assert not g._range_cached(img, 8)
    assert not g.check_range(img, 8)              # 64 * 10000^2 > 2^31
    with pytest.raises(g.GBM3DError):
        g.block_match(img, 8, 3, 4, 4)
    other = img.clone()
    assert not g._range_cached(other, 2)          # another tensor object: no entry


def test_deterministic_repeat():
    img = torch.from_numpy(config_images("c2")[0]).cuda()
    g = _gbm3d()
    a = g.block_match(img, 12, 4, 19, 16, 720000)
    b = g.block_match(img, 12, 4, 19, 16, 720000)
    for x, y in zip(a, b):
        assert torch.equal(x, y)


def test_fuzz_wide():
    """80 random cases per method family: shapes on and off the fast paths (the tensor-core
    product kernels take P8 s3 r<=21 K<=32; the strip kernel its four shapes; the rest the
    direct kernel), natural-looking and uniform images, thresholds from 0 to above the int32
    key range, batched and single calls, all bit-exact against the oracle."""
    from synth import make_image
    rng = np.random.default_rng(2024)
    shapes = [(8, 3), (8, 3), (8, 3), (12, 4), (8, 2), (8, 4), (5, 2), (16, 16), (8, 8), (4, 1)]
    for case in range(80):
        P, s = shapes[case % len(shapes)]
        H = int(rng.integers(P, 120))
        W = int(rng.integers(P, 120))
        r = int(rng.integers(0, 33))
        K = int(rng.integers(1, 65))
        tau = [None, int(rng.integers(0, 400000)), int(rng.integers(0, 1 << 33))][case % 3]
        if case % 2:
            img = make_image(H, W, 6, 2, float(rng.uniform(5, 50)), case)
        else:
            img = special_image("uniform", H, W, seed=case, lo=-150, hi=400)
        _assert_same(_gpu(img, P, s, r, K, tau), oracle.block_match(img, P, s, r, K, tau),
                     f"wide fuzz {case}: {H}x{W} P{P} s{s} r{r} K{K} tau{tau}")


@pytest.mark.parametrize("name,ci", [("c0", 0), ("c1", 1), ("c2", 0)])
def test_cuda_graph_replay_matches_oracle(name, ci):
    """The device entry is capturable in a CUDA graph, including the side streams of the
    appended row / column (fork / join with events); replays on new pixels give the oracle's
    tables."""
    g = _gbm3d()
    cfg = CONFIGS[name]
    c = cfg.calls[ci]
    img = config_images(cfg)[0]
    t = torch.from_numpy(img).cuda()
    Ry, Rx = g.grid_dims(cfg.H, cfg.W, c.patch, c.stride)
    outs = (torch.empty((Ry, Rx, c.K), dtype=torch.int32, device="cuda"),
            torch.empty((Ry, Rx, c.K), dtype=torch.int32, device="cuda"),
            torch.empty((Ry, Rx), dtype=torch.int32, device="cuda"))
    g.block_match(t, c.patch, c.stride, c.radius, c.K, c.tau, check=False, out=outs)  # warm-up
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        g.block_match(t, c.patch, c.stride, c.radius, c.K, c.tau, check=False, out=outs)
    img2 = np.ascontiguousarray(img[::-1, ::-1])     # new pixels, same shape
    t.copy_(torch.from_numpy(img2))
    for o in outs:
        o.fill_(-7)
    graph.replay()
    torch.cuda.synchronize()
    got = tuple(o.cpu().numpy() for o in outs)
    _assert_same(got, oracle.block_match(img2, c.patch, c.stride, c.radius, c.K, c.tau),
                 f"graph replay {name} call {ci}")


def test_fuzz_p12_and_direct_p16():
    """60 random cases on the round's new paths: the patch-12 tensor-core kernel (r <= 21 incl.
    the 64-bit recompute when tau - 1 exceeds the 32-bit key range, r > 21 on the strip
    kernel) and the direct kernel's modular Eq. (2) form at P 12 / 16 (strides with no fast
    kernel), natural-looking and uniform images, single and batched, bit-exact vs the oracle."""
    from synth import make_image
    rng = np.random.default_rng(77)
    g = _gbm3d()
    for case in range(60):
        P, s = [(12, 4), (12, 4), (12, 4), (16, 16), (12, 13), (16, 5)][case % 6]
        H = int(rng.integers(P, 130))
        W = int(rng.integers(P, 130))
        r = int(rng.integers(0, 26))
        K = int(rng.integers(1, 40))
        tau = [None, int(rng.integers(0, 1500000)), int(rng.integers(0, 1 << 33))][case % 3]
        if case % 2:
            img = make_image(H, W, 6, 2, float(rng.uniform(5, 50)), case + 500)
        else:
            img = special_image("uniform", H, W, seed=case + 500, lo=-150, hi=400)
        what = f"p12/p16 fuzz {case}: {H}x{W} P{P} s{s} r{r} K{K} tau{tau}"
        _assert_same(_gpu(img, P, s, r, K, tau), oracle.block_match(img, P, s, r, K, tau), what)
        if case % 10 == 0:
            imgs = np.stack([img, np.ascontiguousarray(img[::-1])])
            i, d, n = g.block_match(torch.from_numpy(imgs).cuda(), P, s, r, K, tau)
            _assert_same((i.cpu().numpy(), d.cpu().numpy(), n.cpu().numpy()),
                         oracle.block_match_batched(imgs, P, s, r, K, tau), what + " batched")


def test_auto_small_jobs_direct():
    """AUTO's latency rule: jobs below the pixel-work threshold (c0) run on the per-reference
    direct kernel alone (one launch), larger ones (c1) on the tile kernels; both give the
    oracle's tables.  Subprocess without GBM3D_NO_SMALL_DIRECT (set for the rest of the suite)."""
    import json, os, subprocess, sys
    code = r'''
import json, sys, torch
import paper_2103_10765_b200 as g
from synth import CONFIGS, config_images
out = {}
for name in ("c0", "c1"):
    c = CONFIGS[name].calls[0]
    img = torch.from_numpy(config_images(name)[0]).cuda()
    i, d, n = g.block_match(img, c.patch, c.stride, c.radius, c.K, c.tau)
    torch.cuda.synchronize()
    out[name] = [g.last_launch_count(), i.cpu().numpy().tolist(), d.cpu().numpy().tolist(),
                 n.cpu().numpy().tolist()]
json.dump(out, sys.stdout)
'''
    env = {k: v for k, v in os.environ.items() if k != "GBM3D_NO_SMALL_DIRECT"}
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stderr[-2000:]
    got = json.loads(r.stdout)
    assert got["c0"][0] == 1          # the direct kernel alone
    assert got["c1"][0] > 1           # tile kernel (+ the appended row / column)
    for name in ("c0", "c1"):
        exp = _oracle_config(name, 0)
        _assert_same(tuple(np.array(x, dtype=np.int32) for x in got[name][1:]), exp,
                     f"AUTO small-job rule {name}")
