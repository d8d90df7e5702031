"""GPU parity of stage-2 collaborative Wiener filtering + aggregation (-m gpu)
against the float64 oracle (oracle/wiener.py).  fp32 arithmetic: transform coefficients reach
8 x 500 x sqrt(32) ~ 2.3e4 (ulp 2e-3); each of the six transform passes adds at most ~8
half-ulp roundings of its partial sums, so a filtered pixel is within ~2e-2 of the exact value
and so is any weighted average of such pixels: ATOL = 2e-2 on a 0..255 scale (W6)."""
import numpy as np
import pytest

import oracle
from oracle import wiener
from synth import CONFIGS, make_image

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ATOL = 2e-2


def _g():
    import paper_2103_10765_b200 as g
    return g


def _case(H, W, n_rect, n_tex, sigma, seed, K, r, s=3, tau=None):
    noisy, clean, sig = make_image(H, W, n_rect, n_tex, sigma, seed, return_clean=True)
    idx, dist, nv = oracle.block_match(clean, 8, s, r, K, tau)  # stage 2 matches on the estimate
    return noisy, clean.astype(np.float32), sig, idx, nv


def _gpu(noisy, basic, idx, nv, sigma):
    g = _g()
    out = g.wiener_stage2(torch.from_numpy(noisy).cuda(), torch.from_numpy(basic).cuda(),
                          torch.from_numpy(idx).cuda(), torch.from_numpy(nv).cuda(), 8, sigma)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("H,W,K,r,sigma,seed", [(64, 64, 16, 19, 25.0, 0), (96, 80, 32, 11, 40.0, 1),
                                                 (72, 64, 8, 7, 10.0, 2), (40, 56, 4, 5, 25.0, 3)])
def test_wiener_parity(H, W, K, r, sigma, seed):
    noisy, basic, sig, idx, nv = _case(H, W, 6, 2, sigma, seed, K, r)
    exp = wiener.stage2(noisy, basic.astype(np.float64), idx, nv, 8, sig)
    got = _gpu(noisy, basic, idx, nv, sig)
    np.testing.assert_allclose(got, exp, atol=ATOL, rtol=0)


def test_wiener_parity_c1_stage2_call():
    """BASELINE c1's stage-2 call shape (256^2, K32, tau = 400 * 64) on the estimate."""
    cfg = CONFIGS["c1"]
    c = cfg.calls[1]
    noisy, clean, sig = make_image(cfg.H, cfg.W, cfg.n_rect, cfg.n_tex, cfg.sigma, cfg.seeds[0],
                                   return_clean=True)
    idx, dist, nv = oracle.block_match(clean, c.patch, c.stride, c.radius, c.K, c.tau)
    exp = wiener.stage2(noisy, clean.astype(np.float64), idx, nv, 8, sig)
    got = _gpu(noisy, clean.astype(np.float32), idx, nv, sig)
    np.testing.assert_allclose(got, exp, atol=ATOL, rtol=0)


def test_wiener_identity_and_batched():
    """sigma = 0 with basic = noisy is the identity (PAPER.md:190 averages copies of each pixel);
    a batch equals per-image calls (per-image sigma)."""
    noisy, basic, sig, idx, nv = _case(48, 64, 5, 1, 25.0, 4, 16, 9)
    got = _gpu(noisy, noisy.astype(np.float32), idx, nv, 0.0)
    np.testing.assert_allclose(got, noisy, atol=ATOL, rtol=0)
    imgs = [_case(48, 48, 5, 1, s, 10 + i, 8, 7) for i, s in enumerate((12.0, 30.0, 45.0))]
    g = _g()
    nz = torch.from_numpy(np.stack([c[0] for c in imgs])).cuda()
    bs = torch.from_numpy(np.stack([c[1] for c in imgs])).cuda()
    ix = torch.from_numpy(np.stack([c[3] for c in imgs])).cuda()
    nvv = torch.from_numpy(np.stack([c[4] for c in imgs])).cuda()
    out = g.wiener_stage2(nz, bs, ix, nvv, 8, [c[2] for c in imgs]).cpu().numpy()
    for i, c in enumerate(imgs):
        exp = wiener.stage2(c[0], c[1].astype(np.float64), c[3], c[4], 8, c[2])
        np.testing.assert_allclose(out[i], exp, atol=ATOL, rtol=0)


def test_wiener_errors():
    g = _g()
    noisy, basic, sig, idx, nv = _case(32, 32, 3, 0, 25.0, 5, 8, 5)
    t = lambda a: torch.from_numpy(a).cuda()
    with pytest.raises(g.GBM3DError):  # K = 6 is not a power of two
        g.wiener_stage2(t(noisy), t(basic), t(np.ascontiguousarray(idx[..., :6])), t(nv), 8, sig)


def test_wiener_full_size_c3_sampled():
    """BASELINE c3's full size (2048^2, P8 s3 r19 K32, groups matched on the clean stand-in of
    the basic estimate by the oracle): the GPU call on the whole image, checked on 16 windows
    of 16 x 16 pixels (4,096 pixels: the four corners, windows across the reference-tile seams,
    random ones) whose values the oracle rebuilds from every group with a block on the window
    (wiener_group of each, the aggregation of PAPER.md:190 restricted to the window)."""
    cfg = CONFIGS["c3"]
    c = cfg.calls[0]
    noisy, clean, sig = make_image(cfg.H, cfg.W, cfg.n_rect, cfg.n_tex, cfg.sigma, cfg.seeds[0],
                                   return_clean=True)
    idx, dist, nv = oracle.block_match(clean, c.patch, c.stride, c.radius, c.K, c.tau)
    got = _gpu(noisy, clean.astype(np.float32), idx, nv, sig)
    H, W = noisy.shape
    N, WS = c.patch, 16
    rng = np.random.default_rng(7)
    wins = [(0, 0), (0, W - WS), (H - WS, 0), (H - WS, W - WS), (40, 16), (88, 1000),
            (1000, 2008), (2040 - WS, 500)]
    wins += [tuple(int(v) for v in rng.integers(0, H - WS, 2)) for _ in range(16 - len(wins))]
    basic = clean.astype(np.float64)
    cy_all, cx_all = idx // W, idx % W
    k_ok = np.arange(c.K)[None, None, :] < nv[..., None]
    for (y0, x0) in wins:
        # groups with a valid block overlapping the window
        hit = k_ok & (cy_all <= y0 + WS - 1) & (cy_all + N > y0) & (cx_all <= x0 + WS - 1) & \
            (cx_all + N > x0)
        num = np.zeros((WS, WS))
        den = np.zeros((WS, WS))
        for i, j in zip(*np.nonzero(hit.any(axis=-1))):
            cy, cx = cy_all[i, j], cx_all[i, j]
            Gz = np.stack([noisy[cy[k]:cy[k] + N, cx[k]:cx[k] + N] for k in range(c.K)])
            Gb = np.stack([basic[cy[k]:cy[k] + N, cx[k]:cx[k] + N] for k in range(c.K)])
            U, w = wiener.wiener_group(Gz, Gb, sig)
            for k in np.nonzero(hit[i, j])[0]:
                ya, yb = max(cy[k], y0), min(cy[k] + N, y0 + WS)
                xa, xb = max(cx[k], x0), min(cx[k] + N, x0 + WS)
                num[ya - y0:yb - y0, xa - x0:xb - x0] += w * U[k, ya - cy[k]:yb - cy[k], xa - cx[k]:xb - cx[k]]
                den[ya - y0:yb - y0, xa - x0:xb - x0] += w
        assert (den > 0).all()
        np.testing.assert_allclose(got[y0:y0 + WS, x0:x0 + WS], num / den, atol=ATOL, rtol=0,
                                   err_msg=f"window {(y0, x0)}")
