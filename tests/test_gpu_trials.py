"""GPU parity of stage 1's translation trials Y_f = (1/H) sum_h S_-h phi(S_h Z) (PAPER.md:
203-205; -m gpu): the library's circular shifts and shift-back average are
bit-exact / fp32-exact against numpy, and the composed trial schedule of ``denoise.stage1``
(shift_trials -> one batched block_match -> stage1_denoise -> unshift_mean) equals the float64
oracle ``oracle.stage1.translation_trials`` element-wise within ATOL = 1e-2 (reading S6), at a
noise level for which no coefficient of any trial's volume lies within 3e-4 (relative) of its
threshold (the keep/zero decisions of both sides then agree, see test_gpu_stage1.py)."""
import numpy as np
import pytest

import oracle
from oracle import stage1
from synth import make_image

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _g():
    import paper_2103_10765_b200 as g
    return g


@pytest.mark.parametrize("B,H,W,shifts", [(1, 64, 64, (0, 2, 4)), (3, 40, 72, (0, 5, 39, 1)),
                                          (2, 17, 9, (8, 0))])
def test_shift_and_unshift_exact(B, H, W, shifts):
    g = _g()
    rng = np.random.default_rng(B * 100 + H)
    imgs = rng.integers(-300, 700, (B, H, W)).astype(np.int16)
    z = g.shift_trials(torch.from_numpy(imgs).cuda(), shifts)
    torch.cuda.synchronize()
    exp = np.concatenate([np.roll(imgs, (h, h), axis=(1, 2)) for h in shifts])
    np.testing.assert_array_equal(z.cpu().numpy(), exp)
    ys = rng.normal(0, 50, (len(shifts) * B, H, W)).astype(np.float32)
    out = g.unshift_mean(torch.from_numpy(ys).cuda(), shifts).cpu().numpy()
    ref = np.mean([np.roll(ys[t * B:(t + 1) * B].astype(np.float64), (-h, -h), axis=(1, 2))
                   for t, h in enumerate(shifts)], axis=0)
    np.testing.assert_allclose(out, ref, atol=1e-4, rtol=1e-6)
    with pytest.raises(g.GBM3DError):
        g.shift_trials(torch.from_numpy(imgs).cuda(), (0, max(H, W)))


@pytest.mark.parametrize("H,W,sigma,seed,trials,K", [(64, 64, 25.0, 34, (0, 2, 4), 8),
                                                     (64, 64, 25.0, 33, (0, 4), 16),
                                                     (48, 64, 40.0, 32, (0, 3), 8)])
def test_translation_trials_parity(H, W, sigma, seed, trials, K):
    from paper_2103_10765_b200 import denoise
    N, r = 8, 16
    noisy, clean, sig = make_image(H, W, 8, 3, sigma, seed, return_clean=True)
    vols = []
    for h in trials:
        Zh = np.roll(noisy, (h, h), axis=(0, 1))
        idx, _d, nv = oracle.block_match(Zh, N, N, r, K, None)
        vols.append(oracle.gather_volume(Zh, idx, N).astype(np.float64))
    for i in range(400):
        s_try = sig * (1 + 1e-3 * i)
        if min(stage1.threshold_margin(V, s_try) for V in vols) > 3e-4:
            break
    else:
        pytest.fail("no decision-stable sigma found")
    exp = stage1.translation_trials(noisy, s_try, N, K, r, trials=trials)
    got = denoise.stage1(torch.from_numpy(noisy).cuda(), s_try, patch=N, K=K, radius=r,
                         trials=trials)
    torch.cuda.synchronize()
    np.testing.assert_allclose(got.cpu().numpy(), exp, atol=1e-2, rtol=0)
