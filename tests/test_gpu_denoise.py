"""The composed G-BM3D denoiser (paper_2103_10765_b200.denoise; -m gpu): sanity of the schedule
(each component's parity is tested on its own): both stages improve on their input, stage 2
improves on stage 1 (Table I's consistent ordering), and a single trial equals
one matching + stage-1 call (up to the order of fp32 atomic reductions)."""
import numpy as np
import pytest

from synth import make_image

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _psnr(x, clean):
    return 10 * np.log10(255.0 ** 2 / np.mean((x - clean) ** 2))


@pytest.mark.parametrize("sigma,seed", [(25.0, 0), (40.0, 1)])
def test_two_stage_improves(sigma, seed):
    from paper_2103_10765_b200 import denoise as dn
    noisy, clean, sig = make_image(128, 128, 12, 4, sigma, seed, return_clean=True)
    z = torch.from_numpy(noisy).cuda()
    basic = dn.stage1(z, sig)
    final = dn.stage2(z, basic, sig)
    torch.cuda.synchronize()
    p0 = _psnr(noisy.astype(np.float64), clean)
    p1 = _psnr(basic.cpu().numpy().astype(np.float64), clean)
    p2 = _psnr(final.cpu().numpy().astype(np.float64), clean)
    assert p1 > p0 + 5 and p2 > p1, (p0, p1, p2)


def test_single_trial_is_one_call():
    import paper_2103_10765_b200 as g
    from paper_2103_10765_b200 import denoise as dn
    noisy, clean, sig = make_image(64, 64, 6, 2, 25.0, 3, return_clean=True)
    z = torch.from_numpy(noisy).cuda()
    a = dn.stage1(z, sig, trials=(0,))           # the paper's N = 16 tiles
    idx, dist, nv = g.block_match(z, 16, 16, 16, 16, None)
    b = g.stage1_denoise(z, idx, nv, 16, sig)
    torch.cuda.synchronize()
    # equal up to the order of the fp32 atomic reductions in the aggregation (run to run)
    np.testing.assert_allclose(a.cpu().numpy(), b.cpu().numpy(), atol=1e-3, rtol=0)


def test_batched_denoise_equals_single_images():
    """A batch [B, H, W] runs every step batched (matching, stage 1, stage 2) and equals the
    per-image calls (up to the order of the fp32 atomic reductions)."""
    from paper_2103_10765_b200.denoise import denoise
    imgs = [make_image(64, 96, 8, 2, 25.0, 10 + i) for i in range(3)]
    z = torch.from_numpy(np.stack(imgs)).cuda()
    yb = denoise(z, 25.0)
    ys = [denoise(z[i].contiguous(), 25.0) for i in range(3)]
    torch.cuda.synchronize()
    for i in range(3):
        np.testing.assert_allclose(yb[i].cpu().numpy(), ys[i].cpu().numpy(), atol=2e-3, rtol=0)
