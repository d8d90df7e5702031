"""GPU parity of the matched-block gather (-m gpu): gbm3d_gather_groups /
gbm3d_gather_volume through the C ABI vs the oracle's plain slice copies, bit-exact (byte
work).  Index tables come from the oracle matcher (small cases) or from the GPU matcher,
whose own parity is tested in test_gpu_parity.py (full-size cases, checked on samples)."""
import numpy as np
import pytest

import oracle
from synth import CONFIGS, config_images

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _g():
    import paper_2103_10765_b200 as g
    return g


@pytest.mark.parametrize("name,ci", [("c0", 0), ("c1", 0), ("c1", 1), ("c2", 0)])
def test_groups_parity_small_configs(name, ci):
    g = _g()
    cfg = CONFIGS[name]
    c = cfg.calls[ci]
    img = config_images(cfg)[0]
    idx, _, _ = oracle.block_match(img, c.patch, c.stride, c.radius, c.K, c.tau)
    got = g.gather_groups(torch.from_numpy(img).cuda(), torch.from_numpy(idx).cuda(), c.patch)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy(), oracle.gather_groups(img, idx, c.patch))


def test_groups_parity_c3_full_size_sampled():
    """c3 (2048^2, K32) in the bench's launch configuration: 1.9 GB of groups, checked on
    4096 sampled references against the oracle's slice copies."""
    g = _g()
    cfg = CONFIGS["c3"]
    c = cfg.calls[0]
    img = config_images(cfg)[0]
    t = torch.from_numpy(img).cuda()
    idx, _, _ = g.block_match(t, c.patch, c.stride, c.radius, c.K, c.tau, check=False)
    grp = g.gather_groups(t, idx, c.patch)
    torch.cuda.synchronize()
    rng = np.random.default_rng(3)
    ys = rng.integers(0, idx.shape[0], 4096)
    xs = rng.integers(0, idx.shape[1], 4096)
    sub_idx = idx.cpu().numpy()[ys, xs][None]  # [1, n, K]
    exp = oracle.gather_groups(img, sub_idx, c.patch)[0]
    got = grp[torch.from_numpy(ys).cuda(), torch.from_numpy(xs).cuda()].cpu().numpy()
    np.testing.assert_array_equal(got, exp)


def test_groups_parity_batched_c4_subset():
    g = _g()
    cfg = CONFIGS["c4"]
    c = cfg.calls[0]
    imgs = config_images(cfg, 4)
    idx = oracle.block_match_batched(imgs, c.patch, c.stride, c.radius, c.K, c.tau)[0]
    got = g.gather_groups(torch.from_numpy(imgs).cuda(), torch.from_numpy(idx).cuda(), c.patch)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy(), oracle.gather_groups(imgs, idx, c.patch))


@pytest.mark.parametrize("H,W,N,r,K", [(256, 256, 8, 19, 16), (96, 160, 8, 11, 8),
                                       (120, 96, 12, 12, 16), (64, 64, 16, 16, 4)])
def test_volume_parity_tiling(H, W, N, r, K):
    """Tiling references (stride = N, N | H, W): the volume V slice-major."""
    g = _g()
    img = config_images(CONFIGS["c1"])[0][:H, :W].copy()
    idx, _, _ = oracle.block_match(img, N, N, r, K, None)
    got = g.gather_volume(torch.from_numpy(img).cuda(), torch.from_numpy(idx).cuda(), N)
    torch.cuda.synchronize()
    v = got.cpu().numpy()
    np.testing.assert_array_equal(v, oracle.gather_volume(img, idx, N))
    np.testing.assert_array_equal(v[0], img)


def test_volume_parity_batched():
    g = _g()
    imgs = config_images(CONFIGS["c4"], 3)[:, :128, :128].copy()
    idx = oracle.block_match_batched(imgs, 8, 8, 19, 16, None)[0]
    got = g.gather_volume(torch.from_numpy(imgs).cuda(), torch.from_numpy(idx).cuda(), 8)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy(), oracle.gather_volume(imgs, idx, 8))


def test_invalid_index_gives_zero_block_and_errors():
    g = _g()
    img = config_images(CONFIGS["c0"])[0]
    idx = np.array([[[0, 64 * 60 + 60, -1, 64 * 64 * 2]]], dtype=np.int32)
    got = g.gather_groups(torch.from_numpy(img).cuda(), torch.from_numpy(idx).cuda(), 8)
    torch.cuda.synchronize()
    got = got.cpu().numpy()[0, 0]
    np.testing.assert_array_equal(got[0], img[:8, :8])
    assert (got[1:] == 0).all()  # (60, 60) leaves the image; negative; beyond the image
    with pytest.raises(g.GBM3DError):
        g.gather_groups(torch.from_numpy(img).cuda(), torch.from_numpy(idx).cuda(), 17)
    with pytest.raises(ValueError):
        g.gather_volume(torch.from_numpy(img[:60, :60].copy()).cuda(),
                        torch.from_numpy(idx).cuda(), 8)


@pytest.mark.parametrize("H,W,s,r,K", [(256, 320, 3, 32, 32), (200, 256, 2, 32, 64), (160, 160, 1, 24, 16)])
def test_groups_parity_wide_windows(H, W, s, r, K):
    """Wide windows and dense grids: a chunk's candidate bounding box exceeds the staging
    buffer, so the kernel retries the chunk's references in halves (down to one reference
    with global loads); the groups must still be exact."""
    g = _g()
    img = config_images(CONFIGS["c3"])[0][:H, :W].copy()
    idx, _, _ = oracle.block_match(img, 8, s, r, K, None)
    got = g.gather_groups(torch.from_numpy(img).cuda(), torch.from_numpy(idx).cuda(), 8)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy(), oracle.gather_groups(img, idx, 8))


def test_groups_parity_global_indices():
    """Indices from anywhere in the image (not a local search): the one-reference groups'
    boxes still exceed the buffer and the blocks come straight from global memory."""
    g = _g()
    rng = np.random.default_rng(5)
    img = rng.integers(-300, 300, (300, 280)).astype(np.int16)
    Ry, Rx, K = 40, 37, 32
    cy = rng.integers(0, 300 - 8 + 1, (Ry, Rx, K))
    cx = rng.integers(0, 280 - 8 + 1, (Ry, Rx, K))
    idx = (cy * 280 + cx).astype(np.int32)
    got = g.gather_groups(torch.from_numpy(img).cuda(), torch.from_numpy(idx).cuda(), 8)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy(), oracle.gather_groups(img, idx, 8))
