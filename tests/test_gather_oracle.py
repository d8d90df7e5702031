"""Pins for the oracle's matched-block gather (-m "not gpu").  The groups are
the 5D tensor of PAPER.md:217, the volume V of PAPER.md:160-164; the checks tie them to a
hand-worked case, to Eq. (1) through the matcher's own distances, to an independent numpy
formulation (sliding windows), and to the closed forms "slice 0 of V is Z" and "a periodic
image's volume repeats Z"."""
import numpy as np
import pytest
from numpy.lib.stride_tricks import sliding_window_view

import oracle
from synth import CONFIGS, config_images, special_image


def test_hand_worked_groups():
    # 4 x 4 image 0..15, patch 2; blocks at raster indices 0, 5, 10 and a pad (= self, 0)
    img = np.arange(16, dtype=np.int16).reshape(4, 4)
    idx = np.array([[[0, 5, 10, 0]]], dtype=np.int32)  # [Ry=1, Rx=1, K=4]
    g = oracle.gather_groups(img, idx, 2)
    assert g.shape == (1, 1, 4, 2, 2)
    np.testing.assert_array_equal(g[0, 0, 0], [[0, 1], [4, 5]])
    np.testing.assert_array_equal(g[0, 0, 1], [[5, 6], [9, 10]])
    np.testing.assert_array_equal(g[0, 0, 2], [[10, 11], [14, 15]])
    np.testing.assert_array_equal(g[0, 0, 3], g[0, 0, 0])


def test_hand_worked_volume():
    # 4 x 4 image, 2 x 2 tiles; tile (0,0) matched to the block at (1,1), tile (1,1) to (0,2)
    img = np.arange(16, dtype=np.int16).reshape(4, 4)
    idx = np.array([[[0, 5], [2, 2]], [[8, 8], [10, 2]]], dtype=np.int32)  # [2, 2, K=2]
    v = oracle.gather_volume(img, idx, 2)
    assert v.shape == (2, 4, 4)
    np.testing.assert_array_equal(v[0], img)
    expect1 = np.array([[5, 6, 2, 3], [9, 10, 6, 7], [8, 9, 2, 3], [12, 13, 6, 7]])
    np.testing.assert_array_equal(v[1], expect1)


@pytest.mark.parametrize("name,ci", [("c0", 0), ("c1", 0), ("c1", 1)])
def test_groups_reproduce_matched_distances(name, ci):
    """Eq. (1): the SSD between block k and block 0 of every group is the matcher's dist[k];
    block 0 is the reference block itself; pads repeat it."""
    cfg = CONFIGS[name]
    c = cfg.calls[ci]
    img = config_images(cfg)[0]
    idx, dist, nv = oracle.block_match(img, c.patch, c.stride, c.radius, c.K, c.tau)
    g = oracle.gather_groups(img, idx, c.patch).astype(np.int64)
    gy = oracle.grid(img.shape[0], c.patch, c.stride)
    gx = oracle.grid(img.shape[1], c.patch, c.stride)
    ref = np.stack([np.stack([img[y:y + c.patch, x:x + c.patch] for x in gx]) for y in gy])
    np.testing.assert_array_equal(g[:, :, 0], ref)
    ssd = ((g - g[:, :, :1]) ** 2).sum(axis=(-1, -2))
    valid = np.arange(c.K)[None, None, :] < nv[..., None]
    np.testing.assert_array_equal(ssd[valid], dist[valid])
    np.testing.assert_array_equal(ssd[~valid], 0)


def test_groups_match_sliding_window_formulation():
    """Independent numpy formulation: sliding_window_view(Z, (N, N))[cy, cx] is Z_x."""
    cfg = CONFIGS["c0"]
    img = config_images(cfg)[0]
    rng = np.random.default_rng(5)
    P = 8
    idx = (rng.integers(0, 64 - P + 1, (20, 20, 16)) * 64 +
           rng.integers(0, 64 - P + 1, (20, 20, 16))).astype(np.int32)
    g = oracle.gather_groups(img, idx, P)
    swv = sliding_window_view(img, (P, P))
    np.testing.assert_array_equal(g, swv[idx // 64, idx % 64])


def test_volume_slice0_is_the_image_and_slices_are_groups():
    """Tiling references (stride = N): slot 0 is the tile itself, so V[.., 0] = Z (PAPER.md:162
    with z = the reference); every slice places group block k at its tile."""
    img = config_images(CONFIGS["c1"])[0][:128, :128].copy()
    N = 8
    idx, dist, nv = oracle.block_match(img, N, N, 11, 8, None)
    v = oracle.gather_volume(img, idx, N)
    np.testing.assert_array_equal(v[0], img)
    g = oracle.gather_groups(img, idx, N)
    for k in range(8):
        tiles = v[k].reshape(16, N, 16, N).transpose(0, 2, 1, 3)
        np.testing.assert_array_equal(tiles, g[:, :, k])


def test_volume_of_periodic_image_repeats_it():
    """An N-periodic image has d = 0 at every lattice displacement, so all K matches of a tile
    are copies of it and every slice of V equals Z."""
    N = 8
    img = special_image("periodic", 64, 64, period=N)
    idx, dist, nv = oracle.block_match(img, N, N, 16, 8, None)
    assert (dist[nv > 0] >= 0).all() and (dist[:, :, :8] == 0).all()
    v = oracle.gather_volume(img, idx, N)
    for k in range(8):
        np.testing.assert_array_equal(v[k], img)
