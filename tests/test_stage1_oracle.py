"""Pins for the oracle's stage-1 global volume hard thresholding (-m "not gpu"):
the bior1.5 filter bank (normalisation, biorthogonality, perfect reconstruction, annihilation
of constants / ramps by the Haar analysis highpass), the Mallat layout and level map, the Haar
cascade, the threshold rule, the total variation on a hand-worked group, and closed forms of
the whole operator (sigma = 0 and constant images reproduce the image)."""
import math

import numpy as np
import pytest

import oracle
from oracle import stage1
from synth import make_image


def test_bior15_filters_normalised_and_biorthogonal():
    assert abs(sum(stage1.H_AN.values()) - math.sqrt(2)) < 1e-15
    assert abs(sum(stage1.H_SY.values()) - math.sqrt(2)) < 1e-15
    assert abs(sum(stage1.G_AN.values())) < 1e-15 and abs(sum(stage1.G_SY.values())) < 1e-15
    # sum_n h~[n] h[n + 2k] = delta_k  and  sum_n g~[n] g[n + 2k] = delta_k
    for k in range(-3, 4):
        lo = sum(v * stage1.H_SY.get(n + 2 * k, 0.0) for n, v in stage1.H_AN.items())
        hi = sum(v * stage1.G_SY.get(n + 2 * k, 0.0) for n, v in stage1.G_AN.items())
        assert abs(lo - (k == 0)) < 1e-15 and abs(hi - (k == 0)) < 1e-15


def test_dwt1_closed_forms_and_reconstruction():
    M = 32
    a, d = stage1.dwt1(np.full(M, 5.0), 0)
    np.testing.assert_allclose(a, 5 * math.sqrt(2), atol=1e-12)
    np.testing.assert_allclose(d, 0, atol=1e-15)
    ramp = np.arange(M, dtype=np.float64)
    a, d = stage1.dwt1(ramp, 0)
    np.testing.assert_allclose(d, -1 / math.sqrt(2), atol=1e-12)  # (x[2k] - x[2k+1]) / sqrt 2
    x = np.random.default_rng(0).normal(size=(M, 3))
    np.testing.assert_allclose(stage1.idwt1(*stage1.dwt1(x, 0), 0), x, atol=1e-12)


@pytest.mark.parametrize("levels", [1, 2, 3])
def test_dwt2_reconstruction_and_level_map(levels):
    X = np.random.default_rng(levels).normal(size=(4, 32, 48))
    C = stage1.dwt2(X, levels)
    np.testing.assert_allclose(stage1.idwt2(C, levels), X, atol=1e-10)
    lev = stage1.spatial_level_map(32, 48, levels)
    for l in range(1, levels + 1):
        n = (lev == l).sum()
        details = 3 * (32 * 48) // 4 ** l
        expect = details + (32 * 48 // 4 ** levels if l == levels else 0)
        assert n == expect


def test_haar_z_partial_depth():
    X = np.arange(8, dtype=np.float64)[:, None, None] * np.ones((1, 2, 2))
    T = stage1.haar_z(X, 2)
    s = math.sqrt(2)
    # level 1 pairs (0,1),(2,3),..; level 2 pairs the sums at 0 and 2, 4 and 6
    np.testing.assert_allclose(T[:, 0, 0], [3.0, -1 / s, -2.0, -1 / s, 11.0, -1 / s, -2.0, -1 / s],
                               atol=1e-12)
    np.testing.assert_allclose(stage1.haar_z(T, 2, inverse=True), X, atol=1e-12)


def test_tv3d_hand_worked():
    G = np.zeros((2, 2, 2))
    G[1, 1, 1] = 3.0
    assert stage1.tv3d(G) == 9.0   # one difference of 3 along each of the three axes
    G[0, 0, 0] = -1.0
    assert stage1.tv3d(G) == 12.0


def test_threshold_keeps_large_and_approximation():
    rng = np.random.default_rng(4)
    V = rng.normal(0, 1, (8, 16, 16))
    U = stage1.w3d_threshold(V, 1e6, 2)   # every detail coefficient under the threshold
    # only the (LL_2, z-approximation) coefficients survive: U is the projection on them
    T = stage1.haar_z(stage1.dwt2(V, 2), 2)
    keep = np.zeros_like(T)
    keep[::4, :4, :4] = T[::4, :4, :4]
    np.testing.assert_allclose(U, stage1.idwt2(stage1.haar_z(keep, 2, inverse=True), 2), atol=1e-10)
    np.testing.assert_allclose(stage1.w3d_threshold(V, 0.0, 2), V, atol=1e-10)


def _tables(img, N, r, K):
    return oracle.block_match(img, N, N, r, K, None)


def test_sigma_zero_reproduces_the_image():
    img = make_image(32, 48, 6, 1, 25.0, 5)
    idx, dist, nv = _tables(img, 8, 9, 8)
    Y = stage1.stage1(img, idx, nv, 8, 0.0)
    np.testing.assert_allclose(Y, img, atol=1e-9)


def test_constant_image_stays():
    img = np.full((32, 32), 41, dtype=np.int16)
    idx, dist, nv = _tables(img, 8, 8, 8)
    Y = stage1.stage1(img, idx, nv, 8, 25.0)
    np.testing.assert_allclose(Y, 41.0, atol=1e-9)


def test_denoises():
    """Sanity (not a pin): stage 1 removes a large part of the noise."""
    noisy, clean, sigma = make_image(64, 64, 6, 2, 25.0, 9, return_clean=True)
    idx, dist, nv = _tables(noisy, 8, 16, 16)
    Y = stage1.stage1(noisy, idx, nv, 8, sigma)
    assert np.mean((Y - clean) ** 2) < 0.6 * np.mean((noisy.astype(np.float64) - clean) ** 2)
