"""Pins for the oracle's stage-2 Wiener filtering (-m "not gpu"): the DCT
against scipy's orthonormal DCT-II, the Haar cascade against a hand-worked case, the shrinkage
against the closed forms of SPEC's examples (sigma = 0 is the identity; T_B = sigma halves a
coefficient), invariants (0 <= W <= 1, energy contraction, orthonormality), and aggregation
closed forms (identity filter reproduces the image; constant images stay constant)."""
import math

import numpy as np
import pytest
import scipy.fft

import oracle
from oracle import wiener
from synth import CONFIGS, make_image


@pytest.mark.parametrize("n", [2, 4, 8, 16])
def test_dct_matches_scipy_orthonormal_dct2(n):
    C = wiener.dct_matrix(n)
    np.testing.assert_allclose(C, scipy.fft.dct(np.eye(n), type=2, norm="ortho", axis=0),
                               atol=1e-14)
    np.testing.assert_allclose(C @ C.T, np.eye(n), atol=1e-14)


def test_haar_hand_worked_and_orthonormal():
    Hm = wiener.haar_matrix(4)
    s = 1 / math.sqrt(2)
    np.testing.assert_allclose(Hm @ np.array([1.0, 2, 3, 4]), [5, -2, -s, -s], atol=1e-14)
    for n in (1, 2, 8, 16, 32):
        Hn = wiener.haar_matrix(n)
        np.testing.assert_allclose(Hn @ Hn.T, np.eye(n), atol=1e-14)
        e = Hn @ np.ones(n)
        np.testing.assert_allclose(e, np.r_[math.sqrt(n), np.zeros(n - 1)], atol=1e-12)


def test_group_transform_round_trip_and_energy():
    rng = np.random.default_rng(0)
    G = rng.normal(0, 50, (16, 8, 8))
    T = wiener.transform_group(G)
    np.testing.assert_allclose(wiener.inverse_group(T), G, atol=1e-10)
    assert abs((T * T).sum() - (G * G).sum()) < 1e-6 * (G * G).sum()


def test_sigma_zero_with_basic_equal_noisy_is_identity():
    rng = np.random.default_rng(1)
    Gz = rng.integers(-100, 300, (16, 8, 8)).astype(np.float64)
    U, w = wiener.wiener_group(Gz, Gz, 0.0)
    np.testing.assert_allclose(U, Gz, atol=1e-10)
    assert w == 1.0


def test_coefficient_equal_to_sigma_is_halved():
    """Constant basic blocks c: T_B has one nonzero coefficient, c N sqrt(K) (DC x DC x scaling);
    with sigma equal to it, W = 1/2 there and 0 elsewhere, so a constant noisy group is halved."""
    K, N, c = 16, 8, 3.0
    Gb = np.full((K, N, N), c)
    sigma = c * N * math.sqrt(K)
    U, w = wiener.wiener_group(Gb.copy(), Gb, sigma)
    np.testing.assert_allclose(U, Gb / 2, atol=1e-12)
    assert abs(w - 1.0 / (sigma * sigma * 0.25)) < 1e-15


def test_shrinkage_bounds_and_contraction():
    rng = np.random.default_rng(2)
    for sigma in (5.0, 25.0, 60.0):
        Gz = rng.normal(100, 40, (32, 8, 8))
        Gb = Gz + rng.normal(0, 10, Gz.shape)
        Tz = wiener.transform_group(Gz)
        U, w = wiener.wiener_group(Gz, Gb, sigma)
        Tu = wiener.transform_group(U)
        Wsh = np.divide(Tu, Tz, out=np.zeros_like(Tu), where=np.abs(Tz) > 1e-6)
        assert Wsh.min() > -1e-9 and Wsh.max() < 1 + 1e-9
        assert (Tu * Tu).sum() <= (Tz * Tz).sum() + 1e-6
        assert w > 0


def _tables(img, P, s, r, K):
    return oracle.block_match(img, P, s, r, K, None)


def test_identity_filter_aggregation_reproduces_the_image():
    """sigma = 0, basic = noisy: every filtered block is the noisy block, so the weighted
    average over the blocks covering a pixel is the pixel itself."""
    img = make_image(40, 48, 6, 0, 25.0, 7)
    idx, dist, nv = _tables(img, 8, 3, 6, 8)
    Y = wiener.stage2(img, img.astype(np.float64), idx, nv, 8, 0.0)
    np.testing.assert_allclose(Y, img, atol=1e-9)


def test_constant_images_stay_constant():
    """A constant image c gives constant groups: their transform has only the DC x scaling
    coefficient T = c N sqrt(K), shrunk by W = T^2 / (T^2 + sigma^2); every block becomes c W
    and so does the estimate, everywhere."""
    c, K, N, sigma = 37.0, 8, 8, 25.0
    img = np.full((32, 32), int(c), dtype=np.int16)
    idx, dist, nv = _tables(img, N, 3, 5, K)
    Y = wiener.stage2(img, img.astype(np.float64), idx, nv, N, sigma)
    T = c * N * math.sqrt(K)
    np.testing.assert_allclose(Y, c * T * T / (T * T + sigma * sigma), atol=1e-9)


def test_pad_blocks_left_out():
    """tau = 0 leaves only the reference in every table (n_valid = 1): the estimate is then the
    plain average of the filtered reference blocks; with sigma = 0 it is the image."""
    img = make_image(32, 40, 4, 0, 25.0, 3)
    idx, dist, nv = oracle.block_match(img, 8, 3, 6, 8, 0)
    assert (nv == 1).all()
    Y = wiener.stage2(img, img.astype(np.float64), idx, nv, 8, 0.0)
    np.testing.assert_allclose(Y, img, atol=1e-9)


def test_denoises_with_clean_basic_estimate():
    """Sanity (not a pin): with the noise-free image as the basic estimate, the estimate is far
    closer to the clean image than the noisy input."""
    noisy, clean, sigma = make_image(64, 64, 6, 2, 25.0, 11, return_clean=True)
    idx, dist, nv = _tables(clean, 8, 3, 11, 16)
    Y = wiener.stage2(noisy, clean.astype(np.float64), idx, nv, 8, sigma)
    assert np.mean((Y - clean) ** 2) < 0.5 * np.mean((noisy.astype(np.float64) - clean) ** 2)
