"""Pins for the CPU oracle (-m "not gpu").  Each test checks the oracle against something
other than itself: hand-worked fixtures, closed forms, a library routine (scipy cdist,
numpy lexsort), Eq. (2) in exact integers, invariants, and exhaustive
enumeration by the independent pure-Python twin.  A plausible mistake (dropped term,
wrong sign or index, transposed operand, off-by-one window, wrong tie order, <= vs <)
fails at least one of these."""
import itertools
import math

import numpy as np
import pytest

import oracle
from oracle import pyoracle
from synth import CONFIGS, config_images, special_image
from tests import golden_io


# ---------------------------------------------------------------- golden (hand-worked)
@pytest.mark.parametrize("ci", [0, 1, 2])
def test_hand_worked_fixture(ci):
    img, cases = golden_io.load("hand_3x3.txt")
    case = cases[ci]
    idx, dist, nv = oracle.block_match(img, case["patch"], case["stride"], case["radius"],
                                       case["K"], case["tau"])
    eidx, edist, env = golden_io.expected_arrays(case)
    np.testing.assert_array_equal(idx, eidx)
    np.testing.assert_array_equal(dist, edist)
    np.testing.assert_array_equal(nv, env)


# ---------------------------------------------------------------- grid / window closed forms
def _grid_count(L, P, s):
    return (L - P) // s + 1 + (1 if (L - P) % s else 0)


def _axis_window(p, last, r):
    return min(last, p + r) - max(0, p - r) + 1


def test_grid_counts_closed_form():
    # SURVEY 8(a) a1 counts: c0 400, c1 7056, c2 15876, c3 463761, c4 28561/img
    expect = {"c0": 400, "c1": 7056, "c2": 15876, "c3": 463761, "c4": 28561}
    for name, cfg in CONFIGS.items():
        P, s = cfg.calls[0].patch, cfg.calls[0].stride
        gy, gx = oracle.grid(cfg.H, P, s), oracle.grid(cfg.W, P, s)
        assert len(gy) * len(gx) == expect[name]
        assert len(gy) == _grid_count(cfg.H, P, s)
        # stride = patch on M with N | M reproduces the paper's (M/N)^2 tiles
    for M, N in [(64, 8), (256, 16), (48, 16)]:
        g = oracle.grid(M, N, N)
        assert list(g) == [p * N for p in range(M // N)]


def test_grid_edge_cases():
    assert list(oracle.grid(8, 8, 3)) == [0]
    assert list(oracle.grid(10, 8, 3)) == [0, 2]
    assert list(oracle.grid(11, 8, 3)) == [0, 3]
    assert list(oracle.grid(9, 2, 20)) == [0, 7]


def _total_evals(H, W, P, s, r):
    ys = [p for p in range(0, H - P + 1, s)] + ([H - P] if (H - P) % s else [])
    xs = [p for p in range(0, W - P + 1, s)] + ([W - P] if (W - P) % s else [])
    wy = [_axis_window(p, H - P, r) for p in ys]
    wx = [_axis_window(p, W - P, r) for p in xs]
    return sum(a * b - 1 for a in wy for b in wx)


def test_eval_counts_closed_form_vs_survey():
    # evals excluding self
    expect = {"c0": 401_556, "c1": 9_789_844, "c2": 23_062_540, "c3": 697_499_800,
              "c4": 2_661_557_760}
    for name, cfg in CONFIGS.items():
        c = cfg.calls[0]
        assert _total_evals(cfg.H, cfg.W, c.patch, c.stride, c.radius) * cfg.B == expect[name]


def test_window_clamp_counts_c0():
    """With K larger than any window and no tau, n_valid = |C(rho)| (clamped window, R2)."""
    img = config_images("c0")[0]
    c = CONFIGS["c0"].calls[0]
    _, _, nv = oracle.block_match(img, c.patch, c.stride, c.radius, 2000, None)
    assert int((nv - 1).sum()) == 401_556
    gy, gx = oracle.grid(64, 8, 3), oracle.grid(64, 8, 3)
    for py, ry in enumerate(gy):
        for px, rx in enumerate(gx):
            assert nv[py, px] == _axis_window(ry, 56, 19) * _axis_window(rx, 56, 19)


# ---------------------------------------------------------------- exhaustive pure-Python twin
def _py_arrays(img, P, s, r, K, tau):
    table, nvalid = pyoracle.block_match(img.tolist(), P, s, r, K, tau)
    idx = np.array([[[e[0] for e in ref] for ref in row] for row in table], np.int32)
    dist = np.array([[[e[1] for e in ref] for ref in row] for row in table], np.int32)
    return idx, dist, np.array(nvalid, np.int32)


def _fuzz_cases(n, seed):
    rng = np.random.default_rng(seed)
    for _ in range(n):
        P = int(rng.integers(1, 6))
        H = int(rng.integers(P, 19))
        W = int(rng.integers(P, 19))
        s = int(rng.integers(1, 6))
        r = int(rng.integers(0, 9))
        K = int(rng.integers(1, 21))
        lo, hi = sorted(int(v) for v in rng.integers(-300, 600, size=2))
        img = rng.integers(lo, hi + 1, size=(H, W)).astype(np.int16)
        mode = int(rng.integers(0, 3))
        tau = None if mode == 0 else (0 if mode == 1 else int(rng.integers(0, 4 * P * P * 100 + 1)))
        yield img, P, s, r, K, tau


@pytest.mark.parametrize("seed", range(6))
def test_exhaustive_python_twin(seed):
    for img, P, s, r, K, tau in _fuzz_cases(8, seed):
        got = oracle.block_match(img, P, s, r, K, tau)
        exp = _py_arrays(img, P, s, r, K, tau)
        for g, e in zip(got, exp):
            np.testing.assert_array_equal(g, e)


def test_int16_extremes_within_precondition():
    # P^2 (max-min)^2 <= 2^31-1  ->  P=2: max-min <= 23170
    rng = np.random.default_rng(5)
    img = rng.choice(np.array([-11585, 11585, 0, 11000], np.int16), size=(9, 11))
    for P, s, r, K in [(2, 1, 3, 6), (2, 2, 9, 40)]:
        got = oracle.block_match(img, P, s, r, K, None)
        exp = _py_arrays(img, P, s, r, K, None)
        for g, e in zip(got, exp):
            np.testing.assert_array_equal(g, e)
    assert int(oracle.block_match(img, 2, 1, 3, 6)[1].max()) <= 2**31 - 1


def test_overflow_detected():
    img = np.array([[-32768, 32767], [32767, -32768], [0, 0]], np.int16)
    with pytest.raises(OverflowError):
        oracle.block_match(img, 2, 1, 1, 2)


# ---------------------------------------------------------------- library routine: scipy cdist
def _all_patches(img, P):
    H, W = img.shape
    v = np.lib.stride_tricks.sliding_window_view(img.astype(np.float64), (P, P))
    return v.reshape((H - P + 1) * (W - P + 1), P * P)


@pytest.mark.parametrize("shape,P,s,r,K,tau", [
    ((20, 24), 4, 2, 5, 12, None), ((17, 23), 3, 3, 6, 40, 2000), ((25, 19), 5, 1, 4, 7, None),
    ((30, 30), 8, 3, 19, 16, None)])
def test_scipy_cdist_and_lexsort(shape, P, s, r, K, tau):
    from scipy.spatial.distance import cdist
    img = special_image("uniform", *shape, seed=11, lo=-200, hi=400)
    H, W = shape
    idx, dist, nv = oracle.block_match(img, P, s, r, K, tau)
    pv = _all_patches(img, P)                     # float64 is exact below 2^53
    nx = W - P + 1
    gy, gx = oracle.grid(H, P, s), oracle.grid(W, P, s)
    refs = [(ry, rx) for ry in gy for rx in gx]
    D = cdist(pv[[ry * nx + rx for ry, rx in refs]], pv, "sqeuclidean")
    cy, cx = np.divmod(np.arange(pv.shape[0]), nx)
    for n, (ry, rx) in enumerate(refs):
        m = (np.abs(cy - ry) <= r) & (np.abs(cx - rx) <= r) & ~((cy == ry) & (cx == rx))
        d = D[n][m]
        if tau is not None:
            keep = d < tau
        else:
            keep = np.ones_like(d, bool)
        cand_idx = (cy[m] * W + cx[m])[keep]
        cand_d = d[keep].astype(np.int64)
        order = np.lexsort((cand_idx, cand_d))[: K - 1]
        py, px = divmod(n, len(gx))
        exp_i = [ry * W + rx] + list(cand_idx[order])
        exp_d = [0] + list(cand_d[order])
        nvalid = len(exp_i)
        exp_i += [ry * W + rx] * (K - nvalid)
        exp_d += [-1] * (K - nvalid)
        np.testing.assert_array_equal(idx[py, px], exp_i)
        np.testing.assert_array_equal(dist[py, px], exp_d)
        assert nv[py, px] == nvalid


# ---------------------------------------------------------------- Eq. (2) in exact integers
def test_eq2_expansion_exact():
    """||f-g||^2 = ||f||^2 + ||g||^2 - 2<f,g> on every listed pair."""
    img = config_images("c0")[0]
    P = 8
    idx, dist, nv = oracle.block_match(img, P, 3, 19, 16)
    H, W = img.shape
    gy, gx = oracle.grid(H, P, 3), oracle.grid(W, P, 3)
    Z = img.astype(np.int64)
    for py, ry in enumerate(gy):
        for px, rx in enumerate(gx):
            f = Z[ry:ry + P, rx:rx + P]
            for k in range(nv[py, px]):
                cy, cx = divmod(int(idx[py, px, k]), W)
                g = Z[cy:cy + P, cx:cx + P]
                assert dist[py, px, k] == (f * f).sum() + (g * g).sum() - 2 * (f * g).sum()


def test_patch_ssd_symmetry_and_self():
    img = special_image("uniform", 12, 13, seed=3)
    for (a, b) in itertools.product([(0, 0), (3, 4), (5, 9)], repeat=2):
        assert oracle.patch_ssd(img, a, b, 4) == oracle.patch_ssd(img, b, a, 4)
        if a == b:
            assert oracle.patch_ssd(img, a, b, 4) == 0


# ---------------------------------------------------------------- closed forms
def test_constant_image_tie_order():
    """All d = 0: self, then the first K-1 window positions in raster order (R4, R5)."""
    img = special_image("constant", 40, 37, value=9)
    P, s, r, K = 8, 3, 5, 16
    idx, dist, nv = oracle.block_match(img, P, s, r, K)
    H, W = img.shape
    for py, ry in enumerate(oracle.grid(H, P, s)):
        for px, rx in enumerate(oracle.grid(W, P, s)):
            win = [cy * W + cx for cy in range(max(0, ry - r), min(H - P, ry + r) + 1)
                   for cx in range(max(0, rx - r), min(W - P, rx + r) + 1)
                   if (cy, cx) != (ry, rx)]
            exp = [ry * W + rx] + win[:K - 1]
            assert list(idx[py, px, :len(exp)]) == exp
            assert np.all(dist[py, px, :len(exp)] == 0)


def test_periodic_image_lattice_matches():
    """Z[y][x] = T[y%p][x%p], distinct T, P >= p: d = 0 exactly on the lattice (a p, b p)."""
    p, P, s, r = 5, 6, 3, 11
    img = special_image("periodic", 41, 44, period=p)
    H, W = img.shape
    K = 64
    idx, dist, nv = oracle.block_match(img, P, s, r, K)
    for py, ry in enumerate(oracle.grid(H, P, s)):
        for px, rx in enumerate(oracle.grid(W, P, s)):
            lat = [cy * W + cx for cy in range(max(0, ry - r), min(H - P, ry + r) + 1)
                   for cx in range(max(0, rx - r), min(W - P, rx + r) + 1)
                   if (cy, cx) != (ry, rx) and (cy - ry) % p == 0 and (cx - rx) % p == 0]
            n = len(lat)
            assert list(idx[py, px, 1:1 + n]) == lat
            assert np.all(dist[py, px, 1:1 + n] == 0)
            assert np.all(dist[py, px, 1 + n:nv[py, px]] > 0)


def test_two_identical_halves():
    """an image made of two identical halves matches across the seam with d=0."""
    rng = np.random.default_rng(4)
    half = rng.integers(0, 255, size=(8, 8)).astype(np.int16)
    img = np.concatenate([half, half], axis=1)
    idx, dist, nv = oracle.block_match(img, 4, 4, 8, 4)
    # ref (0,0) -> (0,8) at d=0 is its best match (distinct random halves elsewhere)
    assert idx[0, 0, 1] == 8 and dist[0, 0, 1] == 0
    assert idx[0, 2, 1] == 0 and dist[0, 2, 1] == 0


def test_single_tile_constant_pads_with_reference():
    """16x16 constant, N=16, K=16 -> one tile, reference repeated (padding)."""
    img = special_image("constant", 16, 16, value=3)
    idx, dist, nv = oracle.block_match(img, 16, 16, 19, 16)
    assert idx.shape == (1, 1, 16)
    assert np.all(idx == 0) and dist[0, 0, 0] == 0 and np.all(dist[0, 0, 1:] == -1)
    assert nv[0, 0] == 1


@pytest.mark.parametrize("K,r,tau", [(1, 19, None), (16, 0, None), (16, 19, 0)])
def test_degenerate_parameters(K, r, tau):
    """K=1 -> self only; r=0 -> self only; tau=0 -> nothing passes the strict cut."""
    img = config_images("c0")[0]
    idx, dist, nv = oracle.block_match(img, 8, 3, r, K, tau)
    assert np.all(nv == 1)
    W = img.shape[1]
    gy, gx = oracle.grid(64, 8, 3), oracle.grid(64, 8, 3)
    self_idx = (gy[:, None] * W + gx[None, :]).astype(np.int32)
    np.testing.assert_array_equal(idx[..., 0], self_idx)
    assert np.all(dist[..., 0] == 0)
    if K > 1:
        np.testing.assert_array_equal(idx[..., 1:], np.repeat(self_idx[..., None], K - 1, -1))
        assert np.all(dist[..., 1:] == -1)


# ---------------------------------------------------------------- invariants
def test_symmetry_global_search():
    """d(p,q) = d(q,p): with stride 1 and a global window every pair appears both ways."""
    img = special_image("uniform", 10, 9, seed=8)
    P = 3
    H, W = img.shape
    n = (H - P + 1) * (W - P + 1)
    idx, dist, nv = oracle.block_match(img, P, 1, max(H, W), n)
    nx = W - P + 1
    M = {}
    for py in range(H - P + 1):
        for px in range(nx):
            a = py * W + px
            for k in range(nv[py, px]):
                M[(a, int(idx[py, px, k]))] = int(dist[py, px, k])
    assert len(M) == n * n
    for (a, b), d in M.items():
        assert M[(b, a)] == d


def test_ordering_threshold_completeness_c1():
    """c1 (stage-1 call): ranks ascending by (d, idx), all kept d < tau, and completeness:
    every window candidate not kept has key > last kept key (checked by direct Eq. (1))."""
    img = config_images("c1")[0][:80, :80]
    c = CONFIGS["c1"].calls[0]
    idx, dist, nv = oracle.block_match(img, c.patch, c.stride, c.radius, c.K, c.tau)
    H, W = img.shape
    gy, gx = oracle.grid(H, c.patch, c.stride), oracle.grid(W, c.patch, c.stride)
    rng = np.random.default_rng(0)
    for py, px in zip(rng.integers(0, len(gy), 40), rng.integers(0, len(gx), 40)):
        n = nv[py, px]
        keys = [(int(dist[py, px, k]), int(idx[py, px, k])) for k in range(1, n)]
        assert keys == sorted(keys)
        assert all(d < c.tau for d, _ in keys)
        ry, rx = gy[py], gx[px]
        kept = set(i for _, i in keys)
        for cy in range(max(0, ry - c.radius), min(H - c.patch, ry + c.radius) + 1):
            for cx in range(max(0, rx - c.radius), min(W - c.patch, rx + c.radius) + 1):
                i = cy * W + cx
                if (cy, cx) == (ry, rx) or i in kept:
                    continue
                d = oracle.patch_ssd(img, (ry, rx), (cy, cx), c.patch)
                if d < c.tau and n == c.K:
                    assert (d, i) > keys[-1]
                elif d < c.tau:
                    pytest.fail("a passing candidate was dropped while slots were free")


def test_fft_cross_correlation_loose_check():
    """Prop. 1 + Eq. (2) via the Fourier identity: correlating the zero-
    padded reference block with the image gives <f, g> at every candidate; rounding the
    floating-point distances recovers the oracle's integers."""
    img = special_image("uniform", 32, 32, seed=2, lo=0, hi=255).astype(np.int64)
    P, r = 8, 6
    idx, dist, nv = oracle.block_match(img.astype(np.int16), P, 8, r, 200)
    M = 32
    F = img.astype(np.float64)
    ones = np.zeros((M, M)); ones[:P, :P] = 1
    norms = np.real(np.fft.ifft2(np.conj(np.fft.fft2(ones)) * np.fft.fft2(F * F)))
    for py, ry in enumerate(oracle.grid(M, P, 8)):
        for px, rx in enumerate(oracle.grid(M, P, 8)):
            G = np.zeros((M, M)); G[:P, :P] = F[ry:ry + P, rx:rx + P]
            ip = np.real(np.fft.ifft2(np.conj(np.fft.fft2(G)) * np.fft.fft2(F)))
            for k in range(nv[py, px]):
                cy, cx = divmod(int(idx[py, px, k]), M)
                d = norms[ry, rx] + norms[cy, cx] - 2 * ip[cy, cx]
                assert abs(d - dist[py, px, k]) < 1e-6 * max(1.0, abs(d)) + 1e-3
                assert math.isclose(round(d), dist[py, px, k])


def test_refs_entry_matches_whole_image():
    """The per-reference entry (used for sampled full-size checks) equals the whole-image
    routine cell by cell (both are the literal definition)."""
    img = config_images("c1")[0][:100, :90]
    idx, dist, nv = oracle.block_match(img, 8, 3, 19, 32, 25600 * 4)
    rng = np.random.default_rng(1)
    py = rng.integers(0, idx.shape[0], 50)
    px = rng.integers(0, idx.shape[1], 50)
    i2, d2, n2 = oracle.block_match_refs(img, 8, 3, 19, 32, 25600 * 4, py, px)
    np.testing.assert_array_equal(i2, idx[py, px])
    np.testing.assert_array_equal(d2, dist[py, px])
    np.testing.assert_array_equal(n2, nv[py, px])
