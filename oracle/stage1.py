"""ORACLE -- TEST INFRASTRUCTURE ONLY.  Stage-1 global volume hard thresholding of G-BM3D
(SURVEY.md 8f-4), float64, written step by step in the paper's order.

PAPER.md:132-149 (section "Global Volume Hard Thresholding") and :154-206 (formal details):
  V      the volume of matched blocks of the tiling references (slice 0 = Z),
  U_h    = S_-h T3D^-1( Upsilon( T3D( S_h V ) ) ),
  U      = (1/H) sum_h U_h, H = 2, h = 0, 1,
  w_pq   = 1 / TV(U_pq),
  Y(x)   = sum w_pq U_pq^x(x) / sum w_pq chi_x(x)        (PAPER.md:190; pads left out, :142),
  Y_f    = (1/H) sum_h S_-h phi(S_h Z)                   (translation trials).
Parameters: 2D biorthogonal 1.5 wavelets in space, Haar along the group,
3 levels, hard thresholds lambda_l = sigma (3.6 - 0.3 l).  Readings S1-S7 in DESIGN.md.

Only tests/ use this; the CUDA path shares no code with it.
"""
from __future__ import annotations

import math

import numpy as np

import oracle

# bior1.5 (Cohen-Daubechies-Feauveau, box synthesis scaling function): analysis lowpass on
# n = -4..5, synthesis lowpass = Haar on n = 0, 1; highpasses by the biorthogonal QMF relations
# g~[n] = (-1)^n h[1-n] (analysis), g[n] = (-1)^n h~[1-n] (synthesis).
_S2 = math.sqrt(2.0)
H_AN = {n: v * _S2 / 256.0 for n, v in zip(range(-4, 6), (3, -3, -22, 22, 128, 128, 22, -22, -3, 3))}
H_SY = {0: 1.0 / _S2, 1: 1.0 / _S2}
G_AN = {n: ((-1) ** n) * H_SY.get(1 - n, 0.0) for n in range(0, 2)}
G_SY = {n: ((-1) ** n) * H_AN.get(1 - n, 0.0) for n in range(-4, 6)}


def dwt1(x: np.ndarray, axis: int):
    """One analysis level along `axis`, periodic: a[k] = sum_n h~[n] x[2k+n],
    d[k] = sum_n g~[n] x[2k+n] (indices mod the length)."""
    x = np.moveaxis(np.asarray(x, dtype=np.float64), axis, 0)
    M = x.shape[0]
    k = np.arange(M // 2)
    a = sum(v * x[(2 * k + n) % M] for n, v in H_AN.items())
    d = sum(v * x[(2 * k + n) % M] for n, v in G_AN.items())
    return np.moveaxis(a, 0, axis), np.moveaxis(d, 0, axis)


def idwt1(a: np.ndarray, d: np.ndarray, axis: int) -> np.ndarray:
    """Synthesis: x[2k+n] += h[n] a[k] + g[n] d[k] (periodic)."""
    a = np.moveaxis(np.asarray(a, dtype=np.float64), axis, 0)
    d = np.moveaxis(np.asarray(d, dtype=np.float64), axis, 0)
    half = a.shape[0]
    M = 2 * half
    x = np.zeros((M,) + a.shape[1:])
    k = np.arange(half)
    # for a fixed tap n the targets (2k + n) mod M, k < M/2, are distinct: one vector update each
    for n, v in H_SY.items():
        x[(2 * k + n) % M] += v * a
    for n, v in G_SY.items():
        x[(2 * k + n) % M] += v * d
    return np.moveaxis(x, 0, axis)


def dwt2(img: np.ndarray, levels: int):
    """2D separable transform of the last two axes (rows then columns of the current LL band,
    Mallat), returned in the usual in-place layout: at level l the LL band of size (H/2^l,
    W/2^l) sits in the top-left corner, its details LH (top-right), HL (bottom-left), HH."""
    out = np.array(img, dtype=np.float64)
    h, w = out.shape[-2:]
    for _ in range(levels):
        band = out[..., :h, :w]
        a, d = dwt1(band, -1)               # along x
        lo = np.concatenate([a, d], axis=-1)
        a2, d2 = dwt1(lo, -2)               # along y
        out[..., :h, :w] = np.concatenate([a2, d2], axis=-2)
        h //= 2
        w //= 2
    return out


def idwt2(coef: np.ndarray, levels: int) -> np.ndarray:
    out = np.array(coef, dtype=np.float64)
    H, W = out.shape[-2:]
    for lev in range(levels, 0, -1):
        h, w = H >> (lev - 1), W >> (lev - 1)
        band = out[..., :h, :w]
        lo = idwt1(band[..., : h // 2, :], band[..., h // 2:, :], -2)
        out[..., :h, :w] = idwt1(lo[..., : w // 2], lo[..., w // 2:], -1)
    return out


def haar_z(V: np.ndarray, levels: int, inverse: bool = False) -> np.ndarray:
    """Orthonormal Haar along axis 0 with `levels` cascade levels, in-place lifting positions
    (level with stride s pairs entries i and i + s for i a multiple of 2s)."""
    X = np.array(V, dtype=np.float64)
    K = X.shape[0]
    strides = [1 << t for t in range(levels)]
    for s in (reversed(strides) if inverse else strides):
        for i in range(0, K, 2 * s):
            a, d = X[i].copy(), X[i + s].copy()
            X[i] = (a + d) / _S2
            X[i + s] = (a - d) / _S2
    return X


def spatial_level_map(H: int, W: int, levels: int) -> np.ndarray:
    """Level of every position of the in-place 2D layout: 1..L for the detail bands, L for the
    final LL band (reading S2), as an int array [H, W]."""
    lev = np.full((H, W), levels, dtype=np.int64)
    h, w = H, W
    for l in range(1, levels + 1):
        lev[:h, :w] = l
        h //= 2
        w //= 2
    lev[:h, :w] = levels  # LL_L
    return lev


def upsilon(T: np.ndarray, sigma: float, levels: int, lam_scale: float = 1.0,
            override=None) -> np.ndarray:
    """Upsilon on a coefficient volume T [K, H, W] in the in-place layout: keep |alpha| >= lambda
     with lambda_l = sigma (3.6 - 0.3 l) for the spatial level l of the
    coefficient (the final LL band counts as level L); the coefficients that are
    approximations both in space (LL_L) and along z are always kept (reading S2).
    ``override`` (tests only): (mask, keep) boolean arrays shaped like T; where mask is set the
    decision is taken from keep -- used to follow a second implementation's decisions on the
    coefficients that lie within rounding of their threshold (no arithmetic changes)."""
    K, H, W = T.shape
    lz = min(levels, int(math.log2(K)))
    lev = spatial_level_map(H, W, levels)
    lam = lam_scale * sigma * (3.6 - 0.3 * lev)
    keep = np.abs(T) >= lam[None]                        # Upsilon
    hL, wL = H >> levels, W >> levels
    zapprox = np.zeros(K, dtype=bool)
    zapprox[:: 1 << lz] = True
    keep[np.ix_(zapprox, np.arange(hL), np.arange(wL))] = True
    if override is not None:
        keep = np.where(override[0], override[1], keep)
    return np.where(keep, T, 0.0)


def w3d_threshold(V: np.ndarray, sigma: float, levels: int, lam_scale: float = 1.0,
                  override=None) -> np.ndarray:
    """T3D^-1( Upsilon( T3D(V) ) ) for one volume V [K, H, W] (readings S1, S2).  `lam_scale`
    (tests only) scales the thresholds, to find the decisions that sit within rounding of them."""
    K = V.shape[0]
    lz = min(levels, int(math.log2(K)))
    T = haar_z(dwt2(V, levels), lz)
    return idwt2(haar_z(upsilon(T, sigma, levels, lam_scale, override), lz, inverse=True), levels)


def spin_coefficients(V: np.ndarray, h: int, levels: int = 3) -> np.ndarray:
    """Tests only: the coefficients T3D(S_h V) that Upsilon sees in cycle spin h."""
    lz = min(levels, int(math.log2(V.shape[0])))
    return haar_z(dwt2(np.roll(V, (h, h, h), axis=(0, 1, 2)), levels), lz)


def threshold_margin(V: np.ndarray, sigma: float, levels: int = 3, shifts=(0, 1)) -> float:
    """Tests only: the smallest relative distance | |alpha| - lambda | / lambda over every
    thresholded coefficient of every cycle spin -- the precision a second implementation needs
    to take all of Upsilon's keep/zero decisions the same way."""
    K, H, W = V.shape
    lz = min(levels, int(math.log2(K)))
    lev = spatial_level_map(H, W, levels)
    lam = sigma * (3.6 - 0.3 * lev)
    best = math.inf
    for h in shifts:
        T = haar_z(dwt2(np.roll(V, (h, h, h), axis=(0, 1, 2)), levels), lz)
        rel = np.abs(np.abs(T) - lam[None]) / lam[None]
        hL, wL = H >> levels, W >> levels
        rel[:: 1 << lz, :hL, :wL] = np.inf  # always kept
        best = min(best, float(rel.min()))
    return best


def filter_volume(V: np.ndarray, sigma: float, levels: int = 3, shifts=(0, 1),
                  lam_scale: float = 1.0, overrides=None) -> np.ndarray:
    """U = (1/H) sum_h S_-h( T3D^-1 Upsilon T3D (S_h V) ), S_h = circular shift by h along all
    three axes (reading S3)."""
    acc = np.zeros(V.shape)
    for i, h in enumerate(shifts):
        Vh = np.roll(V, (h, h, h), axis=(0, 1, 2))
        ov = overrides[i] if overrides is not None else None
        acc += np.roll(w3d_threshold(Vh, sigma, levels, lam_scale, ov), (-h, -h, -h), axis=(0, 1, 2))
    return acc / len(shifts)


def tv3d(G: np.ndarray) -> float:
    """Anisotropic 3D total variation of a group [K, N, N]: sum of |forward differences| along
    the group axis and both block axes (reading S4)."""
    return float(np.abs(np.diff(G, axis=0)).sum() + np.abs(np.diff(G, axis=1)).sum()
                 + np.abs(np.diff(G, axis=2)).sum())


def stage1(noisy: np.ndarray, idx: np.ndarray, n_valid: np.ndarray, patch: int, sigma: float,
           levels: int = 3, shifts=(0, 1), lam_scale: float = 1.0, overrides=None) -> np.ndarray:
    """phi(Z) for tiling references (stride = N): the filtered volume's groups are aggregated
    at their blocks' positions with weights 1 / TV, first n_valid blocks."""
    H, W = noisy.shape
    N = patch
    V = oracle.gather_volume(noisy, idx, N).astype(np.float64)   # [K, H, W]
    U = filter_volume(V, sigma, levels, shifts, lam_scale, overrides)
    Ry, Rx, K = idx.shape
    num = np.zeros((H, W))
    den = np.zeros((H, W))
    for p in range(Ry):
        for q in range(Rx):
            G = U[:, p * N:(p + 1) * N, q * N:(q + 1) * N]
            tv = tv3d(G)
            w = 1.0 / tv if tv > 0 else 1.0
            for k in range(int(n_valid[p, q])):
                cy, cx = divmod(int(idx[p, q, k]), W)
                num[cy:cy + N, cx:cx + N] += w * G[k]
                den[cy:cy + N, cx:cx + N] += w
    return num / den


def translation_trials(noisy: np.ndarray, sigma: float, patch: int, K: int, radius: int,
                       trials=(0, 2, 4), levels: int = 3, shifts=(0, 1)) -> np.ndarray:
    """Y_f = (1/H) sum_h S_-h( phi(S_h Z) ) (Eq. (10)): phi = block matching
    of the shifted image on the tiling grid (stride = N) followed by stage1;
    S_h = circular shift of the image by h pixels along both axes (reading S8)."""
    acc = np.zeros(noisy.shape)
    for h in trials:
        Zh = np.roll(noisy, (h, h), axis=(0, 1))
        idx, _dist, nv = oracle.block_match(Zh, patch, patch, radius, K, None)
        acc += np.roll(stage1(Zh, idx, nv, patch, sigma, levels, shifts), (-h, -h), axis=(0, 1))
    return acc / len(trials)
