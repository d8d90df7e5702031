"""ORACLE -- TEST INFRASTRUCTURE ONLY.  Stage-2 collaborative Wiener filtering of the matched
groups and their aggregation, in float64, written as the definitions.

PAPER.md:210-217 (section "Second Wiener Filter Estimation"): the 3D transform is a 2D DCT in
the block coordinates and a 1D Haar wavelet transform along the group axis; all groups are
transformed at once as a 5D tensor N x N x K x B x B; "the filtering and aggregation rules in
this step match the original algorithm precisely".  The original rules (DESIGN.md readings
W1-W6, following SPEC.md's wiener_filter_groups):
  T = Haar_z o DCT2_xy on the group of the noisy image (T_Z) and of the basic estimate (T_B);
  shrinkage W = T_B^2 / (T_B^2 + sigma^2);  filtered group = T^-1(W . T_Z);
  group weight w = 1 / (sigma^2 ||W||_2^2);
  aggregation (with w_pq): Y(x) = sum_groups sum_blocks w U(x) / sum w chi(x),
  leaving out the pad blocks that fill groups with fewer than K matches.

Only tests/ and bench.py's cpu leg use this; the CUDA path shares no code with it.
"""
from __future__ import annotations

import math

import numpy as np


def dct_matrix(n: int) -> np.ndarray:
    """Orthonormal DCT-II: C[k, i] = a_k cos(pi (2 i + 1) k / (2 n)), a_0 = sqrt(1/n),
    a_k = sqrt(2/n) -- the 2D DCT of a block X is C X C^T."""
    C = np.zeros((n, n))
    for k in range(n):
        a = math.sqrt(1.0 / n) if k == 0 else math.sqrt(2.0 / n)
        for i in range(n):
            C[k, i] = a * math.cos(math.pi * (2 * i + 1) * k / (2 * n))
    return C


def haar_matrix(n: int) -> np.ndarray:
    """Orthonormal Haar transform of length n = 2^L at full dyadic depth, written as the
    usual cascade: at each level the current approximation a (length m) becomes
    [(a[2i] + a[2i+1]) / sqrt 2 ; (a[2i] - a[2i+1]) / sqrt 2] and the recursion continues on
    the first half.  Row 0 is the scaling function (constant 1/sqrt n)."""
    assert n >= 1 and (n & (n - 1)) == 0, "Haar length must be a power of two"
    Hm = np.eye(n)
    m = n
    while m > 1:
        step = np.eye(n)
        blk = np.zeros((m, m))
        s = 1.0 / math.sqrt(2.0)
        for i in range(m // 2):
            blk[i, 2 * i] = s
            blk[i, 2 * i + 1] = s
            blk[m // 2 + i, 2 * i] = s
            blk[m // 2 + i, 2 * i + 1] = -s
        step[:m, :m] = blk
        Hm = step @ Hm
        m //= 2
    return Hm


def transform_group(G: np.ndarray) -> np.ndarray:
    """T(G) for a group G[K, N, N]: DCT2 of every block, then Haar along the group axis."""
    K, N, _ = G.shape
    C = dct_matrix(N)
    Hk = haar_matrix(K)
    D = np.einsum("ki,zij,lj->zkl", C, G, C)
    return np.einsum("yz,zkl->ykl", Hk, D)


def inverse_group(T: np.ndarray) -> np.ndarray:
    K, N, _ = T.shape
    C = dct_matrix(N)
    Hk = haar_matrix(K)
    D = np.einsum("yz,ykl->zkl", Hk, T)  # Hk^T: the transform is orthonormal
    return np.einsum("ki,zkl,lj->zij", C, D, C)


def wiener_group(Gz: np.ndarray, Gb: np.ndarray, sigma: float):
    """One group: returns (filtered blocks [K, N, N], weight).  Readings (W3, W4):
    where T_B^2 + sigma^2 == 0 the shrinkage is 1 (the identity filter); a zero ||W||^2 or
    sigma == 0 gives weight 1."""
    Tz = transform_group(Gz.astype(np.float64))
    Tb = transform_group(Gb.astype(np.float64))
    den = Tb * Tb + sigma * sigma
    Wsh = np.where(den > 0, (Tb * Tb) / np.where(den > 0, den, 1.0), 1.0)
    U = inverse_group(Wsh * Tz)
    n2 = float((Wsh * Wsh).sum())
    w = 1.0 / (sigma * sigma * n2) if (sigma > 0 and n2 > 0) else 1.0
    return U, w


def stage2(noisy: np.ndarray, basic: np.ndarray, idx: np.ndarray, n_valid: np.ndarray,
           patch: int, sigma: float) -> np.ndarray:
    """The stage-2 estimate of one image from its match table idx [Ry, Rx, K] (the matches of
    every reference, slot 0 = the reference) and n_valid [Ry, Rx]: every group is Wiener
    filtered and its first n_valid blocks are aggregated with the group weight (
    pad blocks left out).  Returns float64 [H, W]."""
    H, W = noisy.shape
    N = patch
    Ry, Rx, K = idx.shape
    num = np.zeros((H, W))
    den = np.zeros((H, W))
    for ry in range(Ry):
        for rx in range(Rx):
            cy = idx[ry, rx] // W
            cx = idx[ry, rx] % W
            Gz = np.stack([noisy[cy[k]:cy[k] + N, cx[k]:cx[k] + N] for k in range(K)])
            Gb = np.stack([basic[cy[k]:cy[k] + N, cx[k]:cx[k] + N] for k in range(K)])
            U, w = wiener_group(Gz, Gb, sigma)
            for k in range(int(n_valid[ry, rx])):
                num[cy[k]:cy[k] + N, cx[k]:cx[k] + N] += w * U[k]
                den[cy[k]:cy[k] + N, cx[k]:cx[k] + N] += w
    return num / den
