"""ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain CPU reference for G-BM3D block matching (arXiv 2103.10765).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import this package.  The product path (``paper_2103_10765_b200``) never does,
and this package never imports the product path: the two share no code.

* ``block_match`` -- the C direct loop (``gbm3d_oracle.c``; OpenMP over reference rows).
* ``pyoracle``     -- the same definition in pure Python, for exhaustive tiny checks.

Every function cites the PAPER.md passage it follows; ambiguities use the DESIGN.md
readings R1..R17.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gbm3d_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

ORACLE_ERR_RANGE = -2


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (plain -O2 -fopenmp, no -march: the .so travels to
    the GPU box whose host CPU may differ).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c99",
                               "-Wall", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            i32p = ctypes.POINTER(ctypes.c_int32)
            lib.oracle_block_match.argtypes = [
                ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                ctypes.c_int, ctypes.c_int, ctypes.c_int64, i32p, i32p, i32p, ctypes.c_int]
            lib.oracle_block_match.restype = ctypes.c_int
            lib.oracle_block_match_refs.argtypes = [
                ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                ctypes.c_int, ctypes.c_int, ctypes.c_int64, i32p, i32p, ctypes.c_int, i32p, i32p,
                i32p, ctypes.c_int]
            lib.oracle_block_match_refs.restype = ctypes.c_int
            lib.oracle_grid.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_int)]
            lib.oracle_grid.restype = ctypes.c_int
            lib.oracle_patch_ssd.argtypes = [ctypes.c_void_p] + [ctypes.c_int] * 6
            lib.oracle_patch_ssd.restype = ctypes.c_int64
            lib.oracle_max_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def grid(L: int, P: int, s: int) -> np.ndarray:
    """Reference positions along one axis (step 1, reading R3)."""
    lib = _load()
    n = lib.oracle_grid(L, P, s, None)
    out = (ctypes.c_int * max(n, 1))()
    lib.oracle_grid(L, P, s, out)
    return np.array(out[:n], dtype=np.int64)


def patch_ssd(img: np.ndarray, a: tuple, b: tuple, P: int) -> int:
    """Eq. (1) for one pair of top-left positions."""
    img = np.ascontiguousarray(img, dtype=np.int16)
    return int(_load().oracle_patch_ssd(img.ctypes.data, img.shape[1], a[0], a[1], b[0], b[1], P))


def block_match(img: np.ndarray, patch: int, stride: int, radius: int, K: int,
                tau: Optional[int] = None, threads: int = 0):
    """S^K_pq on the local window with Eq. (1)'s cut
     and P:134's padding.  Returns (idx, dist, n_valid) int32 arrays of
    shapes [Ry, Rx, K], [Ry, Rx, K], [Ry, Rx].  ``tau=None`` = no threshold."""
    img = np.ascontiguousarray(img, dtype=np.int16)
    if img.ndim != 2:
        raise ValueError("oracle.block_match takes one [H, W] image")
    H, W = img.shape
    lib = _load()
    Ry = lib.oracle_grid(H, patch, stride, None)
    Rx = lib.oracle_grid(W, patch, stride, None)
    if Ry == 0 or Rx == 0:
        raise ValueError("image smaller than the patch")
    idx = np.empty((Ry, Rx, K), dtype=np.int32)
    dist = np.empty((Ry, Rx, K), dtype=np.int32)
    nv = np.empty((Ry, Rx), dtype=np.int32)
    i32p = ctypes.POINTER(ctypes.c_int32)
    st = lib.oracle_block_match(
        img.ctypes.data, H, W, patch, stride, radius, K, -1 if tau is None else int(tau),
        idx.ctypes.data_as(i32p), dist.ctypes.data_as(i32p), nv.ctypes.data_as(i32p), int(threads))
    if st == ORACLE_ERR_RANGE:
        raise OverflowError("a patch distance exceeds INT32_MAX (outside the int32 domain, R10)")
    if st != 0:
        raise RuntimeError(f"oracle_block_match failed: {st}")
    return idx, dist, nv


def block_match_refs(img: np.ndarray, patch: int, stride: int, radius: int, K: int,
                     tau: Optional[int], py, px, threads: int = 0):
    """The definition for selected reference grid cells (py[i], px[i]) only.
    Returns (idx [n, K], dist [n, K], n_valid [n])."""
    img = np.ascontiguousarray(img, dtype=np.int16)
    H, W = img.shape
    py = np.ascontiguousarray(py, dtype=np.int32)
    px = np.ascontiguousarray(px, dtype=np.int32)
    n = len(py)
    idx = np.empty((n, K), np.int32)
    dist = np.empty((n, K), np.int32)
    nv = np.empty((n,), np.int32)
    i32p = ctypes.POINTER(ctypes.c_int32)
    st = _load().oracle_block_match_refs(
        img.ctypes.data, H, W, patch, stride, radius, K, -1 if tau is None else int(tau),
        py.ctypes.data_as(i32p), px.ctypes.data_as(i32p), n, idx.ctypes.data_as(i32p),
        dist.ctypes.data_as(i32p), nv.ctypes.data_as(i32p), int(threads))
    if st == ORACLE_ERR_RANGE:
        raise OverflowError("a patch distance exceeds INT32_MAX (outside the int32 domain, R10)")
    if st != 0:
        raise RuntimeError(f"oracle_block_match_refs failed: {st}")
    return idx, dist, nv


def block_match_batched(imgs: np.ndarray, patch: int, stride: int, radius: int, K: int,
                        tau: Optional[int] = None, threads: int = 0):
    outs = [block_match(im, patch, stride, radius, K, tau, threads) for im in imgs]
    return tuple(np.stack([o[i] for o in outs]) for i in range(3))


def gather_groups(img: np.ndarray, idx: np.ndarray, patch: int) -> np.ndarray:
    """The matched blocks of every reference, stacked as the paper's 5D tensor "N x N x K x B x B"
    (the blocks of S^K_pq): out[.., r, k] = Z[cy:cy+N, cx:cx+N] with
    (cy, cx) = divmod(idx[.., r, k], W).  Written as the plain slice copy it is."""
    img = np.asarray(img)
    idx = np.asarray(idx)
    batched = img.ndim == 3
    imgs = img if batched else img[None]
    tabs = idx if batched else idx[None]
    B, H, W = imgs.shape
    out = np.zeros(tabs.shape + (patch, patch), dtype=np.int16)
    for b in range(B):
        flat = tabs[b].reshape(-1)
        o = out[b].reshape(-1, patch, patch)
        for n, c in enumerate(flat):
            cy, cx = divmod(int(c), W)
            o[n] = imgs[b, cy:cy + patch, cx:cx + patch]
    return out if batched else out[0]


def gather_volume(img: np.ndarray, idx: np.ndarray, patch: int) -> np.ndarray:
    """The aggregated 3D volume of matched blocks, for tiling references
    (stride = N, N | M): V[p N + i, q N + j, z] = Z_x[i, j] with x the z-th match of tile (p, q).
    Returned slice-major: out[.., z, y, x] = V[y, x, z]."""
    img = np.asarray(img)
    idx = np.asarray(idx)
    batched = img.ndim == 3
    imgs = img if batched else img[None]
    tabs = idx if batched else idx[None]
    B, H, W = imgs.shape
    N = patch
    K = tabs.shape[-1]
    V = np.zeros((B, H, W, K), dtype=np.int16)  # the paper's index order [x, y, z]
    for b in range(B):
        for p in range(H // N):
            for q in range(W // N):
                for z in range(K):
                    cy, cx = divmod(int(tabs[b, p, q, z]), W)
                    V[b, p * N:(p + 1) * N, q * N:(q + 1) * N, z] = imgs[b, cy:cy + N, cx:cx + N]
    out = np.ascontiguousarray(np.moveaxis(V, 3, 1))
    return out if batched else out[0]
