"""Boundary checks that need no GPU: libgbm3d.so loads, exports every symbol include/gbm3d.h
declares, and host-side validation returns the documented codes without touching CUDA."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_2103_10765_b200 import build
    build.build()
    import paper_2103_10765_b200 as g
    return g, g.load_library()


def _declared():
    src = open(os.path.join(ROOT, "include", "gbm3d.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gbm3d_\w+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    g, lib = _lib()
    names = _declared()
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), n


def test_grid_dims_host():
    g, _ = _lib()
    assert g.grid_dims(64, 64, 8, 3) == (20, 20)
    assert g.grid_dims(2048, 2048, 8, 3) == (681, 681)
    assert g.grid_dims(512, 512, 12, 4) == (126, 126)
    with pytest.raises(g.GBM3DError):
        g.grid_dims(7, 64, 8, 3)


def test_argument_validation_before_any_device_work():
    """Bad arguments return GBM3D_ERR_ARG / UNSUPPORTED with nothing enqueued (no CUDA call
    is made, so this runs without a GPU)."""
    g, lib = _lib()
    dummy = ctypes.c_void_p(0x1000)
    null = ctypes.c_void_p(0)
    none = g.TAU_NONE
    f = lib.gbm3d_block_match_ex
    # (imgs, B, H, W, patch, stride, radius, K, tau, method, idx, dist, nv, stream)
    assert f(null, 1, 64, 64, 8, 3, 19, 16, none, 0, dummy, dummy, null, null) == -1
    assert f(dummy, 1, 64, 64, 8, 3, 19, 16, none, 0, null, dummy, null, null) == -1
    assert f(dummy, 0, 64, 64, 8, 3, 19, 16, none, 0, dummy, dummy, null, null) == -1
    assert f(dummy, 1, 7, 64, 8, 3, 19, 16, none, 0, dummy, dummy, null, null) == -1
    assert f(dummy, 1, 64, 64, 8, 0, 19, 16, none, 0, dummy, dummy, null, null) == -1
    assert f(dummy, 1, 64, 64, 8, 3, -1, 16, none, 0, dummy, dummy, null, null) == -1
    assert f(dummy, 1, 64, 64, 8, 3, 19, 0, none, 0, dummy, dummy, null, null) == -1
    assert f(dummy, 1, 64, 64, 8, 3, 19, 16, -5, 0, dummy, dummy, null, null) == -1
    assert f(dummy, 1, 64, 64, 8, 3, 19, 16, none, 9, dummy, dummy, null, null) == -1
    assert f(dummy, 1, 64, 64, 17, 3, 19, 16, none, 0, dummy, dummy, null, null) == -3
    assert f(dummy, 1, 64, 64, 8, 3, 33, 16, none, 0, dummy, dummy, null, null) == -3
    assert f(dummy, 1, 64, 64, 8, 3, 19, 65, none, 0, dummy, dummy, null, null) == -3
    assert f(dummy, 1, 1 << 16, 1 << 15, 8, 3, 19, 16, none, 0, dummy, dummy, null, null) == -1
    rows = lib.gbm3d_block_match_rows
    # slab lacks the halo rows needed by reference rows [10, 20) -> ERR_ARG
    assert rows(dummy, 10, 40, 200, 64, 8, 3, 19, 16, none, 10, 20, dummy, dummy, null,
                null) == -1
    assert rows(dummy, 0, 200, 200, 64, 8, 3, 19, 16, none, 20, 10, dummy, dummy, null,
                null) == -1
    assert lib.gbm3d_check_range(null, 10, 8, None, null) == -1
    assert lib.gbm3d_strerror(-2).decode().startswith("image range")
    assert "sm_100a" in g.version()


def test_host_workspace_size():
    g, _ = _lib()
    n = g.host_workspace_bytes(64, 512, 512, 8, 3, 16)
    assert n >= 64 * 512 * 512 * 2 + 2 * 64 * 169 * 169 * 16 * 4 + 64 * 169 * 169 * 4


def test_product_path_never_imports_oracle():
    """The product package must not reference the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2103_10765_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), fn
                assert "liboracle" not in txt and "gbm3d_oracle" not in txt, fn


def test_gather_argument_validation_host():
    """gather entries reject bad arguments before any CUDA call (runs without a GPU)."""
    g, lib = _lib()
    d = ctypes.c_void_p(0x1000)
    null = ctypes.c_void_p(0)
    G, V = lib.gbm3d_gather_groups, lib.gbm3d_gather_volume
    # (imgs, B, H, W, patch, idx, Ry, Rx, K, groups, stream)
    assert G(null, 1, 64, 64, 8, d, 20, 20, 16, d, null) == -1
    assert G(d, 1, 64, 64, 8, null, 20, 20, 16, d, null) == -1
    assert G(d, 0, 64, 64, 8, d, 20, 20, 16, d, null) == -1
    assert G(d, 1, 7, 64, 8, d, 20, 20, 16, d, null) == -1
    assert G(d, 1, 64, 64, 8, d, 20, 20, 0, d, null) == -1
    assert G(d, 1, 64, 64, 8, d, -1, 20, 16, d, null) == -1
    assert G(d, 1, 64, 64, 17, d, 20, 20, 16, d, null) == -3
    assert G(d, 1, 64, 64, 8, d, 0, 20, 16, d, null) == 0  # nothing to do
    # (imgs, B, H, W, patch, idx, K, vol, stream): tiling needs patch | H and patch | W
    assert V(d, 1, 60, 64, 8, d, 16, d, null) == -1
    assert V(d, 1, 64, 60, 8, d, 16, d, null) == -1
    assert V(d, 1, 64, 64, 8, null, 16, d, null) == -1
    assert V(d, 1, 64, 64, 32, d, 16, d, null) == -3
