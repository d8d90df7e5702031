"""The C ABI exactly as include/gbm3d.h declares it (-m gpu): gbm3d_block_match and
gbm3d_block_match_batched called through ctypes with raw device pointers, on the legacy default
stream (NULL) and on a created stream, bit-exact against the oracle (c1's two calls, the first 4
images of c4)."""
import ctypes

import numpy as np
import pytest

import oracle
from synth import CONFIGS, config_images

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _lib():
    import paper_2103_10765_b200 as g
    return g.load_library(), g


def _tau(t):
    return (1 << 63) - 1 if t is None else int(t)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


@pytest.mark.parametrize("use_stream", [False, True])
@pytest.mark.parametrize("ci", [0, 1])
def test_gbm3d_block_match_raw(ci, use_stream):
    lib, g = _lib()
    cfg = CONFIGS["c1"]
    c = cfg.calls[ci]
    img = config_images(cfg)[0]
    d_img = torch.from_numpy(img).cuda()
    Ry, Rx = g.grid_dims(cfg.H, cfg.W, c.patch, c.stride)
    idx = torch.full((Ry, Rx, c.K), -7, dtype=torch.int32, device="cuda")
    dist = torch.full_like(idx, -7)
    nv = torch.full((Ry, Rx), -7, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    s = torch.cuda.Stream() if use_stream else None
    handle = ctypes.c_void_p(s.cuda_stream) if s is not None else ctypes.c_void_p(0)
    st = lib.gbm3d_block_match(_ptr(d_img), cfg.H, cfg.W, c.patch, c.stride, c.radius, c.K,
                               _tau(c.tau), _ptr(idx), _ptr(dist), _ptr(nv), handle)
    assert st == 0
    if s is not None:
        s.synchronize()
    torch.cuda.synchronize()
    e = oracle.block_match(img, c.patch, c.stride, c.radius, c.K, c.tau)
    np.testing.assert_array_equal(idx.cpu().numpy(), e[0])
    np.testing.assert_array_equal(dist.cpu().numpy(), e[1])
    np.testing.assert_array_equal(nv.cpu().numpy(), e[2])


@pytest.mark.parametrize("use_stream", [False, True])
def test_gbm3d_block_match_batched_raw(use_stream):
    lib, g = _lib()
    cfg = CONFIGS["c4"]
    c = cfg.calls[0]
    imgs = config_images(cfg, 4)
    d = torch.from_numpy(imgs).cuda()
    B = imgs.shape[0]
    Ry, Rx = g.grid_dims(cfg.H, cfg.W, c.patch, c.stride)
    idx = torch.empty((B, Ry, Rx, c.K), dtype=torch.int32, device="cuda")
    dist = torch.empty_like(idx)
    torch.cuda.synchronize()
    s = torch.cuda.Stream() if use_stream else None
    handle = ctypes.c_void_p(s.cuda_stream) if s is not None else ctypes.c_void_p(0)
    # n_valid is nullable in the ABI
    st = lib.gbm3d_block_match_batched(_ptr(d), B, cfg.H, cfg.W, c.patch, c.stride, c.radius,
                                       c.K, _tau(c.tau), _ptr(idx), _ptr(dist), ctypes.c_void_p(0),
                                       handle)
    assert st == 0
    if s is not None:
        s.synchronize()
    torch.cuda.synchronize()
    gi, gd = idx.cpu().numpy(), dist.cpu().numpy()
    for b in range(B):
        e = oracle.block_match(imgs[b], c.patch, c.stride, c.radius, c.K, c.tau)
        np.testing.assert_array_equal(gi[b], e[0])
        np.testing.assert_array_equal(gd[b], e[1])


def test_raw_entry_errors():
    lib, g = _lib()
    z = torch.zeros((16, 16), dtype=torch.int16, device="cuda")
    out = torch.zeros((4, 4, 4), dtype=torch.int32, device="cuda")
    null = ctypes.c_void_p(0)
    assert lib.gbm3d_block_match(null, 16, 16, 8, 3, 4, 4, _tau(None), _ptr(out), _ptr(out), null,
                                 null) == -1
    assert lib.gbm3d_block_match(_ptr(z), 16, 16, 17, 3, 4, 4, _tau(None), _ptr(out), _ptr(out),
                                 null, null) == -1          # patch > H
    assert lib.gbm3d_block_match(_ptr(z), 16, 16, 8, 3, 40, 4, _tau(None), _ptr(out), _ptr(out),
                                 null, null) == -3          # radius > 32
    assert lib.gbm3d_block_match_batched(_ptr(z), 0, 16, 16, 8, 3, 4, 4, _tau(None), _ptr(out),
                                         _ptr(out), null, null) == -1
