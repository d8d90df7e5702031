"""B200-native block matching for G-BM3D (arXiv 2103.10765) -- Python binding of libgbm3d.so.

Argument marshalling only: every step of the matching runs in the CUDA kernels of
``libgbm3d.so`` (C ABI: ``include/gbm3d.h``).  PyTorch provides device memory and streams.
There is no CPU fallback: if the library is missing or no CUDA device is present, the calls
raise.  See DESIGN.md for the method (section II, Eq. (1), Prop. 1, S^K_pq).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

__all__ = [
    "TAU_NONE", "METHODS", "GBM3DError", "lib_path", "load_library", "grid_dims", "block_match",
    "block_match_rows", "block_match_host", "host_workspace_bytes", "check_range",
    "last_launch_count", "version", "gather_groups", "gather_volume", "wiener_stage2",
    "stage1_denoise", "shift_trials", "unshift_mean", "int_peak",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# GBM3D_LIB: dev override to load an experimental build of the same library.
_LIB_PATH = os.environ.get("GBM3D_LIB") or os.path.join(_HERE, "libgbm3d.so")
TAU_NONE = (1 << 63) - 1  # GBM3D_TAU_NONE
METHODS = {"auto": 0, "ssd": 1, "product": 2, "direct": 3, "product_i8": 4}
_ERR = {0: "ok", -1: "GBM3D_ERR_ARG", -2: "GBM3D_ERR_RANGE", -3: "GBM3D_ERR_UNSUPPORTED",
        -4: "GBM3D_ERR_CUDA"}
_lib = None


class GBM3DError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {_ERR.get(status, status)} ({_strerror(status)})")


def lib_path() -> str:
    return _LIB_PATH


def load_library():
    """Load libgbm3d.so (built in-tree by paper_2103_10765_b200/build.py).  Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: build it with "
                          "`python -m paper_2103_10765_b200.build` (no CPU fallback exists)")
    lib = ctypes.CDLL(_LIB_PATH)
    vp, i32, i64, ip = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.POINTER(ctypes.c_int)
    sig = {
        "gbm3d_grid_dims": (i32, [i32, i32, i32, i32, ip, ip]),
        "gbm3d_block_match": (i32, [vp, i32, i32, i32, i32, i32, i32, i64, vp, vp, vp, vp]),
        "gbm3d_block_match_batched": (i32, [vp, i32, i32, i32, i32, i32, i32, i32, i64, vp, vp,
                                            vp, vp]),
        "gbm3d_block_match_rows": (i32, [vp, i32, i32, i32, i32, i32, i32, i32, i32, i64, i32,
                                         i32, vp, vp, vp, vp]),
        "gbm3d_block_match_ex": (i32, [vp, i32, i32, i32, i32, i32, i32, i32, i64, i32, vp, vp,
                                       vp, vp]),
        "gbm3d_host_workspace_bytes": (ctypes.c_size_t, [i32, i32, i32, i32, i32, i32]),
        "gbm3d_block_match_host": (i32, [vp, i32, i32, i32, i32, i32, i32, i32, i64, vp, vp, vp,
                                         vp, ctypes.c_size_t, vp]),
        "gbm3d_check_range": (i32, [vp, i64, i32, ip, vp]),
        "gbm3d_gather_groups": (i32, [vp, i32, i32, i32, i32, vp, i32, i32, i32, vp, vp]),
        "gbm3d_gather_volume": (i32, [vp, i32, i32, i32, i32, vp, i32, vp, vp]),
        "gbm3d_wiener_workspace_bytes": (ctypes.c_size_t, [i32, i32, i32]),
        "gbm3d_stage1_workspace_bytes": (ctypes.c_size_t, [i32, i32, i32, i32, i32]),
        "gbm3d_stage1_denoise": (i32, [vp, i32, i32, i32, i32, vp, vp, i32, vp, i32, vp, vp,
                                       ctypes.c_size_t, vp]),
        "gbm3d_stage1_denoise_keep": (i32, [vp, i32, i32, i32, i32, vp, vp, i32, vp, i32, vp, vp,
                                            ctypes.c_size_t, vp, vp]),
        "gbm3d_wiener_stage2": (i32, [vp, vp, i32, i32, i32, i32, vp, vp, i32, i32, i32, vp, vp,
                                      vp, ctypes.c_size_t, vp]),
        "gbm3d_shift_trials": (i32, [vp, i32, i32, i32, vp, i32, vp, vp]),
        "gbm3d_unshift_mean": (i32, [vp, i32, i32, i32, i32, vp, vp, vp]),
        "gbm3d_int_peak_ops": (ctypes.c_double, [i32, i32, i32, i32]),
        "gbm3d_int_peak_launch": (i32, [i32, i32, i32, i32, vp, vp]),
        "gbm3d_last_launch_count": (i32, []),
        "gbm3d_strerror": (ctypes.c_char_p, [i32]),
        "gbm3d_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        try:
            fn = getattr(lib, name)
        except AttributeError:
            if os.environ.get("GBM3D_LIB"):  # dev builds of older sources: call-time error
                continue
            raise
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _strerror(status: int) -> str:
    try:
        return load_library().gbm3d_strerror(status).decode()
    except Exception:
        return "?"


def version() -> str:
    return load_library().gbm3d_version().decode()


def last_launch_count() -> int:
    """Kernel launches enqueued by the last successful call on this thread."""
    return int(load_library().gbm3d_last_launch_count())


def grid_dims(H: int, W: int, patch: int, stride: int) -> Tuple[int, int]:
    ry, rx = ctypes.c_int(), ctypes.c_int()
    st = load_library().gbm3d_grid_dims(H, W, patch, stride, ctypes.byref(ry), ctypes.byref(rx))
    if st != 0:
        raise GBM3DError(st, "grid_dims")
    return ry.value, rx.value


def _tau(tau: Optional[int]) -> int:
    return TAU_NONE if tau is None else int(tau)


def _stream_handle(device):
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _on(device):
    """The library launches on the current device: make the tensors' device current for the
    call (a tensor on another GPU than the current one would otherwise fail to launch)."""
    import torch
    return torch.cuda.device(device)


def _check_cuda_int16(t, name):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.int16:
        raise TypeError(f"{name} must be a CUDA torch.int16 tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


# Range checks that passed, per live tensor object: (weakref, version counter, data_ptr, numel)
# -> largest patch that passed (the bound P^2 (max-min)^2 <= 2^31-1 then holds for every smaller
# patch).  A tensor modified in place bumps its version counter, so a stale entry never matches.
_range_ok = {}


def _range_cached(img, patch: int) -> bool:
    e = _range_ok.get(id(img))
    return (e is not None and e[0]() is img and e[1] == img._version and e[2] == img.data_ptr()
            and e[3] == img.numel() and patch <= e[4])


def _range_remember(img, patch: int):
    import weakref
    if len(_range_ok) > 256:
        for k in [k for k, e in _range_ok.items() if e[0]() is None]:
            del _range_ok[k]
        if len(_range_ok) > 256:
            _range_ok.clear()
    _range_ok[id(img)] = (weakref.ref(img), img._version, img.data_ptr(), img.numel(), patch)


def check_range(img, patch: int) -> bool:
    """P^2 (max-min)^2 <= 2^31-1 on the device (reading R10).  Synchronises the stream, except
    when this same tensor object, unmodified since (same version counter), already passed for a
    patch at least as large."""
    _check_cuda_int16(img, "img")
    if _range_cached(img, patch):
        return True
    ok = ctypes.c_int(0)
    with _on(img.device):
        st = load_library().gbm3d_check_range(ctypes.c_void_p(img.data_ptr()), img.numel(), patch,
                                              ctypes.byref(ok), _stream_handle(img.device))
    if st != 0:
        raise GBM3DError(st, "check_range")
    if ok.value:
        _range_remember(img, patch)
    return bool(ok.value)


def _alloc_out(shape, device, out):
    import torch
    if out is not None:
        idx, dist, nv = out
        for t, s, n in ((idx, shape, "idx"), (dist, shape, "dist"), (nv, shape[:-1], "n_valid")):
            if t is None and n == "n_valid":
                continue
            if t.dtype != torch.int32 or tuple(t.shape) != tuple(s) or not t.is_contiguous() \
                    or t.device != device:
                raise ValueError(f"out {n} must be contiguous int32 {tuple(s)} on {device}")
        return idx, dist, nv
    return (torch.empty(shape, dtype=torch.int32, device=device),
            torch.empty(shape, dtype=torch.int32, device=device),
            torch.empty(shape[:-1], dtype=torch.int32, device=device))


def block_match(img, patch: int, stride: int, radius: int, K: int, tau: Optional[int] = None,
                check: bool = True, method: str = "auto", out=None):
    """Block matching of one image [H, W] or a batch [B, H, W] (CUDA int16).

    Returns (idx, dist, n_valid) int32 CUDA tensors of shapes [(B,) Ry, Rx, K] and
    [(B,) Ry, Rx]: slot 0 = the reference (d = 0), slots 1..n_valid-1 = the K-1 nearest
    candidates of the clamped (2 radius + 1)^2 window by (SSD, raster index) with SSD < tau,
    pads = (reference, -1).  Enqueued on torch's current stream.  ``check`` runs the
    range precondition first (``check_range``: a stream synchronisation, skipped for a tensor
    that already passed and was not modified since); callers that know their pixel range pass
    ``check=False`` for a fully asynchronous call."""
    _check_cuda_int16(img, "img")
    batched = img.dim() == 3
    if img.dim() not in (2, 3):
        raise ValueError("img must be [H, W] or [B, H, W]")
    B = img.shape[0] if batched else 1
    H, W = img.shape[-2], img.shape[-1]
    if check and not check_range(img, patch):
        raise GBM3DError(-2, "block_match")
    Ry, Rx = grid_dims(H, W, patch, stride)
    shape = ((B,) if batched else ()) + (Ry, Rx, K)
    idx, dist, nv = _alloc_out(shape, img.device, out)
    with _on(img.device):
        st = load_library().gbm3d_block_match_ex(
            ctypes.c_void_p(img.data_ptr()), B, H, W, patch, stride, radius, K, _tau(tau),
            METHODS[method], ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(dist.data_ptr()),
            ctypes.c_void_p(nv.data_ptr() if nv is not None else 0), _stream_handle(img.device))
    if st != 0:
        raise GBM3DError(st, "block_match")
    return idx, dist, nv


def block_match_rows(slab, slab_y0: int, H: int, W: int, patch: int, stride: int, radius: int,
                     K: int, tau: Optional[int], row_begin: int, row_end: int, out=None):
    """Reference grid rows [row_begin, row_end) of an H x W image whose rows
    [slab_y0, slab_y0 + slab.shape[0]) are in ``slab`` (spatial sharding).
    Global raster indices; outputs [row_end-row_begin, Rx, K]."""
    _check_cuda_int16(slab, "slab")
    if slab.dim() != 2 or slab.shape[1] != W:
        raise ValueError("slab must be [rows, W]")
    _, Rx = grid_dims(H, W, patch, stride)
    idx, dist, nv = _alloc_out((row_end - row_begin, Rx, K), slab.device, out)
    with _on(slab.device):
        st = load_library().gbm3d_block_match_rows(
            ctypes.c_void_p(slab.data_ptr()), slab_y0, slab.shape[0], H, W, patch, stride, radius,
            K, _tau(tau), row_begin, row_end, ctypes.c_void_p(idx.data_ptr()),
            ctypes.c_void_p(dist.data_ptr()),
            ctypes.c_void_p(nv.data_ptr() if nv is not None else 0), _stream_handle(slab.device))
    if st != 0:
        raise GBM3DError(st, "block_match_rows")
    return idx, dist, nv


def host_workspace_bytes(B: int, H: int, W: int, patch: int, stride: int, K: int) -> int:
    return int(load_library().gbm3d_host_workspace_bytes(B, H, W, patch, stride, K))


def block_match_host(h_img, patch: int, stride: int, radius: int, K: int,
                     tau: Optional[int] = None, workspace=None, out=None, device=None):
    """End-to-end entry: host (ideally pinned) int16 [B, H, W] torch tensor in, host int32
    tables out; the library copies in, matches and copies out, blocking until done."""
    import torch
    if h_img.device.type != "cpu" or h_img.dtype != torch.int16 or not h_img.is_contiguous():
        raise TypeError("h_img must be a contiguous CPU torch.int16 tensor")
    x = h_img if h_img.dim() == 3 else h_img.unsqueeze(0)
    B, H, W = x.shape
    Ry, Rx = grid_dims(H, W, patch, stride)
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    device = torch.device(device)
    need = host_workspace_bytes(B, H, W, patch, stride, K)
    if workspace is None:
        workspace = torch.empty(need, dtype=torch.uint8, device=device)
    elif not workspace.is_cuda or workspace.device != device or not workspace.is_contiguous() \
            or workspace.numel() * workspace.element_size() < need:
        raise ValueError(f"workspace must be a contiguous buffer of >= {need} bytes on {device}")
    if out is None:
        pin = torch.cuda.is_available()
        out = (torch.empty((B, Ry, Rx, K), dtype=torch.int32, pin_memory=pin),
               torch.empty((B, Ry, Rx, K), dtype=torch.int32, pin_memory=pin),
               torch.empty((B, Ry, Rx), dtype=torch.int32, pin_memory=pin))
    else:
        # the library copies B Ry Rx K int32 into each host buffer: check before it does
        for t, shp, n in ((out[0], (B, Ry, Rx, K), "idx"), (out[1], (B, Ry, Rx, K), "dist"),
                          (out[2], (B, Ry, Rx), "n_valid")):
            if not isinstance(t, torch.Tensor) or t.device.type != "cpu" or t.dtype != torch.int32 \
                    or tuple(t.shape) != shp or not t.is_contiguous():
                raise ValueError(f"out {n} must be a contiguous CPU int32 tensor {shp}")
    idx, dist, nv = out
    with _on(device):
        st = load_library().gbm3d_block_match_host(
            ctypes.c_void_p(x.data_ptr()), B, H, W, patch, stride, radius, K, _tau(tau),
            ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(dist.data_ptr()),
            ctypes.c_void_p(nv.data_ptr()), ctypes.c_void_p(workspace.data_ptr()),
            workspace.numel() * workspace.element_size(), _stream_handle(device))
    if st != 0:
        raise GBM3DError(st, "block_match_host")
    return out


def _check_cuda_int32(t, name):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.int32:
        raise TypeError(f"{name} must be a CUDA torch.int32 tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def gather_groups(img, idx, patch: int, out=None):
    """Matched-block groups (the 5D tensor of PAPER.md:217): for a table ``idx`` [(B,) Ry, Rx, K]
    of ``block_match`` on ``img`` [(B,) H, W], returns int16 [(B,) Ry, Rx, K, patch, patch] with
    block k of reference (y, x) = the patch whose top-left raster index is idx[.., y, x, k]."""
    import torch
    _check_cuda_int16(img, "img")
    _check_cuda_int32(idx, "idx")
    batched = img.dim() == 3
    B = img.shape[0] if batched else 1
    H, W = img.shape[-2], img.shape[-1]
    if idx.dim() != (4 if batched else 3) or (batched and idx.shape[0] != B):
        raise ValueError("idx must be [(B,) Ry, Rx, K] matching img")
    Ry, Rx, K = idx.shape[-3], idx.shape[-2], idx.shape[-1]
    shape = tuple(idx.shape) + (patch, patch)
    if out is None:
        out = torch.empty(shape, dtype=torch.int16, device=img.device)
    elif out.dtype != torch.int16 or tuple(out.shape) != shape or not out.is_contiguous():
        raise ValueError(f"out must be contiguous int16 {shape}")
    with _on(img.device):
        st = load_library().gbm3d_gather_groups(
            ctypes.c_void_p(img.data_ptr()), B, H, W, patch, ctypes.c_void_p(idx.data_ptr()), Ry,
            Rx, K, ctypes.c_void_p(out.data_ptr()), _stream_handle(img.device))
    if st != 0:
        raise GBM3DError(st, "gather_groups")
    return out


def gather_volume(img, idx, patch: int, out=None):
    """The volume of matched blocks V for tiling references (stride = patch,
    patch | H, W): returns int16 [(B,) K, H, W] with slice k = the k-th matched block of every
    tile placed at the tile's position (slice 0 is the image itself)."""
    import torch
    _check_cuda_int16(img, "img")
    _check_cuda_int32(idx, "idx")
    batched = img.dim() == 3
    B = img.shape[0] if batched else 1
    H, W = img.shape[-2], img.shape[-1]
    K = idx.shape[-1]
    if idx.shape[-3:-1] != (H // patch, W // patch):
        raise ValueError("idx must be the table of the tiling grid (stride = patch)")
    shape = ((B,) if batched else ()) + (K, H, W)
    if out is None:
        out = torch.empty(shape, dtype=torch.int16, device=img.device)
    elif out.dtype != torch.int16 or tuple(out.shape) != shape or not out.is_contiguous():
        raise ValueError(f"out must be contiguous int16 {shape}")
    with _on(img.device):
        st = load_library().gbm3d_gather_volume(
            ctypes.c_void_p(img.data_ptr()), B, H, W, patch, ctypes.c_void_p(idx.data_ptr()), K,
            ctypes.c_void_p(out.data_ptr()), _stream_handle(img.device))
    if st != 0:
        raise GBM3DError(st, "gather_volume")
    return out


def _sigmas(sigma, B: int, device):
    """One float32 noise level per image on `device` (a scalar is broadcast): the kernels read
    sigmas[b] for every b < B, so the length is checked here (the C ABI cannot)."""
    import torch
    sig = torch.as_tensor(sigma, dtype=torch.float32).reshape(-1)
    if sig.numel() == 1:
        sig = sig.expand(B)
    if sig.numel() != B:
        raise ValueError(f"sigma must be a scalar or have one entry per image ({B})")
    return sig.contiguous().to(device)


def _float_out(out, like):
    import torch
    if out is None:
        return torch.empty(like.shape, dtype=torch.float32, device=like.device)
    if out.dtype != torch.float32 or out.shape != like.shape or not out.is_contiguous() \
            or out.device != like.device:
        raise ValueError(f"out must be a contiguous float32 tensor {tuple(like.shape)} on {like.device}")
    return out


def _workspace(ws, need: int, device):
    import torch
    if ws is None:
        return torch.empty(need, dtype=torch.uint8, device=device)
    if not ws.is_cuda or ws.device != device or not ws.is_contiguous() \
            or ws.numel() * ws.element_size() < need:
        raise ValueError(f"workspace must be a contiguous buffer of >= {need} bytes on {device}")
    return ws


def wiener_stage2(noisy, basic, idx, n_valid, patch: int, sigma, out=None, workspace=None):
    """Stage-2 collaborative Wiener estimate from the match
    tables of ``block_match`` (normally run on the basic estimate): noisy int16 and basic
    float32 CUDA tensors [(B,) H, W], sigma a float or one per image.  Returns float32 [(B,) H, W]."""
    import torch
    _check_cuda_int16(noisy, "noisy")
    _check_cuda_int32(idx, "idx")
    _check_cuda_int32(n_valid, "n_valid")
    if basic.dtype != torch.float32 or not basic.is_cuda or basic.shape != noisy.shape \
            or not basic.is_contiguous():
        raise TypeError("basic must be a contiguous CUDA float32 tensor shaped like noisy")
    batched = noisy.dim() == 3
    B = noisy.shape[0] if batched else 1
    H, W = noisy.shape[-2], noisy.shape[-1]
    if idx.dim() != (4 if batched else 3) or (batched and idx.shape[0] != B):
        raise ValueError("idx must be [(B,) Ry, Rx, K] matching noisy")
    Ry, Rx, K = idx.shape[-3], idx.shape[-2], idx.shape[-1]
    if Ry > H - patch + 1 or Rx > W - patch + 1:
        raise ValueError("idx grid larger than the image's reference grid")
    if tuple(n_valid.shape) != tuple(idx.shape[:-1]):
        raise ValueError("n_valid must be idx.shape[:-1]")
    sig = _sigmas(sigma, B, noisy.device)
    out = _float_out(out, noisy)
    need = int(load_library().gbm3d_wiener_workspace_bytes(B, H, W))
    workspace = _workspace(workspace, need, noisy.device)
    with _on(noisy.device):
        st = load_library().gbm3d_wiener_stage2(
            ctypes.c_void_p(noisy.data_ptr()), ctypes.c_void_p(basic.data_ptr()), B, H, W, patch,
            ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(n_valid.data_ptr()), Ry, Rx, K,
            ctypes.c_void_p(sig.data_ptr()), ctypes.c_void_p(out.data_ptr()),
            ctypes.c_void_p(workspace.data_ptr()), need, _stream_handle(noisy.device))
    if st != 0:
        raise GBM3DError(st, "wiener_stage2")
    return out


def stage1_denoise(noisy, idx, n_valid, patch: int, sigma, levels: int = 3, out=None,
                   workspace=None, keep=None):
    """Stage-1 global volume hard thresholding: noisy int16
    CUDA [(B,) H, W], tables of ``block_match(noisy, patch, patch, ...)`` (tiling references).
    Returns the float32 estimate [(B,) H, W]."""
    import torch
    _check_cuda_int16(noisy, "noisy")
    _check_cuda_int32(idx, "idx")
    _check_cuda_int32(n_valid, "n_valid")
    batched = noisy.dim() == 3
    B = noisy.shape[0] if batched else 1
    H, W = noisy.shape[-2], noisy.shape[-1]
    K = idx.shape[-1]
    tiles = ((B,) if batched else ()) + (H // patch, W // patch)
    if patch < 1 or H % patch or W % patch or tuple(idx.shape[:-1]) != tiles:
        raise ValueError(f"idx must be the tiling grid's table {tiles + (K,)} (stride = patch)")
    if tuple(n_valid.shape) != tiles:
        raise ValueError(f"n_valid must be {tiles}")
    sig = _sigmas(sigma, B, noisy.device)
    out = _float_out(out, noisy)
    need = int(load_library().gbm3d_stage1_workspace_bytes(B, H, W, patch, K))
    workspace = _workspace(workspace, need, noisy.device)
    if keep is not None:  # test hook: Upsilon's decisions, uint8 [2, B, K, H, W]
        if keep.dtype != torch.uint8 or tuple(keep.shape) != (2, B, K, H, W) or \
                not keep.is_contiguous() or keep.device != noisy.device:
            raise ValueError(f"keep must be a contiguous uint8 {(2, B, K, H, W)} on {noisy.device}")
    with _on(noisy.device):
        args = [ctypes.c_void_p(noisy.data_ptr()), B, H, W, patch, ctypes.c_void_p(idx.data_ptr()),
                ctypes.c_void_p(n_valid.data_ptr()), K, ctypes.c_void_p(sig.data_ptr()), levels,
                ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(workspace.data_ptr()), need]
        if keep is None:
            st = load_library().gbm3d_stage1_denoise(*args, _stream_handle(noisy.device))
        else:
            st = load_library().gbm3d_stage1_denoise_keep(*args, ctypes.c_void_p(keep.data_ptr()),
                                                          _stream_handle(noisy.device))
    if st != 0:
        raise GBM3DError(st, "stage1_denoise")
    return out


def _shift_array(shifts):
    arr = (ctypes.c_int * len(shifts))(*[int(h) for h in shifts])
    return arr, len(shifts)


def shift_trials(img, shifts, out=None):
    """S_h Z for every translation trial h: img int16 CUDA [(B,) H, W] ->
    int16 [T * B, H, W] (trial-major), image t*B + b = img[b] circularly shifted by (h_t, h_t)."""
    import torch
    _check_cuda_int16(img, "img")
    x = img if img.dim() == 3 else img.unsqueeze(0)
    B, H, W = x.shape
    arr, T = _shift_array(shifts)
    shape = (T * B, H, W)
    if out is None:
        out = torch.empty(shape, dtype=torch.int16, device=img.device)
    elif out.dtype != torch.int16 or tuple(out.shape) != shape or not out.is_contiguous() \
            or out.device != img.device:
        raise ValueError(f"out must be contiguous int16 {shape} on {img.device}")
    with torch.cuda.device(img.device):
        st = load_library().gbm3d_shift_trials(ctypes.c_void_p(x.data_ptr()), B, H, W, arr, T,
                                               ctypes.c_void_p(out.data_ptr()),
                                               _stream_handle(img.device))
    if st != 0:
        raise GBM3DError(st, "shift_trials")
    return out


def unshift_mean(ys, shifts, out=None):
    """(1/T) sum_t S_-h_t(ys[t]) for trial-major float32 CUDA estimates ys [T * B, H, W]:
    returns float32 [B, H, W]."""
    import torch
    if not isinstance(ys, torch.Tensor) or not ys.is_cuda or ys.dtype != torch.float32 \
            or ys.dim() != 3 or not ys.is_contiguous():
        raise TypeError("ys must be a contiguous CUDA float32 tensor [T*B, H, W]")
    arr, T = _shift_array(shifts)
    if ys.shape[0] % T:
        raise ValueError("ys.shape[0] must be a multiple of the number of trials")
    B, H, W = ys.shape[0] // T, ys.shape[1], ys.shape[2]
    if out is None:
        out = torch.empty((B, H, W), dtype=torch.float32, device=ys.device)
    elif out.dtype != torch.float32 or tuple(out.shape) != (B, H, W) or not out.is_contiguous() \
            or out.device != ys.device:
        raise ValueError(f"out must be contiguous float32 {(B, H, W)} on {ys.device}")
    with torch.cuda.device(ys.device):
        st = load_library().gbm3d_unshift_mean(ctypes.c_void_p(ys.data_ptr()), T, B, H, W, arr,
                                               ctypes.c_void_p(out.data_ptr()),
                                               _stream_handle(ys.device))
    if st != 0:
        raise GBM3DError(st, "unshift_mean")
    return out


INT_PEAK_KINDS = {"alu": 0, "fma": 1, "minmax": 2, "mixed": 3}


def int_peak(kind: str, device=None, iters: int = 2000, reps: int = 5) -> float:
    """Measured integer instruction throughput (lane-instructions per second) of one of the
    library's microkernels (``INT_PEAK_KINDS``) on every SM of ``device``: 8 CTAs of 256 threads
    per SM, CUDA-event timed, best of ``reps`` after a warm-up launch."""
    import torch
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    k = INT_PEAK_KINDS[kind]
    nsm = torch.cuda.get_device_properties(device).multi_processor_count
    blocks, threads = nsm * 8, 256
    lib = load_library()
    sink = torch.zeros(blocks, dtype=torch.int32, device=device)
    best = 0.0
    with _on(device):
        stream = torch.cuda.current_stream(device)
        h = ctypes.c_void_p(stream.cuda_stream)
        for rep in range(reps + 1):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            st = lib.gbm3d_int_peak_launch(k, blocks, threads, iters, ctypes.c_void_p(sink.data_ptr()), h)
            e.record(stream)
            if st != 0:
                raise GBM3DError(st, "int_peak")
            e.synchronize()
            if rep:
                best = max(best, lib.gbm3d_int_peak_ops(k, blocks, threads, iters) / (s.elapsed_time(e) * 1e-3))
    return best
