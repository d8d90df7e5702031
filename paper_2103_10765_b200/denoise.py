"""The whole G-BM3D denoiser composed from the library's kernels (section IV-V).

Every arithmetic step runs in libgbm3d.so: block matching (``block_match``), the translation
trials' shifts and averaging (``shift_trials``, ``unshift_mean``), stage-1 global volume hard
thresholding (``stage1_denoise``), stage-2 collaborative Wiener filtering (``wiener_stage2``).
What this module adds is the paper's schedule around them (torch only rounds the basic estimate
to int16 for the second matching):

* stage 1: Y_f = (1/H) sum_h S_-h phi(S_h Z) over the translation trials
  h = 0, N/4, N/2 of the tiling reference grid (each trial matches its shifted image; the
  trials run as one batch through the matching and the thresholding);
* stage 2: matching on the basic estimate (rounded to int16), Wiener
  filtering of the noisy image's groups with the basic estimate's spectra, aggregation.

Parameters default to the paper's: stage 1 uses N = 16 tiles with K = 16 and
the trials h = 0, N/4, N/2, stage 2 N = 8 blocks on a stride-3 grid with K = 32 (the
library's choice: the paper's stage-2 reference blocks tile the image), both with a search
radius of 16 (the paper's window "32").  ``stage1(patch=8)`` gives the N = 8 variant.
"""
from __future__ import annotations

from typing import Optional, Sequence

from . import block_match, shift_trials, stage1_denoise, unshift_mean, wiener_stage2


def stage1(noisy, sigma, patch: int = 16, K: int = 16, radius: int = 16,
           trials: Optional[Sequence[int]] = None, levels: int = 3):
    """Basic estimate Y_f (float32, same shape as ``noisy`` [(B,) H, W] int16 CUDA).  The
    translation trials are stacked into one batch (``shift_trials``), so the matching and the
    global thresholding each run as a single batched call over trials x images, and
    ``unshift_mean`` shifts the estimates back and averages them."""
    import torch
    trials = (0, patch // 4, patch // 2) if trials is None else tuple(trials)
    x = noisy if noisy.dim() == 3 else noisy.unsqueeze(0)
    B = x.shape[0]
    z = shift_trials(x, trials)
    sig = torch.as_tensor(sigma, dtype=torch.float32).reshape(-1)
    sig = (sig.expand(B) if sig.numel() == 1 else sig).repeat(len(trials))
    idx, dist, nv = block_match(z, patch, patch, radius, K, None, check=False)
    y = stage1_denoise(z, idx, nv, patch, sig, levels)
    out = unshift_mean(y, trials)
    return out if noisy.dim() == 3 else out[0]


def stage2(noisy, basic, sigma, patch: int = 8, stride: int = 3, K: int = 32, radius: int = 16):
    """Final estimate from the basic estimate (float32 CUDA, same shape as ``noisy``)."""
    import torch
    est = torch.round(basic).clamp_(-32768, 32767).to(torch.int16).contiguous()
    idx, dist, nv = block_match(est, patch, stride, radius, K, None, check=False)
    return wiener_stage2(noisy, basic.contiguous(), idx, nv, patch, sigma)


def denoise(noisy, sigma, two_stage: bool = True):
    """G-BM3D1 (stage 1 only) or G-BM3D2 (both stages) of int16 CUDA images [(B,) H, W];
    H and W must be multiples of 16 (stage-1 tiling and wavelet levels)."""
    basic = stage1(noisy, sigma)
    return stage2(noisy, basic, sigma) if two_stage else basic
