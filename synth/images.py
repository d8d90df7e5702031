"""Seeded image generator (SURVEY.md 8(d) recipe) and the five BASELINE.json configs.

Draw order (numpy PCG64 ``default_rng(seed)``, all floats float64) -- frozen:
  1. gradient: psi ~ U[0, 2pi), G ~ U[0, 64);  g = G (u - min u)/(max u - min u),
     u = y cos(psi) + x sin(psi)
  2. n_rect rectangles, each: L ~ U[0,255), h ~ Uint[lo,hi), w ~ Uint[lo,hi),
     y0 ~ Uint[0,H), x0 ~ Uint[0,W);  add L on [y0:y0+h, x0:x0+w] (clipped);
     a = sqrt(H W / n_rect), lo = max(2, a//2), hi = max(3, floor(1.5 a))
  3. n_tex textures, each: T ~ U[6,20), theta ~ U[0,pi), phi ~ U[0,2pi),
     side ~ Uint[lo_t,hi_t), y0 ~ Uint[0,H), x0 ~ Uint[0,W);
     add 40 sin(2 pi (x cos theta + y sin theta)/T + phi) on the square;
     a_t = sqrt(H W / n_tex)/2
  4. clean = clip(sum, 0, 255)
  5. sigma ~ U[10, 50) only when the config says so (c4)
  6. img = int16(rint(clean + N(0, sigma^2)))   (round half to even, no clipping)

No block-matching arithmetic lives here (input recipe).
"""
from __future__ import annotations

import dataclasses
import hashlib
import math
from typing import Optional, Sequence

import numpy as np

TAU_NONE = None  # "no threshold" (PAPER.md:73 with tau_match = +inf)


@dataclasses.dataclass(frozen=True)
class MatchCall:
    """One block-matching call: patch N, reference stride, search radius
    (window side 2r+1), K, tau_match."""

    patch: int
    stride: int
    radius: int
    K: int
    tau: Optional[int] = TAU_NONE


@dataclasses.dataclass(frozen=True)
class SynthConfig:
    name: str
    H: int
    W: int
    B: int
    n_rect: int
    n_tex: int
    sigma: Optional[float]  # None -> per-image sigma ~ U[10, 50)
    seeds: Sequence[int]
    calls: Sequence[MatchCall]
    note: str = ""


# BASELINE.json "configs" 0..4 (seeds c0..c3 are our choice, c4 = 0..63 from BASELINE.json).
CONFIGS = {
    "c0": SynthConfig("c0", 64, 64, 1, 6, 0, 25.0, (0,),
                      (MatchCall(8, 3, 19, 16, None),), "64x64, 6 rects + gradient, sigma 25"),
    "c1": SynthConfig("c1", 256, 256, 1, 20, 5, 25.0, (1,),
                      (MatchCall(8, 3, 19, 16, 2500 * 64), MatchCall(8, 3, 19, 32, 400 * 64)),
                      "256x256, 20 rects + 5 textures, sigma 25; stage-1 and stage-2 calls"),
    "c2": SynthConfig("c2", 512, 512, 1, 60, 15, 50.0, (2,),
                      (MatchCall(12, 4, 19, 16, 5000 * 144),), "512x512 high-noise, P12 s4"),
    "c3": SynthConfig("c3", 2048, 2048, 1, 400, 100, 25.0, (3,),
                      (MatchCall(8, 3, 19, 32, None),), "2048x2048, K32, row-sharded at N>1"),
    "c4": SynthConfig("c4", 512, 512, 64, 20, 5, None, tuple(range(64)),
                      (MatchCall(8, 3, 19, 16, None),), "batch of 64 512x512, sigma~U[10,50)"),
}


def _side_bounds(a: float):
    lo = max(2, int(a // 2))
    hi = max(3, int(math.floor(1.5 * a)))
    if hi <= lo:
        hi = lo + 1
    return lo, hi


def make_image(H: int, W: int, n_rect: int, n_tex: int, sigma: Optional[float], seed: int,
               return_clean: bool = False):
    """Draw one int16 [H, W] noisy image following the frozen recipe above."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    # 1. gradient
    psi = rng.uniform(0.0, 2.0 * math.pi)
    G = rng.uniform(0.0, 64.0)
    u = yy * math.cos(psi) + xx * math.sin(psi)
    span = float(u.max() - u.min())
    acc = G * (u - u.min()) / span if span > 0 else np.zeros((H, W))
    # 2. rectangles
    if n_rect > 0:
        lo, hi = _side_bounds(math.sqrt(H * W / n_rect))
        for _ in range(n_rect):
            L = rng.uniform(0.0, 255.0)
            h = int(rng.integers(lo, hi))
            w = int(rng.integers(lo, hi))
            y0 = int(rng.integers(0, H))
            x0 = int(rng.integers(0, W))
            acc[y0:y0 + h, x0:x0 + w] += L
    # 3. textures
    if n_tex > 0:
        lo, hi = _side_bounds(0.5 * math.sqrt(H * W / n_tex))
        for _ in range(n_tex):
            T = rng.uniform(6.0, 20.0)
            th = rng.uniform(0.0, math.pi)
            ph = rng.uniform(0.0, 2.0 * math.pi)
            side = int(rng.integers(lo, hi))
            y0 = int(rng.integers(0, H))
            x0 = int(rng.integers(0, W))
            ys = slice(y0, min(H, y0 + side))
            xs = slice(x0, min(W, x0 + side))
            acc[ys, xs] += 40.0 * np.sin(2.0 * math.pi * (xx[ys, xs] * math.cos(th)
                                                         + yy[ys, xs] * math.sin(th)) / T + ph)
    # 4. clip
    clean = np.clip(acc, 0.0, 255.0)
    # 5. per-image sigma (c4)
    if sigma is None:
        sigma = rng.uniform(10.0, 50.0)
    # 6. noise, round half-to-even, int16 without clipping
    noisy = np.rint(clean + rng.normal(0.0, sigma, (H, W))).astype(np.int16)
    if return_clean:
        return noisy, np.rint(clean).astype(np.int16), float(sigma)
    return noisy


def config_images(cfg: SynthConfig | str, n_images: Optional[int] = None) -> np.ndarray:
    """int16 [B, H, W] stack for a config (first ``n_images`` of the batch if given)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    seeds = list(cfg.seeds)[: (n_images or cfg.B)]
    return np.stack([make_image(cfg.H, cfg.W, cfg.n_rect, cfg.n_tex, cfg.sigma, s) for s in seeds])


def special_image(kind: str, H: int, W: int, seed: int = 0, period: int = 5, value: int = 7,
                  lo: int = -100, hi: int = 100) -> np.ndarray:
    """Test-only images with known matching structure (SURVEY.md 8(c) pins).

    constant    -- every pixel ``value``
    periodic    -- Z[y][x] = T[y % p][x % p] with distinct T entries
    checker     -- +-value checkerboard
    uniform     -- i.i.d. integers in [lo, hi]
    """
    rng = np.random.default_rng(seed)
    if kind == "constant":
        return np.full((H, W), value, dtype=np.int16)
    if kind == "periodic":
        T = rng.permutation(period * period).reshape(period, period).astype(np.int16) * 3 - 20
        yy, xx = np.mgrid[0:H, 0:W]
        return T[yy % period, xx % period].astype(np.int16)
    if kind == "checker":
        yy, xx = np.mgrid[0:H, 0:W]
        return np.where((yy + xx) % 2 == 0, value, -value).astype(np.int16)
    if kind == "uniform":
        return rng.integers(lo, hi + 1, size=(H, W)).astype(np.int16)
    raise ValueError(kind)


def image_sha256(img: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(img, dtype=np.int16).tobytes()).hexdigest()
