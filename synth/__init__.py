"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO block-matching arithmetic: it only draws images.  It is the
one module both sides of the parity check may import ("Input
recipe").  The recipe is SURVEY.md section 8(d), standing in for the paper's
workloads: the paper times unnamed single-channel images of 256^2..4096^2
(Table II) and adds zero-mean i.i.d. Gaussian noise with
sigma = mean(I)/SNR; its 8 test images are not available, so
piecewise-constant rectangles + oriented sinusoidal textures + a gradient, clipped
to 8-bit range, then noised and rounded to int16, play their role.
"""
from .images import (  # noqa: F401
    CONFIGS,
    MatchCall,
    SynthConfig,
    config_images,
    make_image,
    special_image,
)
