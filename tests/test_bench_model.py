"""The bench's closed-form counts and roofline models (-m "not gpu"): evaluation and reference
counts of the five BASELINE configs against SURVEY.md 8(a) and an independent enumeration,
A_eval of SURVEY 8(d), and the stage-1 traffic model of DESIGN.md 7.7."""
import itertools

import pytest

import bench
from synth import CONFIGS


def _brute(H, W, P, s, r):
    """Windows by direct enumeration of the grid and of the clamped candidate positions."""
    def grid(L):
        g = list(range(0, L - P + 1, s))
        if g[-1] != L - P:
            g.append(L - P)
        return g
    ev = 0
    gy, gx = grid(H), grid(W)
    for y, x in itertools.product(gy, gx):
        ny = sum(1 for cy in range(y - r, y + r + 1) if 0 <= cy <= H - P)
        nx = sum(1 for cx in range(x - r, x + r + 1) if 0 <= cx <= W - P)
        ev += ny * nx - 1
    return ev, len(gy) * len(gx)


@pytest.mark.parametrize("name,evals,refs", [("c0", 401_556, 400), ("c1", 9_789_844, 7_056),
                                             ("c2", 23_062_540, 15_876),
                                             ("c3", 697_499_800, 463_761)])
def test_total_evals_match_survey(name, evals, refs):
    c = CONFIGS[name].calls[0]
    cfg = CONFIGS[name]
    assert bench.total_evals(cfg.H, cfg.W, c.patch, c.stride, c.radius) == (evals, refs)


def test_c4_evals_per_batch():
    cfg = CONFIGS["c4"]
    c = cfg.calls[0]
    ev, refs = bench.total_evals(cfg.H, cfg.W, c.patch, c.stride, c.radius)
    assert ev * cfg.B == 2_661_557_760 and refs * cfg.B == 1_827_904


@pytest.mark.parametrize("H,W,P,s,r", [(37, 53, 8, 3, 5), (64, 64, 12, 4, 19), (30, 31, 8, 3, 32),
                                       (45, 61, 5, 2, 6)])
def test_total_evals_brute_force(H, W, P, s, r):
    assert bench.total_evals(H, W, P, s, r) == _brute(H, W, P, s, r)


def test_a_eval():
    # 3 s^2 + s + 1 int32 ops per evaluation of the SSD form
    assert bench.a_eval(3) == 31 and bench.a_eval(4) == 53 and bench.a_eval(1) == 5
