"""ORACLE (pure-Python twin) -- TEST INFRASTRUCTURE ONLY.

The same definition as gbm3d_oracle.c, written independently with Python integers
(no overflow possible) and ``sorted``.  Used for exhaustive checks on tiny inputs.
Steps follow PAPER.md: grid (reading R3), clamped window (R2),
Eq. (1) distance, strict tau cut (R6), (d, idx) order (R5), self in slot 0
and padding with the reference block (R4/R7).
"""
from __future__ import annotations


def grid(L, P, s):
    pos = list(range(0, L - P + 1, s))
    if pos[-1] != L - P:
        pos.append(L - P)
    return pos


def ssd(img, ay, ax, by, bx, P):
    return sum((int(img[ay + i][ax + j]) - int(img[by + i][bx + j])) ** 2
               for i in range(P) for j in range(P))


def block_match(img, P, s, r, K, tau=None):
    """Returns nested lists: table[py][px] = list of K (idx, d) pairs, and n_valid[py][px]."""
    H, W = len(img), len(img[0])
    table, nvalid = [], []
    for ry in grid(H, P, s):
        trow, nrow = [], []
        for rx in grid(W, P, s):
            cands = []
            for cy in range(max(0, ry - r), min(H - P, ry + r) + 1):
                for cx in range(max(0, rx - r), min(W - P, rx + r) + 1):
                    if (cy, cx) == (ry, rx):
                        continue
                    d = ssd(img, ry, rx, cy, cx, P)
                    if tau is None or d < tau:
                        cands.append((d, cy * W + cx))
            cands.sort()
            out = [(ry * W + rx, 0)] + [(i, d) for d, i in cands[:K - 1]]
            nrow.append(len(out))
            out += [(ry * W + rx, -1)] * (K - len(out))
            trow.append(out)
        table.append(trow)
        nvalid.append(nrow)
    return table, nvalid
