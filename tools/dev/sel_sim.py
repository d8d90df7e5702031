"""Dev: CPU simulation of the tc16 selector protocol on real c3 tiles: insertion rounds per
selector warp (sum over staged rows of the max pass count over lanes) for row orders and gate
policies.  Not part of the product; distances computed directly with numpy."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from synth import CONFIGS, config_images

S, r, P, K = 3, 19, 8, 32
KL = K - 1
TY, TX = 16, 8
img = config_images(CONFIGS["c3"])[0].astype(np.int64)
H, W = img.shape
NT = 15 * S + 2 * r + 1


def tile_dists(ky0, kx0):
    gy0, gx0 = S * ky0 - r, S * kx0 - r
    D = np.full((TY, TX, NT, 64), np.iinfo(np.int64).max, dtype=np.int64)
    # patch sums via integral of squared differences per displacement is slow; direct is fine
    for a in range(TY):
        for b in range(TX):
            ry, rx = S * (ky0 + a), S * (kx0 + b)
            f = img[ry:ry + P, rx:rx + P]
            for t in range(S * a, S * a + 2 * r + 1):
                cy = gy0 + t
                if cy < 0 or cy > H - P:
                    continue
                for j in range(S * b, S * b + 2 * r + 1):
                    cx = gx0 + j
                    if cx < 0 or cx > W - P or (cy == ry and cx == rx):
                        continue
                    g = img[cy:cy + P, cx:cx + P]
                    D[a, b, t, j] = ((f - g) ** 2).sum()
    return D


def tile_dists_fast(ky0, kx0):
    gy0, gx0 = S * ky0 - r, S * kx0 - r
    D = np.full((TY, TX, NT, 64), np.iinfo(np.int64).max, dtype=np.int64)
    from numpy.lib.stride_tricks import sliding_window_view as swv
    pat = swv(img, (P, P))  # [H-P+1, W-P+1, P, P]
    for a in range(TY):
        for b in range(TX):
            ry, rx = S * (ky0 + a), S * (kx0 + b)
            f = img[ry:ry + P, rx:rx + P]
            t0, t1 = S * a, S * a + 2 * r
            j0, j1 = S * b, S * b + 2 * r
            cy0, cy1 = max(0, gy0 + t0), min(H - P, gy0 + t1)
            cx0, cx1 = max(0, gx0 + j0), min(W - P, gx0 + j1)
            blk = pat[cy0:cy1 + 1, cx0:cx1 + 1]
            d = ((blk - f) ** 2).sum(axis=(2, 3))
            D[a, b, cy0 - gy0:cy1 - gy0 + 1, cx0 - gx0:cx1 - gx0 + 1] = d
            D[a, b, ry - gy0, rx - gx0] = np.iinfo(np.int64).max
    return D


def row_seq(order, t_lo=0, t_hi=NT - 1):
    n = t_hi - t_lo + 1
    if order == "raster":
        return list(range(t_lo, t_hi + 1))
    st = max(1, int(0.618 * n))
    while np.gcd(st, n) != 1:
        st += 1
    seq = [t_lo + (s * st) % n for s in range(n)]
    if order == "scr":
        return seq
    a1, b1 = 11 * S, min(2 * r, 12 * S - 1)
    a2, b2 = max(15 * S, 7 * S + 2 * r + 1), 12 * S + 2 * r
    f = [(a1 + b1) // 2, (a2 + b2) // 2]
    return f + [t for t in seq if t not in f]


def simulate(D, order="fill", lag=2, key_sorted=True):
    INF = np.iinfo(np.int64).max
    res = []
    for w in range(4):
        wt0, wt1 = S * 4 * w, S * (4 * w + 3) + 2 * r
        lanes = [(4 * w + (l >> 3), l & 7) for l in range(32)]
        lists = [[] for _ in range(32)]
        gates_hist = []  # gate after each processed row
        rounds = inserts = useful = 0
        u = 0
        for t in row_seq(order):
            if t < wt0 or t > wt1:
                continue
            filling = any(len(L) < KL for L in lists)
            if u == 0:
                g = [INF] * 32
            elif filling:
                g = gates_hist[-1]
            else:
                g = gates_hist[max(0, u - lag)] if u - lag >= 0 else gates_hist[0]
                g = gates_hist[max(0, u - 1 - (lag - 1))]
            pc = []
            for l, (a, b) in enumerate(lanes):
                drow = D[a, b, t]
                cand = [(int(drow[j]), (t - S * a) * 39 + (j - S * b)) for j in range(64)
                        if drow[j] != INF and drow[j] < g[l]]
                pc.append(len(cand))
                before = list(lists[l])
                lists[l] = sorted(lists[l] + cand)[:KL]
                useful += len(set(lists[l]) - set(before))
            rounds += max(pc)
            inserts += sum(pc)
            gates_hist.append([(L[-1][0] + 1 if len(L) == KL else INF) for L in lists])
            u += 1
        res.append((rounds, inserts, useful))
    return res


if __name__ == "__main__":
    rng = np.random.default_rng(1)
    tiles = [(int(rng.integers(2, 40)) * 16, int(rng.integers(3, 80)) * 8) for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3)]
    for order in ["fill", "scr", "raster"]:
        for lag in [1, 2, 4]:
            tot = np.zeros(3)
            for ky0, kx0 in tiles:
                D = tile_dists_fast(ky0, kx0)
                tot += np.array(simulate(D, order, lag)).sum(0)
            n = 4 * len(tiles)
            print(f"{order:6s} lag {lag}: rounds/warp {tot[0]/n:7.1f}  inserts/ref {tot[1]/n/32:7.1f}  balanced rounds {tot[1]/n/32:7.1f} useful/ref {tot[2]/n/32:6.1f}")


def simulate_grouped(D, G=2, lag_groups=1, order="fill", first_single=True):
    """Rows processed in groups of G: masks of a group use the gates published after group
    (g - lag_groups); rounds per group = max over lanes of the group's total passes."""
    INF = np.iinfo(np.int64).max
    res = []
    for w in range(4):
        wt0, wt1 = S * 4 * w, S * (4 * w + 3) + 2 * r
        lanes = [(4 * w + (l >> 3), l & 7) for l in range(32)]
        rows = [t for t in row_seq(order) if wt0 <= t <= wt1]
        groups = ([rows[:1]] + [rows[i:i + G] for i in range(1, len(rows), G)]) if first_single else \
            [rows[i:i + G] for i in range(0, len(rows), G)]
        lists = [[] for _ in range(32)]
        hist = []
        rounds = inserts = 0
        for gi, grp in enumerate(groups):
            if gi == 0:
                g = [INF] * 32
            else:
                g = hist[max(0, gi - lag_groups)]
            pc = [0] * 32
            for t in grp:
                for l, (a, b) in enumerate(lanes):
                    drow = D[a, b, t]
                    m = (drow != INF) & (drow < g[l])
                    js = np.nonzero(m)[0]
                    cand = [(int(drow[j]), (t - S * a) * 39 + (j - S * b)) for j in js]
                    pc[l] += len(cand)
                    lists[l] = sorted(lists[l] + cand)[:KL]
            rounds += max(pc)
            inserts += sum(pc)
            hist.append([(L[-1][0] + 1 if len(L) == KL else INF) for L in lists])
        res.append((rounds, inserts))
    return res
