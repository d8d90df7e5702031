"""Dev: CPU model of selector strategies for the tc16 matcher on real c3 tiles.

Strategy "list" is the round-1 protocol (running gate, per-row insertion rounds, bulk rows).
Strategy "buf" appends passing keys to a per-lane buffer and merges the buffer into the sorted
list only when some lane's buffer holds >= TH keys (the gate is refreshed at merges).  Costs are
warp instructions of one selector warp, from a rough per-operation model.  Not product code."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np

from sel_sim import KL, S, r, row_seq, tile_dists_fast

INF = np.iinfo(np.int64).max
SIDE = 2 * r + 1


def quarter_keys(D, w):
    """keys[l][t] = int64 array of (d << 11 | code) for the lane's window columns of row t."""
    out = []
    for l in range(32):
        a, b = 4 * w + (l >> 3), l & 7
        rows = {}
        for t in range(S * a, S * a + 2 * r + 1):
            drow = D[a, b, t]
            js = np.arange(S * b, S * b + 2 * r + 1)
            d = drow[js]
            ok = d != INF
            code = (t - S * a) * SIDE + (js - S * b)
            rows[t] = (d[ok] << 11) | code[ok]
        out.append(rows)
    return out


def sim_list(K, rows, lag=1, bulk_min=16):
    L = [np.empty(0, np.int64) for _ in range(32)]
    gates = [[INF] * 32]
    cost = rounds = inserts = 0
    for u, t in enumerate(rows):
        g = gates[max(0, len(gates) - lag)] if u > 0 else gates[0]
        pc = []
        for l in range(32):
            k = K[l].get(t)
            if k is None:
                pc.append(0)
                continue
            p = k[(k >> 11) < g[l]]
            pc.append(len(p))
            L[l] = np.sort(np.concatenate([L[l], p]))[:KL]
        m = max(pc)
        inserts += sum(pc)
        if m >= bulk_min:
            cost += 1150
        else:
            rounds += (m + 1) // 2
            cost += 25 + ((m + 1) // 2) * 70
        gates.append([(int(x[-1] >> 11) + 1 if len(x) == KL else INF) for x in L])
    return cost, rounds, inserts


def sim_buf(K, rows, TH=24, chunk=16, append_cost=10, first_th=1):
    L = [np.empty(0, np.int64) for _ in range(32)]
    buf = [[] for _ in range(32)]
    g = [INF] * 32
    cost = appends = merges = 0
    chunk_cost = {8: 230, 16: 340, 32: 700}[chunk]
    for u, t in enumerate(rows):
        pc = []
        for l in range(32):
            k = K[l].get(t)
            if k is None:
                pc.append(0)
                continue
            p = k[(k >> 11) < g[l]]
            pc.append(len(p))
            buf[l].extend(p.tolist())
        m = max(pc)
        appends += sum(pc)
        cost += 20 + m * append_cost
        mb = max(len(b) for b in buf)
        th = first_th if any(len(x) < KL for x in L) else TH
        if mb >= th or u == len(rows) - 1:
            if mb:
                cost += 30 + -(-mb // chunk) * chunk_cost
                merges += 1
            for l in range(32):
                L[l] = np.sort(np.concatenate([L[l], np.array(buf[l], np.int64)]))[:KL]
                buf[l] = []
            g = [(int(x[-1] >> 11) + 1 if len(x) == KL else INF) for x in L]
    return cost, merges, appends


if __name__ == "__main__":
    rng = np.random.default_rng(1)
    nt = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    tiles = [(int(rng.integers(2, 40)) * 16, int(rng.integers(3, 80)) * 8) for _ in range(nt)]
    quarters = []
    for ky0, kx0 in tiles:
        D = tile_dists_fast(ky0, kx0)
        for w in range(4):
            wt0, wt1 = S * 4 * w, S * (4 * w + 3) + 2 * r
            rows = [t for t in row_seq("fill") if wt0 <= t <= wt1]
            quarters.append((quarter_keys(D, w), rows))
    n = len(quarters)
    c = np.array([sim_list(K, rows) for K, rows in quarters]).sum(0) / n
    print(f"list      : cost/warp {c[0]:8.0f}  rounds {c[1]:6.1f}  inserts/ref {c[2]/32:6.1f}")
    for chunk in (8, 16, 32):
        for TH in (8, 16, 24, 32, 48):
            c = np.array([sim_buf(K, rows, TH, chunk) for K, rows in quarters]).sum(0) / n
            print(f"buf c{chunk:2d} th{TH:2d}: cost/warp {c[0]:8.0f}  merges {c[1]:5.1f}  appends/ref {c[2]/32:6.1f}")


def orders_study(quarters):
    """inserts/ref (exact running gate, lag 1) for several candidate-row orders."""
    for name in ("fill", "centre", "oracle", "antioracle"):
        tot = np.zeros(3)
        for K, rows in quarters:
            if name == "centre":
                c = (min(rows) + max(rows)) / 2
                rows = sorted(rows, key=lambda t: (abs(t - c), t))
            elif name in ("oracle", "antioracle"):
                cnt = {t: 0 for t in rows}
                for l in range(32):
                    allk = np.concatenate([K[l][t] for t in K[l]])
                    top = set(np.sort(allk)[:KL].tolist())
                    for t in K[l]:
                        cnt[t] += sum(1 for x in K[l][t].tolist() if x in top)
                rows = sorted(rows, key=lambda t: -cnt[t] if name == "oracle" else cnt[t])
            tot += np.array(sim_list(K, rows))
        n = len(quarters)
        print(f"order {name:10s}: cost/warp {tot[0]/n:8.0f} rounds {tot[1]/n:6.1f} inserts/ref {tot[2]/n/32:6.1f}")
