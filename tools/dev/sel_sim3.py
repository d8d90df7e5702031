"""Dev: CPU model of a balanced selector for tc16 (per-lane backlog of passing keys; insertion
rounds run only while some lane's backlog exceeds CAP, every lane inserting from its own backlog
in each round) against the round-1/2 protocol (sim_list).  Not product code."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np

from sel_sim import KL, S, r, row_seq, tile_dists_fast
from sel_sim2 import INF, quarter_keys, sim_list


def sim_bal(K, rows, cap=4, append_cost=8, round_cost=80, bulk_min=16, row_cost=25):
    L = [np.empty(0, np.int64) for _ in range(32)]
    B = [[] for _ in range(32)]
    cost = rounds = inserts = appends = 0
    gate = lambda l: (int(L[l][-1] >> 11) if len(L[l]) == KL else INF)
    for u, t in enumerate(rows):
        pc = []
        ps = []
        for l in range(32):
            k = K[l].get(t)
            if k is None:
                pc.append(0); ps.append(None)
                continue
            p = k[(k >> 11) < gate(l)]
            pc.append(len(p)); ps.append(p)
        m = max(pc)
        cost += row_cost
        if m >= bulk_min:
            cost += 1150
            for l in range(32):
                if ps[l] is not None:
                    L[l] = np.sort(np.concatenate([L[l], ps[l], np.array(B[l], np.int64)]))[:KL]
                    B[l] = []
            continue
        appends += sum(pc)
        cost += m * append_cost
        for l in range(32):
            if ps[l] is not None:
                B[l].extend(ps[l].tolist())
        last = u == len(rows) - 1
        while max(len(b) for b in B) > (0 if last else cap):
            rounds += 1
            cost += round_cost
            for l in range(32):
                take, B[l] = B[l][:2], B[l][2:]
                take = [x for x in take if (x >> 11) < gate(l)]
                inserts += len(take)
                if take:
                    L[l] = np.sort(np.concatenate([L[l], np.array(take, np.int64)]))[:KL]
    return cost, rounds, appends


if __name__ == "__main__":
    rng = np.random.default_rng(1)
    nt = int(sys.argv[1]) if len(sys.argv) > 1 else 2
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
    print(f"list    : cost/warp {c[0]:8.0f}  rounds {c[1]:6.1f}  inserts/ref {c[2]/32:6.1f}")
    for cap in (0, 2, 4, 8, 16, 64):
        c = np.array([sim_bal(K, rows, cap) for K, rows in quarters]).sum(0) / n
        print(f"bal c{cap:2d}  : cost/warp {c[0]:8.0f}  rounds {c[1]:6.1f}  appends/ref {c[2]/32:6.1f}")
