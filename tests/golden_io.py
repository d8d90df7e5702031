"""Parser for the hand-worked fixtures in tests/golden/ (format documented in each file)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    img_rows, cases, cur = [], [], None
    mode = None
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            if line == "image":
                mode = "image"
                continue
            if line.startswith("case"):
                mode = "case"
                kv = dict(t.split("=") for t in line.split()[1:])
                cur = {"patch": int(kv["patch"]), "stride": int(kv["stride"]),
                       "radius": int(kv["radius"]), "K": int(kv["K"]),
                       "tau": None if kv["tau"] == "none" else int(kv["tau"]), "refs": []}
                cases.append(cur)
                continue
            if mode == "image":
                img_rows.append([int(v) for v in line.split()])
            elif mode == "case":
                head, rest = line.split(":", 1)
                _, py, px = head.split()
                slots_s, nv_s = rest.split(";")
                slots = [tuple(int(v) for v in s.split()) for s in slots_s.split("|")]
                cur["refs"].append((int(py), int(px), slots, int(nv_s.split()[1])))
    return np.array(img_rows, dtype=np.int16), cases


def expected_arrays(case):
    ny = max(r[0] for r in case["refs"]) + 1
    nx = max(r[1] for r in case["refs"]) + 1
    K = case["K"]
    idx = np.zeros((ny, nx, K), np.int32)
    dist = np.zeros((ny, nx, K), np.int32)
    nv = np.zeros((ny, nx), np.int32)
    for py, px, slots, n in case["refs"]:
        idx[py, px] = [s[0] for s in slots]
        dist[py, px] = [s[1] for s in slots]
        nv[py, px] = n
    return idx, dist, nv
