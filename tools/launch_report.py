"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into the text kept
under profiles/: share of device time per kernel, then every launch with its grid.
Usage: python tools/launch_report.py launches.csv "command line" > profiles/rNN_launches.txt"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]
data = [dict(zip(h, r)) for r in rows[i + 1:] if len(r) == len(h)]
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}
agg = collections.defaultdict(lambda: [0, 0.0])
per = []
for d in data:
    ms = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
    name = d["Kernel Name"][:70]
    agg[name][0] += 1
    agg[name][1] += ms
    per.append((ms, d.get("Grid Size", ""), name))
tot = sum(v[1] for v in agg.values())
print(f"# ncu --metrics gpu__time_duration.sum --clock-control none -c 400 of\n#   {sys.argv[2]}")
print("# (cold-cache, serialised launches: compare SHARES, not absolutes)")
print(f"# total device time of listed launches: {tot:.3f} ms")
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{100 * v / tot:6.2f}%  {v:10.3f} ms {c:4d} launches  {v / c:8.4f} ms/launch  {n}")
print("\n# per launch")
for ms, grid, name in per:
    print(f"{ms:10.4f} ms  grid {grid:>16s}  {name}")
