"""Summarise an ncu report's SASS source page: time (stall samples) and instructions by code
region, with stall-reason breakdowns.  Usage: python tools/ncu_regions.py report.ncu-rep [B]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
ci = h.index("Instructions Executed")
si = h.index("Warp Stall Sampling (All Samples)")
ti = h.index("Avg. Threads Executed")
stall = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
tot = sum(int(r[ci]) for r in data)
stot = sum(int(r[si]) for r in data)
print(f"instructions {tot:.4g}  samples {stot}  sass {len(data)}")
for s in range(0, len(data), B):
    blk = data[s:s + B]
    ins = sum(int(r[ci]) for r in blk)
    smp = sum(int(r[si]) for r in blk)
    if smp / stot < 0.01:
        continue
    st = collections.Counter()
    for r in blk:
        for i in stall:
            st[h[i][6:]] += int(r[i] or 0)
    ops = collections.Counter()
    for r in blk:
        t = r[1].strip().split()
        op = t[1] if t[0].startswith("@") else t[0]
        ops[op.split(".")[0]] += int(r[ci])
    act = sum(float(r[ti] or 0) * int(r[ci]) for r in blk) / max(ins, 1)
    print(f"[{s:5d},{s+B:5d}) inst {ins/tot*100:5.1f}% time {smp/stot*100:5.1f}% lanes {act:4.1f} | "
          + " ".join(f"{k}:{v/smp*100:.0f}" for k, v in st.most_common(4)) + " | "
          + " ".join(f"{k}:{v/ins*100:.0f}" for k, v in ops.most_common(5)))
