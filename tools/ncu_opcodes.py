"""Warp-instruction mix by SASS opcode for one kernel of an ncu report.
Usage: python tools/ncu_opcodes.py report.ncu-rep function-substring [topN]"""
import collections
import csv
import io
import subprocess
import sys

rep, want = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
cnt = collections.Counter()
func = ""
h = None
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Kernel Name":
        func = r[1]
        continue
    if r and r[0] == "Address":
        h = r
        continue
    if want not in func or h is None or len(r) < 6:
        continue
    op = r[1].split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1] if len(op) > 1 else o
    try:
        cnt[o.split(".")[0]] += int(r[h.index("Instructions Executed")] or 0)
    except ValueError:
        pass
tot = sum(cnt.values()) or 1
print(f"total warp-instructions {tot:.4g}")
for o, v in cnt.most_common(top):
    print(f"{o:10s} {100 * v / tot:5.1f}%  {v:.4g}")
