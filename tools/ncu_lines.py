"""Per-CUDA-source-line totals (stall samples, warp instructions) from an ncu report.
Usage: python tools/ncu_lines.py report.ncu-rep [topN] [function-substring]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
want = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
smp = collections.Counter()
ins = collections.Counter()
text = {}
fname = ""
hdr = None
func = ""
for r in rows:
    if r and r[0] == "Function Name":
        func = r[1]
        continue
    if want and want not in func:
        continue
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or not r[0].isdigit():
        continue
    key = (fname, int(r[0]))
    text[key] = r[1].strip()
    try:
        smp[key] += int(r[4] or 0)
        ins[key] += int(r[7] or 0)
    except ValueError:
        pass
tot = sum(smp.values()) or 1
itot = sum(ins.values()) or 1
print(f"samples {tot} warp-instructions {itot:.4g}")
for key, v in smp.most_common(top):
    print(f"{key[0]}:{key[1]:<5d} {100 * v / tot:5.1f}% smp {100 * ins[key] / itot:5.1f}% ins | {text[key][:80]}")
