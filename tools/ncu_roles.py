"""Stall-sample breakdown of one kernel by code region (line ranges of one source file).
Usage: python tools/ncu_roles.py report.ncu-rep function-substring file.cuh name:first_line ...
Lines from other files count under that file's name."""
import collections
import csv
import io
import subprocess
import sys

rep, want, src = sys.argv[1], sys.argv[2], sys.argv[3]
cuts = [(a.split(":")[0], int(a.split(":")[1])) for a in sys.argv[4:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
func = fname = ""
h = None
agg = collections.defaultdict(collections.Counter)
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Function Name":
        func = r[1]
        continue
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        h = r
        continue
    if want not in func or h is None or not r or not r[0].isdigit():
        continue
    ln = int(r[0])
    reg = fname
    if fname == src:
        reg = "?"
        for name, first in cuts:
            if ln >= first:
                reg = name
    for i, n in enumerate(h):
        if n.startswith("stall_") and "Not Issued" not in n:
            try:
                agg[reg][n[6:]] += int(r[i] or 0)
            except ValueError:
                pass
    try:
        agg[reg]["_ins"] += int(r[7] or 0)
    except ValueError:
        pass
tot = sum(sum(v for k, v in c.items() if k != "_ins") for c in agg.values()) or 1
itot = sum(c["_ins"] for c in agg.values()) or 1
for reg, c in sorted(agg.items(), key=lambda x: -sum(v for k, v in x[1].items() if k != "_ins")):
    s = sum(v for k, v in c.items() if k != "_ins") or 1
    top = ", ".join(f"{k} {100 * v / s:.0f}%" for k, v in c.most_common(8) if k != "_ins")
    print(f"{reg:22s} {100 * s / tot:5.1f}% smp {100 * c['_ins'] / itot:5.1f}% ins | {top}")
