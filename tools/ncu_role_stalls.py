"""Stall reasons and instruction counts per kernel role, by SASS address range: the range of a
role is spanned by the SASS of its CUDA source lines (inlined helpers inside it included).
Usage: python tools/ncu_role_stalls.py report.ncu-rep file.cuh name:first-last [name:first-last ...]"""
import collections
import csv
import io
import subprocess
import sys

rep, fname = sys.argv[1], sys.argv[2]
roles = []
for a in sys.argv[3:]:
    n, rng = a.split(":")
    lo, hi = (int(x) for x in rng.split("-"))
    roles.append((n, lo, hi))
cs = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                    capture_output=True, text=True).stdout
addr_lines = collections.defaultdict(list)  # role -> addresses
cur_file, cur_line = "", None
for r in csv.reader(io.StringIO(cs)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0].isdigit():
        cur_line = int(r[0])
        continue
    if r[0] == "" and len(r) > 3 and r[2].startswith("0x") and cur_file == fname and cur_line:
        for n, lo, hi in roles:
            if lo <= cur_line <= hi:
                addr_lines[n].append(int(r[2], 16))
ranges = {n: (min(v), max(v)) for n, v in addr_lines.items() if v}
ss = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                    capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(ss)))
h, data = rows[1], rows[2:]
ci, si = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
stall = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
tot_s = sum(int(r[si]) for r in data)
tot_i = sum(int(r[ci]) for r in data)
for n, (lo, hi) in ranges.items():
    sel = [r for r in data if lo <= int(r[0], 16) <= hi]
    smp = sum(int(r[si]) for r in sel)
    ins = sum(int(r[ci]) for r in sel)
    st = collections.Counter()
    for r in sel:
        for i in stall:
            st[h[i][6:]] += int(r[i] or 0)
    ops = collections.Counter()
    for r in sel:
        t = r[1].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
        ops[op.split(".")[0]] += int(r[ci])
    top = ", ".join(f"{k} {100 * v / max(smp, 1):.0f}%" for k, v in st.most_common(6))
    topo = ", ".join(f"{k} {v / 1e6:.1f}M" for k, v in ops.most_common(8))
    print(f"{n:10s} {hex(lo)}-{hex(hi)}: {100 * smp / tot_s:5.1f}% samples, {ins / 1e6:7.1f}M warp-instr "
          f"({100 * ins / tot_i:4.1f}%) | {top}\n           ops: {topo}")
