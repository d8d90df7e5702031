"""Build profiles/ncu_counters.json (what bench.py reports under "ncu" and roofline.traffic)
from the ncu --set full captures of tools/capture_r02.sh, tagged with the build id of the
library that was captured.  Usage: python tools/make_ncu_counters.py gpurun_out/build_id.txt
c3=gpurun_out/prof_c3.ncu-rep c4=gpurun_out/prof_c4.ncu-rep"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
bid = open(sys.argv[1]).read().split("src ")[-1].strip()
out = {"build": bid, "source": "ncu --set full --clock-control none, one launch of the step's "
                                "dominant kernel (match_tc16 for c3 / c4, match_tcp for c2), "
                                "tools/capture_r02.sh"}
keep = ("kernel", "duration_s", "dram_bytes", "dram_gbs", "alu_pipe_pct", "fma_pipe_pct",
        "lsu_pipe_pct", "issue_active_pct", "ipc_active", "inst_executed", "sm_clock_hz",
        "shared_wavefronts", "shared_bank_conflicts", "shared_gbs_upper", "shared_pipe_pct",
        "achieved_occupancy_pct", "registers_per_thread")
for arg in sys.argv[2:]:
    name, rep = arg.split("=", 1)
    js = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, name],
                        capture_output=True, text=True, check=True).stdout
    d = json.loads(js)
    out[name] = {k: d.get(k) for k in keep}
with open(os.path.join(ROOT, "profiles", "ncu_counters.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
