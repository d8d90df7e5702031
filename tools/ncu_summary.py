"""Extract the numbers the bench and DESIGN.md cite from an `ncu --set full` report.
Usage: python tools/ncu_summary.py report.ncu-rep [name]  -> JSON on stdout."""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
m = dict(zip(hdr, vals))
u = dict(zip(hdr, units))


def num(k):
    v = m.get(k, "").replace(",", "")
    try:
        return float(v)
    except ValueError:
        return None


def scaled(k):
    v, unit = num(k), u.get(k, "")
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
            "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
            "s": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9, "B": 1, "hz": 1, "Khz": 1e3, "Mhz": 1e6,
            "Ghz": 1e9, "KHz": 1e3, "MHz": 1e6, "GHz": 1e9}.get(unit, 1)
    return None if v is None else v * mult


out = {
    "kernel": m.get("Kernel Name"),
    "duration_s": scaled("gpu__time_duration.sum"),
    "dram_read_bytes": scaled("dram__bytes_read.sum"),
    "dram_write_bytes": scaled("dram__bytes_write.sum"),
    "registers_per_thread": num("launch__registers_per_thread"),
    "block_size": num("launch__block_size"),
    "grid_size": num("launch__grid_size"),
    "shared_mem_per_block_bytes": scaled("launch__shared_mem_per_block_dynamic"),
    "achieved_occupancy_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "ipc_active": num("sm__inst_executed.avg.per_cycle_active"),
    "issue_active_pct": num("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
    "inst_issued_pct": num("sm__inst_issued.avg.pct_of_peak_sustained_active"),
    "inst_executed": num("smsp__inst_executed.sum"),
    "alu_pipe_pct": num("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    "fma_pipe_pct": num("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
    "lsu_pipe_pct": num("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    "sm_clock_hz": scaled("smsp__cycles_elapsed.avg.per_second"),
    "shared_ld_wavefronts": num("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"),
    "shared_bank_conflicts": num("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    "shared_wavefronts": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    "shared_pipe_pct": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
}
# shared-memory bandwidth: every wavefront moves up to 128 B (32 banks x 4 B)
if out["shared_wavefronts"] is not None and out["duration_s"]:
    out["shared_gbs_upper"] = out["shared_wavefronts"] * 128 / out["duration_s"] / 1e9
if out["dram_read_bytes"] is not None and out["duration_s"]:
    out["dram_gbs"] = (out["dram_read_bytes"] + (out["dram_write_bytes"] or 0)) / out["duration_s"] / 1e9
if out["dram_read_bytes"] is not None and out["dram_write_bytes"] is not None:
    out["dram_bytes"] = out["dram_read_bytes"] + out["dram_write_bytes"]
out["units"] = {k: u.get(k) for k in ("gpu__time_duration.sum", "dram__bytes_read.sum")}
if len(sys.argv) > 2:
    out["name"] = sys.argv[2]
print(json.dumps(out, indent=1))
