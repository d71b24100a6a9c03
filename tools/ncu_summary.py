"""Summarise an ncu report: headline metrics, stall reasons, per-source-line instruction counts.
usage: python tools/ncu_summary.py report.ncu-rep [n_units_for_per_unit_counts]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0


def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
items = dict(zip(raw[0], raw[2]))
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
          "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
          "smsp__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
          "sm__warps_active.avg.pct_of_peak_sustained_active"]:
    if k in items:
        print(f"{k:70s} {items[k]}")
stalls = sorted(((float(v), h) for h, v in items.items()
                 if re.search(r"smsp__average_warps_issue_stalled_.*_per_issue_active.ratio", h) and v), reverse=True)
print("stalls (per issued inst):", ", ".join(f"{h.split('stalled_')[1].split('_per')[0]}={v:.2f}" for v, h in stalls[:8]))
rows = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source", "cuda,sass"]))))
cur = None
hdr = None
out = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":
        out.append((cur, int(r[0]), r[1].strip(), float(r[4] or 0), float(r[7] or 0)))
tot_i = sum(o[4] for o in out) or 1
tot_s = sum(o[3] for o in out) or 1
print(f"warp instructions per unit: {tot_i / units:.0f}")
for o in sorted(out, key=lambda o: -o[4])[:28]:
    print(f"{o[4] / units:9.0f} {o[4] / tot_i * 100:5.1f}%i {o[3] / tot_s * 100:5.1f}%s {o[0]}:{o[1]} {o[2][:80]}")
