"""Per-source-line stall samples, instructions and shared wavefronts from an ncu report.
usage: python tools/ncu_lines.py report.ncu-rep [units] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = hdr = None
out = []
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        ix = {h: i for i, h in enumerate(r)}
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":
        def f(name):
            i = ix.get(name)
            try:
                return float(r[i]) if i is not None and r[i] not in ("", "-") else 0.0
            except ValueError:
                return 0.0
        out.append((cur, int(r[0]), r[1].strip(), f("Warp Stall Sampling (All Samples)"), f("Instructions Executed"),
                    f("L1 Wavefronts Shared"), f("L1 Wavefronts Shared Ideal")))
ts = sum(o[3] for o in out) or 1
ti = sum(o[4] for o in out)
tw = sum(o[5] for o in out)
print(f"per unit: instructions {ti / units:.0f}  shared wavefronts {tw / units:.0f} (ideal {sum(o[6] for o in out) / units:.0f})")
for o in sorted(out, key=lambda o: -o[3])[:top]:
    print(f"stall {o[3] / ts * 100:5.1f}%  instr {o[4] / units:8.0f}  wf {o[5] / units:7.0f}  {o[0]}:{o[1]} {o[2][:72]}")
