"""Write profiles/traffic.json from ncu --set full captures: DRAM bytes (read + write) and shared-memory
wavefronts per launch for each kernel mode, with the capture date and the kernel build (git commit).
usage: python tools/traffic_json.py key=report.ncu-rep [key=report.ncu-rep ...]"""
import csv
import datetime
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path = os.path.join(ROOT, "profiles", "traffic.json")
out = json.load(open(path)) if os.path.exists(path) else {}
src = out.setdefault("source", {})
for arg in sys.argv[1:]:
    key, rep = arg.split("=", 1)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    m = dict(zip(rows[0], rows[2]))
    unit = rows[1][rows[0].index("dram__bytes_read.sum")]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
    out[key] = (float(m["dram__bytes_read.sum"]) + float(m["dram__bytes_write.sum"])) * scale
    out[key + "_smem_wavefronts"] = float(m["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"])
    src[key] = os.path.relpath(rep, ROOT)
src["how"] = ("ncu --set full --clock-control none, dram__bytes_read.sum + dram__bytes_write.sum and "
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum, one fused launch (A.v + v^T.A) over 1024 "
              "config-2 batches")
out["captured"] = datetime.date.today().isoformat()
out["kernel_build"] = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"], capture_output=True,
                                     text=True).stdout.strip()
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out, indent=1))
