"""Write the per-kernel DRAM traffic that bench.py reports as roofline.traffic.

usage: python tools/ncu_traffic.py REPORT.ncu-rep OUT.json "capture description"
Reads one launch per kernel from an `ncu --set full` report (dram__bytes_read.sum,
dram__bytes_write.sum, gpu__time_duration.sum, FP64 pipe, warps, L2 hit rate)."""
import csv
import json
import math
import subprocess
import sys

M = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
     "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
     "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "lts__t_sector_hit_rate.pct"]
rep, out, desc = sys.argv[1], sys.argv[2], sys.argv[3]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(txt.splitlines()))
h, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3}


def val(row, m):
    i = h.index(m)
    try:
        v = float(row[i])
    except ValueError:
        return None
    if math.isnan(v):
        return None
    return v * scale.get(units[i], 1.0)


kern = {}
for row in rows[2:]:
    name = row[h.index("Kernel Name")].split("(")[0].split("<")[0].replace("void ", "").strip()
    name = name.split("::")[-1]
    if name in kern:
        continue
    kern[name] = {"dram_read_bytes": val(row, M[0]), "dram_write_bytes": val(row, M[1]),
                  "duration_ms": val(row, M[2]), "fp64_pipe_pct": val(row, M[3]),
                  "warps_active_per_sm": val(row, M[4]), "registers": val(row, M[5]),
                  "l2_hit_pct": val(row, M[6])}
json.dump({"capture": desc, "kernels": kern}, open(out, "w"), indent=1)
print(json.dumps(kern, indent=1))
