"""Share of the step per kernel from an ncu launch list (--metrics gpu__time_duration.sum --csv).
usage: python tools/launch_share.py launches.csv"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
ui = h.index("Metric Unit")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
    v = float(r[vi].replace(",", ""))
    v *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1.0)
    tot[name] += v
    cnt[name] += 1
s = sum(tot.values())
print(f"{sum(cnt.values())} launches, {s:.1f} ms")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"| {k} | {100 * v / s:.1f} % | {cnt[k]} | {v / cnt[k]:.3f} ms |")
