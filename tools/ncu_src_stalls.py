"""Summarise an `ncu --page source --csv --print-source sass` export: stall reasons
per region of the SASS (ranges split at the given instruction indices) and the top
instructions.  usage: python tools/ncu_src_stalls.py file.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) >= len(hdr)]
# the export repeats the listing once per source view; keep the first copy
addrs = [r[0] for r in data]
if addrs.count(addrs[0]) > 1:
    data = data[:addrs.index(addrs[0], 1)]
reasons = [h for h in hdr[30:47]]
ri = [hdr.index(h) for h in reasons]
si = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
num = lambda s: int(s) if s.strip().isdigit() else 0
tot = sum(num(r[si]) for r in data)
agg = {h: sum(num(r[j]) for r in data) for h, j in zip(reasons, ri)}
print(f"instructions={len(data)} samples={tot}")
print("  ".join(f"{k[6:]}={100 * v / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1]) if v))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for i in sorted(sorted(range(len(data)), key=lambda i: -num(data[i][si]))[:top]):
    r = data[i]
    rs = sorted(((num(r[j]), h[6:]) for h, j in zip(reasons, ri)), reverse=True)[:2]
    print(f"{i:5d} {100 * num(r[si]) / tot:5.2f}% ex={num(r[ie]):>10d} {r[1].strip()[:60]:60s} {rs}")
