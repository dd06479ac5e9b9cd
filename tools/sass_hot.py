"""Summarise an ncu source page (SASS, --csv) by stall reason and hot spots.
usage: ncu -i X.ncu-rep --page source --csv --print-source sass > s.csv
       python tools/sass_hot.py s.csv [top]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = Counter()
for d in data:
    for c in stall_cols:
        tot[c] += int(d[c] or 0)
S = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
print("total samples", S)
for c, v in tot.most_common():
    if v:
        print(f"  {c:28s} {v:8d} {100 * v / S:5.1f}%")
print()
hot = sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:top]
for d in hot:
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    why = sorted(((int(d[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    print(f"{d['Address'][-5:]} {s:6d} {100 * s / S:4.1f}%  {d['Source'].strip()[:60]:60s} "
          + " ".join(f"{c}={v}" for v, c in why if v))
