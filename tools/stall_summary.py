"""Per-region stall breakdown of an ncu source page (SASS):
python tools/stall_summary.py <source.csv> — groups instructions into the
regions delimited by the kernel's mbarrier waits and prints, per region, the
total samples and the top stall reasons (used for profiles/*_stalls.md)."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = Counter()
by_op = Counter()
insts = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    samples = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    st = {k: int(r[ix[k]] or 0) for k in stalls}
    insts.append((r[ix["Address"]], src, samples, st))
    for k, v in st.items():
        tot[k] += v
    by_op[op.split(".")[0]] += samples
allS = sum(tot.values())
print(f"total stall samples {allS}")
for k, v in tot.most_common(10):
    print(f"  {k:24s} {100 * v / allS:5.1f}%")
print("samples by opcode:")
for k, v in by_op.most_common(15):
    print(f"  {k:14s} {100 * v / allS:5.1f}%")
print("hottest instructions:")
for a, src, s, st in sorted(insts, key=lambda x: -x[2])[:25]:
    top = ", ".join(f"{k[6:]} {v}" for k, v in Counter(st).most_common(2) if v)
    print(f"  {s:7d} {src[:70]:70s} {top}")
