"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Address" in r and "Source" in r][0]
h, data = rows[hi], rows[hi + 1:]
si, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
ie = h.index("Instructions Executed")
data = [r for r in data if len(r) > si and r[si].strip().isdigit()]
tot = sum(int(r[si]) for r in data) or 1
print("samples", tot, "instructions", sum(int(r[ie] or 0) for r in data))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for k, r in sorted(enumerate(data), key=lambda kr: -int(kr[1][si]))[:n]:
    print(f"{int(r[si]):6d} {100 * int(r[si]) / tot:5.1f}% #{k:5d} exec={r[ie]:>8s}  {r[src].strip()[:80]}")
