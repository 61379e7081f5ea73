"""Top SASS instructions by warp-stall samples from an ncu report's source page.

    python tools/ncu_sass_hot.py report.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ci = {k: i for i, k in enumerate(h)}
col = ci["Warp Stall Sampling (All Samples)"]
data = []
for idx, r in enumerate(rows[2:]):
    try:
        data.append((float(r[col]), idx, r[ci["Address"]], r[ci["Source"]].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
print(f"total samples {tot:.0f}, instructions {len(data)}")
for s, idx, addr, src in sorted(data, reverse=True)[:n]:
    print(f"{s:6.0f} {100 * s / tot:5.1f}%  #{idx:5d} {src[:90]}")
