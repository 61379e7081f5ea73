"""Condense the ncu evidence of one round into profiles/.

    python tools/profile_summary.py <round-tag>   (reads gpurun_out/)

Writes profiles/<tag>_launches.csv (per-launch list, steady-state step),
profiles/<tag>_kernels.md (per-kernel metrics of the --set full captures),
and profiles/ncu_traffic.json (DRAM bytes per launch of each captured kernel,
read by bench.py for the roofline `traffic` field).
"""
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from launches import load  # noqa: E402
from ncu_summary import metrics  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
if tag.startswith("-"):
    sys.exit(__doc__)
src = os.path.join(ROOT, "gpurun_out")
dst = os.path.join(ROOT, "profiles")
os.makedirs(dst, exist_ok=True)

# launch list
L = load(os.path.join(src, "launches.csv"))
shutil.copy(os.path.join(src, "launches.csv"), os.path.join(dst, f"{tag}_launches_raw.csv"))
with open(os.path.join(dst, f"{tag}_launches.csv"), "w") as f:
    f.write("kernel,duration_ns,dram_read_bytes,dram_write_bytes\n")
    for n, m in L:
        f.write(f"{n},{m.get('gpu__time_duration.sum', 0):.0f},{m.get('dram__bytes_read.sum', 0):.0f},"
                f"{m.get('dram__bytes_write.sum', 0):.0f}\n")

# full captures
traffic = {}
lines = [f"# ncu --set full captures ({tag})", "",
         "One steady-state launch of each kernel of the C4 replay step, captured with",
         "`ncu --set full --clock-control none --import-source on` (tools/gpu_round.sh).",
         "ncu replays each kernel with flushed caches: durations are cold-cache and serialised.", ""]
for fn in sorted(os.listdir(src)):
    if not (fn.startswith("prof_") and fn.endswith(".ncu-rep")):
        continue
    name = fn[5:-8]
    rep = os.path.join(src, fn)
    shutil.copy(rep, os.path.join(dst, f"{tag}_{fn}"))
    res, top = metrics(rep)
    rd = float(res.get("dram__bytes_read.sum", 0) or 0)
    wr = float(res.get("dram__bytes_write.sum", 0) or 0)
    traffic[name] = rd + wr  # bytes (ncu_summary normalises units)
    lines.append(f"## {name}")
    for k, v in res.items():
        lines.append(f"- `{k}` = {v}")
    lines.append("- top stalls (warps per issue): " + ", ".join(f"{k}={x:.2f}" for x, k in top))
    lines.append("")
with open(os.path.join(dst, f"{tag}_kernels.md"), "w") as f:
    f.write("\n".join(lines) + "\n")
with open(os.path.join(dst, "ncu_traffic.json"), "w") as f:
    json.dump(traffic, f, indent=1, sort_keys=True)
print("wrote", dst, sorted(traffic))
