"""Emulated strong scaling of C4 (rank 0 of an N-GPU job alone on one GPU):
reads gpurun_out/emu_<N>.json (graph timing) and emu_ph_<N>.json (--phases)
written by tools/evidence_scaling.sh and prints the markdown table committed
under profiles/."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = os.path.join(ROOT, "gpurun_out")


def last(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


rows = []
for n in (1, 2, 4, 8):
    try:
        d, p = last(os.path.join(out, f"emu_{n}.json")), last(os.path.join(out, f"emu_ph_{n}.json"))
    except (OSError, ValueError, IndexError) as e:
        sys.exit(f"missing emulation output for N={n}: {e}")
    ph = p["phases_ms"]
    rows.append((n, d["ms_per_step"] * 1e3, ph.get("insert_sample_gather", 0) * 1e3,
                 ph.get("loss", 0) * 1e3, d["value"], d["config"]["workload"]))
base = rows[0][1]
print("| N | rank-0 step (µs, graph) | insert+sample+gather (µs, eager phases) | loss + finalize (µs) "
      "| job tokens/s | strong-scaling efficiency N=1 step / (N x step) |")
print("|---|---|---|---|---|---|")
for n, st, f, l, v, _ in rows:
    print(f"| {n} | {st:.1f} | {f:.1f} | {l:.1f} | {v:.3g} | {base / (n * st):.2f} |")
print()
for n, *_, w in rows:
    print(f"- N={n}: {w}")
