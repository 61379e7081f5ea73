"""Build an A/B variant of the library with extra nvcc defines:
    python tools/build_variant.py <name> -DFOO=1 ...
-> paper_2604_08706_b200/libreplay_b200_<name>.so (use with tools/ab.sh <name>)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2604_08706_b200"))
import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(B.HERE, f"libreplay_b200_{name}.so")
cmd = [B.NVCC, *B.FLAGS, *defs, "-o", out, *[os.path.join(B.CSRC, s) for s in B.SOURCES]]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr[-3000:])
print(out)
