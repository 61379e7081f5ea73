"""Build libreplay_b200.so in-tree for sm_100a (nvcc -shared)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libreplay_b200.so")
SOURCES = ["rng.cu", "buffer.cu", "loss.cu", "queue.cu", "ledger.cu"]
HEADERS = ["common.cuh", "rng_internal.cuh", "buffer_internal.cuh", "stream_copy.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--shared", "-Xcompiler", "-fPIC",
    "-Xcompiler", "-fvisibility=hidden", "-Xptxas", "-v",
    "-I", os.path.join(ROOT, "include"), "-I", CSRC,
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps += [os.path.join(ROOT, "include", "replay_b200.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, debug_clocks: bool = False) -> str:
    lib = LIB.replace(".so", "_clocks.so") if debug_clocks else LIB
    if not force and not debug_clocks and not _stale():
        return LIB
    extra = ["-DRB_PHASE_CLOCKS"] if debug_clocks else []
    cmd = [NVCC, *FLAGS, *extra, "-o", lib + ".tmp", *[os.path.join(CSRC, s) for s in SOURCES]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stderr[-6000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    os.replace(lib + ".tmp", lib)
    if verbose:
        print(r.stderr)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                debug_clocks="--clocks" in sys.argv))
