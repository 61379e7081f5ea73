"""Phase clocks (globaltimer, ns) of k_sample_prio on the C4 buffer shape
(debug library built with -DRB_PHASE_CLOCKS: python paper_2604_08706_b200/build.py --clocks)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["REPLAY_B200_LIB"] = os.path.join(ROOT, "paper_2604_08706_b200", "libreplay_b200_clocks.so")
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2604_08706_b200 import _lib  # noqa: E402
from tools.prio_probe import run  # noqa: E402

_lib.lib.rb_debug_phase_clocks.argtypes = [C.c_void_p]
for cap, batch in [(16384, 4096), (16384, 512), (1024, 4096), (1024, 1024)]:  # one shard
    us = run(cap, batch, "priority_with_replacement", (1, 65536, 4096), iters=5)
    torch.cuda.synchronize()
    out = (C.c_longlong * 64)()
    _lib.check(_lib.lib.rb_debug_phase_clocks(out))
    ck = list(out)
    names = {9: "weights", 10: "scan", 11: "twist", 12: "words+rank", 13: "modulo",
             15: "search", 14: "shard0 end"}
    print(f"cap={cap} batch={batch} call {us:.1f} us:",
          " ".join(f"{nm}={(ck[i] - ck[8]) / 1e3:.1f}" for i, nm in names.items()), "(us from start)")
