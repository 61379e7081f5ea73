"""Phase clocks of the single-CTA kernels on the C4 workload (debug library)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["REPLAY_B200_LIB"] = os.path.join(ROOT, "paper_2604_08706_b200", "libreplay_b200_clocks.so")
sys.path.insert(0, ROOT)
sys.argv = ["bench.py", "--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu-baseline"]
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_08706_b200 import _lib  # noqa: E402

_lib.lib.rb_debug_phase_clocks.argtypes = [C.c_void_p]
args = bench.argparse.Namespace(steps=3, warmup=3, config=os.environ.get("CFG", "c4"), no_e2e=True, graph=False)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    res, buf, wl, rng = bench.run_ours(args, 0, 1, None)
torch.cuda.synchronize()
out = (C.c_longlong * 64)()
_lib.check(_lib.lib.rb_debug_phase_clocks(out))
ck = list(out)
mhz = 1.9e3
def show(name, idx):
    base = ck[idx[0]]
    print(name)
    for a, b in zip(idx, idx[1:]):
        print(f"  phase {a}->{b}: {ck[b] - ck[a]:8d} cycles ({(ck[b] - ck[a]) / mhz:7.2f} us @1.9GHz)")
show("k_sample_draw (0 start, 1 end)", [0, 1])
show("k_insert_route_fifo (20 start,21 phase1,22 after sync,23 metadata,24 end)", [20, 21, 22, 23, 24])
show("k_sample_map_coop (30 start,31 slots,32 after sync,33 scan)", [30, 31, 32, 33])
print("phases_ms", res["phases_ms"])
