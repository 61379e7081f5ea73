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
args = bench.argparse.Namespace(steps=3, warmup=3, config=os.environ.get("CFG", "c4"), no_e2e=True)
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
show("k_sample_with (0 start,1 draws done,2 map start,3 slots,4 offsets,5 units)", [0, 1, 2, 3, 4, 5])
show("k_insert_route (10 start,11 lengths,12 adv,13 risk,14 route,15 units,16 end)", [10, 11, 12, 13, 14, 15, 16])
print("phases_ms", res["phases_ms"])
