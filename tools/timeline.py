"""Per-kernel GPU timeline of one C4 replay step (debug library, global timer).

Runs warm-up steps eagerly, resets the timeline, runs one more step and
prints each kernel's [start, end] relative to the step's first kernel."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["REPLAY_B200_LIB"] = os.environ.get("TIMELINE_LIB") or os.path.join(
    ROOT, "paper_2604_08706_b200", "libreplay_b200_clocks.so")
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_08706_b200 import _lib  # noqa: E402

_lib.lib.rb_debug_timeline.argtypes = [C.c_void_p, C.c_int]
_lib.lib.rb_debug_timeline_loss.argtypes = [C.c_void_p, C.c_int]
NAMES = ["route_fifo", "payload", "draw", "map", "gather", "loss", "gen"]
steps = int(os.environ.get("STEPS", "4"))
args = bench.argparse.Namespace(steps=steps, warmup=3, config=os.environ.get("CFG", "c4"),
                                no_e2e=True, graph=os.environ.get("GRAPH", "0") == "1", check=False)
out = (C.c_ulonglong * 64)()
out2 = (C.c_ulonglong * 64)()


def reset():
    _lib.check(_lib.lib.rb_debug_timeline(out, 1))
    _lib.check(_lib.lib.rb_debug_timeline_loss(out2, 1))


args.pre_timed = reset
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    res, buf, wl, rng = bench.run_ours(args, 0, int(os.environ.get("EMU_WORLD", "1")), None)
torch.cuda.synchronize()
_lib.check(_lib.lib.rb_debug_timeline(out, 0))
_lib.check(_lib.lib.rb_debug_timeline_loss(out2, 0))
t = list(out)
t[10], t[11] = out2[10], out2[11]
print("(timeline spans all timed steps; first start .. last end per kernel)")
t0 = min(t[2 * k] for k in range(len(NAMES)) if t[2 * k] != 2**64 - 1)
for k, n in enumerate(NAMES):
    a, b = t[2 * k], t[2 * k + 1]
    if a == 2**64 - 1:
        continue
    ls = t[32 + k] if k != 5 else out2[32 + k]
    print(f"{n:12s} start {(a - t0) / 1e3:9.2f} us  last CTA start {(ls - t0) / 1e3:9.2f} us"
          f"  end {(b - t0) / 1e3:9.2f} us")
print("phases_ms", res["phases_ms"], "ms_per_step", res["ms_per_step"])
_lib.lib.rb_debug_phase_clocks.argtypes = [C.c_void_p]
ck = (C.c_longlong * 64)()
_lib.check(_lib.lib.rb_debug_phase_clocks(ck))
lb = (C.c_longlong * 2)()
_lib.check(_lib.lib.rb_debug_locb(lb))
print("local twist blocks (locb - qhi0; -1 none):", list(lb))
names = {40: "map t0 start", 41: "map0 enter", 42: "map0 after local twist", 46: "map0 after draws",
         47: "map0 after L loads", 43: "map0 after loads",
         44: "map0 after lookback", 45: "map0 end", 49: "map1 enter", 50: "map1 after local twist",
         54: "map1 after draws", 55: "map1 after L loads",
         51: "map1 after loads", 52: "map1 after lookback", 53: "map1 end", 58: "finalize start",
         59: "finalize end", 60: "route0 loads+validation", 61: "route0 verdict",
         62: "route0 records written", 63: "route0 done-count", 56: "route last CTA start",
         57: "route done flag"}
names.update({i: f"clock {i}" for i in range(64) if i not in names})
for i, nm in sorted(names.items()):
    if ck[i] > 0:
        print(f"  {nm:22s} {(ck[i] - t0) / 1e3:9.2f} us")
