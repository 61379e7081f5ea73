"""Phase clocks of k_route_fifo in a record-level step (debug library): CUDA
graph of record-level steps (insert + sample, C5 N=84 T=1 shape), clocks of
the last step relative to the route's first CTA start."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["REPLAY_B200_LIB"] = os.path.join(ROOT, "paper_2604_08706_b200", "libreplay_b200_clocks.so")
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2604_08706_b200 as rb  # noqa: E402
from paper_2604_08706_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
N, T, B, G = 84, 1, 504, 8
buf = rb.ShardedReplayBuffer(T, N, max_tokens=0)
buf.set_stream(s.cuda_stream)
rng = rb.Rng(1).stream("buffer_sampling")


def make(nid, n):
    ids = torch.arange(nid, nid + n, dtype=torch.int64, device=dev)
    return dict(rollout_id=ids, reward=(ids % 3 == 0).to(torch.float64),
                group_offsets=torch.arange(0, n + 1, G, dtype=torch.int64, device=dev))


buf.insert(**make(0, 88), assume_unique=True)
plan = [make(1000 + 64 * i, 32) for i in range(12)]
for p in plan[:3]:
    buf.insert(**p, assume_unique=True)
    buf.sample_device(B, rng)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
    for p in plan[3:]:
        buf.insert(**p, assume_unique=True)
        buf.sample_device(B, rng)
torch.cuda.synchronize()
g.replay()
torch.cuda.synchronize()
_lib.lib.rb_debug_phase_clocks.argtypes = [C.c_void_p]
ck = (C.c_longlong * 64)()
_lib.check(_lib.lib.rb_debug_phase_clocks(ck))
t0 = ck[30]
names = {30: "route start", 31: "flags+fence+barrier", 32: "ctl loaded", 60: "loads+validation",
         61: "verdict", 62: "records written", 63: "done-count", 56: "last CTA start",
         57: "done flag", 40: "map t0 start", 41: "map0 enter", 46: "map0 after draws",
         47: "map0 after L loads", 44: "map0 after lookback", 45: "map0 end", 58: "finalize start",
         59: "finalize end"}
for i, nm in sorted(names.items(), key=lambda kv: ck[kv[0]]):
    if ck[i] > 0:
        print(f"  {nm:22s} {(ck[i] - t0) / 1e3:8.2f} us")
