"""Phase clocks of k_posbias_par in a C2-shaped record-level step (debug
library): buffer 84, one shard, positive bias delta = 0.5, 160 records per
insert in groups of 8 (about half correct), then a sample of 512; a CUDA
graph of such steps, clocks of the last step relative to the kernel's start."""
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
N, B, G, R = 84, 512, 8, int(os.environ.get("PB_R", "160"))
buf = rb.ShardedReplayBuffer(1, N, "uniform_with_replacement", "positive_bias", 0.5, max_tokens=0)
buf.set_stream(s.cuda_stream)
rng = rb.Rng(1).stream("buffer_sampling")


def make(nid, n):
    ids = torch.arange(nid, nid + n, dtype=torch.int64, device=dev)
    return dict(rollout_id=ids, reward=((ids * 7) % 5 < 2).to(torch.float64),
                group_offsets=torch.arange(0, n + 1, G, dtype=torch.int64, device=dev))


buf.insert(**make(1, 88), assume_unique=True)
nid = [1000]


def plan(k):
    out = []
    for _ in range(k):
        out.append(make(nid[0], R))
        nid[0] += 1000
    return out


for p in plan(3):
    buf.insert(**p, assume_unique=True)
    buf.sample_device(B, rng)
torch.cuda.synchronize()
buf.check()
graphs, keep = [], []
for _ in range(4):  # fresh ids in every graph: each is replayed once
    ps = plan(9)
    keep.append(ps)  # the graphs read these tensors
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
        for p in ps:
            buf.insert(**p, assume_unique=True)
            buf.sample_device(B, rng)
    graphs.append(g)
torch.cuda.synchronize()
graphs[0].replay()
torch.cuda.synchronize()
buf.check()
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st.record(s)
for g in graphs[1:]:
    g.replay()
en.record(s)
torch.cuda.synchronize()
buf.check()
print(f"R={R}  step (insert + sample) {st.elapsed_time(en) * 1e3 / 27:8.2f} us")
_lib.lib.rb_debug_phase_clocks.argtypes = [C.c_void_p]
ck = (C.c_longlong * 64)()
_lib.check(_lib.lib.rb_debug_phase_clocks(ck))
t0 = ck[20]
names = {20: "posbias start", 29: "after griddepcontrol.wait", 21: "state loaded + verdict", 22: "rings in smem", 23: "victims",
         24: "slots (pointer jumping)", 25: "queues rewritten", 26: "records written",
         27: "order materialised", 28: "done", 40: "map t0 start", 41: "map0 enter",
         46: "map0 after draws", 47: "map0 after L loads", 44: "map0 after lookback",
         45: "map0 end", 58: "finalize start", 59: "finalize end"}
for i, nm in sorted(names.items(), key=lambda kv: ck[kv[0]]):
    if ck[i] > 0:
        print(f"  {nm:26s} {(ck[i] - t0) / 1e3:8.2f} us")
