"""C5 latency anatomy: per-step time of a CUDA graph of K record-level steps
(insert + sample), of K samples alone and of K inserts alone (N=84, T=1)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2604_08706_b200 as rb  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
N, T, B, G, K = int(os.environ.get("N", 84)), int(os.environ.get("T", 1)), 504, 8, 100


def make(nid, n, step):
    ids = torch.arange(nid, nid + n, dtype=torch.int64, device=dev)
    rew = (torch.rand(n, device=dev) < 0.5).to(torch.float64)
    return dict(rollout_id=ids, reward=rew, group_id=ids // G,
                creation_step=torch.full((n,), step, dtype=torch.int64, device=dev),
                group_offsets=torch.arange(0, n + 1, G, dtype=torch.int64, device=dev))


for mode in ("both", "sample", "insert"):
    buf = rb.ShardedReplayBuffer(T, N, max_tokens=0)
    buf.set_stream(stream.cuda_stream)
    rng = rb.Rng(1).stream("buffer_sampling")
    buf.insert(**make(0, N + N % G, 0), assume_unique=True)
    plan = [make(10**6 + i * 64, 32, i + 1) for i in range(K + 3)]

    def step(p):
        if mode != "sample":
            buf.insert(**p, assume_unique=True)
        if mode != "insert":
            buf.sample_device(B, rng)

    for p in plan[:3]:
        step(p)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream, capture_error_mode="relaxed"):
        for p in plan[3:]:
            step(p)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    buf.check()
    print(f"{mode:7s} {e0.elapsed_time(e1) / K * 1e3:6.2f} us/step")
