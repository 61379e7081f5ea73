"""Time one sampling call (rb_sample, device outputs only) of the
priority_with_replacement strategy against uniform_with_replacement on the
C4 (16384 / B = 4096, one shard and 8 shards) and C3 (1024 / B = 1024) buffer
shapes, metadata only.  Back-to-back eager calls: host launch overhead included.
CUDA events on the buffer's stream (torch's current stream), after warm-up.

    python tools/prio_probe.py  ->  one JSON line per (shape, strategy)
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(cap, batch, strategy, prio, iters=50, shards=1):
    import torch

    import paper_2604_08706_b200 as rb

    b = rb.ShardedReplayBuffer(shards, cap, strategy=strategy)
    b.set_stream(torch.cuda.current_stream().cuda_stream)
    if prio is not None:
        b.set_priority(*prio)
    rs = np.random.default_rng(1)
    g = 16
    n = cap
    b.insert(rollout_id=np.arange(n, dtype=np.uint64), reward=rs.integers(0, 2, n).astype(np.float64),
             prompt_id=np.arange(n) // g, group_id=np.arange(n) // g,
             group_offsets=np.arange(0, n + 1, g), assume_unique=True)
    rng = rb.Rng(3).stream("buffer_sampling")
    for _ in range(5):
        b.sample_device(batch, rng)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        b.sample_device(batch, rng)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters


def main():
    for cap, batch, shape, shards in [(16384, 4096, "C4", 1), (1024, 1024, "C3", 1),
                                      (16384, 4096, "C4 in 8 shards", 8)]:
        for strategy, prio in [("uniform_with_replacement", None),
                               ("priority_with_replacement", (1, 0, 0)),
                               ("priority_with_replacement", (1, 65536, 4096))]:
            us = run(cap, batch, strategy, prio, shards=shards)
            print(json.dumps({"shape": shape, "capacity": cap, "batch": batch, "shards": shards,
                              "strategy": strategy, "priority": prio,
                              "us_per_sample_call": round(us, 2)}), flush=True)


if __name__ == "__main__":
    main()
