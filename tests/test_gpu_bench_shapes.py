"""Parity at the benchmarked shapes.

* bench.py itself, on each BASELINE config at its full shape, through the
  default kernels it times (C4: k_route_fifo -> k_insert_payload_tma ->
  k_sample_fused -> k_gather -> k_loss_grpo_buf, captured in a CUDA graph):
  three warm-up and three timed steps, then its --check leg replays the
  whole schedule through the CPU oracle and compares the last step's sampled
  trajectories, packed offsets and tokens, dL/dlogp (rtol 1e-5) and
  objective, and the final contents of every shard (use counts, frozen
  advantages).
* the GRPO fast path (fp32 ratio, one ex2 per token) against the oracle's
  fp64 reference arithmetic (bandit.cpp:375-406) with |logp_now - logp_old|
  spread over 1e-3 .. 79 with both signs and both signs of the advantage, on
  trajectories long enough to span several work units (> 2048 tokens).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from tests.harness import Producer, StepConfig, insert_groups

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(config, *extra):
    if not torch.cuda.is_available():
        pytest.fail("GPU test requested but CUDA is not available")
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", config, "--steps", "3",
           "--warmup", "3", "--no-e2e", "--no-cpu-baseline", *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    return line


@pytest.mark.parametrize("config", ["c4", "c1", "c2", "c3", "c4prio"])
def test_bench_step_matches_oracle_at_full_shape(config):
    line = _bench(config)
    chk = line["parity_check"]
    assert line["parity"] == "ok", (line["parity"], chk)
    assert chk["tokens_checked"] > 0
    assert chk["dlogp_max_rel_err"] <= 1e-5


def test_bench_c4_eager_matches_oracle():
    """The same C4 steps launched eagerly (no CUDA graph)."""
    line = _bench("c4", "--eager")
    assert line["parity"] == "ok", line["parity_check"]


@pytest.mark.parametrize("ratio_sign", [1, -1])
def test_grpo_fast_path_large_log_ratio(oracle, ratio_sign):
    from paper_2604_08706_b200 import Rng, ShardedReplayBuffer

    cfg = StepConfig(capacity=64, shards=1, batch=48, group=8, lmax=5000, ragged=True, seed=29)
    buf = ShardedReplayBuffer(1, cfg.capacity, max_tokens=cfg.lmax)
    buf.set_stream(torch.cuda.current_stream().cuda_stream)
    ob = oracle.buffer(1, cfg.capacity)
    prod = Producer(cfg, oracle)
    while ob.size() < cfg.capacity:
        rec, length, tok, lpo, toff, _ = prod.groups(2, 0)
        insert_groups(buf, rec, toff, tok, lpo, cfg.group, "cuda:0")
        for r in rec:
            ob.push(r)
    buf.sample_device(cfg.batch, Rng(cfg.seed).stream("buffer_sampling"))
    orec = ob.sample(cfg.batch, oracle.rng(cfg.seed).stream("buffer_sampling"))[0]
    ids, lens, off = buf.batch_ids()
    assert np.array_equal(ids, orec["rollout_id"])
    assert int(lens.max()) > 2048, "needs multi-unit trajectories"
    total = int(off[-1])
    _, lpo, _ = oracle.synth_payload(cfg.seed, ids, lens)
    rs = np.random.default_rng(5 + ratio_sign)
    mag = 10.0 ** rs.uniform(-3.0, np.log10(79.0), total)
    sign = np.where(rs.random(total) < 0.5, -1.0, 1.0) * ratio_sign
    lpn = (lpo.astype(np.float64) + sign * mag).astype(np.float32)
    pad = total + 8
    lpn_d = torch.zeros(pad, dtype=torch.float32, device="cuda:0")
    lpn_d[:total] = torch.from_numpy(lpn)
    dl = torch.zeros(pad, dtype=torch.float32, device="cuda:0")
    torch.cuda.synchronize()
    st = buf.loss_grpo(lpn_d, dl, 0.2, 0.28)
    d_want, obj, inc, exc = oracle.loss_grpo_tokens(lpn, lpo, orec["advantage"], off, 0.2, 0.28)
    got = dl[:total].cpu().numpy()
    assert (st.included, st.excluded) == (inc, exc)
    assert (orec["advantage"] > 0).any() and (orec["advantage"] < 0).any()
    live = np.abs(d_want) > 1e-30  # normal fp32 range (denormals: absolute check below)
    assert live.sum() > 1000, "both branches must carry live gradients"
    rel = np.abs(got - d_want) / np.abs(np.where(live, d_want, 1.0))
    assert float(rel[live].max()) <= 1e-5, float(rel[live].max())
    assert float(np.abs(got[~live] - d_want[~live]).max(initial=0.0)) <= 1e-37
    assert abs(st.objective - obj) <= 1e-5 * max(1.0, abs(obj)), (st.objective, obj)


@pytest.mark.parametrize("owned", [False, True])
def test_bench_two_ranks_strong_scaled(owned):
    """bench.py's N-GPU path end to end with 2 processes (torchrun, gloo, both on
    cuda:0 — the test box has one GPU): C4 split over 2 shards, one per rank,
    the loss statistics all-reduced, and each rank's --check leg against the
    oracle's replay of the whole job (owned: each rank received only its
    shard's records)."""
    import socket

    if not torch.cuda.is_available():
        pytest.fail("GPU test requested but CUDA is not available")
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu-baseline"]
    if owned:
        cmd.append("--owned")
    env = dict(os.environ, RB_BENCH_SAME_GPU="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["parity"] == "ok", line["parity_check"]
