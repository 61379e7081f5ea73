"""Device replay diagnostics (rb_batch_staleness_hist / rb_use_count_hist,
SURVEY.md §8f-1) against the same metrics computed from the sampled records
and the resident contents on the host, summarised through the reference's
summarize() (metrics.cpp:37-39, 185-202)."""
import numpy as np
import pytest
import torch

from tests.harness import Producer, StepConfig, insert_groups

pytestmark = pytest.mark.gpu

CASES = {
    "fifo": dict(capacity=96, shards=3, batch=42, group=8, lmax=17, ragged=True, seed=51),
    "posbias_wo": dict(capacity=64, shards=2, batch=24, group=8, lmax=9, ragged=True, seed=52,
                       retention="positive_bias", delta=0.5,
                       strategy="uniform_without_replacement"),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_diagnostics_match_host(oracle, reference, case):
    if not torch.cuda.is_available():
        pytest.fail("GPU test requested but CUDA is not available")
    from paper_2604_08706_b200 import Rng, ShardedReplayBuffer, summarize_hist

    cfg = StepConfig(**CASES[case])
    buf = ShardedReplayBuffer(cfg.shards, cfg.capacity, cfg.strategy, cfg.retention, cfg.delta,
                              max_tokens=cfg.lmax)
    buf.set_stream(torch.cuda.current_stream().cuda_stream)
    rng = Rng(cfg.seed).stream("buffer_sampling")
    prod = Producer(cfg, oracle)
    for step in range(12):
        rec, length, tok, lpo, toff, _ = prod.groups(3 if step < 6 else 1, step)
        insert_groups(buf, rec, toff, tok, lpo, cfg.group, "cuda:0")
        recs = buf.sample(cfg.batch, rng)
        use_step = step + 3
        h, s = buf.staleness_hist(use_step, max_bin=63)
        st = use_step - recs["creation_step"].astype(np.int64)
        assert (st >= 0).all() and st.max() < 63
        assert np.array_equal(h, np.bincount(st, minlength=64).astype(np.uint64))
        assert s == int(st.sum())
        assert summarize_hist(h, s) == reference.summarize(st.astype(np.float64))
        uh, us = buf.use_count_hist(max_bin=31)
        uses = np.concatenate([buf.shard_contents(i)["use_count"] for i in range(cfg.shards)])
        assert np.array_equal(uh, np.bincount(np.minimum(uses, 31), minlength=32).astype(np.uint64))
        assert us == int(uses.astype(np.int64).sum())


def test_diagnostics_reject_bad_bins():
    from paper_2604_08706_b200 import ShardedReplayBuffer

    buf = ShardedReplayBuffer(1, 8, max_tokens=4)
    with pytest.raises(ValueError, match="max_bin"):
        buf.use_count_hist(max_bin=5000)
