"""Binary checkpoint / resume of the device buffer (rb_snapshot / rb_restore,
SURVEY.md §8f-3) and of the RNG position (rb_rng_get_state / set_state):
a buffer restored from a snapshot, with the stream restored from the saved
state, continues exactly like the original — samples, gathered payload,
final contents and text dump — for host and device snapshot memory."""
import numpy as np
import pytest
import torch

from tests.harness import Producer, StepConfig, insert_groups

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rb():
    if not torch.cuda.is_available():
        pytest.fail("GPU test requested but CUDA is not available")
    import paper_2604_08706_b200 as rb

    return rb

CASES = {
    "fifo": dict(capacity=96, shards=3, batch=24, group=8, lmax=33, ragged=True, seed=41),
    "posbias": dict(capacity=64, shards=2, batch=16, group=8, lmax=21, ragged=True, seed=42,
                    retention="positive_bias", delta=0.5),
}


def _drive(buf, rng, prod_state, cfg, ora, steps, record):
    """Insert the producer's groups and sample; returns (records, tokens) per step."""
    prod, lengths = prod_state
    out = []
    debt = 0.0
    for step in range(steps):
        debt += cfg.per_step
        ng = int(debt // cfg.group)
        debt -= ng * cfg.group
        if ng:
            rec, length, tok, lpo, toff, _ = prod.groups(ng, 100 + step)
            for r, L in zip(rec, length):
                lengths[int(r["rollout_id"])] = int(L)
            insert_groups(buf, rec, toff, tok, lpo, cfg.group, "cuda:0")
        recs = buf.sample(cfg.batch, rng)
        tot = int(sum(lengths[int(i)] for i in recs["rollout_id"]))
        pad = (tot + 3) // 4 * 4 + 4
        gt = torch.zeros(pad, dtype=torch.int32, device="cuda:0")
        gl = torch.zeros(pad, dtype=torch.float32, device="cuda:0")
        torch.cuda.synchronize()
        buf.gather(gt, gl, None)
        buf.synchronize()
        out.append((recs, gt[:tot].cpu().numpy(), gl[:tot].cpu().numpy()))
    return out


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("where", ["host", "device"])
def test_snapshot_restore_continues_identically(rb, oracle, case, where):
    from oracle.pyoracle import same_records
    from paper_2604_08706_b200 import Rng, ShardedReplayBuffer

    cfg = StepConfig(**CASES[case])
    mk = lambda: ShardedReplayBuffer(cfg.shards, cfg.capacity, cfg.strategy,  # noqa: E731
                                     cfg.retention, cfg.delta, max_tokens=cfg.lmax)
    a = mk()
    a.set_stream(torch.cuda.current_stream().cuda_stream)
    rng = Rng(cfg.seed).stream("buffer_sampling")
    prod = Producer(cfg, oracle)
    lengths = {}
    while a.size() < cfg.capacity:
        rec, length, tok, lpo, toff, _ = prod.groups(1, 0)
        for r, L in zip(rec, length):
            lengths[int(r["rollout_id"])] = int(L)
        insert_groups(a, rec, toff, tok, lpo, cfg.group, "cuda:0")
    _drive(a, rng, (prod, lengths), cfg, oracle, 3, None)
    # checkpoint
    n = a.snapshot().nbytes
    snap = a.snapshot() if where == "host" else a.snapshot(torch.empty(n, dtype=torch.uint8,
                                                                       device="cuda:0"))
    state = rng.get_state()
    prod2, lengths2 = Producer(cfg, oracle), dict(lengths)
    prod2.next_id, prod2.next_group, prod2.prompt = prod.next_id, prod.next_group, prod.prompt
    # resume into a fresh buffer and a fresh stream object
    b = mk()
    b.set_stream(torch.cuda.current_stream().cuda_stream)
    b.restore(snap)
    rng2 = Rng(12345)
    rng2.set_state(state)
    assert b.dump() == a.dump()
    ra = _drive(a, rng, (prod, lengths), cfg, oracle, 5, None)
    rb2 = _drive(b, rng2, (prod2, lengths2), cfg, oracle, 5, None)
    for step, ((x, xt, xl), (y, yt, yl)) in enumerate(zip(ra, rb2)):
        assert same_records(x, y), f"records differ at step {step}"
        assert np.array_equal(xt, yt) and np.array_equal(xl, yl), f"payload differs at step {step}"
    assert a.dump() == b.dump()
    assert rng.draws == rng2.draws


def test_restore_rejects_other_shape(rb):
    from paper_2604_08706_b200 import ShardedReplayBuffer

    a = ShardedReplayBuffer(2, 32, max_tokens=8)
    b = ShardedReplayBuffer(2, 64, max_tokens=8)
    with pytest.raises(ValueError, match="different shape"):
        b.restore(a.snapshot())
    with pytest.raises(ValueError, match="truncated"):
        a.restore(a.snapshot()[:16])
    junk = a.snapshot()
    junk[:8] = 0
    with pytest.raises(ValueError, match="not a buffer snapshot"):
        a.restore(junk)
