"""A rank holding some of the shards (shard_range) receives the full inbound
batch with its token payload in pinned host memory: only its own records'
ranges are staged (one batched copy, rb_insert), and everything it stores,
samples and gathers equals the same buffer fed device inputs — ragged and
fixed lengths, first and last shard, FIFO and positive bias."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _batch(rng, start, n, lmax, ragged):
    lens = rng.integers(1, lmax + 1, n) if ragged else np.full(n, lmax)
    toff = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=toff[1:])
    tot = int(toff[-1])
    tok = rng.integers(-2**31, 2**31 - 1, tot, dtype=np.int64).astype(np.int32)
    lpo = rng.standard_normal(tot).astype(np.float32)
    ids = np.arange(start, start + n, dtype=np.uint64)
    rew = (rng.random(n) < 0.5).astype(np.float64)
    goff = np.arange(0, n + 1, 4, dtype=np.int64)
    return dict(rollout_id=ids, reward=rew, group_offsets=goff, tok_offsets=toff, tokens=tok,
                logp_old=lpo)


@pytest.mark.parametrize("shard", [0, 2])
@pytest.mark.parametrize("ragged", [True, False])
@pytest.mark.parametrize("retention", ["plain_fifo", "positive_bias"])
def test_partial_shard_host_payload_matches_device(shard, ragged, retention):
    if not torch.cuda.is_available():
        pytest.fail("GPU test requested but CUDA is not available")
    from paper_2604_08706_b200 import Rng, ShardedReplayBuffer

    T, N, lmax, B = 3, 96, 70, 30
    delta = 0.5 if retention == "positive_bias" else 0.0
    mk = lambda: ShardedReplayBuffer(T, N, "uniform_with_replacement", retention, delta,  # noqa: E731
                                     max_tokens=lmax, shard_range=(shard, shard + 1))
    host, dev = mk(), mk()
    rng = np.random.default_rng(7 + shard)
    start = 1
    for step in range(6):
        n = 44 if step else 100
        b = _batch(rng, start, n, lmax, ragged)
        start += n
        hb = {k: (torch.from_numpy(v).pin_memory() if k in ("tokens", "logp_old", "tok_offsets")
                  else v) for k, v in b.items()}
        # offsets on the host (pinned) so the ranges are known; payload pinned
        host.insert(**hb, assume_unique=True)
        dev.insert(**{k: torch.from_numpy(v).cuda() for k, v in b.items()}, assume_unique=True)
        host.check()
        dev.check()
        assert host.dump() == dev.dump()
        g1, g2 = Rng(3 + step).stream("s"), Rng(3 + step).stream("s")
        host.sample_device(B, g1)
        dev.sample_device(B, g2)
        outs = []
        for buf in (host, dev):
            tok = torch.zeros(B * lmax + 8, dtype=torch.int32, device="cuda")
            lpo = torch.zeros(B * lmax + 8, dtype=torch.float32, device="cuda")
            off = torch.zeros(B // T + 1, dtype=torch.int64, device="cuda")
            buf.gather(tok, lpo, off)
            buf.synchronize()
            outs.append((tok.cpu().numpy(), lpo.cpu().numpy(), off.cpu().numpy()))
        (t1, l1, o1), (t2, l2, o2) = outs
        assert np.array_equal(o1, o2)
        tot = int(o1[-1])
        assert tot > 0
        assert np.array_equal(t1[:tot], t2[:tot]) and np.array_equal(l1[:tot], l2[:tot])
