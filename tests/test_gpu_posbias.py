"""Positive-bias retention with ids promised new (k_posbias_par: validation,
advantages and the queue update in one launch, the update as scans) against
the oracle's push-by-push restatement of replay_buffer.cpp:98-133: evicted
id of every push and the arrival order of every shard after every insert,
for correctness patterns that keep W empty, keep it full, and mix."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rb():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test requested but CUDA is not available")
    import paper_2604_08706_b200 as rb

    return rb


def _correct(pattern, n, g):
    if pattern == "all_correct":
        return np.ones(n, bool)
    if pattern == "all_wrong":
        return np.zeros(n, bool)
    p = {"random": 0.5, "mostly_correct": 0.9, "mostly_wrong": 0.1}[pattern]
    return g.random(n) < p


CASES = [
    # (per-shard capacity, shards, delta, pattern, batch sizes)
    (84, 1, 0.5, "random", [84, 162, 161, 1, 7, 300]),
    (84, 1, 0.5, "all_correct", [84, 40, 200]),
    (84, 1, 0.5, "all_wrong", [84, 40, 200]),
    (32, 2, 0.75, "mostly_correct", [64, 256, 18, 512]),
    (32, 2, 0.25, "mostly_wrong", [64, 256, 18, 512]),
    (48, 3, 0.0, "random", [144, 50, 600]),       # fresh_slots = C: the reserve is empty
    (16, 4, 0.9, "random", [10, 54, 300, 2]),      # the first batch fills part-way (sequential)
    (1000, 2, 0.4, "random", [2000, 3000, 640, 8001]),  # 8001 > 4096 per shard: fallback path
    (4096, 1, 0.5, "mostly_wrong", [4096, 4096, 1000]),  # the largest shard in shared memory
    (7, 5, 0.5, "random", [35, 4, 100, 1000]),
]


@pytest.mark.parametrize("C,T,delta,pattern,batches", CASES)
def test_posbias_unique_insert_matches_oracle(rb, oracle, C, T, delta, pattern, batches):
    g = np.random.default_rng(C * 7 + T)
    buf = rb.ShardedReplayBuffer(T, C * T, "uniform_with_replacement", "positive_bias", delta)
    obuf = oracle.buffer(T, C * T, "uniform_with_replacement", "positive_bias", delta)
    from oracle.pyoracle import RECORD_DTYPE

    nid = 1
    for bsz in batches:
        bsz += bsz % 2  # whole groups of 2
        ids = np.arange(nid, nid + bsz, dtype=np.uint64)
        nid += bsz + int(g.integers(0, 3))
        corr = _correct(pattern, bsz, g)
        reward = corr.astype(np.float64)
        goff = np.arange(0, bsz + 1, 2, dtype=np.int64)
        ev = np.zeros(bsz, np.uint64)
        buf.insert(rollout_id=ids, reward=reward, group_offsets=goff, evicted=ev,
                   assume_unique=True)
        buf.synchronize()
        buf.check()
        recs = np.zeros(bsz, RECORD_DTYPE)
        recs["rollout_id"] = ids
        recs["reward"] = reward
        recs["is_correct"] = corr
        for i in range(bsz):
            e = obuf.push(recs[i])
            want = np.iinfo(np.uint64).max if e is None else int(e["rollout_id"])
            assert int(ev[i]) == want, f"batch {bsz}: push {i} evicted {ev[i]}, want {want}"
        for s in range(T):
            got = buf.shard_contents(s)
            exp = obuf.shard_contents(s)
            assert np.array_equal(got["rollout_id"], exp["rollout_id"]), f"shard {s} order"
            assert np.array_equal(got["is_correct"], exp["is_correct"])
    # the materialised order drives sampling: a few draws agree with the oracle
    grng = rb.Rng(3).stream("buffer_sampling")
    orng = oracle.rng(3).stream("buffer_sampling")
    grec, gsh, gix = buf.sample(4 * T, grng, with_index=True)
    orec, osh, oix = obuf.sample(4 * T, orng)
    assert np.array_equal(grec["rollout_id"], orec["rollout_id"])


def test_posbias_unique_rejects_non_increasing_ids(rb):
    buf = rb.ShardedReplayBuffer(2, 16, "uniform_with_replacement", "positive_bias", 0.5)
    ids = np.arange(1, 17, dtype=np.uint64)
    buf.insert(rollout_id=ids, reward=np.ones(16), group_offsets=np.arange(0, 17, 2),
               assume_unique=True)
    buf.check()
    before = [buf.shard_contents(s)["rollout_id"].copy() for s in range(2)]
    bad = np.array([20, 19, 21, 22], np.uint64)
    buf.insert(rollout_id=bad, reward=np.ones(4), group_offsets=np.arange(0, 5, 2),
               assume_unique=True)
    with pytest.raises(ValueError, match="ASSUME_UNIQUE"):
        buf.check()
    for s in range(2):  # nothing applied
        assert np.array_equal(buf.shard_contents(s)["rollout_id"], before[s])


def test_posbias_unique_with_given_advantages(rb, oracle):
    """Advantages / group means supplied by the caller (no group offsets): the
    one-launch path stores them as given (frozen at insertion)."""
    from oracle.pyoracle import RECORD_DTYPE

    g = np.random.default_rng(5)
    buf = rb.ShardedReplayBuffer(2, 64, "uniform_with_replacement", "positive_bias", 0.5)
    obuf = oracle.buffer(2, 64, "uniform_with_replacement", "positive_bias", 0.5)
    nid = 1
    for bsz in (64, 50, 130):
        ids = np.arange(nid, nid + bsz, dtype=np.uint64)
        nid += bsz
        corr = g.random(bsz) < 0.4
        adv = g.normal(size=bsz)
        gm = g.random(bsz)
        ev = np.zeros(bsz, np.uint64)
        buf.insert(rollout_id=ids, reward=corr.astype(np.float64), advantage=adv, group_mean=gm,
                   evicted=ev, assume_unique=True)
        buf.synchronize()
        buf.check()
        recs = np.zeros(bsz, RECORD_DTYPE)
        recs["rollout_id"] = ids
        recs["reward"] = corr
        recs["is_correct"] = corr
        recs["advantage"] = adv
        for i in range(bsz):
            e = obuf.push(recs[i])
            want = np.iinfo(np.uint64).max if e is None else int(e["rollout_id"])
            assert int(ev[i]) == want
    for s in range(2):
        got, want = buf.shard_contents(s), obuf.shard_contents(s)
        assert np.array_equal(got["rollout_id"], want["rollout_id"])
        assert np.array_equal(got["advantage"], want["advantage"])
