"""The device UseEvent ledger (rb_ledger_*, csrc/ledger.cu) against the
UNMODIFIED reference's MetricsLedger and diagnostics (oracle/_ref):
replay_counts, global_use_order and steps_since_last_use
(metrics.cpp:123-170) bit-exact, including the MT19937-64 draws of the
per-batch shuffles (the Rng continues identically afterwards), events
recorded from the sampler (replay_buffer.cpp:205-215), and the reference's
validation errors (metrics.cpp:44-69)."""
import numpy as np
import pytest

from oracle.pyoracle import RECORD_DTYPE

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rb():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test requested but CUDA is not available")
    import paper_2604_08706_b200 as rb

    return rb


def random_events(seed, n_batches, max_batch, n_ids):
    rs = np.random.default_rng(seed)
    ev = []
    bid = 0
    for b in range(n_batches):
        m = int(rs.integers(1, max_batch + 1))
        use_step = int(rs.integers(0, n_batches // 2 + 1))  # several batches share a step
        ids = rs.integers(0, n_ids, m)
        ranks = rs.permutation(m)  # recorded out of rank order
        for i in range(m):
            cstep = int(rs.integers(0, use_step + 1))
            ev.append((int(ids[i]), cstep, use_step, bid, int(ranks[i])))
        bid += int(rs.integers(1, 4))  # gaps between batch ids
    return ev


def compare_diagnostics(rb, ours, theirs, reference, seed):
    e = ours.events()
    t = theirs.events()
    assert e.shape[0] == t.shape[0]
    for k, name in enumerate(["rollout_id", "creation_step", "use_step", "batch_id",
                              "within_batch_rank"]):
        assert np.array_equal(e[name].astype(np.int64), t[:, k]), name
    for inc in (True, False):
        ids, cnt = ours.replay_counts(inc)
        rids, rcnt = theirs.replay_counts(inc)
        assert np.array_equal(ids, rids) and np.array_equal(cnt, rcnt), inc
    g = rb.Rng(seed).stream("ledger")
    r = reference.rng(seed).stream("ledger")
    assert np.array_equal(ours.global_use_order(g), theirs.global_use_order(r))
    idx, gap, has = ours.steps_since_last_use(g)
    ridx, rgap, rhas = theirs.steps_since_last_use(r)
    assert np.array_equal(idx, ridx)
    assert np.array_equal(has, rhas)
    assert np.array_equal(gap[has == 1], rgap[rhas == 1])
    # both streams consumed exactly the same draws
    assert g.next_u64() == r.next_u64()


@pytest.mark.parametrize("seed,n_batches,max_batch,n_ids", [(1, 6, 9, 20), (2, 40, 300, 500),
                                                            (3, 12, 5000, 3000), (4, 1, 1, 1)])
def test_ledger_diagnostics_match_reference(rb, reference, seed, n_batches, max_batch, n_ids):
    ours, theirs = rb.MetricsLedger(), reference.ledger()
    gen = np.arange(0, n_ids + 50, 3, dtype=np.uint64)  # some never used, some used never noted
    ours.note_generated(gen)
    for i in gen:
        theirs.note_generated(i)
    ev = random_events(seed, n_batches, max_batch, n_ids)
    arr = np.array(ev, dtype=[("rollout_id", "<u8"), ("creation_step", "<i8"), ("use_step", "<i8"),
                              ("batch_id", "<i8"), ("within_batch_rank", "<i8")])
    ours.record_use(arr)
    for x in ev:
        theirs.record_use(*x)
    compare_diagnostics(rb, ours, theirs, reference, seed + 100)


def test_ledger_from_the_sampler_matches_reference(rb, reference, oracle):
    """sample(batch, rng, &ledger, batch_id, use_step) on both sides."""
    shards, cap, batch, G = 2, 64, 32, 8
    buf = rb.ShardedReplayBuffer(shards, cap)
    rbuf = reference.buffer(shards, cap)
    grng, rrng = rb.Rng(9).stream("buffer_sampling"), reference.rng(9).stream("buffer_sampling")
    ours, theirs = rb.MetricsLedger(), reference.ledger()
    nid = 0
    for step in range(14):
        n = G * (cap // G if step == 0 else 3)
        ids = np.arange(nid, nid + n, dtype=np.uint64)
        nid += n
        reward, _, blp = oracle.synth_meta(5, ids, 4, False)
        rec = np.zeros(n, RECORD_DTYPE)
        rec["rollout_id"] = ids
        rec["group_id"] = ids // G
        rec["creation_step"] = step
        rec["policy_version"] = step
        rec["reward"] = reward
        rec["is_correct"] = reward == 1.0
        rec["behavior_logprob"] = blp
        for g0 in range(0, n, G):
            rec["advantage"][g0:g0 + G] = reference.group_advantages(reward[g0:g0 + G])
        buf.insert(rollout_id=ids, reward=reward, group_id=ids // G,
                   creation_step=np.full(n, step, np.int64), policy_version=np.full(n, step, np.int64),
                   behavior_logprob=blp, group_offsets=np.arange(0, n + 1, G, dtype=np.int64))
        ours.note_generated(ids)
        for r in rec:
            rbuf.push(r)
            theirs.note_generated(int(r["rollout_id"]))
        if step == 0:
            continue
        buf.sample_device(batch, grng)
        ours.record_batch(buf, batch_id=10 * step, use_step=step + 2)
        _, ev = rbuf.sample(batch, rrng, with_events=True, batch_id=10 * step, use_step=step + 2)
        for x in ev:
            theirs.record_use(*[int(v) for v in x])
    compare_diagnostics(rb, ours, theirs, reference, 17)


def test_ledger_validation_errors(rb, reference):
    ours, theirs = rb.MetricsLedger(), reference.ledger()
    ours.note_generated(np.array([5, 6], np.uint64))
    with pytest.raises(ValueError, match="rollout 6 noted as generated twice"):
        ours.note_generated(np.array([7, 6], np.uint64))
    ev = np.zeros(3, dtype=[("rollout_id", "<u8"), ("creation_step", "<i8"), ("use_step", "<i8"),
                            ("batch_id", "<i8"), ("within_batch_rank", "<i8")])
    ev["rollout_id"] = [1, 2, 3]
    ev["use_step"] = [4, 4, 4]
    ev["creation_step"] = [1, 9, 0]  # the second precedes its creation
    ev["within_batch_rank"] = [0, 1, 2]
    with pytest.raises(ValueError, match="use event for rollout 2 precedes its creation step"):
        ours.record_use(ev)
    assert len(ours) == 1  # the events before it are recorded, as in the reference
    with pytest.raises(ValueError, match=r"duplicate batch slot \(batch 0, rank 0\)"):
        ours.record_use(ev[:1])
    # use-before-creation from the sampler: detected on the device, reported
    # by the next synchronising call, which keeps the events before it
    buf = rb.ShardedReplayBuffer(1, 16)
    ids = np.arange(100, 116, dtype=np.uint64)
    buf.insert(rollout_id=ids, reward=np.ones(16), creation_step=np.full(16, 50, np.int64),
               group_offsets=np.array([0, 8, 16], np.int64))
    buf.sample_device(4, rb.Rng(1))
    led = rb.MetricsLedger()
    led.record_batch(buf, batch_id=0, use_step=3)
    with pytest.raises(ValueError, match="precedes its creation step"):
        led.check()
    assert len(led) == 0
