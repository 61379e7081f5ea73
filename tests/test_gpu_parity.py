"""Parity of the CUDA library (through its C-ABI) against the pinned oracle
and the golden fixtures generated from the compiled reference.  GPU only."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD_DIR = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def rb():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test requested but CUDA is not available")
    import paper_2604_08706_b200 as rb

    return rb


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(GOLD_DIR, "golden.npz"))


def make_record(rid, correct=True, step=0):
    """test_buffer_core.cpp:23-36"""
    from oracle.pyoracle import RECORD_DTYPE

    r = np.zeros(1, RECORD_DTYPE)[0]
    r["rollout_id"] = rid
    r["prompt_id"] = rid % 7
    r["group_id"] = rid // 4
    r["creation_step"] = step
    r["policy_version"] = step
    r["reward"] = 1.0 if correct else 0.0
    r["is_correct"] = correct
    r["behavior_logprob"] = -1.25 - 0.001 * rid
    r["advantage"] = 0.5 if correct else -0.5
    return r


def ids(recs):
    return [int(x) for x in recs["rollout_id"]]


# ------------------------------------------------------------------ RNG
@pytest.mark.parametrize("count", [1, 311, 312, 313, 1000, 5000])
def test_device_mt_stream_matches_oracle(rb, oracle, count):
    for seed in (1, 2, 5489):
        g = rb.Rng(seed).stream("buffer_sampling")
        o = oracle.rng(seed).stream("buffer_sampling")
        got = g.fill_u64(count)
        want = np.array([o.next_u64() for _ in range(count)], np.uint64)
        assert np.array_equal(got, want)
        # the stream continues seamlessly on the host after device draws
        assert g.next_u64() == o.next_u64()
        assert g.draws == count + 1


def test_rng_golden(rb, golden):
    for seed in range(1, 6):
        r = rb.Rng(seed).stream("buffer_sampling")
        assert r.seed() == int(golden[f"rng_s{seed}_seed"])
        np.testing.assert_array_equal(r.fill_u64(700), golden[f"rng_s{seed}_raw"])
        assert [r.below(84) for _ in range(300)] == list(golden[f"rng_s{seed}_below84"])
        assert [r.below(16384) for _ in range(300)] == list(golden[f"rng_s{seed}_below16384"])
        np.testing.assert_array_equal(r.sample_without_replacement(100, 37),
                                      golden[f"rng_s{seed}_swor_100_37"])
    k = rb.Rng(5489)
    k.fill_u64(9999)
    assert k.next_u64() == int(golden["rng_kat_10000"]) == 9981545732273789042


# ------------------------------------------------------------------ buffer known answers
def test_fifo_cap3_and_round_robin(rb):
    b = rb.ShardedReplayBuffer(1, 3)
    assert b.push(make_record(1)) is None
    b.push(make_record(2))
    b.push(make_record(3))
    assert int(b.push(make_record(4))["rollout_id"]) == 1
    assert ids(b.shard_contents(0)) == [2, 3, 4]
    b2 = rb.ShardedReplayBuffer(2, 6)
    for i in range(1, 7):
        b2.push(make_record(i))
    assert ids(b2.shard_contents(0)) == [1, 3, 5] and ids(b2.shard_contents(1)) == [2, 4, 6]


def test_constructor_validation(rb):
    """test_buffer_core.cpp:87-99"""
    for args in ((0, 4), (2, 0), (3, 8)):
        with pytest.raises(ValueError):
            rb.ShardedReplayBuffer(*args)
    for d in (1.5, -0.1):
        with pytest.raises(ValueError):
            rb.ShardedReplayBuffer(1, 4, retention="positive_bias", delta=d)


def test_positive_bias_worked_example(rb):
    arrivals = [(9, 0), (8, 1), (7, 1), (6, 0), (5, 1), (4, 1), (3, 0), (2, 1), (1, 0), (0, 0)]
    b = rb.ShardedReplayBuffer(1, 8, retention="positive_bias", delta=0.75)
    for i, c in arrivals:
        b.push(make_record(i, bool(c)))
    assert ids(b.shard_contents(0)) == [8, 7, 5, 4, 3, 2, 1, 0]


def test_positive_bias_vs_oracle_random(rb, oracle):
    rs = np.random.default_rng(5)
    for delta in (0.0, 0.25, 1 / 3, 0.5, 0.75, 1.0):
        for cap in (1, 3, 8):
            g = rb.ShardedReplayBuffer(1, cap, retention="positive_bias", delta=delta)
            o = oracle.buffer(1, cap, retention="positive_bias", delta=delta)
            for i in range(5 * cap + 5):
                r = make_record(i, bool(rs.random() < 0.4))
                eg, eo = g.push(r), o.push(r)
                assert (eg is None) == (eo is None)
                if eg is not None:
                    assert int(eg["rollout_id"]) == int(eo["rollout_id"])
                assert ids(g.shard_contents(0)) == ids(o.shard_contents(0))


def test_duplicate_ids(rb):
    """test_buffer_core.cpp:263-274 — rejected before mutation, evicted ids may recur."""
    b = rb.ShardedReplayBuffer(1, 2)
    b.push(make_record(10))
    with pytest.raises(ValueError, match="already stored"):
        b.push(make_record(10))
    b.push(make_record(11))
    assert int(b.push(make_record(12))["rollout_id"]) == 10
    b.push(make_record(10))
    with pytest.raises(ValueError):
        b.push(make_record(12))
    assert ids(b.shard_contents(0)) == [12, 10]


def test_batched_duplicate_applies_prefix(rb):
    from oracle.pyoracle import RECORD_DTYPE

    b = rb.ShardedReplayBuffer(2, 8)
    recs = np.array([make_record(i) for i in (1, 2, 3, 2, 5)], RECORD_DTYPE)
    with pytest.raises(ValueError):
        b.insert(rollout_id=recs["rollout_id"].copy(), reward=recs["reward"].copy(),
                 advantage=recs["advantage"].copy())
    assert sorted(ids(b.shard_contents(0)) + ids(b.shard_contents(1))) == [1, 2, 3]
    assert b.route_cursor() == 1


def test_assume_unique_violation_is_sticky(rb):
    """RB_INSERT_ASSUME_UNIQUE: a broken promise applies nothing and is reported later."""
    from oracle.pyoracle import RECORD_DTYPE

    b = rb.ShardedReplayBuffer(2, 8)
    recs = np.array([make_record(i) for i in (1, 2, 3)], RECORD_DTYPE)
    b.insert(rollout_id=recs["rollout_id"].copy(), reward=recs["reward"].copy(),
             advantage=recs["advantage"].copy(), assume_unique=True)
    b.check()
    bad = np.array([make_record(i) for i in (4, 4)], RECORD_DTYPE)
    b.insert(rollout_id=bad["rollout_id"].copy(), reward=bad["reward"].copy(),
             advantage=bad["advantage"].copy(), assume_unique=True)
    with pytest.raises(ValueError, match="ASSUME_UNIQUE"):
        b.check()
    b.check()  # cleared
    assert sorted(ids(b.shard_contents(0)) + ids(b.shard_contents(1))) == [1, 2, 3]


@pytest.mark.parametrize("where", [1, 4500, -1])
def test_assume_unique_violation_split_validation(rb, where):
    """Batches above 4096 records split the route's validation over its CTAs:
    a broken promise in any CTA's slice still applies nothing, and the next
    valid batch goes through (the verdict counters are reset)."""
    b = rb.ShardedReplayBuffer(2, 64)
    n = 5000
    ids_ = np.arange(1, n + 1, dtype=np.uint64)
    if where >= 0:
        ids_[where] = ids_[where - 1]  # not strictly increasing
    goff = np.arange(0, n + 1, 8, dtype=np.int64)
    goff[-1] = n
    if where < 0:
        goff[300] = goff[299] + 1  # a group of one
    rew = (np.arange(n) % 3 == 0).astype(np.float64)
    b.insert(rollout_id=ids_, reward=rew, group_offsets=goff, assume_unique=True)
    with pytest.raises(ValueError, match="ASSUME_UNIQUE|group"):
        b.check()
    b.check()
    assert b.size() == 0
    good = np.arange(1, n + 1, dtype=np.uint64)
    goff = np.arange(0, n + 1, 8, dtype=np.int64)
    goff[-1] = n
    b.insert(rollout_id=good, reward=rew, group_offsets=goff, assume_unique=True)
    b.check()
    assert sorted(ids(b.shard_contents(0)) + ids(b.shard_contents(1))) == list(range(n - 63, n + 1))


def test_sample_validation(rb):
    """test_buffer_core.cpp:347-359"""
    b = rb.ShardedReplayBuffer(2, 8, strategy="uniform_without_replacement")
    r = rb.Rng(5)
    b.push(make_record(1))
    with pytest.raises(ValueError, match="empty shard"):
        b.sample(2, r)
    b.push(make_record(2))
    with pytest.raises(ValueError):
        b.sample(0, r)
    with pytest.raises(ValueError):
        b.sample(3, r)
    with pytest.raises(ValueError, match="occupancy"):
        b.sample(4, r)
    b.sample(2, r)


def test_unused_first_worked_example(rb):
    """test_buffer_core.cpp:361-381"""
    b = rb.ShardedReplayBuffer(1, 8, strategy="unused_first_without_replacement")
    for i in range(1, 6):
        b.push(make_record(i))
    r = rb.Rng(17)
    assert ids(b.sample(2, r)) == [5, 4]
    assert ids(b.sample(2, r)) == [3, 2]
    got = ids(b.sample(4, r))
    assert got[0] == 1 and len(set(got[1:])) == 3


def test_ledger_events(rb):
    """test_buffer_core.cpp:383-401"""
    b = rb.ShardedReplayBuffer(2, 8)
    for i in range(6):
        b.push(make_record(i, True, 3))
    recs, ev = b.sample(4, rb.Rng(2), ledger=True, batch_id=7, use_step=9)
    assert list(ev["rollout_id"]) == list(recs["rollout_id"])
    assert all(ev["creation_step"] == 3) and all(ev["use_step"] == 9) and all(ev["batch_id"] == 7)
    assert list(ev["within_batch_rank"]) == [0, 1, 2, 3]


def test_uniform_frequencies(rb):
    """test_buffer_core.cpp:301-318 (device draws, 1e5 selections)."""
    b = rb.ShardedReplayBuffer(1, 100)
    for i in range(100):
        b.push(make_record(i))
    r = rb.Rng(12345)
    counts = np.zeros(100)
    for _ in range(20):
        counts += np.bincount(b.sample(5000, r)["rollout_id"].astype(np.int64), minlength=100)
    freq = counts / counts.sum()
    assert np.all(np.abs(freq - 0.01) <= 0.003)


# ------------------------------------------------------------------ golden schedules
SCHEDS = ["c1_fifo_with", "c2_posbias_with", "c5_t3_fifo_with", "t3_posbias_without",
          "t2_unused_first", "t4_posbias_one_third"]


@pytest.mark.parametrize("name", SCHEDS)
def test_schedule_golden_push_by_push(rb, oracle, golden, name):
    """Record-level traces of the reference (evictions, sampled ids + use counts, dump)."""
    from oracle.pyoracle import same_records
    from oracle.workload import ScheduleConfig, run_schedule

    meta = json.load(open(os.path.join(GOLD_DIR, "schedules.json")))
    cfg = ScheduleConfig(**meta["schedules"][name])
    b = rb.ShardedReplayBuffer(cfg.shards, cfg.capacity, cfg.strategy, cfg.retention, cfg.delta)
    r = rb.Rng(cfg.seed).stream("buffer_sampling")
    tr = run_schedule(b, r, cfg, meta["steps"], oracle)
    for k, v in tr.items():
        np.testing.assert_array_equal(v, golden[f"sched_{name}_{k}"], err_msg=k)
    final = np.concatenate([b.shard_contents(s) for s in range(cfg.shards)])
    assert same_records(final, golden[f"sched_{name}_final_shards"])
    assert b.dump() == bytes(golden[f"sched_{name}_dump"]).decode()


@pytest.mark.parametrize("name", ["c1_fifo_with", "t3_posbias_without", "t2_unused_first"])
def test_dump_load_round_trip(rb, golden, name):
    """test_buffer_core.cpp:425-452 on the golden dumps of the reference."""
    text = bytes(golden[f"sched_{name}_dump"]).decode()
    b = rb.ShardedReplayBuffer.load(text)
    assert b.dump() == text


def test_load_rejects_corrupt(rb):
    with pytest.raises(ValueError):
        rb.ShardedReplayBuffer.load("not a dump")
    b = rb.ShardedReplayBuffer(2, 4)
    b.push(make_record(1))
    b.push(make_record(2))
    good = b.dump()
    with pytest.raises(ValueError, match="duplicate rollout id"):
        rb.ShardedReplayBuffer.load(good + "1,1,0,0,0,1,1,-1.251,0.5,0\n")
    with pytest.raises(ValueError):
        rb.ShardedReplayBuffer.load(good.replace("# route_cursor = 0", "# route_cursor = 5"))


# ------------------------------------------------------------------ advantages / losses
def test_group_advantages_bit_exact(rb, golden):
    got = rb.group_advantages(golden["adv_rewards"], golden["adv_offsets"])
    np.testing.assert_array_equal(got, golden["adv_out"])
    with pytest.raises(ValueError):
        rb.group_advantages(np.array([1.0]))


def test_grpo_records_golden(rb, golden):
    recs = golden["loss_records"]
    d, st = rb.grpo_records(golden["loss_logp_now"], recs["behavior_logprob"], recs["advantage"],
                            0.2, 0.28)
    assert st.excluded == int(golden["grpo_excluded"])
    assert st.objective == pytest.approx(float(golden["grpo_obj"]), rel=1e-12, abs=1e-14)
    np.testing.assert_allclose(d, golden["grpo_dlogp"], rtol=1e-10, atol=1e-15)


def test_asymre_records_golden(rb, golden):
    recs = golden["loss_records"]
    d, st = rb.asymre_records(golden["loss_logp_now"], recs["reward"], golden["loss_group_mean"])
    assert st.objective == pytest.approx(float(golden["asymre_obj"]), rel=1e-12, abs=1e-14)
    np.testing.assert_allclose(d, golden["asymre_dlogp"], rtol=1e-10, atol=1e-15)


def test_grpo_known_answers(rb):
    """test_bandit.cpp:301-330, 374-398."""
    lp = np.log(0.5)
    d, st = rb.grpo_records([lp], [lp - np.log(1.5)], [1.0])
    assert st.objective == pytest.approx(1.2, rel=1e-12) and d[0] == 0.0
    d, st = rb.grpo_records([lp], [lp - np.log(1.5)], [-1.0])
    assert st.objective == pytest.approx(-1.5, rel=1e-12) and d[0] != 0.0
    d, st = rb.grpo_records([lp, lp], [lp, -2000.0], [1.0, 1.0])
    assert (st.excluded, st.included) == (1, 1) and st.objective == pytest.approx(1.0)
    with pytest.raises(ValueError):
        rb.grpo_records([lp], [lp], [1.0], eps_low=-0.1)


@pytest.mark.parametrize("ragged", [False, True])
def test_grpo_tokens_vs_oracle(rb, oracle, ragged):
    rs = np.random.default_rng(7)
    n = 300
    lens = rs.integers(1, 700, n) if ragged else np.full(n, 512)
    off = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    tot = int(off[-1])
    lpo = (-rs.uniform(0, 6, tot)).astype(np.float32)
    lpn = (lpo + rs.normal(0, 0.15, tot)).astype(np.float32)
    lpn[::9973] = np.float32(np.inf)  # excluded tokens
    lpn[5] = lpo[5] + np.float32(np.log(1.2))  # at a clip edge
    adv = rs.normal(size=n)
    adv[::11] = 0.0
    d, st = rb.grpo_tokens(lpn, lpo, adv, off, 0.2, 0.2)
    dw, obj, inc, exc = oracle.loss_grpo_tokens(lpn, lpo, adv, off, 0.2, 0.2)
    assert (st.included, st.excluded) == (inc, exc) and exc > 0
    assert st.objective == pytest.approx(obj, rel=1e-5)
    np.testing.assert_allclose(d, dw, rtol=1e-5, atol=1e-12)
    gm = rs.uniform(0, 1, n)
    rew = rs.integers(0, 2, n).astype(np.float64)
    lpn2 = (lpo + rs.normal(0, 0.15, tot)).astype(np.float32)
    d2, st2 = rb.asymre_tokens(lpn2, rew, gm, off, -0.1)
    dw2, obj2 = oracle.loss_asymre_tokens(lpn2, rew, gm, off, -0.1)
    assert st2.objective == pytest.approx(obj2, rel=1e-6)
    np.testing.assert_allclose(d2, dw2, rtol=1e-6, atol=1e-12)


# ------------------------------------------------------------------ the replay step
STEP_CASES = {
    "c1_shape_small": dict(capacity=84, shards=1, batch=64, group=8, lmax=48, ragged=False),
    "c2_posbias_asymre": dict(capacity=84, shards=1, batch=64, group=8, lmax=40, ragged=True,
                              retention="positive_bias", delta=0.5, loss="asymre", seed=2),
    "c3_ragged": dict(capacity=128, shards=1, batch=64, group=16, lmax=257, ragged=True, seed=3),
    "c4_sharded": dict(capacity=256, shards=4, batch=64, group=16, lmax=96, ragged=True, seed=4),
    "c4_sharded_unique": dict(capacity=256, shards=4, batch=64, group=16, lmax=96, ragged=True,
                              seed=14, assume_unique=True),
    "c3_ragged_unique": dict(capacity=128, shards=1, batch=64, group=16, lmax=257, ragged=True,
                             seed=13, assume_unique=True),
    "big_batch_unique": dict(capacity=32, shards=2, batch=16, group=8, lmax=12, ragged=True,
                             seed=18, workers=16, trainers=1, mu=1.0, assume_unique=True),
    "host_inputs": dict(capacity=60, shards=3, batch=30, group=6, lmax=33, ragged=True, seed=5,
                        device_inputs=False),
    "without_repl": dict(capacity=96, shards=2, batch=32, group=8, lmax=20, ragged=True, seed=6,
                         strategy="uniform_without_replacement"),
    "unused_first_posbias": dict(capacity=96, shards=2, batch=32, group=8, lmax=20, ragged=True,
                                 seed=7, strategy="unused_first_without_replacement",
                                 retention="positive_bias", delta=0.2),
    "big_batch_evicts_in_batch": dict(capacity=32, shards=2, batch=16, group=8, lmax=12,
                                      ragged=True, seed=8, workers=16, trainers=1, mu=1.0),
    "posbias_in_batch": dict(capacity=32, shards=2, batch=16, group=8, lmax=12, ragged=True,
                             seed=9, workers=16, trainers=1, mu=1.0, retention="positive_bias",
                             delta=0.75),
    # insert -> sample with no host sync: the sampler overlaps the running
    # route / payload kernels and maps the new records from the insert's plan
    "c4_unique_overlap": dict(capacity=256, shards=4, batch=64, group=16, lmax=96, ragged=True,
                              seed=21, assume_unique=True, overlap=True),
    "c3_unique_overlap_big": dict(capacity=512, shards=1, batch=2048, group=16, lmax=33,
                                  ragged=True, seed=22, assume_unique=True, overlap=True),
    # more shards than the samplers cache per-shard state for (64 / 128)
    "many_shards_unique": dict(capacity=130 * 3, shards=130, batch=260, group=10, lmax=9,
                               ragged=True, seed=23, assume_unique=True, overlap=True),
    "many_shards": dict(capacity=70 * 2, shards=70, batch=140, group=10, lmax=9, ragged=True,
                        seed=24),
    "posbias_delta_one": dict(capacity=48, shards=3, batch=24, group=8, lmax=10, ragged=True,
                              seed=25, retention="positive_bias", delta=1.0, assume_unique=True),
    # positive bias with ids promised new: one-launch parallel queue update (k_posbias_par)
    "posbias_unique_c2": dict(capacity=84, shards=1, batch=64, group=8, lmax=40, ragged=True,
                              retention="positive_bias", delta=0.5, loss="asymre", seed=51,
                              assume_unique=True),
    "posbias_unique_in_batch": dict(capacity=32, shards=2, batch=16, group=8, lmax=12,
                                    ragged=True, seed=52, workers=16, trainers=1, mu=1.0,
                                    retention="positive_bias", delta=0.75, assume_unique=True),
    "posbias_unique_overlap": dict(capacity=600, shards=3, batch=96, group=8, lmax=33,
                                   ragged=True, seed=53, retention="positive_bias", delta=0.5,
                                   assume_unique=True, overlap=True),
    "posbias_delta_zero": dict(capacity=48, shards=3, batch=24, group=8, lmax=10, ragged=True,
                               seed=26, retention="positive_bias", delta=0.0),
    # insert -> sample -> gather with no host sync: the gather is a dependent
    # of the sampler (k_gather_early) and overlaps it and the payload copy
    "early_gather_c4": dict(capacity=256, shards=4, batch=64, group=16, lmax=96, ragged=True,
                            seed=31, assume_unique=True, overlap=True, early_gather=True),
    "early_gather_long": dict(capacity=48, shards=2, batch=32, group=8, lmax=4200, ragged=True,
                              seed=32, assume_unique=True, overlap=True, early_gather=True),
    "early_gather_fixed_len": dict(capacity=64, shards=1, batch=48, group=8, lmax=2052,
                                   ragged=False, seed=33, assume_unique=True, overlap=True,
                                   early_gather=True),
    "early_gather_many_shards": dict(capacity=130 * 3, shards=130, batch=260, group=10, lmax=9,
                                     ragged=True, seed=34, assume_unique=True, overlap=True,
                                     early_gather=True),
    # more than 4096 records per insert: the route splits its validation
    "split_validation_unique": dict(capacity=1024, shards=2, batch=64, group=8, lmax=6,
                                    ragged=True, seed=36, workers=80, trainers=1, mu=1.0,
                                    assume_unique=True, overlap=True),
    "early_gather_not_unique": dict(capacity=96, shards=3, batch=48, group=8, lmax=40,
                                    ragged=True, seed=35, early_gather=True),
    # packed-range gather / loss (packed_range.cuh): trajectories of 1-2
    # tokens put > PK_SL selections in one CTA's run (the unstaged search), of
    # 1-5 tokens make almost every warp unit straddle selections
    "tiny_traj_unstaged": dict(capacity=512, shards=1, batch=4096, group=8, lmax=2, ragged=True,
                               seed=41, assume_unique=True),
    "tiny_traj_sharded": dict(capacity=512, shards=2, batch=2048, group=8, lmax=5, ragged=True,
                              seed=42),
    "tiny_traj_asymre": dict(capacity=256, shards=1, batch=2048, group=8, lmax=3, ragged=True,
                             seed=43, loss="asymre", assume_unique=True),
    "one_token_fixed": dict(capacity=64, shards=1, batch=1024, group=8, lmax=1, ragged=False,
                            seed=44),
    # rows longer than 4096 tokens: LSU payload, chunk-major gather, claimed
    # loss units by default; the alternatives through their switches
    "long_rows": dict(capacity=64, shards=2, batch=64, group=8, lmax=9000, ragged=True, seed=45,
                      assume_unique=True),
    "long_rows_switches": dict(capacity=64, shards=1, batch=48, group=8, lmax=8500, ragged=True,
                               seed=46, env={"RB_LOSS_CHUNK_MAJOR": "1", "RB_NO_CHUNK_MAJOR": "1",
                                             "RB_PAYLOAD_TMA_LONG": "1"}),
    "long_rows_cm_loss": dict(capacity=64, shards=1, batch=48, group=8, lmax=8500, ragged=True,
                              seed=47, assume_unique=True, env={"RB_LOSS_CHUNK_MAJOR": "1"}),
}


@pytest.mark.parametrize("case", sorted(STEP_CASES))
def test_replay_step_parity(rb, oracle, case, monkeypatch):
    from tests.harness import StepConfig, run_step_parity

    cfg = dict(STEP_CASES[case])
    if cfg.get("early_gather"):
        monkeypatch.setenv("RB_EARLY_GATHER", "1")  # read at buffer creation
    for k, v in cfg.pop("env", {}).items():
        monkeypatch.setenv(k, v)

    counts = run_step_parity(StepConfig(**cfg), steps=12, ora=oracle)
    assert counts["samples"] > 0 and counts["tokens"] > 0


@pytest.mark.parametrize("case", ["c4_unique_overlap", "c3_unique_overlap_big", "many_shards",
                                  "early_gather_c4", "host_inputs"])
def test_side_lookahead_matches(rb, oracle, case, monkeypatch):
    """The Rng's side-stream ring lookahead (taken above 8192 draws per call)
    forced on every call: same stream, selections, payload and losses; host
    draws after device sampling continue the stream (it is joined first)."""
    from tests.harness import StepConfig, run_step_parity

    monkeypatch.setenv("RB_LOOKAHEAD_MIN_DRAWS", "0")
    if STEP_CASES[case].get("early_gather"):
        monkeypatch.setenv("RB_EARLY_GATHER", "1")
    counts = run_step_parity(StepConfig(**STEP_CASES[case]), steps=10, ora=oracle)
    assert counts["samples"] > 0


@pytest.mark.parametrize("switch", ["RB_NO_PDL", "RB_PAYLOAD_LSU", "RB_NO_LOOKAHEAD",
                                    "RB_TMA_CTAS", "RB_NO_ROUTE_PDL"])
@pytest.mark.parametrize("case", ["c4_unique_overlap", "c3_unique_overlap_big"])
def test_env_switches_do_not_change_results(rb, oracle, case, switch, monkeypatch):
    """Every performance switch leaves the results bit-identical."""
    from tests.harness import StepConfig, run_step_parity

    monkeypatch.setenv(switch, "1")
    counts = run_step_parity(StepConfig(**STEP_CASES[case]), steps=8, ora=oracle)
    assert counts["samples"] > 0


def test_side_lookahead_rng_continues_on_host(rb, oracle, monkeypatch):
    monkeypatch.setenv("RB_LOOKAHEAD_MIN_DRAWS", "0")
    buf = rb.ShardedReplayBuffer(2, 64)
    obuf = oracle.buffer(2, 64)
    for i in range(1, 65):
        r = make_record(i)
        buf.push(r)
        obuf.push(r)
    g = rb.Rng(7).stream("buffer_sampling")
    o = oracle.rng(7).stream("buffer_sampling")
    for _ in range(5):
        buf.sample_device(2000, g)
        obuf.sample(2000, o)
    buf.synchronize()
    assert [g.next_u64() for _ in range(3)] == [o.next_u64() for _ in range(3)]
    assert g.draws == 5 * 2000 + 3


@pytest.mark.parametrize("case", ["c4_unique_overlap", "c3_unique_overlap_big", "many_shards",
                                  "early_gather_c4", "early_gather_long"])
def test_forced_draw_replay_matches(rb, oracle, case, monkeypatch):
    """The sampler's exact-replay path (taken for real only after a below()
    rejection, probability ~n/2^64) forced on every CTA gives the same
    stream, selections and losses (env read at buffer creation)."""
    from tests.harness import StepConfig, run_step_parity

    monkeypatch.setenv("RB_DEBUG_FORCE_DRAW_REPLAY", "1")
    if STEP_CASES[case].get("early_gather"):
        monkeypatch.setenv("RB_EARLY_GATHER", "1")
    counts = run_step_parity(StepConfig(**STEP_CASES[case]), steps=6, ora=oracle)
    assert counts["samples"] > 0
