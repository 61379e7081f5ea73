"""Pins the C restatement (oracle/replay_oracle.c) before anything trusts it.

(1) known answers from the reference's own tests (test_rng.cpp,
    test_buffer_core.cpp, test_bandit.cpp — cited per test),
(2) golden fixtures generated from the compiled reference
    (tests/golden/make_golden.py), and
(3) live differential runs against oracle/_ref when it is built here.
"""
import os

import numpy as np
import pytest

from oracle.pyoracle import RECORD_DTYPE, OracleError, same_records
from oracle.workload import ScheduleConfig, run_schedule

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def make_record(rid, correct=True, step=0):
    """test_buffer_core.cpp:23-36"""
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


# ---------------------------------------------------------------- RNG
def test_mt19937_64_kat(oracle):
    r = oracle.rng(5489)  # [rand.predef]: 10000th output of the default-seeded engine
    for _ in range(9999):
        r.next_u64()
    assert r.next_u64() == 9981545732273789042


def test_rng_golden(oracle, golden):
    for seed in range(1, 6):
        r = oracle.rng(seed).stream("buffer_sampling")
        assert r.seed == int(golden[f"rng_s{seed}_seed"])
        assert [r.next_u64() for _ in range(700)] == [int(x) for x in golden[f"rng_s{seed}_raw"]]
        assert [r.below(84) for _ in range(300)] == [int(x) for x in golden[f"rng_s{seed}_below84"]]
        assert [r.below(16384) for _ in range(300)] == [
            int(x) for x in golden[f"rng_s{seed}_below16384"]]
        assert list(r.sample_without_replacement(100, 37)) == list(golden[f"rng_s{seed}_swor_100_37"])
    assert oracle.rng(99).stream("cell", 7).seed == int(golden["rng_stream_idx_seed"])
    # SURVEY.md §8a a8 probe: Rng(1).stream("buffer_sampling") first below(84) draws
    s = oracle.rng(1).stream("buffer_sampling")
    assert s.seed == 12401569385529067767
    assert [s.below(84) for _ in range(4)] == [35, 37, 58, 7]


def test_rng_streams_position_independent(oracle):
    """test_rng.cpp:28-48"""
    parent = oracle.rng(99)
    fresh = parent.stream("metrics")
    for _ in range(17):
        parent.next_u64()
    later = parent.stream("metrics")
    assert [fresh.next_u64() for _ in range(20)] == [later.next_u64() for _ in range(20)]
    assert oracle.hash_name("metrics") != oracle.hash_name("training")
    with pytest.raises(OracleError):
        oracle.rng(1).below(0)


# ---------------------------------------------------------------- buffer known answers
def test_fifo_cap3(oracle):
    """test_buffer_core.cpp:101-112"""
    b = oracle.buffer(1, 3)
    assert b.push(make_record(1)) is None
    assert b.push(make_record(2)) is None
    assert b.push(make_record(3)) is None
    assert int(b.push(make_record(4))["rollout_id"]) == 1
    assert ids(b.shard_contents(0)) == [2, 3, 4]


def test_round_robin(oracle):
    """test_buffer_core.cpp:114-142"""
    b = oracle.buffer(2, 6)
    for i in range(1, 7):
        b.push(make_record(i))
    assert ids(b.shard_contents(0)) == [1, 3, 5]
    assert ids(b.shard_contents(1)) == [2, 4, 6]


def test_positive_bias_worked_example(oracle):
    """test_buffer_core.cpp:172-185"""
    arrivals = [(9, 0), (8, 1), (7, 1), (6, 0), (5, 1), (4, 1), (3, 0), (2, 1), (1, 0), (0, 0)]
    b = oracle.buffer(1, 8, retention="positive_bias", delta=0.75)
    for i, c in arrivals:
        b.push(make_record(i, bool(c)))
    assert ids(b.shard_contents(0)) == [8, 7, 5, 4, 3, 2, 1, 0]


def retained_reference(history, cap, delta):
    """Full-history oracle of test_buffer_core.cpp:51-83."""
    n = len(history)
    if n <= cap:
        return [h[0] for h in history]
    cs = int(np.floor(delta * cap + 1e-9))
    fs = cap - cs
    keep = set(range(n - fs, n))
    taken = 0
    for i in range(n - fs - 1, -1, -1):
        if taken >= cs:
            break
        if history[i][1]:
            keep.add(i)
            taken += 1
    for i in range(n - fs - 1, -1, -1):
        if len(keep) >= cap:
            break
        keep.add(i)
    return [history[i][0] for i in sorted(keep)]


def test_positive_bias_full_history(oracle):
    """test_buffer_core.cpp:187-209"""
    rng = oracle.rng(99)
    for delta in (0.0, 0.25, 1 / 3, 0.5, 0.6, 0.75, 1.0):
        for cap in (1, 2, 3, 4, 8):
            for p in (0.2, 0.5, 0.8):
                b = oracle.buffer(1, cap, retention="positive_bias", delta=delta)
                hist = []
                for i in range(6 * cap + 7):
                    c = rng.uniform01() < p
                    hist.append((i, c))
                    b.push(make_record(i, c))
                    assert ids(b.shard_contents(0)) == retained_reference(hist, cap, delta)


def test_duplicate_ids(oracle):
    """test_buffer_core.cpp:263-274"""
    b = oracle.buffer(1, 2)
    b.push(make_record(10))
    with pytest.raises(OracleError):
        b.push(make_record(10))
    b.push(make_record(11))
    assert int(b.push(make_record(12))["rollout_id"]) == 10
    b.push(make_record(10))
    with pytest.raises(OracleError):
        b.push(make_record(12))


def test_sample_validation_and_unused_first(oracle):
    """test_buffer_core.cpp:347-381"""
    b = oracle.buffer(2, 8, strategy="uniform_without_replacement")
    r = oracle.rng(5)
    b.push(make_record(1))
    with pytest.raises(OracleError):
        b.sample(2, r)
    b.push(make_record(2))
    for bad in (3, 4):
        with pytest.raises(OracleError):
            b.sample(bad, r)
    b.sample(2, r)
    u = oracle.buffer(1, 8, strategy="unused_first_without_replacement")
    for i in range(1, 6):
        u.push(make_record(i))
    r = oracle.rng(17)
    assert ids(u.sample(2, r)[0]) == [5, 4]
    assert ids(u.sample(2, r)[0]) == [3, 2]
    got = ids(u.sample(4, r)[0])
    assert got[0] == 1 and len(set(got[1:])) == 3 and all(2 <= x <= 5 for x in got[1:])


# ---------------------------------------------------------------- golden schedules
SCHEDS = ["c1_fifo_with", "c2_posbias_with", "c5_t3_fifo_with", "t3_posbias_without",
          "t2_unused_first", "t4_posbias_one_third"]


@pytest.mark.parametrize("name", SCHEDS)
def test_schedule_golden(oracle, golden, name):
    import json

    meta = json.load(open(os.path.join(os.path.dirname(GOLDEN), "schedules.json")))
    cfg = ScheduleConfig(**meta["schedules"][name])
    b = oracle.buffer(cfg.shards, cfg.capacity, cfg.strategy, cfg.retention, cfg.delta)
    r = oracle.rng(cfg.seed).stream("buffer_sampling")
    tr = run_schedule(b, r, cfg, meta["steps"], oracle)
    for k, v in tr.items():
        np.testing.assert_array_equal(v, golden[f"sched_{name}_{k}"], err_msg=k)
    final = np.concatenate([b.shard_contents(s) for s in range(cfg.shards)])
    assert same_records(final, golden[f"sched_{name}_final_shards"])


# ---------------------------------------------------------------- advantages / losses
def test_group_advantages_golden(oracle, golden):
    r, off, want = golden["adv_rewards"], golden["adv_offsets"], golden["adv_out"]
    got = np.concatenate([oracle.group_advantages(r[off[i]:off[i + 1]])
                          for i in range(len(off) - 1)])
    np.testing.assert_array_equal(got, want)  # bit-exact fp64
    np.testing.assert_allclose(oracle.group_advantages([1, 0, 1, 0]), [1, -1, 1, -1], rtol=1e-12)
    with pytest.raises(OracleError):
        oracle.group_advantages([1.0])


def test_grpo_records_golden(oracle, golden):
    recs = golden["loss_records"]
    d, obj, inc, exc = oracle.loss_grpo_records(golden["loss_logp_now"], recs["behavior_logprob"],
                                                recs["advantage"], 0.2, 0.28)
    assert exc == int(golden["grpo_excluded"])
    assert obj == pytest.approx(float(golden["grpo_obj"]), rel=1e-12, abs=1e-14)
    np.testing.assert_allclose(d, golden["grpo_dlogp"], rtol=1e-10, atol=1e-15)


def test_asymre_records_golden(oracle, golden):
    recs = golden["loss_records"]
    d, obj = oracle.loss_asymre_records(golden["loss_logp_now"], recs["reward"],
                                        golden["loss_group_mean"], -0.1)
    assert obj == pytest.approx(float(golden["asymre_obj"]), rel=1e-12, abs=1e-14)
    np.testing.assert_allclose(d, golden["asymre_dlogp"], rtol=1e-10, atol=1e-15)


def test_grpo_known_answers(oracle):
    """test_bandit.cpp:301-330 and 374-398 at the record level."""
    lp = np.log(0.5)
    d, obj, inc, exc = oracle.loss_grpo_records([lp], [lp - np.log(1.5)], [1.0])
    assert obj == pytest.approx(1.2, rel=1e-12) and d[0] == 0.0
    d, obj, _, _ = oracle.loss_grpo_records([lp], [lp - np.log(1.5)], [-1.0])
    assert obj == pytest.approx(-1.5, rel=1e-12) and d[0] != 0.0
    d, obj, inc, exc = oracle.loss_grpo_records([lp, lp], [lp, -2000.0], [1.0, 1.0])
    assert exc == 1 and inc == 1 and obj == pytest.approx(1.0, rel=1e-12)


def test_token_loss_reduces_to_records_at_L1(oracle):
    rs = np.random.default_rng(3)
    n = 500
    lpo = (-rs.uniform(0, 5, n)).astype(np.float32)
    lpn = (lpo + rs.normal(0, 0.2, n)).astype(np.float32)
    adv = rs.normal(size=n)
    off = np.arange(n + 1, dtype=np.int64)
    d, obj, inc, exc = oracle.loss_grpo_tokens(lpn, lpo, adv, off)
    d2, obj2, inc2, exc2 = oracle.loss_grpo_records(lpn.astype(np.float64),
                                                    lpo.astype(np.float64), adv)
    assert (inc, exc) == (inc2, exc2) and obj == obj2
    np.testing.assert_array_equal(d, d2.astype(np.float32))


# ---------------------------------------------------------------- live differential
@pytest.mark.ref
def test_differential_vs_reference(oracle, reference):
    rs = np.random.default_rng(11)
    for trial in range(30):
        shards = int(rs.integers(1, 5))
        cap = shards * int(rs.integers(1, 12))
        strat = ["uniform_with_replacement", "uniform_without_replacement",
                 "unused_first_without_replacement"][trial % 3]
        ret = "positive_bias" if trial % 2 else "plain_fifo"
        delta = float(rs.choice([0.0, 0.2, 0.25, 1 / 3, 0.5, 0.7, 1.0]))
        a = oracle.buffer(shards, cap, strat, ret, delta)
        b = reference.buffer(shards, cap, strat, ret, delta)
        ra, rb = oracle.rng(trial), reference.rng(trial)
        nid = 0
        for _ in range(200):
            if rs.random() < 0.7:
                rec = make_record(nid if rs.random() < 0.9 else max(0, nid - 3), rs.random() < 0.4)
                nid += 1
                ea = eb = None
                try:
                    ea = a.push(rec)
                except OracleError:
                    with pytest.raises(OracleError):
                        b.push(rec)
                    continue
                eb = b.push(rec)
                assert (ea is None) == (eb is None)
                if ea is not None:
                    assert same_records(ea, eb)
            else:
                k = shards * int(rs.integers(1, 4))
                try:
                    sa = a.sample(k, ra)[0]
                except OracleError:
                    with pytest.raises(OracleError):
                        b.sample(k, rb)
                    continue
                sb = b.sample(k, rb)
                assert same_records(sa, sb)
        for s in range(shards):
            assert same_records(a.shard_contents(s), b.shard_contents(s))
