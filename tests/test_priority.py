"""priority_with_replacement — the north star's prioritised-sampling CDF.

Builder extension: the reference samples uniformly (replay_buffer.cpp:135-182)
and its "positive bias" is a retention rule (replay_buffer.cpp:106-128), so
there is no reference implementation of a weighted sampler.  Parity is pinned
two ways: (1) with unit weights the strategy IS the reference's
uniform_with_replacement, draw for draw — checked against the compiled
reference (oracle/_ref); (2) with real weights the oracle's C restatement is
checked against an independent numpy restatement here, and the GPU kernel
(k_sample_prio) against the oracle, bit-exact, through the whole replay step.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle.pyoracle import RECORD_DTYPE, OracleError, same_records


def make_record(rid, reward, adv, step=0):
    r = np.zeros(1, RECORD_DTYPE)[0]
    r["rollout_id"] = rid
    r["prompt_id"] = rid % 7
    r["group_id"] = rid // 4
    r["creation_step"] = step
    r["policy_version"] = step
    r["reward"] = reward
    r["is_correct"] = reward > 0
    r["behavior_logprob"] = -1.25 - 0.001 * rid
    r["advantage"] = adv
    return r


def weights_np(recs, base, adv_scale, pos_bonus):
    """include/replay_b200.h rb_set_priority, restated in numpy."""
    a = np.abs(recs["advantage"].astype(np.float64))
    a = np.where(np.isnan(a), 0.0, np.minimum(a, 32768.0))
    w = np.uint64(base) + (a * float(adv_scale)).astype(np.uint64)
    w = w + np.where(recs["reward"] > 0, np.uint64(pos_bonus), np.uint64(0))
    return w.astype(np.uint64)


def random_records(rs, n, start=0):
    out = []
    for i in range(n):
        adv = float(rs.choice([0.0, rs.normal() * 2.0, 40000.0 * rs.choice([-1, 1])]))
        out.append(make_record(start + i, float(rs.choice([0.0, 1.0, -0.5])), adv, step=i))
    return out


# ------------------------------------------------------------------ CPU: oracle
def test_set_priority_validation(oracle):
    b = oracle.buffer(1, 8, "priority_with_replacement", "plain_fifo", 0.0)
    with pytest.raises(OracleError, match="base"):
        b.set_priority(0, 0, 0)
    with pytest.raises(OracleError, match="adv_scale"):
        b.set_priority(1, 65537, 0)
    b.set_priority(1, 65536, 7)


@pytest.mark.parametrize("prio", [(1, 0, 0), (1, 4096, 0), (5, 65536, 100000), (1000, 3, 1)])
def test_oracle_matches_numpy_restatement(oracle, prio):
    rs = np.random.default_rng(sum(prio))
    shards, cap = 3, 3 * 50
    b = oracle.buffer(shards, cap, "priority_with_replacement", "plain_fifo", 0.0)
    b.set_priority(*prio)
    for r in random_records(rs, 190):
        b.push(r)
    contents = [b.shard_contents(s) for s in range(shards)]
    rng_a, rng_b = oracle.rng(9).stream("buffer_sampling"), oracle.rng(9).stream("buffer_sampling")
    for _ in range(4):
        got, gsh, gix = b.sample(shards * 37, rng_a)
        want_sh, want_ix = [], []
        for s in range(shards):
            cdf = np.cumsum(weights_np(contents[s], *prio), dtype=np.uint64)
            for _ in range(37):
                x = rng_b.below(int(cdf[-1]))
                want_sh.append(s)
                want_ix.append(int(np.searchsorted(cdf, np.uint64(x), side="right")))
        assert gsh.tolist() == want_sh and gix.tolist() == want_ix
        for s, i in zip(gsh, gix):  # use counts move with the draws
            contents[s][i]["use_count"] += 1


def test_oracle_weights_shape_the_distribution(oracle):
    """The empirical frequencies follow w_i / W (a chi-square bound)."""
    b = oracle.buffer(1, 16, "priority_with_replacement", "plain_fifo", 0.0)
    b.set_priority(1, 64, 500)
    rs = np.random.default_rng(3)
    recs = [make_record(i, float(i % 3 == 0), float(rs.uniform(-4, 4))) for i in range(16)]
    for r in recs:
        b.push(r)
    w = weights_np(np.array(recs, RECORD_DTYPE), 1, 64, 500).astype(np.float64)
    p = w / w.sum()
    rng = oracle.rng(4)
    counts = np.zeros(16)
    n = 0
    for _ in range(40):
        _, _, ix = b.sample(1000, rng)
        counts += np.bincount(ix, minlength=16)
        n += 1000
    chi2 = float(((counts - n * p) ** 2 / (n * p)).sum())
    assert chi2 < 45.0, chi2  # 15 dof: P(chi2 > 45) ~ 1e-4


@pytest.mark.ref
def test_unit_weights_are_the_reference_uniform_sampler(oracle, reference):
    """priority_with_replacement with weights (1, 0, 0) == the compiled
    reference's uniform_with_replacement (replay_buffer.cpp:141-145), record
    for record, including eviction interplay and shard order."""
    rs = np.random.default_rng(17)
    for trial in range(12):
        shards = int(rs.integers(1, 5))
        cap = shards * int(rs.integers(1, 12))
        ret = "positive_bias" if trial % 2 else "plain_fifo"
        a = oracle.buffer(shards, cap, "priority_with_replacement", ret, 0.5)
        b = reference.buffer(shards, cap, "uniform_with_replacement", ret, 0.5)
        ra, rb = oracle.rng(trial), reference.rng(trial)
        for i in range(150):
            if rs.random() < 0.7:
                rec = make_record(i, float(rs.random() < 0.4), 0.25)
                ea, eb = a.push(rec), b.push(rec)
                assert (ea is None) == (eb is None)
            else:
                k = shards * int(rs.integers(1, 4))
                try:
                    sa = a.sample(k, ra)[0]
                except OracleError:
                    with pytest.raises(OracleError):
                        b.sample(k, rb)
                    continue
                assert same_records(sa, b.sample(k, rb))


# ------------------------------------------------------------------ GPU
PRIO_CASES = {
    "adv_two_shards": dict(capacity=96, shards=2, batch=32, group=8, lmax=20, ragged=True,
                           seed=61, priority=(1, 4096, 0)),
    "bonus_posbias": dict(capacity=84, shards=3, batch=48, group=8, lmax=24, ragged=True,
                          seed=62, retention="positive_bias", delta=0.5, loss="asymre",
                          priority=(3, 1000, 50000)),
    "unit_weights_unique": dict(capacity=128, shards=1, batch=64, group=16, lmax=40,
                                ragged=True, seed=63, assume_unique=True, priority=(1, 0, 0)),
    "many_shards": dict(capacity=70 * 2, shards=70, batch=140, group=10, lmax=9, ragged=True,
                        seed=64, priority=(2, 65536, 7)),
    # shards above 24576 records: CDF and guide table in global scratch (k_sample_prio<false>)
    "cdf_in_global_memory": dict(capacity=2 * 25600, shards=2, batch=1024, group=16, lmax=4,
                                 ragged=True, seed=66, assume_unique=True, prompts=64,
                                 priority=(1, 30000, 2048)),
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(PRIO_CASES))
def test_priority_step_matches_oracle(name):
    """insert -> prioritised sample -> gather -> loss, bit-exact sampled
    (shard, index) pairs and records against the oracle every step."""
    from oracle.pyoracle import Oracle
    from tests.harness import StepConfig, run_step_parity

    cfg = StepConfig(strategy="priority_with_replacement", **PRIO_CASES[name])
    counts = run_step_parity(cfg, steps=5, ora=Oracle())
    assert counts["samples"] == 5 * cfg.batch


@pytest.mark.gpu
def test_priority_c4_shape_sampler():
    """The C4 shape (16384 trajectories, B = 4096): 32 CDF chunks and 14 MT
    blocks per call, sampled (shard, index) pairs bit-exact vs the oracle."""
    from oracle.pyoracle import Oracle
    from tests.harness import StepConfig, run_step_parity

    cfg = StepConfig(capacity=16384, shards=1, batch=4096, group=16, lmax=4, ragged=True,
                     seed=65, prompts=256, assume_unique=True,
                     strategy="priority_with_replacement", priority=(1, 65536, 4096))
    run_step_parity(cfg, steps=3, ora=Oracle(), check_every=3)


@pytest.mark.gpu
def test_priority_gpu_api():
    """Validation messages, and unit weights draw exactly as the uniform
    sampler on the device (same pushes, same seed)."""
    import paper_2604_08706_b200 as rb

    b = rb.ShardedReplayBuffer(2, 16, strategy="priority_with_replacement")
    assert b.strategy() == "priority_with_replacement" and b.priority() == (1, 0, 0)
    with pytest.raises(ValueError, match="base"):
        b.set_priority(0, 0, 0)
    with pytest.raises(ValueError, match="adv_scale"):
        b.set_priority(1, 70000, 0)
    u = rb.ShardedReplayBuffer(2, 16, strategy="uniform_with_replacement")
    rs = np.random.default_rng(5)
    for r in random_records(rs, 21):
        b.push(r)
        u.push(r)
    rp, ru = rb.Rng(8), rb.Rng(8)
    for _ in range(3):
        gp, sp, ip = b.sample(10, rp, with_index=True)
        gu, su, iu = u.sample(10, ru, with_index=True)
        assert np.array_equal(sp, su) and np.array_equal(ip, iu)
    # weighted: every record with |A| = 40000 (clamped to 2^15) dominates
    b.set_priority(1, 65536, 0)
    _, sh, ix = b.sample(200, rp, with_index=True)
    heavy = set()
    for s in range(2):
        c = b.shard_contents(s)
        heavy |= {(s, i) for i in range(len(c)) if abs(c[i]["advantage"]) > 30000}
    frac = np.mean([(int(s), int(i)) in heavy for s, i in zip(sh, ix)])
    assert heavy and frac > 0.9, frac


@pytest.mark.gpu
def test_priority_mass_owned_shards():
    """rb_priority_mass: exact per-shard sums; a process holding shard 1 of 3
    reports zeros for the others (its contribution to the all-reduce)."""
    import paper_2604_08706_b200 as rb

    recs = random_records(np.random.default_rng(4), 40)
    full = rb.ShardedReplayBuffer(3, 30, strategy="priority_with_replacement")
    part = rb.ShardedReplayBuffer(3, 30, strategy="priority_with_replacement",
                                  shard_range=(1, 2))
    for b in (full, part):
        b.set_priority(1, 65536, 12345)
        for r in recs:
            b.push(r)
    want = np.array([weights_np(full.shard_contents(s), 1, 65536, 12345).sum(dtype=np.uint64)
                     for s in range(3)], np.uint64)
    assert np.array_equal(full.priority_mass(), want)
    assert np.array_equal(part.priority_mass(), np.array([0, want[1], 0], np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["adv_two_shards", "bonus_posbias"])
def test_priority_multi_shard_fallback(name, monkeypatch):
    """Several shards are drawn in one pass that assumes no below() rejection;
    a rejection (probability < W/2^64 per draw) falls back to the exact
    shard-by-shard loop over the same ring.  RB_DEBUG_FORCE_DRAW_REPLAY forces
    that fallback after every optimistic pass: still bit-exact."""
    from oracle.pyoracle import Oracle
    from tests.harness import StepConfig, run_step_parity

    monkeypatch.setenv("RB_DEBUG_FORCE_DRAW_REPLAY", "1")
    cfg = StepConfig(strategy="priority_with_replacement", **PRIO_CASES[name])
    run_step_parity(cfg, steps=4, ora=Oracle())


@pytest.mark.gpu
def test_priority_eight_shards_c4_shape():
    """C4 split into 8 shards (16384 records, 512 draws each): the
    all-shards-at-once pass, bit-exact vs the oracle."""
    from oracle.pyoracle import Oracle
    from tests.harness import StepConfig, run_step_parity

    cfg = StepConfig(capacity=16384, shards=8, batch=4096, group=16, lmax=4, ragged=True,
                     seed=67, prompts=256, assume_unique=True,
                     strategy="priority_with_replacement", priority=(1, 65536, 4096))
    run_step_parity(cfg, steps=3, ora=Oracle(), check_every=3)
