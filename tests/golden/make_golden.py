"""Generate the golden fixtures in tests/golden/ by running the UNMODIFIED
reference library (oracle/_ref/libreplab_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile).

    python tests/golden/make_golden.py

The reference's own tests hold no sampled-index or RNG vectors (SURVEY.md
§4), so these fixtures are produced from the reference itself and then
used to pin both the C restatement (oracle/) and the CUDA library.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import RECORD_DTYPE, Oracle, Reference, build_oracle, canon  # noqa: E402
from oracle.workload import ScheduleConfig, run_schedule  # noqa: E402

# Schedules: C1/C2 of SURVEY.md §8d at the record level, plus multi-shard and
# without-replacement variants exercising every branch of pick_indices.
SCHEDULES = {
    "c1_fifo_with": ScheduleConfig(capacity=84, shards=1, batch=512, group=8, seed=1),
    "c2_posbias_with": ScheduleConfig(capacity=84, shards=1, batch=512, group=8, seed=2,
                                      retention="positive_bias", delta=0.5),
    "c5_t3_fifo_with": ScheduleConfig(capacity=252, shards=3, batch=504, group=8, seed=3,
                                      workers=5, trainers=3),
    "t3_posbias_without": ScheduleConfig(capacity=252, shards=3, batch=126, group=8, seed=4,
                                         strategy="uniform_without_replacement",
                                         retention="positive_bias", delta=0.2),
    "t2_unused_first": ScheduleConfig(capacity=84, shards=2, batch=42, group=8, seed=5,
                                      strategy="unused_first_without_replacement",
                                      workers=2, trainers=3),
    "t4_posbias_one_third": ScheduleConfig(capacity=96, shards=4, batch=64, group=16, seed=6,
                                           retention="positive_bias", delta=1.0 / 3.0,
                                           workers=7, trainers=1),
}
STEPS = 40


def seq_ratio_golden(ref: Reference) -> dict:
    """Sequence-level GRPO: ragged token trajectories whose
    record-level inputs are logp_now = sum_t logp_now_t and behavior_logprob =
    sum_t logp_old_t (fp64, token order), run through the reference's own
    grpo_loss_grad (bandit.cpp:363-408) by the 2-arm embedding.  Every token of
    trajectory i must get the record's dL/dlogp."""
    rs = np.random.default_rng(2604)
    n = 48
    lens = rs.integers(1, 41, n)
    off = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    tot = int(off[-1])
    lpo = (-rs.uniform(0.005, 0.2, tot)).astype(np.float32)
    lpn = (lpo.astype(np.float64) + rs.normal(0.0, 0.02, tot)).astype(np.float32)
    lpn = np.minimum(lpn, np.float32(-1e-4))
    recs = np.zeros(n, RECORD_DTYPE)
    blp = np.array([float(np.sum(lpo[off[i]:off[i + 1]].astype(np.float64))) for i in range(n)])
    want = np.zeros(n)
    for i in range(n):  # sequential fp64 sums, token order
        a = b = 0.0
        for t in range(off[i], off[i + 1]):
            a += float(lpn[t])
            b += float(lpo[t])
        want[i], blp[i] = a, b
    recs["behavior_logprob"] = blp
    recs["advantage"] = rs.normal(size=n)
    recs["advantage"][::11] = 0.0
    used, d, obj, exc = ref.loss_records("grpo", want, recs, eps_low=0.2, eps_high=0.28)
    return {"seq_offsets": off, "seq_logp_old": lpo, "seq_logp_now": lpn, "seq_blp": blp,
            "seq_adv": recs["advantage"].copy(), "seq_logp_used": used, "seq_dlogp_record": d,
            "seq_obj": np.float64(obj), "seq_excluded": np.int64(exc)}


def main():
    build_oracle(with_ref=True)
    if "--seq-only" in sys.argv:
        np.savez_compressed(os.path.join(HERE, "golden_seq.npz"), **seq_ratio_golden(Reference()))
        print("wrote", os.path.join(HERE, "golden_seq.npz"))
        return
    ref = Reference()
    ora = Oracle()
    out = {}

    # --- RNG: raw engine outputs, below() and Fisher-Yates per seed
    for seed in range(1, 6):
        r = ref.rng(seed).stream("buffer_sampling")
        out[f"rng_s{seed}_seed"] = np.uint64(r.seed)
        out[f"rng_s{seed}_raw"] = np.array([r.next_u64() for _ in range(700)], np.uint64)
        out[f"rng_s{seed}_below84"] = np.array([r.below(84) for _ in range(300)], np.uint64)
        out[f"rng_s{seed}_below16384"] = np.array([r.below(16384) for _ in range(300)],
                                                  np.uint64)
        out[f"rng_s{seed}_swor_100_37"] = r.sample_without_replacement(100, 37)
    idx = ref.rng(99).stream("cell", 7)
    out["rng_stream_idx_seed"] = np.uint64(idx.seed)
    out["rng_kat_10000"] = np.uint64(0)
    k = ref.rng(5489)
    for _ in range(9999):
        k.next_u64()
    out["rng_kat_10000"] = np.uint64(k.next_u64())

    # --- group advantages on random binary / real rewards
    rs = np.random.default_rng(7)
    groups = [rs.integers(0, 2, size=int(rs.integers(2, 17))).astype(np.float64)
              for _ in range(60)]
    groups += [rs.normal(size=int(rs.integers(2, 17))) for _ in range(20)]
    groups += [np.ones(8), np.zeros(2), np.array([1.0, 0.0, 1.0, 0.0])]
    flat = np.concatenate(groups)
    offs = np.zeros(len(groups) + 1, np.int64)
    np.cumsum([len(g) for g in groups], out=offs[1:])
    out["adv_rewards"] = flat
    out["adv_offsets"] = offs
    out["adv_out"] = np.concatenate([ref.group_advantages(g) for g in groups])

    # --- record-level losses through the reference's own grpo/asymre_loss_grad
    n = 256
    recs = np.zeros(n, RECORD_DTYPE)
    lp_old = -rs.uniform(0.05, 4.0, n)
    lp_want = np.log(np.clip(np.exp(lp_old) * np.exp(rs.normal(0, 0.15, n)), 1e-6, 0.999))
    recs["behavior_logprob"] = lp_old
    recs["advantage"] = rs.normal(size=n)
    recs["advantage"][::17] = 0.0
    recs["reward"] = rs.integers(0, 2, n)
    gmean = rs.uniform(0, 1, n)
    used, d, obj, exc = ref.loss_records("grpo", lp_want, recs, eps_low=0.2, eps_high=0.28)
    out["loss_records"] = recs
    out["loss_logp_now"] = used
    out["loss_group_mean"] = gmean
    out["grpo_dlogp"] = d
    out["grpo_obj"] = np.float64(obj)
    out["grpo_excluded"] = np.int64(exc)
    used2, d2, obj2, _ = ref.loss_records("asymre", lp_want, recs, group_mean=gmean, delta_v=-0.1)
    assert np.array_equal(used, used2)
    out["asymre_dlogp"] = d2
    out["asymre_obj"] = np.float64(obj2)

    # --- replay schedules (push/evict/sample traces)
    meta = {}
    for name, cfg in SCHEDULES.items():
        buf = ref.buffer(cfg.shards, cfg.capacity, cfg.strategy, cfg.retention, cfg.delta)
        rng = ref.rng(cfg.seed).stream("buffer_sampling")
        tr = run_schedule(buf, rng, cfg, STEPS, ora)
        for k2, v in tr.items():
            out[f"sched_{name}_{k2}"] = v
        out[f"sched_{name}_final_shards"] = canon(np.concatenate(
            [buf.shard_contents(s) for s in range(cfg.shards)]))
        out[f"sched_{name}_dump"] = np.frombuffer(buf.dump().encode(), np.uint8)
        meta[name] = cfg.__dict__
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    np.savez_compressed(os.path.join(HERE, "golden_seq.npz"), **seq_ratio_golden(ref))
    with open(os.path.join(HERE, "schedules.json"), "w") as f:
        json.dump({"steps": STEPS, "schedules": meta}, f, indent=1, sort_keys=True)
    print("wrote", os.path.join(HERE, "golden.npz"))


if __name__ == "__main__":
    main()
