"""The oracle's GRPO normalisation modes (oracle/replay_oracle.c
or_loss_grpo_tokens_mode), pinned against the compiled reference:

* sequence ratio (mode 2) equals the reference's own record-level
  grpo_loss_grad (bandit.cpp:363-408) with logp = sum_t logp_now_t and
  behavior_logprob = sum_t logp_old_t, on every token of the trajectory
  (tests/golden/golden_seq.npz, made by tests/golden/make_golden.py from
  oracle/_ref);
* at L = 1 all three modes reduce to the record form;
* the per-sequence mean (mode 1) against a direct restatement, with
  excluded tokens and a fully excluded sequence.
"""
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def golden_seq():
    return np.load(os.path.join(HERE, "golden", "golden_seq.npz"))


def test_seq_ratio_matches_reference_records(oracle, golden_seq):
    g = golden_seq
    off = g["seq_offsets"]
    d, obj, inc, exc = oracle.loss_grpo_tokens_mode(g["seq_logp_now"], g["seq_logp_old"],
                                                    g["seq_adv"], off, 2, blp=g["seq_blp"],
                                                    eps_low=0.2, eps_high=0.28)
    want = np.repeat(g["seq_dlogp_record"], np.diff(off)).astype(np.float32)
    np.testing.assert_allclose(d, want, rtol=1e-6, atol=1e-12)
    assert abs(obj - float(g["seq_obj"])) <= 1e-12 * max(1.0, abs(float(g["seq_obj"])))
    assert exc == int(g["seq_excluded"]) and inc == off.size - 1 - exc
    # behavior_logprob defaults to sum_t logp_old: the same answer here
    d2, obj2, _, _ = oracle.loss_grpo_tokens_mode(g["seq_logp_now"], g["seq_logp_old"],
                                                  g["seq_adv"], off, 2, eps_low=0.2, eps_high=0.28)
    assert np.array_equal(d2, d) and obj2 == obj


def test_modes_reduce_to_records_at_length_one(oracle):
    rs = np.random.default_rng(3)
    n = 300
    lpo = (-rs.uniform(0.01, 3.0, n)).astype(np.float32)
    lpn = (lpo + rs.normal(0, 0.2, n)).astype(np.float32)
    adv = rs.normal(size=n)
    adv[::7] = 0.0
    off = np.arange(n + 1, dtype=np.int64)
    ref = oracle.loss_grpo_records(lpn.astype(np.float64), lpo.astype(np.float64), adv, 0.2, 0.28)
    for mode in (0, 1, 2):
        d, obj, inc, exc = oracle.loss_grpo_tokens_mode(lpn, lpo, adv, off, mode, eps_low=0.2,
                                                        eps_high=0.28)
        assert np.array_equal(d, ref[0].astype(np.float32)), mode
        assert obj == pytest.approx(ref[1], rel=1e-14) and (inc, exc) == (ref[2], ref[3])


def _seq_mean_restated(lpn, lpo, adv, off, lo, hi):
    terms, coefs, ns = [], [], []
    for i in range(off.size - 1):
        t_sum, n = 0.0, 0
        c_i = []
        for t in range(off[i], off[i + 1]):
            r = np.exp(float(lpn[t]) - float(lpo[t]))
            if not np.isfinite(r):
                c_i.append(0.0)
                continue
            n += 1
            cl = min(max(r, lo), hi)
            if r * adv[i] <= cl * adv[i]:
                t_sum += r * adv[i]
                c_i.append(adv[i] * r)
            else:
                t_sum += cl * adv[i]
                c_i.append(0.0)
        terms.append(t_sum / n if n else None)
        coefs.append(c_i)
        ns.append(n)
    S = sum(1 for n in ns if n)
    obj = sum(t for t in terms if t is not None) / S
    d = np.concatenate([np.array([-c / (n * S) if n else 0.0 for c in ci])
                        for ci, n in zip(coefs, ns)]).astype(np.float32)
    return d, obj, S


def test_seq_mean_with_exclusions(oracle):
    rs = np.random.default_rng(11)
    lens = rs.integers(1, 30, 40)
    off = np.zeros(41, np.int64)
    np.cumsum(lens, out=off[1:])
    tot = int(off[-1])
    lpo = (-rs.uniform(0.01, 2.0, tot)).astype(np.float32)
    lpn = (lpo + rs.normal(0, 0.3, tot)).astype(np.float32)
    lpn[5] = np.inf
    lpn[off[7]:off[8]] = np.nan  # a fully excluded sequence
    adv = rs.normal(size=40)
    d, obj, inc, exc = oracle.loss_grpo_tokens_mode(lpn, lpo, adv, off, 1, eps_low=0.2,
                                                    eps_high=0.28)
    dw, objw, S = _seq_mean_restated(lpn, lpo, adv, off, 0.8, 1.28)
    np.testing.assert_allclose(d, dw, rtol=1e-6, atol=1e-12)
    assert obj == pytest.approx(objw, rel=1e-12)
    assert inc == S == 39 and exc == 1 + int(lens[7])
