"""GRPO normalisation modes on the GPU.

* sequence ratio: rb_grpo_tokens_ex at L > 1 against the reference's own
  record-level grpo_loss_grad (tests/golden/golden_seq.npz, from oracle/_ref)
  within 1e-5;
* both sequence modes through the buffer (k_loss_grpo_seq_buf: logp_old from
  the slot rows, behavior_logprob from the record column) and over explicit
  arrays against the oracle (or_loss_grpo_tokens_mode), with excluded
  tokens, a fully excluded sequence, device and host buffers, and the
  one-collective finalize at world size 1.
"""
import os

import numpy as np
import pytest
import torch

from tests.harness import Producer, StepConfig, insert_groups

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
MODES = {"seq_mean": 1, "seq_ratio": 2}


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU test requested but CUDA is not available")


def test_seq_ratio_stateless_matches_reference_golden():
    _need_gpu()
    import paper_2604_08706_b200 as rb

    g = np.load(os.path.join(HERE, "golden", "golden_seq.npz"))
    off = g["seq_offsets"]
    for dev in (False, True):
        args = [g["seq_logp_now"], g["seq_logp_old"], g["seq_adv"], off]
        if dev:
            args = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in args]
        out = torch.zeros(int(off[-1]) + 4, dtype=torch.float32, device="cuda") if dev else None
        d, st = rb.grpo_tokens(*args, eps_low=0.2, eps_high=0.28, mode="seq_ratio",
                               behavior_logprob=g["seq_blp"], out=out)
        d = d[: int(off[-1])].cpu().numpy() if dev else d
        want = np.repeat(g["seq_dlogp_record"], np.diff(off))
        np.testing.assert_allclose(d, want, rtol=1e-5, atol=1e-12)
        assert st.objective == pytest.approx(float(g["seq_obj"]), rel=1e-5)
        assert st.excluded == int(g["seq_excluded"])


@pytest.mark.parametrize("mode", sorted(MODES))
def test_stateless_modes_match_oracle_with_exclusions(oracle, mode):
    _need_gpu()
    import paper_2604_08706_b200 as rb

    rs = np.random.default_rng(17)
    n = 60
    lens = rs.integers(1, 700, n)
    off = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    tot = int(off[-1])
    lpo = (-rs.uniform(0.001, 0.05, tot)).astype(np.float32)
    lpn = (lpo + rs.normal(0, 0.01, tot)).astype(np.float32)
    lpn[3] = np.inf
    lpn[off[9]:off[10]] = np.nan
    adv = rs.normal(size=n)
    d, st = rb.grpo_tokens(lpn, lpo, adv, off, 0.2, 0.28, mode=mode)
    dw, obj, inc, exc = oracle.loss_grpo_tokens_mode(lpn, lpo, adv, off, MODES[mode], eps_low=0.2,
                                                     eps_high=0.28)
    np.testing.assert_allclose(d, dw, rtol=1e-5, atol=1e-12)
    assert (st.included, st.excluded) == (inc, exc)
    assert st.objective == pytest.approx(obj, rel=1e-5)


@pytest.mark.parametrize("mode", sorted(MODES))
@pytest.mark.parametrize("shards", [1, 2])
@pytest.mark.parametrize("host_io", [False, True])
def test_buffer_modes_match_oracle(oracle, mode, shards, host_io):
    _need_gpu()
    from paper_2604_08706_b200 import LossStats, Rng, ShardedReplayBuffer

    cfg = StepConfig(capacity=96, shards=shards, batch=32 * shards, group=8, lmax=3000,
                     ragged=True, seed=41 + shards)
    buf = ShardedReplayBuffer(shards, cfg.capacity, max_tokens=cfg.lmax)
    buf.set_stream(torch.cuda.current_stream().cuda_stream)
    ob = oracle.buffer(shards, cfg.capacity)
    prod = Producer(cfg, oracle)
    while ob.size() < cfg.capacity:
        rec, length, tok, lpo, toff, _ = prod.groups(3, 0)
        insert_groups(buf, rec, toff, tok, lpo, cfg.group, "cuda:0", assume_unique=True)
        for r in rec:
            ob.push(r)
    buf.sample_device(cfg.batch, Rng(cfg.seed).stream("buffer_sampling"))
    orec = ob.sample(cfg.batch, oracle.rng(cfg.seed).stream("buffer_sampling"))[0]
    ids, lens, off = buf.batch_ids()
    assert np.array_equal(ids, orec["rollout_id"])
    total = int(off[-1])
    _, lpo, _ = oracle.synth_payload(cfg.seed, ids, lens)
    lpn = oracle.synth_logp_now(cfg.seed, 1, ids, off)
    # short sequences so the sequence ratio is not always clipped
    lpn[2] = np.float32(np.inf)
    k = int(np.argmin(lens[1:])) + 1
    lpn[off[k]:off[k + 1]] = np.nan  # a fully excluded sequence
    pad = total + 8
    if host_io:
        lpn_a = np.zeros(pad, np.float32)
        lpn_a[:total] = lpn
        dl = np.zeros(pad, np.float32)
    else:
        lpn_a = torch.zeros(pad, dtype=torch.float32, device="cuda:0")
        lpn_a[:total] = torch.from_numpy(lpn)
        dl = torch.zeros(pad, dtype=torch.float32, device="cuda:0")
        torch.cuda.synchronize()
    st = buf.loss_grpo(lpn_a, dl, 0.2, 0.28, mode=mode)
    got = dl[:total] if host_io else dl[:total].cpu().numpy()
    # the buffer path takes behavior_logprob from the record (= sum of logp_old here)
    dw, obj, inc, exc = oracle.loss_grpo_tokens_mode(lpn, lpo, orec["advantage"], off, MODES[mode],
                                                     blp=orec["behavior_logprob"], eps_low=0.2,
                                                     eps_high=0.28)
    np.testing.assert_allclose(got, dw, rtol=1e-5, atol=1e-12)
    assert (st.included, st.excluded) == (inc, exc)
    assert st.objective == pytest.approx(obj, rel=1e-5)
    if mode == "seq_ratio":
        assert (dw != 0).any(), "no live sequence gradient: test data too far off-policy"
    if not host_io:  # world size 1: the one-collective finalize leaves the result alone
        vec = torch.zeros(3, dtype=torch.float64, device="cuda:0")
        buf.loss_set_reduce_vector(vec)
        buf.loss_grpo(lpn_a, dl, 0.2, 0.28, mode=mode)
        out = LossStats()
        buf.loss_finalize_vec(dl, vec, out)
        np.testing.assert_allclose(dl[:total].cpu().numpy(), dw, rtol=1e-5, atol=1e-12)
        assert (out.included, out.excluded) == (inc, exc)
        assert out.objective == pytest.approx(obj, rel=1e-5)
        buf.loss_set_reduce_vector(None)
