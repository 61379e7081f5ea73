"""Error and normalisation paths (round-2 advisor findings):

* an asynchronous (RB_INSERT_ASSUME_UNIQUE) insert rejected on the device
  freezes the fused sampler (and the prioritised one) enqueued behind it — no use counts, no RNG
  consumption — and the next synchronising call reports the error; the
  buffer then continues exactly like the reference, which never applied the
  rejected push (replay_buffer.cpp:85-88);
* rb_loss_finalize / rb_loss_finalize_vec after AsymRE keep the reference's
  objective sum(coef * logp) / B (bandit.cpp:436);
* the GRPO normalisation is applied once: a finalize after the
  single-process local fix (or a second finalize) leaves dlogp unchanged;
* misaligned device arrays are rejected with RB_EINVAL instead of faulting.
"""
import numpy as np
import pytest
import torch

from tests.harness import Producer, StepConfig, insert_groups

pytestmark = pytest.mark.gpu


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU test requested but CUDA is not available")


def _fill(cfg, oracle):
    from paper_2604_08706_b200 import ShardedReplayBuffer

    buf = ShardedReplayBuffer(cfg.shards, cfg.capacity, cfg.strategy, cfg.retention, cfg.delta,
                              max_tokens=cfg.lmax)
    buf.set_stream(torch.cuda.current_stream().cuda_stream)
    ob = oracle.buffer(cfg.shards, cfg.capacity, cfg.strategy, cfg.retention, cfg.delta)
    prod = Producer(cfg, oracle)
    while ob.size() < cfg.capacity:
        rec, length, tok, lpo, toff, _ = prod.groups(2, 0)
        insert_groups(buf, rec, toff, tok, lpo, cfg.group, "cuda:0", assume_unique=True)
        for r in rec:
            ob.push(r)
    return buf, ob, prod


@pytest.mark.parametrize("strategy", ["uniform_with_replacement", "priority_with_replacement"])
@pytest.mark.parametrize("shards", [1, 3])
def test_rejected_async_insert_freezes_sampler(oracle, shards, strategy):
    _need_gpu()
    from oracle.pyoracle import same_records
    from paper_2604_08706_b200 import Rng

    cfg = StepConfig(capacity=48 * shards, shards=shards, batch=12 * shards, group=4, lmax=40,
                     ragged=True, seed=7, strategy=strategy)
    buf, ob, prod = _fill(cfg, oracle)
    grng = Rng(cfg.seed).stream("buffer_sampling")
    orng = oracle.rng(cfg.seed).stream("buffer_sampling")
    # a batch whose ids are not new: rejected on the device, nothing applied
    rec, length, tok, lpo, toff, _ = prod.groups(3, 1)
    bad = rec.copy()
    bad["rollout_id"] = bad["rollout_id"][::-1].copy()  # decreasing: violates the promise
    insert_groups(buf, bad, toff, tok, lpo, cfg.group, "cuda:0", assume_unique=True, overlap=True)
    buf.sample_device(cfg.batch, grng)  # overlaps the rejected insert: must freeze
    draws = grng.draws
    with pytest.raises(ValueError, match="ASSUME_UNIQUE"):
        buf.check()
    assert grng.draws == draws
    assert buf.batch_total_tokens() == 0
    for s in range(shards):  # the reference never applied the push
        assert same_records(buf.shard_contents(s), ob.shard_contents(s)), f"shard {s}"
    # the stream continues where the reference's does
    for _ in range(3):
        grec, gsh, gix = buf.sample(cfg.batch, grng, with_index=True)
        orec, osh, oix = ob.sample(cfg.batch, orng)
        assert np.array_equal(gix, oix) and np.array_equal(gsh, osh)
        assert same_records(grec, orec)


@pytest.mark.parametrize("strategy", ["uniform_with_replacement", "priority_with_replacement"])
def test_rejected_async_insert_reported_by_host_sample(oracle, strategy):
    _need_gpu()
    from paper_2604_08706_b200 import Rng

    cfg = StepConfig(capacity=32, shards=1, batch=8, group=4, lmax=16, ragged=False, seed=3,
                     strategy=strategy)
    buf, ob, prod = _fill(cfg, oracle)
    rec, length, tok, lpo, toff, _ = prod.groups(2, 1)
    bad = rec.copy()
    bad["rollout_id"][:] = 0  # already stored
    insert_groups(buf, bad, toff, tok, lpo, cfg.group, "cuda:0", assume_unique=True, overlap=True)
    with pytest.raises(ValueError):
        buf.sample(cfg.batch, Rng(cfg.seed).stream("buffer_sampling"))
    buf.check()  # cleared


def _loss_batch(oracle, seed=11):
    from paper_2604_08706_b200 import Rng

    cfg = StepConfig(capacity=64, shards=1, batch=32, group=8, lmax=50, ragged=True, seed=seed)
    buf, ob, prod = _fill(cfg, oracle)
    buf.sample_device(cfg.batch, Rng(cfg.seed).stream("buffer_sampling"))
    ids, lens, off = buf.batch_ids()
    total = int(off[-1])
    lpn = oracle.synth_logp_now(cfg.seed, 1, ids, off)
    rec = ob.sample(cfg.batch, oracle.rng(cfg.seed).stream("buffer_sampling"))[0]
    return buf, lpn, total, off, rec


def test_asymre_finalize_keeps_reference_objective(oracle):
    _need_gpu()
    from paper_2604_08706_b200 import LossStats

    buf, lpn, total, off, rec = _loss_batch(oracle)
    pad = total + 8
    lpn_d = torch.zeros(pad, dtype=torch.float32, device="cuda:0")
    lpn_d[:total] = torch.from_numpy(lpn)
    dl = torch.zeros(pad, dtype=torch.float32, device="cuda:0")
    torch.cuda.synchronize()
    st = buf.loss_asymre(lpn_d, dl, -0.1)
    want = st.objective
    assert np.isfinite(want) and want != 0.0
    st2 = buf.loss_finalize(dl, st)  # world size 1: reduced stats == local stats
    assert st2.objective == pytest.approx(want, rel=1e-15)
    vec = torch.zeros(3, dtype=torch.float64, device="cuda:0")
    buf.loss_set_reduce_vector(vec)
    buf.loss_asymre(lpn_d, dl, -0.1)
    out = LossStats()
    buf.loss_finalize_vec(dl, vec, out)
    assert out.objective == pytest.approx(want, rel=1e-15)
    buf.loss_set_reduce_vector(None)


def test_grpo_normalisation_applied_once(oracle):
    _need_gpu()
    from paper_2604_08706_b200 import LossStats

    buf, lpn, total, off, rec = _loss_batch(oracle, seed=13)
    lpn = lpn.copy()
    lpn[total // 2] = np.float32(np.inf)  # one excluded token: the local fix rescales
    pad = total + 8
    lpn_d = torch.zeros(pad, dtype=torch.float32, device="cuda:0")
    lpn_d[:total] = torch.from_numpy(lpn)
    dl = torch.zeros(pad, dtype=torch.float32, device="cuda:0")
    torch.cuda.synchronize()
    st = buf.loss_grpo(lpn_d, dl, 0.2, 0.28)
    assert st.excluded == 1
    d_want, obj, inc, exc = oracle.loss_grpo_tokens(lpn, _lpo(oracle, rec, off), rec["advantage"],
                                                    off, 0.2, 0.28)
    once = dl[:total].cpu().numpy().copy()
    np.testing.assert_allclose(once, d_want, rtol=1e-5, atol=1e-12)
    buf.loss_finalize(dl, st)  # generic multi-rank code at world size 1
    buf.loss_finalize(dl, st)
    assert np.array_equal(dl[:total].cpu().numpy(), once), "normalisation applied twice"
    vec = torch.zeros(3, dtype=torch.float64, device="cuda:0")
    buf.loss_set_reduce_vector(vec)
    buf.loss_grpo(lpn_d, dl, 0.2, 0.28)
    buf.loss_finalize_vec(dl, vec, LossStats())
    assert np.array_equal(dl[:total].cpu().numpy(), once)
    buf.loss_set_reduce_vector(None)


def _lpo(oracle, rec, off):
    lens = np.diff(off)
    _, lpo, _ = oracle.synth_payload(13, rec["rollout_id"], lens)
    return lpo


def test_misaligned_device_arrays_rejected(oracle):
    _need_gpu()
    buf, lpn, total, off, rec = _loss_batch(oracle, seed=17)
    out = torch.zeros(total + 16, dtype=torch.int32, device="cuda:0")
    with pytest.raises(ValueError, match="16-byte aligned"):
        buf.gather(out[1:], None, None)
    lp = torch.zeros(total + 16, dtype=torch.float32, device="cuda:0")
    with pytest.raises(ValueError, match="16-byte aligned"):
        buf.loss_grpo(lp[1:], lp[4:], 0.2, 0.2)
    buf.gather(out[4:], None, None)  # 16-byte aligned slices are fine
    buf.check()
