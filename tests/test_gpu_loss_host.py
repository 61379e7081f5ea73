"""The losses with HOST logp_now / dlogp buffers (the chunked upload / kernel /
download pipeline of run_loss, loss.cu) give exactly the device-buffer result:
dlogp bit-identical per token, the same included / excluded counts, the
objective within fp64 summation-order noise — for pageable and pinned host
memory, GRPO and AsymRE, with and without an excluded (non-finite) token
(which takes the rescale-and-re-download path)."""
import numpy as np
import pytest
import torch

from tests.harness import Producer, StepConfig, insert_groups

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def batch(oracle):
    if not torch.cuda.is_available():
        pytest.fail("GPU test requested but CUDA is not available")
    from paper_2604_08706_b200 import Rng, ShardedReplayBuffer

    cfg = StepConfig(capacity=256, shards=2, batch=96, group=8, lmax=300, ragged=True, seed=61)
    buf = ShardedReplayBuffer(cfg.shards, cfg.capacity, cfg.strategy, cfg.retention, cfg.delta,
                              max_tokens=cfg.lmax)
    buf.set_stream(torch.cuda.current_stream().cuda_stream)
    prod = Producer(cfg, oracle)
    while buf.size() < cfg.capacity:
        rec, length, tok, lpo, toff, _ = prod.groups(4, 0)
        insert_groups(buf, rec, toff, tok, lpo, cfg.group, "cuda:0")
    buf.sample_device(cfg.batch, Rng(cfg.seed).stream("buffer_sampling"))
    ids, lens, off = buf.batch_ids()
    total = int(off[-1])
    lpn = oracle.synth_logp_now(cfg.seed, 1, ids, off)
    return buf, lpn, total


def _run(buf, kind, lpn_arr, dl_arr):
    if kind == "grpo":
        return buf.loss_grpo(lpn_arr, dl_arr, 0.2, 0.28)
    return buf.loss_asymre(lpn_arr, dl_arr, -0.1)


@pytest.mark.parametrize("kind", ["grpo", "asymre"])
@pytest.mark.parametrize("memory", ["pageable", "pinned"])
@pytest.mark.parametrize("excluded", [False, True])
def test_host_buffer_loss_matches_device(batch, kind, memory, excluded):
    buf, lpn0, total = batch
    lpn = lpn0.copy()
    if excluded:
        lpn[total // 3] = np.float32(np.inf)
    pad = total + 8
    lpn_d = torch.zeros(pad, dtype=torch.float32, device="cuda:0")
    lpn_d[:total] = torch.from_numpy(lpn)
    dl_d = torch.zeros(pad, dtype=torch.float32, device="cuda:0")
    torch.cuda.synchronize()
    st_d = _run(buf, kind, lpn_d, dl_d)
    buf.synchronize()
    want = dl_d[:total].cpu().numpy()
    if memory == "pageable":
        lpn_h = np.zeros(pad, np.float32)
        lpn_h[:total] = lpn
        dl_h = np.full(pad, -5.0, np.float32)
        st_h = _run(buf, kind, lpn_h, dl_h)
        got, tail = dl_h[:total], dl_h[total:]
    else:
        lpn_h = torch.zeros(pad, dtype=torch.float32).pin_memory()
        lpn_h[:total] = torch.from_numpy(lpn)
        dl_h = torch.full((pad,), -5.0, dtype=torch.float32).pin_memory()
        st_h = _run(buf, kind, lpn_h, dl_h)
        got, tail = dl_h[:total].numpy(), dl_h[total:].numpy()
    assert np.array_equal(got, want), "host-buffer dlogp differs from the device path"
    assert (tail == -5.0).all(), "wrote past the batch"
    assert (st_h.included, st_h.excluded) == (st_d.included, st_d.excluded)
    if kind == "grpo":
        assert st_d.excluded == (1 if excluded else 0)
    if np.isfinite(st_d.objective):
        assert abs(st_h.objective - st_d.objective) <= 1e-12 * max(1.0, abs(st_d.objective))
    else:  # AsymRE has no exclusion: a non-finite logp_now reaches the objective
        assert st_h.objective == st_d.objective


@pytest.mark.parametrize("excluded", [False, True])
def test_async_host_outputs(batch, excluded):
    """rb_set_async_outputs: the pinned dlogp download completes after
    synchronize(); back-to-back calls reuse the staging area safely."""
    buf, lpn0, total = batch
    lpn = lpn0.copy()
    if excluded:
        lpn[total // 5] = np.float32(np.inf)
    pad = total + 8
    lpn_d = torch.zeros(pad, dtype=torch.float32, device="cuda:0")
    lpn_d[:total] = torch.from_numpy(lpn)
    dl_d = torch.zeros(pad, dtype=torch.float32, device="cuda:0")
    torch.cuda.synchronize()
    st_d = _run(buf, "grpo", lpn_d, dl_d)
    buf.synchronize()
    want = dl_d[:total].cpu().numpy()
    lpn_h = torch.zeros(pad, dtype=torch.float32).pin_memory()
    lpn_h[:total] = torch.from_numpy(lpn)
    outs = [torch.full((pad,), -5.0, dtype=torch.float32).pin_memory() for _ in range(3)]
    buf.set_async_outputs(True)
    try:
        for o in outs:  # three calls in a row, no synchronisation between them
            st = _run(buf, "grpo", lpn_h, o)
            assert (st.included, st.excluded) == (st_d.included, st_d.excluded)
        buf.synchronize()
    finally:
        buf.set_async_outputs(False)
    for o in outs:
        np.testing.assert_array_equal(o[:total].numpy(), want)


def test_async_host_gather(batch):
    """rb_set_async_outputs with a pinned host gather: the packed tokens /
    logp_old drain on the copy stream (complete after synchronize()) while
    the next calls run; gather -> loss -> gather with no synchronisation
    between them reuses the staging area safely."""
    buf, lpn0, total = batch
    pad = total + 8
    tok_d = torch.zeros(pad, dtype=torch.int32, device="cuda:0")
    lpo_d = torch.zeros(pad, dtype=torch.float32, device="cuda:0")
    off_d = torch.zeros(buf.batch_size() + 1, dtype=torch.int64, device="cuda:0")
    buf.gather(tok_d, lpo_d, off_d)
    buf.synchronize()
    lpn_h = torch.zeros(pad, dtype=torch.float32).pin_memory()
    lpn_h[:total] = torch.from_numpy(lpn0)
    dl_h = torch.zeros(pad, dtype=torch.float32).pin_memory()
    toks = [torch.full((pad,), -7, dtype=torch.int32).pin_memory() for _ in range(2)]
    lpos = [torch.full((pad,), -7.0, dtype=torch.float32).pin_memory() for _ in range(2)]
    offs = [torch.zeros(buf.batch_size() + 1, dtype=torch.int64).pin_memory() for _ in range(2)]
    buf.set_async_outputs(True)
    try:
        for i in range(2):
            buf.gather(toks[i], lpos[i], offs[i])
            assert int(offs[i][-1]) == total  # the offsets are synchronous
            _run(buf, "grpo", lpn_h, dl_h)
        buf.synchronize()
    finally:
        buf.set_async_outputs(False)
    for i in range(2):
        assert np.array_equal(toks[i][:total].numpy(), tok_d[:total].cpu().numpy())
        assert np.array_equal(lpos[i][:total].numpy(), lpo_d[:total].cpu().numpy())
        assert (toks[i][total:].numpy() == -7).all()
