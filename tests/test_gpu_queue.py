"""GPU TransferQueue (transfer_queue.hpp:12-35) with payload: LIFO order,
all-or-nothing groups under back-pressure, unbounded growth, and the packed
token payload of popped records against the synthetic producer."""
import numpy as np
import pytest
import torch

from tests.harness import Producer, StepConfig

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rb():
    if not torch.cuda.is_available():
        pytest.fail("GPU test requested but CUDA is not available")
    import paper_2604_08706_b200 as rb

    return rb


@pytest.mark.parametrize("capacity", [None, 40])
def test_lifo_with_payload_vs_stack(rb, oracle, capacity):
    cfg = StepConfig(group=8, lmax=37, ragged=True, seed=51)
    q = rb.TransferQueue(capacity, max_tokens=cfg.lmax)
    prod = Producer(cfg, oracle)
    stack, lengths = [], {}
    rng = np.random.default_rng(5)
    for step in range(60):
        if rng.random() < 0.55:
            rec, length, tok, lpo, toff, _ = prod.groups(1, step)
            ok = q.push_group(rec, toff, tok, lpo)
            expect = capacity is None or len(stack) + len(rec) <= capacity
            assert ok == expect
            if ok:
                for r, L in zip(rec, length):
                    stack.append(r.copy())
                    lengths[int(r["rollout_id"])] = int(L)
        else:
            k = int(rng.integers(1, 12))
            pad = k * cfg.lmax + 8
            t = torch.zeros(pad, dtype=torch.int32, device="cuda:0")
            lp = torch.zeros(pad, dtype=torch.float32, device="cuda:0")
            off = torch.zeros(k + 1, dtype=torch.int64, device="cuda:0")
            torch.cuda.synchronize()
            got, n = q.pop_batch(k, t, lp, off)
            want = [stack.pop() for _ in range(min(k, len(stack)))]
            assert n == len(want)
            assert [int(x) for x in got["rollout_id"]] == [int(w["rollout_id"]) for w in want]
            if n:
                ids = got["rollout_id"]
                lens = np.array([lengths[int(i)] for i in ids], np.int64)
                tok_w, lpo_w, _ = oracle.synth_payload(cfg.seed, ids, lens)
                tot = int(lens.sum())
                assert np.array_equal(off[:n + 1].cpu().numpy()[-1:], [tot])
                assert np.array_equal(t[:tot].cpu().numpy(), tok_w)
                assert np.array_equal(lp[:tot].cpu().numpy(), lpo_w)
        assert q.size() == len(stack)


def test_queue_validation(rb):
    with pytest.raises(ValueError):
        rb.TransferQueue(0)
    q = rb.TransferQueue(4, max_tokens=3)
    rec = np.zeros(1, rb.RECORD_DTYPE)
    with pytest.raises(ValueError, match="max_tokens"):
        q.push(rec, tokens=np.arange(5, dtype=np.int32), logp_old=np.zeros(5, np.float32))
    assert q.size() == 0 and q.pop() is None
