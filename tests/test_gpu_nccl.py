"""rb_allreduce_loss_stats: the step's one collective issued by the library
on its own stream through an NCCL communicator taken from torch's
ProcessGroupNCCL (world size 1 on the single GPU of the test box: the
all-reduce is the identity, so the result must equal rb_loss_finalize_vec
on the un-reduced vector), plus its error contract."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def comm():
    import torch.distributed as dist

    if not torch.cuda.is_available():
        pytest.fail("GPU test requested but CUDA is not available")
    torch.cuda.set_device(0)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    x = torch.ones(1, device="cuda:0")
    dist.all_reduce(x)  # the communicator exists once a collective ran
    torch.cuda.synchronize()
    ptr = dist.group.WORLD._get_backend(torch.device("cuda"))._comm_ptr()
    assert ptr
    yield ptr
    dist.destroy_process_group()


def _loaded_buffer(rb, oracle, seed):
    """One sampled batch (with an excluded token) and its packed logp_now."""
    from tests.harness import Producer, StepConfig

    cfg = StepConfig(capacity=64, shards=1, batch=32, group=8, lmax=40, ragged=True, seed=seed)
    buf = rb.ShardedReplayBuffer(1, 64, max_tokens=40)
    buf.set_stream(torch.cuda.current_stream().cuda_stream)
    prod = Producer(cfg, oracle)
    rec, length, tok, lpo, toff, _ = prod.groups(8, 0)
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    buf.insert(rollout_id=t(rec["rollout_id"].copy()), reward=t(rec["reward"].copy()),
               group_offsets=t(np.arange(0, 65, 8, dtype=np.int64)), tok_offsets=t(toff),
               tokens=t(tok), logp_old=t(lpo), assume_unique=True)
    buf.sample_device(32, rb.Rng(seed).stream("buffer_sampling"))
    tot = buf.batch_total_tokens()
    pad = (tot + 3) // 4 * 4 + 4
    gen = torch.Generator(device="cuda").manual_seed(seed)
    lpn = torch.randn(pad, device="cuda", generator=gen).mul_(0.1).sub_(1.0)
    lpn[3] = float("inf")  # one excluded token: the finalize rescales
    return buf, lpn, pad


def test_allreduce_loss_stats_equals_finalize_vec(comm, oracle):
    import paper_2604_08706_b200 as rb

    outs = []
    for use_nccl in (False, True):
        buf, lpn, pad = _loaded_buffer(rb, oracle, seed=5)
        vec = torch.zeros(3, dtype=torch.float64, device="cuda")
        buf.loss_set_reduce_vector(vec)
        dl = torch.zeros(pad, device="cuda")
        st = rb.LossStats()
        buf.loss_grpo(lpn, dl, 0.2, 0.2, stats=False)
        if use_nccl:
            buf.allreduce_loss_stats(comm, dl, st)
        else:
            buf.loss_finalize_vec(dl, vec, st)
        buf.synchronize()
        outs.append((dl.cpu().numpy(), st.objective, st.included, st.excluded, vec.cpu().numpy()))
    (d0, o0, i0, e0, v0), (d1, o1, i1, e1, v1) = outs
    assert e0 == e1 == 1 and i0 == i1 and o0 == o1
    assert np.array_equal(d0, d1) and np.array_equal(v0, v1)


def test_allreduce_loss_stats_needs_a_registered_vector(comm, oracle):
    import paper_2604_08706_b200 as rb

    buf, lpn, pad = _loaded_buffer(rb, oracle, seed=6)
    dl = torch.zeros(pad, device="cuda")
    buf.loss_grpo(lpn, dl, 0.2, 0.2, stats=False)
    from paper_2604_08706_b200._lib import ReplayError

    with pytest.raises(ReplayError, match="register a reduce vector"):
        buf.allreduce_loss_stats(comm, dl)
    with pytest.raises(ValueError, match="NULL communicator"):
        buf.allreduce_loss_stats(0, dl)


def test_allreduce_priority_mass(comm):
    """rb_allreduce_priority_mass at world size 1: the identity over
    rb_priority_mass, which equals the numpy sum of the record weights."""
    import paper_2604_08706_b200 as rb
    from tests.test_priority import random_records, weights_np

    buf = rb.ShardedReplayBuffer(3, 60, strategy="priority_with_replacement")
    buf.set_priority(2, 4096, 777)
    for r in random_records(np.random.default_rng(3), 50):
        buf.push(r)
    want = np.array([weights_np(buf.shard_contents(s), 2, 4096, 777).sum(dtype=np.uint64)
                     for s in range(3)], np.uint64)
    assert np.array_equal(buf.priority_mass(), want)
    dev = torch.full((3,), -1, dtype=torch.int64, device="cuda:0")
    buf.allreduce_priority_mass(comm, dev)
    torch.cuda.synchronize()
    assert np.array_equal(dev.cpu().numpy().view(np.uint64), want)
    with pytest.raises(ValueError, match="device vector"):
        buf.allreduce_priority_mass(comm, np.zeros(3, np.uint64))
