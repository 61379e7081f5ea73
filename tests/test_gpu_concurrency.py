"""The reference's thread-safety contract: every ShardedReplayBuffer method
holds one mutex (replay_buffer.cpp:84, 188; replay_buffer.hpp:106-107), so
concurrent producers and a consumer see ONE total order of pushes and
samples, and a batched push (a whole group, async_sim.cpp:175-187,
bandit.cpp:596-607) is atomic.

Producers insert whole groups from several host threads while a consumer
samples; afterwards the test finds a serial order of the same calls that the
CPU oracle replays to exactly the consumer's observed samples (greedy
linearisation: the insert order is read back from the buffer's arrival
order, each sample is placed at the earliest insert prefix that reproduces
it), and checks the final shard contents."""
import threading

import numpy as np
import pytest

from oracle.pyoracle import RECORD_DTYPE, same_records

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rb():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test requested but CUDA is not available")
    import paper_2604_08706_b200 as rb

    return rb

G = 8          # group size
SEED = 77


def make_batch(ora, first_id, gid, step):
    ids = np.arange(first_id, first_id + G, dtype=np.uint64)
    reward, _, blp = ora.synth_meta(SEED, ids, 4, False)
    rec = np.zeros(G, RECORD_DTYPE)
    rec["rollout_id"] = ids
    rec["group_id"] = gid
    rec["prompt_id"] = gid % 5
    rec["creation_step"] = step
    rec["policy_version"] = step
    rec["reward"] = reward
    rec["is_correct"] = reward == 1.0
    rec["behavior_logprob"] = blp
    rec["advantage"] = ora.group_advantages(reward)
    return rec


def insert(buf, rec):
    buf.insert(rollout_id=rec["rollout_id"], reward=rec["reward"], prompt_id=rec["prompt_id"],
               group_id=rec["group_id"], creation_step=rec["creation_step"],
               policy_version=rec["policy_version"], behavior_logprob=rec["behavior_logprob"],
               group_offsets=np.array([0, G], np.int64))


def replay(ora, shards, cap, warm, order, batch):
    """Oracle replay of a serial order: ('i', rec) / ('s', None) events."""
    ob = ora.buffer(shards, cap)
    orng = ora.rng(SEED).stream("buffer_sampling")
    for rec in warm:
        for r in rec:
            ob.push(r)
    outs = []
    for kind, rec in order:
        if kind == "i":
            for r in rec:
                ob.push(r)
        else:
            outs.append(ob.sample(batch, orng)[0])
    return ob, outs


@pytest.mark.parametrize("shards", [1, 2])
def test_concurrent_producers_and_sampler_linearise(rb, oracle, shards):
    producers, per_producer, samples, batch = 4, 6, 12, 4 * shards
    warm = [make_batch(oracle, 0, 0, 0)]  # every shard non-empty before the race
    base = len(warm)
    batches = {p: [make_batch(oracle, (base + p * per_producer + k) * G, base + p * per_producer + k, 1)
                   for k in range(per_producer)] for p in range(producers)}
    cap = (base + producers * per_producer) * G  # nothing is evicted: arrival order = push order
    buf = rb.ShardedReplayBuffer(shards, cap, "uniform_with_replacement", "plain_fifo", 0.0)
    rng = rb.Rng(SEED).stream("buffer_sampling")
    for rec in warm:
        insert(buf, rec)
    got, errors = [], []
    start = threading.Barrier(producers + 1)

    def produce(p):
        try:
            start.wait()
            for rec in batches[p]:
                insert(buf, rec)
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    def consume():
        try:
            start.wait()
            for _ in range(samples):
                got.append(buf.sample(batch, rng))
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    th = [threading.Thread(target=produce, args=(p,)) for p in range(producers)]
    th.append(threading.Thread(target=consume))
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    assert len(got) == samples

    # push order from the arrival order: round-robin routing from cursor 0
    # puts push k in shard k % T at rank k // T (replay_buffer.cpp:89-90)
    push_of = {}
    for s in range(shards):
        for rank, r in enumerate(buf.shard_contents(s)):
            push_of[int(r["rollout_id"])] = rank * shards + s
    assert len(push_of) == cap
    by_first = {int(rec["rollout_id"][0]): rec for rec in sum(batches.values(), [])}
    for first, rec in by_first.items():  # a batched push is atomic: consecutive pushes, in order
        ks = [push_of[int(i)] for i in rec["rollout_id"]]
        assert ks == list(range(ks[0], ks[0] + G)), f"group {first} interleaved: {ks}"
    ins_order = sorted(by_first, key=lambda f: push_of[f])
    for p in range(producers):  # and each producer's program order holds
        mine = [int(b["rollout_id"][0]) for b in batches[p]]
        assert [f for f in ins_order if f in mine] == mine

    # place every sample at the earliest insert prefix the oracle reproduces it at
    order, placed = [], 0
    for si in range(samples):
        while True:
            cand = order + [("s", None)]
            _, outs = replay(oracle, shards, cap, warm, cand, batch)
            if same_records(outs[-1], got[si]):
                order = cand
                break
            assert placed < len(ins_order), f"sample {si}: no serial order reproduces it"
            order.append(("i", by_first[ins_order[placed]]))
            placed += 1
    order += [("i", by_first[f]) for f in ins_order[placed:]]
    ob, outs = replay(oracle, shards, cap, warm, order, batch)
    for si in range(samples):
        assert same_records(outs[si], got[si])
    for s in range(shards):  # use counts included
        assert same_records(buf.shard_contents(s), ob.shard_contents(s)), f"shard {s}"


def test_gather_dlpack_hand_off(rb, oracle):
    """rb_gather_dlpack: the packed batch handed to torch through DLPack,
    identical to rb_gather into caller arrays; unconsumed capsules free
    their tensors."""
    import gc

    import torch

    from tests.harness import Producer, StepConfig, insert_groups

    cfg = StepConfig(capacity=64, shards=1, batch=48, group=8, lmax=37, ragged=True, seed=5)
    buf = rb.ShardedReplayBuffer(1, cfg.capacity, max_tokens=cfg.lmax)
    prod = Producer(cfg, oracle)
    rec, length, tok, lpo, toff, _ = prod.groups(cfg.capacity // cfg.group, 0)
    insert_groups(buf, rec, toff, tok, lpo, cfg.group, None)
    rng = rb.Rng(3).stream("buffer_sampling")
    buf.sample(cfg.batch, rng)
    caps = buf.gather_dlpack()
    t, lp, off = (torch.from_dlpack(c) for c in caps)
    assert t.is_cuda and t.dtype == torch.int32 and lp.dtype == torch.float32
    assert off.dtype == torch.int64 and off.numel() == cfg.batch + 1
    tot = int(off[-1])
    assert t.numel() == tot == lp.numel()
    ref_t = torch.empty(tot + 8, dtype=torch.int32, device="cuda")
    ref_l = torch.empty(tot + 8, dtype=torch.float32, device="cuda")
    ref_o = torch.empty(cfg.batch + 1, dtype=torch.int64, device="cuda")
    buf.gather(ref_t, ref_l, ref_o)
    buf.synchronize()
    assert torch.equal(t, ref_t[:tot]) and torch.equal(lp, ref_l[:tot]) and torch.equal(off, ref_o)
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(20):  # never consumed: the capsule destructor releases them
        buf.gather_dlpack()
    gc.collect()
    torch.cuda.synchronize()
    assert torch.cuda.mem_get_info()[0] >= free0 - (8 << 20)
