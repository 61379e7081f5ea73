"""World-size-2 check (gloo, CPU) of the multi-GPU decomposition of the
replay step: every rank holds the replicated metadata of all
T shards and regenerates the same MT19937-64 stream, owns the payload of one
shard, evaluates the token loss over its own selections and all-reduces the
24-byte statistics {objective_sum, included, excluded}.  The per-rank
results, stitched together, must equal the single-process replay step.

The arithmetic is the CPU oracle's (the CUDA kernels implement the same
split: shard_begin/shard_end, rb_loss_finalize); this pins the host-side
decomposition the N-GPU bench relies on.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.harness import Producer, StepConfig

CFG = dict(capacity=64, shards=2, batch=32, group=8, lmax=40, ragged=True, seed=21)
STEPS = 6


def _local_partials(ora, cfg, rng_seed_step, orec, off, lengths, lo, hi):
    """Un-normalised GRPO partials of selections [lo, hi) (token form)."""
    ids = orec["rollout_id"][lo:hi]
    lens = np.array([lengths[int(i)] for i in ids], np.int64)
    loff = np.zeros(len(ids) + 1, np.int64)
    np.cumsum(lens, out=loff[1:])
    _, lpo, _ = ora.synth_payload(cfg.seed, ids, lens)
    lpn = ora.synth_logp_now(cfg.seed, rng_seed_step, ids, loff)
    if len(ids) and loff[-1] > 3:
        lpn[2] = np.float32(np.inf)  # one excluded token per shard
    d, obj, inc, exc = ora.loss_grpo_tokens(lpn, lpo, orec["advantage"][lo:hi], loff,
                                            cfg.eps_low, cfg.eps_high)
    coef = -d.astype(np.float64) * inc if inc else np.zeros_like(d, np.float64)
    return coef, obj * inc, inc, exc


def _run(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.pyoracle import Oracle

    ora = Oracle()
    cfg = StepConfig(**CFG)
    buf = ora.buffer(cfg.shards, cfg.capacity)  # metadata of ALL shards (replicated)
    rng = ora.rng(cfg.seed).stream("buffer_sampling")
    prod = Producer(cfg, ora)
    lengths = {}

    def push(ng, step):
        rec, length, *_ = prod.groups(ng, step)
        for r, L in zip(rec, length):
            lengths[int(r["rollout_id"])] = int(L)
            buf.push(r)

    while buf.size() < cfg.capacity:
        push(1, 0)
    out = []
    debt = 0.0
    for step in range(STEPS):
        debt += cfg.per_step
        ng = 0
        while debt >= cfg.group:
            ng += 1
            debt -= cfg.group
        if ng:
            push(ng, step)
        orec, osh, _ = buf.sample(cfg.batch, rng)
        per = cfg.batch // world
        lo, hi = rank * per, (rank + 1) * per  # shard-major: this rank's shard
        assert np.all(osh[lo:hi] == rank)
        coef, obj_sum, inc, exc = _local_partials(ora, cfg, step + 1, orec, None, lengths, lo, hi)
        stats = torch.tensor([obj_sum, float(inc), float(exc)], dtype=torch.float64)
        dist.all_reduce(stats)
        g_obj, g_inc, g_exc = stats.tolist()
        dl = (-coef / g_inc).astype(np.float32)
        out.append((dl, g_obj / g_inc, int(g_inc), int(g_exc)))
    q.put((rank, out))
    dist.destroy_process_group()


def _single_process():
    from oracle.pyoracle import Oracle

    ora = Oracle()
    cfg = StepConfig(**CFG)
    buf = ora.buffer(cfg.shards, cfg.capacity)
    rng = ora.rng(cfg.seed).stream("buffer_sampling")
    prod = Producer(cfg, ora)
    lengths = {}

    def push(ng, step):
        rec, length, *_ = prod.groups(ng, step)
        for r, L in zip(rec, length):
            lengths[int(r["rollout_id"])] = int(L)
            buf.push(r)

    while buf.size() < cfg.capacity:
        push(1, 0)
    res = []
    debt = 0.0
    for step in range(STEPS):
        debt += cfg.per_step
        ng = 0
        while debt >= cfg.group:
            ng += 1
            debt -= cfg.group
        if ng:
            push(ng, step)
        orec, _, _ = buf.sample(cfg.batch, rng)
        per = cfg.batch // 2
        ids_all, lpn_all, lpo_all, adv_all = [], [], [], []
        lens_all = []
        for lo, hi in ((0, per), (per, 2 * per)):  # same exclusion injection per shard
            ids = orec["rollout_id"][lo:hi]
            lens = np.array([lengths[int(i)] for i in ids], np.int64)
            loff = np.zeros(len(ids) + 1, np.int64)
            np.cumsum(lens, out=loff[1:])
            _, lpo, _ = ora.synth_payload(cfg.seed, ids, lens)
            lpn = ora.synth_logp_now(cfg.seed, step + 1, ids, loff)
            if len(ids) and loff[-1] > 3:
                lpn[2] = np.float32(np.inf)
            ids_all.append(ids)
            lens_all.append(lens)
            lpn_all.append(lpn)
            lpo_all.append(lpo)
        lens = np.concatenate(lens_all)
        off = np.zeros(len(lens) + 1, np.int64)
        np.cumsum(lens, out=off[1:])
        d, obj, inc, exc = ora.loss_grpo_tokens(np.concatenate(lpn_all), np.concatenate(lpo_all),
                                                orec["advantage"], off, cfg.eps_low, cfg.eps_high)
        res.append((d, obj, inc, exc, int(off[per])))
    return res


@pytest.mark.timeout(300)
def test_two_rank_decomposition_matches_single_process():
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_run, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = _single_process()
    for step, (d, obj, inc, exc, split) in enumerate(want):
        d0, o0, i0, e0 = got[0][step]
        d1, o1, i1, e1 = got[1][step]
        assert (i0, e0) == (i1, e1) == (inc, exc) and exc == 2
        assert o0 == pytest.approx(obj, rel=1e-12) and o1 == pytest.approx(obj, rel=1e-12)
        np.testing.assert_allclose(np.concatenate([d0, d1]), d, rtol=1e-6, atol=1e-12)
        assert len(d0) == split


# ---------------------------------------------------------------- priority mass
def _prio_run(rank, world, port, q):
    """Each rank: the replicated oracle buffer, its own shard's mass only
    (rb_priority_mass's contribution), then the all-reduce."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.pyoracle import Oracle
    from tests.test_priority import random_records, weights_np

    ora = Oracle()
    buf = ora.buffer(world, 40 * world, "priority_with_replacement", "plain_fifo", 0.0)
    buf.set_priority(3, 2048, 99)
    for r in random_records(np.random.default_rng(8), 70 * world):
        buf.push(r)
    mass = torch.zeros(world, dtype=torch.int64)
    mass[rank] = int(weights_np(buf.shard_contents(rank), 3, 2048, 99).sum(dtype=np.uint64))
    dist.all_reduce(mass)
    # the prioritised draws of this rank's shard from the shared stream
    rng = ora.rng(5).stream("buffer_sampling")
    _, sh, ix = buf.sample(world * 16, rng)
    q.put((rank, (mass.numpy().copy(), ix[sh == rank].copy())))
    dist.destroy_process_group()


def test_two_rank_priority_mass_allreduce():
    """World size 2 (gloo): the all-reduced per-shard masses equal the
    single-process masses, and each rank's slice of the prioritised draws
    equals the single-process draws of its shard (B/T per shard)."""
    import socket

    from oracle.pyoracle import Oracle
    from tests.test_priority import random_records, weights_np

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_prio_run, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ora = Oracle()
    buf = ora.buffer(2, 80, "priority_with_replacement", "plain_fifo", 0.0)
    buf.set_priority(3, 2048, 99)
    for r in random_records(np.random.default_rng(8), 140):
        buf.push(r)
    want = [int(weights_np(buf.shard_contents(s), 3, 2048, 99).sum(dtype=np.uint64))
            for s in range(2)]
    _, sh, ix = buf.sample(32, ora.rng(5).stream("buffer_sampling"))
    for rank in range(2):
        mass, own = got[rank]
        assert mass.tolist() == want
        assert np.array_equal(own, ix[sh == rank])
