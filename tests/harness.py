"""Replay-step parity harness: the CUDA library vs the CPU oracle, step by step.

Drives both through the same schedule (train()'s production/warm-up loop,
bandit.cpp:568-691, with T shards as in simulate(), async_sim.cpp:138-139)
on the synthetic workload of include/replay_synth.h and compares, every
step: evicted ids per push, sampled records (ids + post-increment use
counts, i.e. the MT19937-64 stream and arrival-order mapping), the packed
token gather, and the GRPO / AsymRE token losses.

Used by tests/test_gpu_*.py and __graft_entry__.smoke().
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from oracle.pyoracle import RECORD_DTYPE, Oracle, same_records


@dataclass
class StepConfig:
    capacity: int = 64
    shards: int = 1
    batch: int = 32
    group: int = 8
    lmax: int = 64
    ragged: bool = True
    workers: int = 5
    trainers: int = 3
    mu: float = 5.28
    strategy: str = "uniform_with_replacement"
    retention: str = "plain_fifo"
    delta: float = 0.0
    seed: int = 1
    loss: str = "grpo"
    eps_low: float = 0.2
    eps_high: float = 0.28
    delta_v: float = -0.1
    prompts: int = 16
    device_inputs: bool = True   # torch CUDA tensors (hot path) vs numpy host arrays
    assume_unique: bool = False  # RB_INSERT_ASSUME_UNIQUE (closed-form FIFO insert kernels)
    overlap: bool = False        # no host sync between insert and sample (evicted ids to the device)
    early_gather: bool = False   # sample with no host outputs, gather right away (overlapped gather)
    priority: tuple | None = None  # (base, adv_scale, pos_bonus) of priority_with_replacement

    @property
    def per_step(self):
        return self.workers * self.batch / (self.mu * self.trainers)


class Producer:
    """Whole groups with monotone ids; advantages left to the device."""

    def __init__(self, cfg: StepConfig, ora: Oracle):
        self.cfg, self.o = cfg, ora
        self.next_id = 0
        self.next_group = 0
        self.prompt = 0

    def groups(self, ngroups: int, step: int):
        c = self.cfg
        n = ngroups * c.group
        ids = np.arange(self.next_id, self.next_id + n, dtype=np.uint64)
        reward, length, blp = self.o.synth_meta(c.seed, ids, c.lmax, c.ragged)
        gid = np.repeat(np.arange(self.next_group, self.next_group + ngroups), c.group).astype(np.uint64)
        prompt = (self.prompt + np.repeat(np.arange(ngroups), c.group)) % c.prompts
        adv = np.zeros(n)
        gmean = np.zeros(n)
        for g in range(ngroups):
            sl = slice(g * c.group, (g + 1) * c.group)
            adv[sl] = self.o.group_advantages(reward[sl])
            m = 0.0
            for r in reward[sl]:
                m += float(r)
            gmean[sl] = m / c.group
        rec = np.zeros(n, RECORD_DTYPE)
        rec["rollout_id"] = ids
        rec["prompt_id"] = prompt
        rec["group_id"] = gid
        rec["creation_step"] = step
        rec["policy_version"] = step
        rec["reward"] = reward
        rec["is_correct"] = reward == 1.0
        rec["behavior_logprob"] = blp
        rec["advantage"] = adv
        tok, lpo, toff = self.o.synth_payload(c.seed, ids, length)
        self.next_id += n
        self.next_group += ngroups
        self.prompt = (self.prompt + ngroups) % c.prompts
        return rec, length, tok, lpo, toff, gmean


def _to(x, dev):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).to(dev) if dev else x


def insert_groups(buf, rec, toff, tok, lpo, group, dev, assume_unique=False, overlap=False):
    n = rec.shape[0]
    goff = np.arange(0, n + 1, group, dtype=np.int64)
    # overlap: no evicted-id output (its copy would serialise the stream) and
    # nothing waits for the insert; evictions are checked through the samples
    # and the final shard contents instead
    ev = None if overlap else np.zeros(n, np.uint64)
    buf.insert(rollout_id=_to(rec["rollout_id"].copy(), dev), prompt_id=_to(rec["prompt_id"].copy(), dev),
               group_id=_to(rec["group_id"].copy(), dev),
               creation_step=_to(rec["creation_step"].copy(), dev),
               policy_version=_to(rec["policy_version"].copy(), dev),
               reward=_to(rec["reward"].copy(), dev),
               behavior_logprob=_to(rec["behavior_logprob"].copy(), dev),
               group_offsets=_to(goff, dev), tok_offsets=_to(toff, dev), tokens=_to(tok, dev),
               logp_old=_to(lpo, dev), evicted=ev, assume_unique=assume_unique)
    if assume_unique and not overlap:
        buf.synchronize()  # the evicted-id copy is asynchronous
        buf.check()
    return ev


def run_step_parity(cfg: StepConfig, steps: int, ora: Oracle | None = None, check_every: int = 1):
    """Returns a dict of per-check counters; raises AssertionError on mismatch."""
    import torch

    from paper_2604_08706_b200 import Rng, ShardedReplayBuffer

    ora = ora or Oracle()
    dev = "cuda:0" if cfg.device_inputs else None
    gbuf = ShardedReplayBuffer(cfg.shards, cfg.capacity, cfg.strategy, cfg.retention, cfg.delta,
                               max_tokens=cfg.lmax)
    if dev:  # inputs are copied to the device on torch's stream: run the library on it too
        gbuf.set_stream(torch.cuda.current_stream().cuda_stream)
    obuf = ora.buffer(cfg.shards, cfg.capacity, cfg.strategy, cfg.retention, cfg.delta)
    if cfg.priority is not None:
        gbuf.set_priority(*cfg.priority)
        obuf.set_priority(*cfg.priority)
    grng = Rng(cfg.seed).stream("buffer_sampling")
    orng = ora.rng(cfg.seed).stream("buffer_sampling")
    prod = Producer(cfg, ora)
    lengths, gmeans = {}, {}
    counts = {"pushes": 0, "evictions": 0, "samples": 0, "tokens": 0, "excluded": 0}

    def push_groups(ngroups, step):
        rec, length, tok, lpo, toff, gmean = prod.groups(ngroups, step)
        for i, r in enumerate(rec):
            lengths[int(r["rollout_id"])] = int(length[i])
            gmeans[int(r["rollout_id"])] = gmean[i]
        ev = insert_groups(gbuf, rec, toff, tok, lpo, cfg.group, dev, cfg.assume_unique,
                           cfg.overlap)
        if cfg.overlap:
            for r in rec:
                e = obuf.push(r)
                counts["pushes"] += 1
                counts["evictions"] += e is not None
            return
        for i, r in enumerate(rec):
            e = obuf.push(r)
            want = np.uint64(np.iinfo(np.uint64).max) if e is None else e["rollout_id"]
            assert ev[i] == want, f"eviction mismatch at push {counts['pushes']}: {ev[i]} vs {want}"
            counts["pushes"] += 1
            counts["evictions"] += e is not None

    while obuf.size() < cfg.capacity:
        push_groups(1, 0)
    debt = 0.0
    for step in range(steps):
        debt += cfg.per_step
        ng = 0
        while debt >= float(cfg.group):
            ng += 1
            debt -= float(cfg.group)
        if ng:
            push_groups(ng, step)
        if cfg.early_gather:
            # insert -> sample -> gather enqueued back to back (outputs allocated
            # first): the gather runs as a dependent of the sampler and overlaps it
            cap = cfg.batch * cfg.lmax + 8
            eg = [torch.full((cap,), -7, dtype=torch.int32, device="cuda:0"),
                  torch.full((cap,), -7.0, dtype=torch.float32, device="cuda:0"),
                  torch.zeros(cfg.batch + 1, dtype=torch.int64, device="cuda:0")]
            gbuf.sample_device(cfg.batch, grng)
            gbuf.gather(*eg)
            gbuf.check()
            orec, osh, oix = obuf.sample(cfg.batch, orng)
            gids, glens, _ = gbuf.batch_ids()
            assert np.array_equal(gids, orec["rollout_id"]), f"sampled ids mismatch step {step}"
        else:
            grec, gsh, gix = gbuf.sample(cfg.batch, grng, with_index=True)
            if cfg.overlap:
                gbuf.check()
            orec, osh, oix = obuf.sample(cfg.batch, orng)
            assert np.array_equal(gsh, osh) and np.array_equal(gix, oix), f"sample index mismatch step {step}"
            assert same_records(grec, orec), f"sampled records mismatch step {step}"
        counts["samples"] += cfg.batch
        if step % check_every and not cfg.early_gather:
            continue
        # ---- gather
        ids = orec["rollout_id"]
        lens = np.array([lengths[int(i)] for i in ids], np.int64)
        off = np.zeros(len(ids) + 1, np.int64)
        np.cumsum(lens, out=off[1:])
        tot = int(off[-1])
        tok_want, lpo_want, _ = ora.synth_payload(cfg.seed, ids, lens)
        pad = (tot + 3) // 4 * 4 + 4
        gt = torch.zeros(pad, dtype=torch.int32, device="cuda:0")
        gl = torch.zeros(pad, dtype=torch.float32, device="cuda:0")
        go = torch.zeros(len(ids) + 1, dtype=torch.int64, device="cuda:0")
        if cfg.early_gather:
            gt, gl, go = eg
            assert int(gt[tot].item()) == -7 and float(gl[tot].item()) == -7.0, "gather overran"
        else:
            torch.cuda.synchronize()  # inputs written on torch's stream
            gbuf.gather(gt, gl, go)
            gbuf.synchronize()  # the library runs on its own stream
        go_h = go.cpu().numpy()[: len(off)]
        if not np.array_equal(go_h, off):
            bad = np.nonzero(go_h != off)[0]
            raise AssertionError(f"packed offsets mismatch step {step}: {bad.size} entries from "
                                 f"{bad[0]}: got {go_h[bad[:4]]} want {off[bad[:4]]}")
        assert np.array_equal(gt[:tot].cpu().numpy(), tok_want), f"gathered tokens mismatch step {step}"
        assert np.array_equal(gl[:tot].cpu().numpy(), lpo_want), f"gathered logp_old mismatch step {step}"
        counts["tokens"] += tot
        # ---- loss
        lpn = ora.synth_logp_now(cfg.seed, step + 1, ids, off)
        if cfg.loss == "grpo" and step % 5 == 3 and tot > 2:  # exercise exclusion
            lpn[1] = np.float32(np.inf)
        lpn_d = torch.zeros(pad, dtype=torch.float32, device="cuda:0")
        lpn_d[:tot] = torch.from_numpy(lpn)
        dl = torch.zeros(pad, dtype=torch.float32, device="cuda:0")
        torch.cuda.synchronize()
        if cfg.loss == "grpo":
            st = gbuf.loss_grpo(lpn_d, dl, cfg.eps_low, cfg.eps_high)
            d_want, obj, inc, exc = ora.loss_grpo_tokens(lpn, lpo_want, orec["advantage"], off,
                                                         cfg.eps_low, cfg.eps_high)
            assert (st.included, st.excluded) == (inc, exc), (st.included, st.excluded, inc, exc)
            counts["excluded"] += exc
        else:
            st = gbuf.loss_asymre(lpn_d, dl, cfg.delta_v)
            gm = np.array([gmeans[int(i)] for i in ids])
            d_want, obj = ora.loss_asymre_tokens(lpn, orec["reward"], gm, off, cfg.delta_v)
        gbuf.synchronize()
        got = dl[:tot].cpu().numpy()
        np.testing.assert_allclose(got, d_want, rtol=1e-5, atol=1e-12,
                                   err_msg=f"dlogp mismatch step {step}")
        assert abs(st.objective - obj) <= 1e-5 * max(1.0, abs(obj)), (st.objective, obj)
    for s in range(cfg.shards):  # final state, arrival order per shard
        assert same_records(gbuf.shard_contents(s), obuf.shard_contents(s)), f"shard {s} contents"
    return counts
