"""Record-level replay schedule used by the tests and the golden-fixture generator.

TEST INFRASTRUCTURE ONLY.  Restates the production / warm-up / sample loop of
train() (bandit.cpp:568-691): warm-up fills the buffer to capacity with whole
groups created at step 0 (609-615); each step adds W*B/(mu*T) records to a
debt and pushes whole groups while the debt covers one (617-640); then
samples B records from the "buffer_sampling" stream (576, 641).  The
trajectories are the synthetic workload of include/replay_synth.h (the
bandit policy is out of scope).  Works with any buffer object
exposing push(record) -> evicted|None and sample(B, rng) -> records.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .pyoracle import RECORD_DTYPE


@dataclass
class ScheduleConfig:
    capacity: int = 84
    shards: int = 1
    batch: int = 512
    group: int = 8
    workers: int = 5
    trainers: int = 3
    mu: float = 5.28
    lmax: int = 1
    ragged: bool = False
    strategy: str = "uniform_with_replacement"
    retention: str = "plain_fifo"
    delta: float = 0.0
    seed: int = 1
    prompts: int = 64

    @property
    def per_step_production(self) -> float:
        return self.workers * self.batch / (self.mu * self.trainers)


@dataclass
class Producer:
    """Emits whole groups with monotone ids (bandit.cpp:596-607)."""

    cfg: ScheduleConfig
    oracle: object
    next_id: int = 0
    next_group: int = 0
    prompt_cursor: int = 0
    group_mean: dict = field(default_factory=dict)

    def group(self, step: int):
        c = self.cfg
        ids = np.arange(self.next_id, self.next_id + c.group, dtype=np.uint64)
        reward, length, blp = self.oracle.synth_meta(c.seed, ids, c.lmax, c.ragged)
        adv = self.oracle.group_advantages(reward)
        mean = 0.0
        for r in reward:  # bandit.cpp:316-318, sequential
            mean += float(r)
        mean /= c.group
        rec = np.zeros(c.group, RECORD_DTYPE)
        rec["rollout_id"] = ids
        rec["prompt_id"] = self.prompt_cursor
        rec["group_id"] = self.next_group
        rec["creation_step"] = step
        rec["policy_version"] = step
        rec["reward"] = reward
        rec["is_correct"] = reward == 1.0
        rec["behavior_logprob"] = blp
        rec["advantage"] = adv
        self.group_mean[self.next_group] = mean
        self.prompt_cursor = (self.prompt_cursor + 1) % c.prompts
        self.next_group += 1
        self.next_id += c.group
        return rec, length


def run_schedule(buf, rng, cfg: ScheduleConfig, steps: int, oracle) -> dict:
    """Drive `buf` through warm-up + `steps` replay steps; return the trace."""
    prod = Producer(cfg, oracle)
    evicted_warm = []
    while buf.size() < cfg.capacity:
        rec, _ = prod.group(0)
        for r in rec:
            ev = buf.push(r)
            evicted_warm.append(-1 if ev is None else int(ev["rollout_id"]))
    debt = 0.0
    pushes_per_step, evicted, sampled = [], [], []
    for step in range(steps):
        debt += cfg.per_step_production
        ev_step = []
        while debt >= float(cfg.group):
            rec, _ = prod.group(step)
            for r in rec:
                ev = buf.push(r)
                ev_step.append(-1 if ev is None else int(ev["rollout_id"]))
            debt -= float(cfg.group)
        batch = buf.sample(cfg.batch, rng)
        if isinstance(batch, tuple):
            batch = batch[0]
        pushes_per_step.append(len(ev_step))
        evicted.extend(ev_step)
        sampled.append(np.stack([batch["rollout_id"].astype(np.int64),
                                 batch["use_count"].astype(np.int64)], axis=1))
    return {
        "evicted_warm": np.asarray(evicted_warm, np.int64),
        "pushes_per_step": np.asarray(pushes_per_step, np.int64),
        "evicted": np.asarray(evicted, np.int64),
        "sampled": np.stack(sampled) if sampled else np.zeros((0, cfg.batch, 2), np.int64),
        "final_size": np.int64(buf.size()),
    }
