#!/usr/bin/env python
"""bench.py — replay-step tokens/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c4|c3|c1|c2] [--no-e2e] [--no-cpu-baseline]

A step is one replay step of the path: insert the step's
freshly produced groups (device advantages, eviction), sample B trajectories
(MT19937-64 "buffer_sampling" stream), ragged-gather their tokens, and
evaluate the per-token GRPO loss + dL/dlogp.  The workload is C4 of
SURVEY.md §8d by default (buffer 16384 sharded over the N GPUs, 256 prompts
x G=16 = 4096 trajectories/step, 4096 tokens each, (W,T)=(5,3), mu=5.28).
logp_now comes from a synthetic trainer stand-in run between the two
phases (its time is reported separately and excluded from the step time).
Inputs are synthetic (include/replay_synth.h), resident in HBM before the
timed region; the buffer (537 MB) and per-step traffic exceed the 126 MB L2.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")

CONFIGS = {
    "c4": dict(name="C4: buffer 16384 trajectories sharded over the GPUs, 256 prompts x G=16 "
                    "per step, 4096-token responses, FIFO, uniform with replacement, GRPO",
               capacity=16384, batch=4096, group=16, lmax=4096, ragged=False,
               retention="plain_fifo", delta=0.0, loss="grpo"),
    "c3": dict(name="C3: buffer 1024, G=16, 64 prompts, ragged U{1..8192} tokens, 1 GPU, GRPO",
               capacity=1024, batch=1024, group=16, lmax=8192, ragged=True,
               retention="plain_fifo", delta=0.0, loss="grpo"),
    "c3fixed": dict(name="C3 shape with fixed 4096-token responses (diagnostic)",
                    capacity=1024, batch=1024, group=16, lmax=4096, ragged=False,
                    retention="plain_fifo", delta=0.0, loss="grpo"),
    "c1": dict(name="C1: buffer 84, (W,T)=(5,3), G=8, 64 prompts, 1024 tokens, GRPO",
               capacity=84, batch=512, group=8, lmax=1024, ragged=False,
               retention="plain_fifo", delta=0.0, loss="grpo"),
    "c5": dict(name="C5: staleness/reuse sweep W in {1,2,4,8}, T in {1,2,4} shards, buffer "
                    "84..4092, B=504 (63 prompts x G=8), record level (insert+evict+sample)",
               capacity=0, batch=504, group=8, lmax=0, ragged=False, retention="plain_fifo",
               delta=0.0, loss="none"),
    "c2": dict(name="C2: C1 + positive-bias retention (delta=0.5) + AsymRE",
               capacity=84, batch=512, group=8, lmax=1024, ragged=False,
               retention="positive_bias", delta=0.5, loss="asymre"),
}
# C4 with the prioritised-sampling CDF (builder extension, include/replay_b200.h
# rb_set_priority): w = 1 + floor(4096 |A|) + 4096 [reward > 0]
CONFIGS["c4prio"] = dict(CONFIGS["c4"], name=CONFIGS["c4"]["name"].replace(
    "uniform with replacement", "priority_with_replacement (w = 1 + 4096|A| + 4096[r > 0])"),
    strategy="priority_with_replacement", priority=(1, 4096, 4096))
W_WORKERS, T_TRAINERS, MU, SEED = 5, 3, 5.28, 1
EPS_LOW, EPS_HIGH, DELTA_V = 0.2, 0.2, -0.1


def algorithmic_bytes(t_ins, t_samp, r, b, loss):
    """16*T_ins + b_loss*T_samp + 64*R + 32*B (b_loss 20 GRPO / 16 AsymRE)."""
    return 16 * t_ins + (20 if loss == "grpo" else 16) * t_samp + 64 * r + 32 * b


def peaks():
    try:
        p = json.load(open(PEAKS_PATH))
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------- schedule
def schedule(cfg, steps):
    """Groups produced before step 0 (warm-up fill) and per step (bandit.cpp:609-640)."""
    g = cfg["group"]
    warm = math.ceil(cfg["capacity"] / g)
    per = W_WORKERS * cfg["batch"] / (MU * T_TRAINERS)
    debt, out = 0.0, []
    for _ in range(steps):
        debt += per
        n = 0
        while debt >= g:
            n += 1
            debt -= g
        out.append(n)
    return warm, out


class Clocks:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every
    ~0.5 ms while the timed region runs (nvidia-smi's 100 ms floor is longer
    than the timed region itself)."""

    NAMES = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
             "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
             "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
             "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
             "hw_power_brake": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, gpu):
        self.gpu, self.sm, self.reasons, self.max_mhz = gpu, [], set(), None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            idx = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(self.gpu)).split(",")[self.gpu]) \
                if os.environ.get("CUDA_VISIBLE_DEVICES", "").replace(",", "").isdigit() else self.gpu
            self.h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.nv = nv
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.nv = None
        return self

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, const in self.NAMES.items():
                    if r & getattr(nv, const):
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                break
            time.sleep(0.0005)

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join(timeout=2)

    def summary(self):
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml"}


# ---------------------------------------------------------------- our arm
class Workload:
    """Pre-generated inbound batches (device) for every step."""

    def __init__(self, cfg, nsteps, dev, stream):
        import torch

        from tools import synth

        self.cfg = cfg
        g = cfg["group"]
        warm, per_step = schedule(cfg, nsteps)
        self.batches = []
        nid, ngid = 0, 0
        prompts = cfg["batch"] // g
        plan = [(warm, 0)] + [(n, s) for s, n in enumerate(per_step)]
        for ngroups, step in plan:
            n = ngroups * g
            ids = torch.arange(nid, nid + n, dtype=torch.int64, device=dev)
            reward = torch.empty(n, dtype=torch.float64, device=dev)
            length = torch.empty(n, dtype=torch.int32, device=dev)
            blp = torch.empty(n, dtype=torch.float64, device=dev)
            synth.fill_meta(SEED, ids, cfg["lmax"], cfg["ragged"], reward, length, blp, stream)
            toff = torch.zeros(n + 1, dtype=torch.int64, device=dev)
            toff[1:] = torch.cumsum(length.to(torch.int64), 0)
            tot = int(toff[-1])
            pad = (tot + 3) // 4 * 4 + 4
            tokens = torch.empty(pad, dtype=torch.int32, device=dev)
            lpo = torch.empty(pad, dtype=torch.float32, device=dev)
            synth.fill_payload(SEED, ids, toff, tokens, lpo, stream)
            gid = torch.arange(ngid, ngid + ngroups, dtype=torch.int64, device=dev).repeat_interleave(g)
            b = dict(rollout_id=ids, reward=reward, behavior_logprob=blp,
                     group_id=gid, prompt_id=gid % prompts,
                     creation_step=torch.full((n,), step, dtype=torch.int64, device=dev),
                     policy_version=torch.full((n,), step, dtype=torch.int64, device=dev),
                     group_offsets=torch.arange(0, n + 1, g, dtype=torch.int64, device=dev),
                     tok_offsets=toff, tokens=tokens, logp_old=lpo)
            self.batches.append((b, n, tot))
            nid += n
            ngid += ngroups
        torch.cuda.synchronize()
        self.warm = self.batches[0]
        self.steps = self.batches[1:]

    def make_owned(self, rank, T):
        """Owned-metadata job (rb_insert_owned): every batch reduced to the records
        the round robin routes to shard `rank` (arrival positions = rank mod T
        from the cursor, replay_buffer.cpp:89-90), with their group advantages
        (computed by the producer from the whole group, bandit.cpp:276-294);
        `n_global` is the global batch size.  Prepared outside the timed region."""
        import torch

        import paper_2604_08706_b200 as rb

        cursor = 0
        out = []
        for b, n, _ in self.batches:
            dev = b["rollout_id"].device
            adv = torch.empty(n, dtype=torch.float64, device=dev)
            rb.group_advantages(b["reward"], b["group_offsets"], out=adv)
            j0 = (rank - cursor) % T
            idx = torch.arange(j0, n, T, device=dev)
            toff = b["tok_offsets"]
            lens = (toff[1:] - toff[:-1])[idx]
            ooff = torch.zeros(idx.numel() + 1, dtype=torch.int64, device=dev)
            ooff[1:] = torch.cumsum(lens, 0)
            tot = int(ooff[-1])
            # token gather indices: start of each own row + position within it
            starts = torch.repeat_interleave(toff[:-1][idx], lens)
            pos = torch.arange(tot, device=dev) - torch.repeat_interleave(ooff[:-1], lens)
            src = starts + pos
            pad = (tot + 3) // 4 * 4 + 4
            tok = torch.zeros(pad, dtype=torch.int32, device=dev)
            lpo = torch.zeros(pad, dtype=torch.float32, device=dev)
            tok[:tot] = b["tokens"][src]
            lpo[:tot] = b["logp_old"][src]
            o = {k: b[k][idx].contiguous() for k in ("rollout_id", "reward", "behavior_logprob",
                                                     "group_id", "prompt_id", "creation_step",
                                                     "policy_version")}
            o.update(advantage=adv[idx].contiguous(), tok_offsets=ooff, tokens=tok, logp_old=lpo,
                     n_global=n)
            out.append((o, int(idx.numel()), tot))
            cursor = (cursor + n) % T
        torch.cuda.synchronize()
        self.owned = True
        self.full = self.batches
        self.batches = out
        self.warm = out[0]
        self.steps = out[1:]


def scaled_cfg(cfg, world, weak=False):
    """The N-GPU job (BASELINE.json configs[3]).

    Strong scaling (default): the single-GPU workload itself — the buffer of
    `capacity` trajectories and the batch of `batch` draws — split into N
    shards, one per GPU (round-robin routing, replay_buffer.cpp:89-90; B/N
    draws per shard, replay_buffer.cpp:193-204).  Per-GPU payload, gather and
    loss work shrink as 1/N.

    Weak scaling (--weak): every GPU holds one shard of the single-GPU size
    and serves the single-GPU batch, so the job is N x the single-GPU
    workload."""
    if world == 1:
        return dict(cfg, scaling="weak")
    c = dict(cfg)
    tag = cfg["name"].split(":")[0]
    if weak:
        c["capacity"] = cfg["capacity"] * world
        c["batch"] = cfg["batch"] * world
        c["scaling"] = "weak"
        c["name"] = (f"{tag} per GPU x {world}: buffer {c['capacity']} "
                     f"trajectories in {world} shards of {cfg['capacity']} (one per GPU), "
                     f"{c['batch'] // cfg['group']} prompts x G={cfg['group']} per step, "
                     f"{cfg['lmax']}-token responses, {cfg['retention']}, {cfg['loss']}")
    else:
        c["scaling"] = "strong"
        c["name"] = (f"{tag} over {world} GPUs: buffer {cfg['capacity']} trajectories in "
                     f"{world} shards of {cfg['capacity'] // world} (one per GPU), "
                     f"{cfg['batch'] // cfg['group']} prompts x G={cfg['group']} per step "
                     f"({cfg['batch'] // world} draws per shard), {cfg['lmax']}-token responses, "
                     f"{cfg['retention']}, {cfg['loss']}")
    return c


def config_dict(cfg, world):
    """The `config` object of the JSON line — identical for both arms."""
    return {"workload": cfg["name"], "buffer": cfg["capacity"], "shards": world,
            "batch": cfg["batch"], "group": cfg["group"], "tokens_per_traj": cfg["lmax"],
            "ragged": cfg["ragged"], "retention": cfg["retention"], "delta": cfg["delta"],
            "sampling": cfg.get("strategy", "uniform_with_replacement"),
            "W": W_WORKERS, "T": T_TRAINERS, "mu": MU, "loss": cfg["loss"],
            "l2": "inputs larger than L2 (buffer + per-step traffic >> 126 MB); the trainer "
                  "stand-in ends with a 256 MB read, so the loss reads logp_now from HBM",
            "parallelism": f"shard{world}"}


def run_ours(args, rank, world, dist):
    import torch

    import paper_2604_08706_b200 as rb
    from tools import synth

    cfg = scaled_cfg(CONFIGS[args.config], world, getattr(args, "weak", False))
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    T, N, B = world, cfg["capacity"], cfg["batch"]
    assert N % T == 0 and B % T == 0, "config not divisible by the GPU count"
    buf = rb.ShardedReplayBuffer(T, N, cfg.get("strategy", "uniform_with_replacement"),
                                 cfg["retention"], cfg["delta"],
                                 max_tokens=cfg["lmax"], shard_range=(rank, rank + 1))
    if cfg.get("priority"):
        buf.set_priority(*cfg["priority"])
    buf.set_stream(sh)
    rng = rb.Rng(SEED).stream("buffer_sampling")
    K, Wm = args.steps, args.warmup
    wl = Workload(cfg, K + Wm, dev, sh)
    owned = getattr(args, "owned", False) and T > 1
    if owned:  # each rank holds and routes only its own shard's records
        wl.make_owned(rank, T)
        buf.set_owned_metadata()
    # warm-up fill (bandit.cpp:609-615)
    b, n, _ = wl.warm
    if owned:
        buf.insert(**b, assume_unique=True)
        n = 0  # inserted whole
    for lo in range(0, n, 4096):
        hi = min(n, lo + 4096)
        part = {k: v for k, v in b.items() if k not in ("group_offsets", "tok_offsets", "tokens", "logp_old")}
        part = {k: v[lo:hi] for k, v in part.items()}
        goff = torch.arange(0, hi - lo + 1, cfg["group"], dtype=torch.int64, device=dev)
        toff = (b["tok_offsets"][lo:hi + 1] - b["tok_offsets"][lo]).contiguous()
        o0 = int(b["tok_offsets"][lo])
        buf.insert(**part, group_offsets=goff, tok_offsets=toff,
                   tokens=b["tokens"][o0:].contiguous(), logp_old=b["logp_old"][o0:].contiguous(),
                   assume_unique=True)
    buf.check()
    per_rank = B // T
    max_local = per_rank * cfg["lmax"]
    pad = max_local + 8
    packed_tok = torch.empty(pad, dtype=torch.int32, device=dev)
    lpn = torch.empty(pad, dtype=torch.float32, device=dev)
    dlogp = torch.empty(pad, dtype=torch.float32, device=dev)
    off = torch.empty(per_rank + 1, dtype=torch.int64, device=dev)
    sel_ids = torch.empty(per_rank, dtype=torch.int64, device=dev)
    stats = torch.zeros(5, dtype=torch.float64, device=dev)  # rb_loss_stats (40 B)
    red3 = torch.zeros(3, dtype=torch.float64, device=dev)   # multi-GPU reduce vector (24 B)
    if world > 1:
        buf.loss_set_reduce_vector(red3)
    # N > 1 over NCCL: the library issues the step's one collective itself
    # (rb_allreduce_loss_stats on the buffer's stream, torch's communicator)
    comm = None
    if dist is not None and dist.get_backend() == "nccl":
        dist.all_reduce(red3)  # the communicator exists once a collective ran
        torch.cuda.synchronize()
        comm = dist.group.WORLD._get_backend(dev)._comm_ptr()
    # The trainer stand-in ends with a 256 MB read: the 126 MB L2 holds none of
    # logp_now when the loss starts (a real trainer's forward would have moved
    # far more data through L2 in between).
    l2buf = torch.ones(64 << 20, dtype=torch.float32, device=dev)
    l2out = torch.empty((), dtype=torch.float32, device=dev)

    def standin(i):
        buf.batch_ids_device(sel_ids)
        synth.logp_now(SEED, i + 1, sel_ids, off, lpn, sh)
        torch.sum(l2buf, dim=0, out=l2out)

    def step(i, ev=None):
        # Timing events only at phase boundaries that are not kernel->kernel
        # programmatic (PDL) edges: insert -> sample -> gather is one chain.
        b, n, tot = wl.steps[i]
        if ev:
            ev[0].record(stream)
        if n:
            buf.insert(**b, assume_unique=True)
        buf.sample_device(B, rng)
        buf.gather(packed_tok, None, off)
        if ev:
            ev[1].record(stream)
        # --- synthetic trainer stand-in (not part of the replay step)
        standin(i)
        if ev:
            ev[2].record(stream)
        buf.loss_grpo(lpn, dlogp, EPS_LOW, EPS_HIGH, stats=stats) if cfg["loss"] == "grpo" else \
            buf.loss_asymre(lpn, dlogp, DELTA_V, stats=stats)
        if world > 1:  # one collective: the registered {objective_sum, included, excluded}
            if comm:
                buf.allreduce_loss_stats(comm, dlogp, stats)
            else:
                if dist is not None:  # gloo (CPU tests)
                    dist.all_reduce(red3)
                else:  # emulated rank 0: the sum over N ranks alike (the collective's result)
                    red3.mul_(world)
                buf.loss_finalize_vec(dlogp, red3, stats)
        if ev:
            ev[3].record(stream)

    for i in range(Wm):
        step(i)
    buf.check()
    torch.cuda.synchronize()
    use_graph = args.graph and dist is None  # one process (N = 1, or an emulated rank)
    phase_events = not use_graph or getattr(args, "phases", False)
    evs = [[torch.cuda.Event(enable_timing=True, external=use_graph) for _ in range(4)]
           for _ in range(K)] if phase_events else [None] * K
    graph = None
    if use_graph:
        # The K timed steps (each with its own inbound batch) are captured once
        # and launched once: no host launch overhead inside the timed region.
        # Without per-phase events inside the graph the step time is the
        # graph's time minus that of a second graph holding the same K
        # trainer stand-ins alone (the stand-in is not part of the step).
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream, capture_error_mode="relaxed"):
            for i in range(K):
                step(Wm + i, evs[i])
        g_standin = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_standin, stream=stream, capture_error_mode="relaxed"):
            for i in range(K):
                standin(Wm + i)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    if getattr(args, "pre_timed", None):  # tools/timeline.py hook
        args.pre_timed()
    e_all = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    with Clocks(torch.cuda.current_device()) as clk:
        t0 = time.perf_counter()
        e_all[0].record(stream)
        if graph is not None:
            graph.replay()
        else:
            for i in range(K):
                step(Wm + i, evs[i])
        e_all[1].record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    if graph is not None:
        e_all[2].record(stream)
        g_standin.replay()
        e_all[3].record(stream)
        torch.cuda.synchronize()
    # Parity of the timed run against the CPU oracle (outside the timed region)
    check = None
    if getattr(args, "check", True):
        torch.cuda.synchronize()
        check = parity_check(cfg, wl, Wm + K, buf, rank, world, packed_tok, lpn, dlogp, stats,
                             owned=owned)
        if dist is not None:
            ok = torch.tensor([1 if check["parity"] == "ok" else 0], dtype=torch.int32, device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok) == 0 and check["parity"] == "ok":
                check["parity"] = "MISMATCH on another rank"
    # Dominant kernel timed alone (roofline.achieved): loss launches on the
    # last batch, each bracketed by CUDA events on the launching stream, with
    # a 256 MB read between launches so no launch starts with the previous
    # one's data in the 126 MB L2 (a read leaves no dirty lines to write back).
    n_kern = min(K, 50)
    lossf = (lambda: buf.loss_grpo(lpn, dlogp, EPS_LOW, EPS_HIGH, stats=stats)) \
        if cfg["loss"] == "grpo" else (lambda: buf.loss_asymre(lpn, dlogp, DELTA_V, stats=stats))
    flush = torch.ones(64 << 20, dtype=torch.float32, device=dev)
    flush_out = torch.empty((), dtype=torch.float32, device=dev)
    lossf()
    torch.cuda.synchronize()
    e_k = [[torch.cuda.Event(enable_timing=True, external=graph is not None) for _ in range(2)]
           for _ in range(n_kern)]

    def kernel_loop():
        for i in range(n_kern):
            torch.sum(flush, dim=0, out=flush_out)
            e_k[i][0].record(stream)
            lossf()
            e_k[i][1].record(stream)

    if graph is not None:
        g_loss = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_loss, stream=stream, capture_error_mode="relaxed"):
            kernel_loop()
        torch.cuda.synchronize()
        g_loss.replay()
    else:
        kernel_loop()
    torch.cuda.synchronize()
    loss_kernel_ms = float(np.mean([a.elapsed_time(b) for a, b in e_k]))
    del flush
    if dist is not None:
        dist.barrier()
    buf.check()
    total_ms = e_all[0].elapsed_time(e_all[1])
    if phase_events:
        ph = np.array([[evs[i][j].elapsed_time(evs[i][j + 1]) for j in range(3)] for i in range(K)])
        # phases: insert+sample+gather, stand-in, loss  (ms)
        mean = {k: float(ph[:, j].mean())
                for j, k in enumerate(["insert_sample_gather", "standin", "loss"])}
    if graph is not None and not phase_events:
        standin_ms = e_all[2].elapsed_time(e_all[3]) / K
        ms = total_ms / K - standin_ms
        mean = {"step": ms, "standin": standin_ms,
                "method": "graph(K steps) - graph(K stand-ins), CUDA events on the stream"}
    else:
        ms = float(ph[:, [0, 2]].sum(1).mean())
    if dist is not None:
        t = torch.tensor([ms, wall], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, wall = float(t[0]), float(t[1])
    # token / byte accounting (global)
    t_samp = B * cfg["lmax"] if not cfg["ragged"] else None
    if t_samp is None:
        t_samp = buf.batch_total_tokens() * T
    ins = [wl.steps[Wm + i] for i in range(K)]
    R = float(np.mean([x[1] for x in ins]))
    T_ins = float(np.mean([x[2] for x in ins]))
    alg = algorithmic_bytes(T_ins, t_samp, R, B, cfg["loss"])
    hbm, peak_kind = peaks()
    value = t_samp / (ms * 1e-3)
    # dominant kernel: the loss (12 B/token GRPO: logp_old, logp_now read + dlogp write)
    loss_bytes = (12 if cfg["loss"] == "grpo" else 8) * (t_samp / T)
    roof = {"bound": "hbm", "kernel": "k_loss_grpo_buf" if cfg["loss"] == "grpo" else "k_loss_asymre_buf",
            "achieved": loss_bytes / (loss_kernel_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
            "kernel_ms": loss_kernel_ms, "algorithmic_bytes_per_launch": loss_bytes,
            "timing": f"{n_kern} launches on the last batch, events around each, 256 MB read between",
            "peak_kind": peak_kind}
    roof["frac"] = roof["achieved"] / hbm
    roof["traffic"] = load_traffic(roof["kernel"])
    roof["step"] = {"algorithmic_bytes": alg / T, "achieved_gbs": alg / T / (ms * 1e-3) / 1e9,
                    "frac": alg / T / (ms * 1e-3) / 1e9 / hbm}
    res = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": K,
        "warmup": Wm, "ms_per_step": ms, "higher_is_better": True, "scaling": cfg["scaling"],
        "vs_baseline": None, "dtype": "fp32", "data": "synthetic (include/replay_synth.h)",
        "config": config_dict(cfg, world),
        "accounting": {"inserted_per_step": R, "sampled_tokens_per_step": t_samp,
                       "algorithmic_bytes_per_step": alg},
        "phases_ms": mean, "step_excludes": "synthetic trainer stand-in (logp_now), phases_ms.standin",
        "wall_ms_per_step_incl_standin": wall * 1e3 / K,
        "roofline": roof,
        "gpu_launches": launches_per_step(cfg, world) * K,
        "gpu_launches_per_step": launches_per_step(cfg, world),
        "launch_mode": "cuda_graph (K steps captured once, launched once)" if use_graph else "eager",
        "clocks": clk.summary(),
    }
    if check is not None:
        res["parity"] = check.pop("parity")
        res["parity_check"] = dict(check, method="last timed step vs the CPU oracle replaying the "
                                                  "whole schedule (oracle/replay_oracle.c)")
    return res, buf, wl, rng


def parity_check(cfg, wl, nsteps, buf, rank, world, packed_tok, lpn, dlogp, stats, owned=False):
    """Outside the timed region: replay the whole schedule (warm-up fill + every
    warm-up and timed step) through the CPU oracle (oracle/, the checker) and
    compare the LAST step's sampled trajectories, packed offsets and tokens,
    dL/dlogp (rtol 1e-5, the north star's tolerance) and objective, plus the
    final shard contents (ids, use counts, frozen advantages) of every shard
    (replay_buffer.cpp:83-217, bandit.cpp:276-294, 363-438)."""
    import torch

    from oracle.pyoracle import RECORD_DTYPE, Oracle, same_records

    t0 = time.perf_counter()
    ora = Oracle()
    T, N, B, G = world, cfg["capacity"], cfg["batch"], cfg["group"]
    ob = ora.buffer(T, N, cfg.get("strategy", "uniform_with_replacement"), cfg["retention"],
                    cfg["delta"])
    if cfg.get("priority"):
        ob.set_priority(*cfg["priority"])
    orng = ora.rng(SEED).stream("buffer_sampling")
    gmean_of = {}

    def push_batch(b, n):
        if not n:
            return
        h = {k: v.cpu().numpy() for k, v in b.items() if k not in ("tokens", "logp_old")}
        rec = np.zeros(n, RECORD_DTYPE)
        for k in ("rollout_id", "prompt_id", "group_id", "creation_step", "policy_version",
                  "reward", "behavior_logprob"):
            rec[k] = h[k]
        rec["is_correct"] = h["reward"] == 1.0
        rw = h["reward"].reshape(-1, G)
        m = np.zeros(rw.shape[0])
        for k in range(G):  # bandit.cpp:316-318, the sequential sum
            m += rw[:, k]
        m /= G
        for gi in range(n // G):
            rec["advantage"][gi * G:(gi + 1) * G] = ora.group_advantages(rw[gi])
        for i, r in enumerate(rec):
            gmean_of[int(r["rollout_id"])] = m[i // G]
            ob.push(r)

    full = wl.full if owned else wl.batches  # the oracle replays the global batches
    push_batch(full[0][0], full[0][1])
    orec = None
    for i in range(nsteps):
        b, n, _ = full[1 + i]
        push_batch(b, n)
        orec, _, _ = ob.sample(B, orng)
    per = B // T
    own = orec[rank * per:(rank + 1) * per]
    ids, lens, off = buf.batch_ids()
    res = {"checked_step": nsteps - 1, "shards_checked": 1 if owned else T}
    bad = []
    if not np.array_equal(ids, own["rollout_id"]):
        bad.append("sampled ids")
    _, want_len, _ = ora.synth_meta(SEED, own["rollout_id"], cfg["lmax"], cfg["ragged"])
    want_off = np.zeros(per + 1, np.int64)
    np.cumsum(want_len.astype(np.int64), out=want_off[1:])
    if not np.array_equal(off, want_off):
        bad.append("packed offsets")
    tot = int(want_off[-1])
    tok_want, lpo_want, _ = ora.synth_payload(SEED, own["rollout_id"], want_len)
    if not np.array_equal(packed_tok[:tot].cpu().numpy(), tok_want):
        bad.append("packed tokens")
    lpn_h = lpn[:tot].cpu().numpy()
    if not np.array_equal(lpn_h, ora.synth_logp_now(SEED, nsteps, own["rollout_id"], want_off)):
        bad.append("trainer stand-in logp_now")
    got = dlogp[:tot].cpu().numpy()
    st = stats.cpu()
    obj = float(st[1])
    if cfg["loss"] == "grpo":
        d_want, obj_want, inc, exc = ora.loss_grpo_tokens(lpn_h, lpo_want, own["advantage"],
                                                          want_off, EPS_LOW, EPS_HIGH)
        sti = st.view(torch.int64)
        if world > 1:  # the per-rank oracle call normalises by this rank's included tokens
            d_want = (d_want.astype(np.float64) * (inc / float(sti[2]))).astype(np.float32)
        res["included"], res["excluded"] = int(sti[2]), int(sti[3])
        if world == 1 and (res["included"], res["excluded"]) != (inc, exc):
            bad.append("included/excluded counts")
    else:
        gm = np.array([gmean_of[int(i)] for i in own["rollout_id"]])
        d_want, obj_want = ora.loss_asymre_tokens(lpn_h, own["reward"], gm, want_off, DELTA_V)
        if world > 1:
            d_want = d_want / np.float32(world)
    denom = np.maximum(np.abs(d_want), 1e-30)
    rel = float(np.max(np.abs(got - d_want) / denom)) if tot else 0.0
    res["dlogp_max_rel_err"] = rel
    if not np.allclose(got, d_want, rtol=1e-5, atol=1e-12):
        bad.append("dlogp")
    if world == 1:
        res["objective_rel_err"] = abs(obj - obj_want) / max(1.0, abs(obj_want))
        if res["objective_rel_err"] > 1e-5:
            bad.append("objective")
    for s in ([rank] if owned else range(T)):  # an owned-metadata rank holds its shard only
        if not same_records(buf.shard_contents(s), ob.shard_contents(s)):
            bad.append(f"shard {s} contents")
    res["parity"] = "ok" if not bad else "MISMATCH: " + ", ".join(bad)
    res["tokens_checked"] = tot
    res["oracle_s"] = round(time.perf_counter() - t0, 1)
    return res


def launches_per_step(cfg, world):
    """Library kernels of one timed step (the stand-in's kernels are not counted):
    FIFO (ids promised unique): k_route_fifo, k_insert_payload_tma, k_sample_fused,
    k_gather, loss; positive bias (ids promised unique): k_posbias_par,
    k_insert_payload, k_sample_fused, k_gather, loss; + k_finalize_vec
    (rb_loss_finalize_vec / rb_allreduce_loss_stats, whose NCCL kernel is not
    ours) per step on more than one rank; + k_ring_lookahead above 8192 draws
    per call.  priority_with_replacement: k_sample_prio + k_sample_map in place
    of k_sample_fused (and no ring lookahead)."""
    if cfg.get("strategy") == "priority_with_replacement":
        return 6 + (1 if world > 1 else 0)
    n = 5
    return n + (1 if world > 1 else 0) + (1 if cfg["batch"] > 8192 else 0)


def load_traffic(kernel):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(p)).get(kernel)
    except Exception:
        return None


def run_e2e(args, buf, wl, rng, cfg, world=1, dist=None, rank=0):
    """Same metric through the C-ABI with HOST (pinned) buffers, copies timed."""
    import torch

    import paper_2604_08706_b200 as rb  # noqa: F401

    B = cfg["batch"]
    nloc = B // world  # selections held by this rank
    K = min(args.steps, 8)
    steps = wl.steps[-K:] if len(wl.steps) >= K else wl.steps
    host = []
    for b, n, tot in steps:
        hb = {k: (v.cpu().pin_memory() if hasattr(v, "cpu") else v) for k, v in b.items()}
        host.append((hb, n, tot))
    pad = B * cfg["lmax"] + 8  # upper bound (ragged batches differ per step)
    # the dlogp download of step i drains while step i+1's insert uploads
    # (the other PCIe direction); every step's copies complete inside the
    # timed region (device-wide synchronise at its end)
    buf.set_async_outputs(True)
    tok_h = torch.empty(pad, dtype=torch.int32).pin_memory()
    off_h = torch.empty(B + 1, dtype=torch.int64).pin_memory()
    dl_h = torch.empty(pad, dtype=torch.float32).pin_memory()
    # logp_now from the host: the stand-in's output for the current batch,
    # produced once (untimed) and re-used; its values do not change the work.
    lpn_h = torch.empty(pad, dtype=torch.float32).pin_memory()
    buf.sample_device(B, rng)
    buf.gather(tok_h, None, off_h)
    ids = torch.empty(nloc, dtype=torch.int64, device="cuda")
    offd = off_h[:nloc + 1].cuda()
    lpn_d = torch.empty(pad, dtype=torch.float32, device="cuda")
    from tools import synth

    buf.batch_ids_device(ids)
    synth.logp_now(SEED, 99, ids, offd, lpn_d, buf.stream())
    torch.cuda.synchronize()
    lpn_h.copy_(lpn_d.cpu())
    # re-insert the same inbound batches needs fresh ids: shift them (pinned,
    # prepared outside the timed region like every other host input)
    shift = 10**12
    plan = []
    for r in range(2):  # r = 0: warm-up pass (staging buffers are allocated once)
        for j, (hb, n, tot) in enumerate(host):
            hb2 = dict(hb)
            hb2["rollout_id"] = (hb["rollout_id"] + shift * (1 + r * len(host) + j)).pin_memory()
            plan.append((r, hb2, n))

    def e2e_step(hb2, n):
        if n:
            buf.insert(**hb2, assume_unique=True)  # ids new and increasing, as on the device path
        buf.sample_device(B, rng)
        buf.gather(tok_h, None, off_h)
        st = buf.loss_grpo(lpn_h, dl_h, EPS_LOW, EPS_HIGH) if cfg["loss"] == "grpo" else \
            buf.loss_asymre(lpn_h, dl_h, DELTA_V)
        _ = st.objective  # device->host read of the step's result
        return int(off_h[nloc])  # this rank's sampled tokens (offsets already on the host)

    for r, hb2, n in plan:
        if r == 0:
            e2e_step(hb2, n)
    # bytes that cross PCIe per insert: every column, and of the token
    # payload only this rank's records' ranges (round-robin from the cursor)
    cursor = buf.route_cursor()
    T = buf.num_shards()

    def h2d_insert(hb2, n, c0):
        meta = sum(v.numel() * v.element_size() for k, v in hb2.items()
                   if hasattr(v, "numel") and k not in ("tokens", "logp_old"))
        toff = hb2["tok_offsets"].numpy()
        lens = np.diff(toff)
        if "n_global" in hb2:  # an owned batch holds this rank's records only
            return meta + int(lens.sum()) * 8
        own = ((c0 + np.arange(n)) % T) == rank if T > 1 else np.ones(n, bool)
        return meta + int(lens[own].sum()) * 8

    h2d = d2h = 0
    done_tokens = 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for r, hb2, n in plan:
        if r == 0:
            continue
        tot_s = e2e_step(hb2, n)
        done_tokens += tot_s
        h2d += (h2d_insert(hb2, n, cursor) if n else 0) + tot_s * 4
        cursor = (cursor + n) % T
        d2h += tot_s * 4 * 2 + (B + 1) * 8 + 40
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / len(host)
    buf.set_async_outputs(False)
    if world > 1:  # whole job: tokens of every rank over the slowest rank's time
        if dist is not None:  # device tensors: NCCL reduces CUDA memory only
            t = torch.tensor([float(done_tokens), dt], dtype=torch.float64, device="cuda")
            dist.all_reduce(t[0:1])
            dist.all_reduce(t[1:2], op=dist.ReduceOp.MAX)
            done_tokens, dt = float(t[0]), float(t[1])
        else:  # emulated rank 0: every rank alike
            done_tokens *= world
        h2d, d2h = h2d * world, d2h * world
    return {"value": done_tokens / len(host) / dt, "unit": "tokens/s", "ms_per_step": dt * 1e3,
            "h2d_bytes_per_step": h2d // len(host), "d2h_bytes_per_step": d2h // len(host),
            "steps": len(host), "path": "rb_insert/rb_sample/rb_gather/rb_loss_* with pinned host "
                                        "buffers (copies inside the timed region; the loss "
                                        "pipelines its upload/download in chunks; its dlogp "
                                        "download overlaps the next step's insert upload, "
                                        "rb_set_async_outputs)"}


# ---------------------------------------------------------------- C5 sweep
C5_W = (1, 2, 4, 8)
C5_T = (1, 2, 4)
C5_N = (84, 756, 4092)


def c5_cpu(T, N, W, steps):
    import ctypes as C

    from oracle.pyoracle import REF_SO

    L = C.CDLL(REF_SO)
    L.ref_c5_run.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_double, C.c_uint64,
                             C.c_uint64, C.c_int, C.c_double, C.c_uint64, C.c_int,
                             C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
    sec, rec = C.c_double(), C.c_uint64()
    if L.ref_c5_run(T, N, W, T_TRAINERS, MU, 504, 8, 0, 0.0, SEED, steps, C.byref(sec), C.byref(rec)):
        raise RuntimeError("ref_c5_run failed")
    return rec.value / sec.value


def run_c5(args):
    """Record-level (W,T) sweep: insert (route + eviction + advantages) and
    sample through the library, T shards on one GPU (simulate() semantics,
    async_sim.cpp:138-139), timed as one CUDA graph of K steps; the
    unmodified reference buffer on 1 host core beside it."""
    import torch

    import paper_2604_08706_b200 as rb

    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream()
    B, G = 504, 8
    K = max(args.steps, 20)
    rows = []
    for N in C5_N:
        for T in C5_T:
            for W in C5_W:
                print(f"c5: N={N} T={T} W={W}", file=sys.stderr, flush=True)
                buf = rb.ShardedReplayBuffer(T, N, "uniform_with_replacement", "plain_fifo", 0.0,
                                             max_tokens=0)
                buf.set_stream(stream.cuda_stream)
                rng = rb.Rng(SEED).stream("buffer_sampling")
                per = W * B / (MU * T_TRAINERS)
                nid = [0]

                def batch(ng, step):
                    n = ng * G
                    ids = torch.arange(nid[0], nid[0] + n, dtype=torch.int64, device=dev)
                    nid[0] += n
                    rew = (torch.rand(n, device=dev) < 0.5).to(torch.float64)
                    return dict(rollout_id=ids, reward=rew, group_id=ids // G,
                                creation_step=torch.full((n,), step, dtype=torch.int64, device=dev),
                                group_offsets=torch.arange(0, n + 1, G, dtype=torch.int64, device=dev))

                buf.insert(**batch(-(-N // G), 0), assume_unique=True)
                debt, plan = 0.0, []
                for i in range(K + 3):
                    debt += per
                    ng = int(debt // G)
                    debt -= ng * G
                    plan.append(batch(ng, i + 1) if ng else None)
                ins = sum(int(p["rollout_id"].numel()) for p in plan[3:] if p is not None)

                def step(p):
                    if p is not None:
                        buf.insert(**p, assume_unique=True)
                    buf.sample_device(B, rng)

                for p in plan[:3]:
                    step(p)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream, capture_error_mode="relaxed"):
                    for p in plan[3:]:
                        step(p)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(stream)
                g.replay()
                e1.record(stream)
                torch.cuda.synchronize()
                buf.check()
                ms = e0.elapsed_time(e1) / K
                gpu = (ins + K * B) / (ms * K * 1e-3)
                cpu = None if args.no_cpu_baseline else c5_cpu(T, N, W, 20)
                rows.append({"W": W, "T": T, "N": N, "us_per_step": ms * 1e3,
                             "gpu_records_per_s": gpu, "cpu_records_per_s": cpu,
                             "gpu_over_cpu": gpu / cpu if cpu else None})
                del g, buf
    gm = float(np.exp(np.mean([np.log(r["gpu_records_per_s"]) for r in rows])))
    return {"metric": "C5 eviction+sampling throughput: (inserted+sampled) records/s, geometric "
                      "mean over the sweep", "value": gm, "unit": "records/s", "n_gpus": 1,
            "steps": K, "warmup": 3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": CONFIGS["c5"]["name"], "W": C5_W, "T": C5_T, "N": C5_N,
                       "B": B, "G": G, "mu": MU},
            "cpu_baseline": {"kind": "reference", "cores": 1,
                             "sample": "20 steps of the same schedule through the unmodified "
                                       "replab ShardedReplayBuffer per configuration"},
            "sweep": rows}


# ---------------------------------------------------------------- CPU arm
def cpu_reference(cfg, steps, warmup, threads=0, budget_s=90.0, shards=1):
    """The reference's CPU path (oracle/_ref: unmodified replab buffer/sampler/
    group_advantages + restated token loss) on the host cores."""
    import ctypes as C

    from oracle.pyoracle import REF_SO, RECORD_DTYPE, Oracle

    if not os.path.exists(REF_SO):
        from oracle.pyoracle import build_oracle

        build_oracle(with_ref=True)
    L = C.CDLL(REF_SO)
    vp = C.c_void_p
    L.ref_bench_new.restype = vp
    L.ref_bench_new.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_double, C.c_int,
                                C.c_uint64, C.c_int]
    L.ref_bench_free.argtypes = [vp]
    L.ref_bench_threads.argtypes = [vp]
    L.ref_bench_phase_a.argtypes = [vp, C.c_uint64, C.c_uint64, vp, vp, vp, vp, C.c_uint64, vp, vp, vp]
    L.ref_bench_phase_b.argtypes = [vp, vp, C.c_double, C.c_double, vp, vp, vp, vp]
    L.ref_last_error.restype = C.c_char_p
    ora = Oracle()
    h = L.ref_bench_new(shards, cfg["capacity"], 0, 1 if cfg["retention"] == "positive_bias" else 0,
                        cfg["delta"], cfg["lmax"], SEED, threads)
    if not h:
        raise RuntimeError(L.ref_last_error().decode())
    nthreads = L.ref_bench_threads(h)
    g = cfg["group"]
    warm, per_step = schedule(cfg, steps + warmup)
    nid = [0]
    ngid = [0]

    def make(ngroups, step):
        n = ngroups * g
        ids = np.arange(nid[0], nid[0] + n, dtype=np.uint64)
        reward, length, blp = ora.synth_meta(SEED, ids, cfg["lmax"], cfg["ragged"])
        tok, lpo, toff = ora.synth_payload(SEED, ids, length)
        rec = np.zeros(n, RECORD_DTYPE)
        rec["rollout_id"] = ids
        rec["group_id"] = np.repeat(np.arange(ngid[0], ngid[0] + ngroups), g)
        rec["prompt_id"] = rec["group_id"] % (cfg["batch"] // g)
        rec["creation_step"] = step
        rec["policy_version"] = step
        rec["reward"] = reward
        rec["is_correct"] = reward == 1.0
        rec["behavior_logprob"] = blp
        nid[0] += n
        ngid[0] += ngroups
        return rec, toff, tok, lpo

    B = cfg["batch"]
    maxtok = B * cfg["lmax"]
    out_ids = np.zeros(B, np.uint64)
    out_tok = np.zeros(maxtok, np.int32)
    out_off = np.zeros(B + 1, np.int64)
    dl = np.zeros(maxtok, np.float32)
    obj, inc, exc = C.c_double(), C.c_int64(), C.c_int64()

    def phase_a(rec, toff, tok, lpo):
        st = L.ref_bench_phase_a(h, rec.shape[0], g, rec.ctypes.data, toff.ctypes.data,
                                 tok.ctypes.data, lpo.ctypes.data, B, out_ids.ctypes.data,
                                 out_tok.ctypes.data, out_off.ctypes.data)
        if st:
            raise RuntimeError(L.ref_last_error().decode())

    rec, toff, tok, lpo = make(warm, 0)
    phase_a(rec, toff, tok, lpo)
    times = []
    spent = 0.0
    for i, n_i in enumerate(per_step):
        # inputs made untimed, one step at a time; the timed steps stop once
        # `budget_s` of timed work is done (a bounded sample of the run)
        if i >= warmup and times and spent >= budget_s:
            break
        rec, toff, tok, lpo = make(n_i, i)
        t0 = time.perf_counter()
        phase_a(rec, toff, tok, lpo)
        ta = time.perf_counter() - t0
        lpn = ora.synth_logp_now(SEED, i + 1, out_ids, out_off)  # stand-in, untimed
        t1 = time.perf_counter()
        st = L.ref_bench_phase_b(h, lpn.ctypes.data, EPS_LOW, EPS_HIGH, dl.ctypes.data,
                                 C.byref(obj), C.byref(inc), C.byref(exc))
        tb = time.perf_counter() - t1
        if st:
            raise RuntimeError(L.ref_last_error().decode())
        if i >= warmup:
            times.append(ta + tb)
            spent += ta + tb
    L.ref_bench_free(h)
    tok_per_step = int(out_off[-1])
    mean = float(np.mean(times))
    return {"value": tok_per_step / mean, "unit": "tokens/s", "cores": nthreads,
            "ms_per_step": mean * 1e3, "steps": len(times),
            "cpu": cpu_model()}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--no-check", dest="check", action="store_false",
                    help="skip the parity check of the last timed step against the CPU oracle")
    ap.add_argument("--eager", dest="graph", action="store_false",
                    help="launch the timed steps eagerly instead of from a CUDA graph")
    ap.add_argument("--phases", action="store_true",
                    help="record CUDA events at the phase boundaries (front end | stand-in | "
                         "loss) inside the graph; the step is the sum of the front end and loss")
    ap.add_argument("--owned", action="store_true",
                    help="N > 1: each rank receives and routes only its own shard's records "
                         "(rb_set_owned_metadata / rb_insert_owned) instead of the whole batch")
    ap.add_argument("--weak", action="store_true",
                    help="N > 1: weak scaling (N x the single-GPU buffer and batch) instead of "
                         "splitting the single-GPU workload over the N GPUs")
    ap.add_argument("--emulate-world", type=int, default=0,
                    help="diagnostic: run rank 0 of an N-GPU job alone on one GPU (no "
                         "collective); the line predicts the N-GPU step")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    emulated = args.emulate_world > 1 and world == 1
    if emulated:
        world = args.emulate_world
    cfg = scaled_cfg(CONFIGS[args.config], world, args.weak)

    if args.impl == "reference":
        if rank != 0:
            return
        if cfg.get("strategy", "uniform_with_replacement") == "priority_with_replacement":
            print(json.dumps({"impl": "reference", "unavailable": "the reference has no "
                              "prioritised sampler (replay_buffer.cpp:135-182 is uniform)"}))
            return
        # bounded sample of the same job's steps (at most ~90 s of timed
        # steps); N shards for an N-GPU job, like our arm
        r = cpu_reference(cfg, args.steps, args.warmup, shards=world)
        line = {"metric": METRIC, "value": r["value"], "unit": "tokens/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
                "higher_is_better": True, "scaling": cfg["scaling"], "vs_baseline": None,
                "dtype": "fp32", "data": "synthetic (include/replay_synth.h)", "impl": "reference",
                "config": config_dict(cfg, world),
                "cpu_baseline": {"value": r["value"], "unit": "tokens/s", "cores": r["cores"],
                                 "kind": "reference",
                                 "sample": f"{r['steps']} {args.config.upper()} replay steps of "
                                           f"the same job ({r['cpu']}), {world} shard(s); record "
                                           "ops through the unmodified replab library, token "
                                           "payload/gather/loss restated"},
                "e2e": {"value": r["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch

    # RB_BENCH_SAME_GPU=1 (test aid): every rank on cuda:0 with gloo, to
    # exercise the sharded path on a one-GPU box (not a performance number)
    same_gpu = os.environ.get("RB_BENCH_SAME_GPU") == "1"
    if same_gpu:
        local = 0
    torch.cuda.set_device(local)
    if args.config == "c5":  # record-level sweep (one GPU; not the headline metric)
        if rank == 0:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                print(json.dumps(run_c5(args)), flush=True)
        return
    dist = None
    if world > 1 and not emulated:
        import torch.distributed as dist

        if same_gpu:
            dist.init_process_group("gloo")
        else:
            # NCCL's own log (stderr) shows nranks / the NVLink(S) transport
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()  # a real stream handle (not the legacy default)
    with torch.cuda.stream(stream):
        res, buf, wl, rng = run_ours(args, rank, world, dist)
        if not args.no_e2e and getattr(wl, "owned", False):
            res["e2e"] = {"skipped": "--owned: the replayed batches' shard positions change with "
                                     "the cursor; run without --owned for the e2e figure"}
        elif not args.no_e2e:
            res["e2e"] = run_e2e(args, buf, wl, rng, cfg, world, dist, rank)
    if emulated:
        res["emulated"] = (f"rank 0 of a {world}-GPU job alone on one GPU, no collective: "
                           "a prediction of the N-GPU step, not a measurement")
    if (rank == 0 and world == 1 and not args.no_cpu_baseline
            and cfg.get("strategy", "uniform_with_replacement") != "priority_with_replacement"):
        try:
            r = cpu_reference(cfg, args.cpu_steps, 1)
            res["cpu_baseline"] = {"value": r["value"], "unit": "tokens/s", "cores": r["cores"],
                                   "kind": "reference",
                                   "sample": f"{r['steps']} full {args.config.upper()} replay steps "
                                             f"after 1 warm-up ({r['cpu']})"}
        except Exception as e:  # noqa: BLE001
            res["cpu_baseline"] = {"value": None, "unavailable": str(e)[:200]}
    if rank == 0:
        print(json.dumps(res), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
