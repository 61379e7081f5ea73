"""World-size-2 run of the CUDA replay step with one buffer shard per rank
(DESIGN.md §6), both ranks on cuda:0 and gloo for the 24-byte loss
all-reduce (the only collective of the path): every rank replicates the
metadata of all shards and regenerates the same MT19937-64 stream, owns the
payload of its shard, gathers and evaluates its own selections, all-reduces
{objective_sum, included, excluded} and finalises dlogp.  Checked against
the single-process CPU oracle: sampled records, the owned packed tokens, the
globally normalised dlogp and the objective.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.harness import Producer, StepConfig

pytestmark = pytest.mark.gpu

CASES = {
    "fifo_unique": dict(capacity=128, shards=2, batch=32, group=8, lmax=40, ragged=True, seed=31,
                        assume_unique=True),
    "posbias": dict(capacity=96, shards=2, batch=32, group=8, lmax=24, ragged=True, seed=32,
                    retention="positive_bias", delta=0.5),
}
STEPS = 6


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(rank, world, port, case, q, one_collective=False):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        vec3 = torch.zeros(3, dtype=torch.float64, device="cuda:0")
        from oracle.pyoracle import Oracle, same_records
        from paper_2604_08706_b200 import Rng, ShardedReplayBuffer

        cfg = StepConfig(**CASES[case])
        ora = Oracle()
        obuf = ora.buffer(cfg.shards, cfg.capacity, cfg.strategy, cfg.retention, cfg.delta)
        orng = ora.rng(cfg.seed).stream("buffer_sampling")
        gbuf = ShardedReplayBuffer(cfg.shards, cfg.capacity, cfg.strategy, cfg.retention,
                                   cfg.delta, max_tokens=cfg.lmax, shard_range=(rank, rank + 1))
        # the library on torch's stream: the inputs torch copies to the device
        # are ordered before the kernels that read them
        gbuf.set_stream(torch.cuda.current_stream().cuda_stream)
        grng = Rng(cfg.seed).stream("buffer_sampling")
        prod = Producer(cfg, ora)
        lengths = {}
        dev = "cuda:0"

        def push(ng, step):
            rec, length, tok, lpo, toff, _ = prod.groups(ng, step)
            for r, L in zip(rec, length):
                lengths[int(r["rollout_id"])] = int(L)
                obuf.push(r)
            n = rec.shape[0]
            t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
            gbuf.insert(rollout_id=t(rec["rollout_id"].copy()), prompt_id=t(rec["prompt_id"].copy()),
                        group_id=t(rec["group_id"].copy()),
                        creation_step=t(rec["creation_step"].copy()),
                        policy_version=t(rec["policy_version"].copy()),
                        reward=t(rec["reward"].copy()),
                        behavior_logprob=t(rec["behavior_logprob"].copy()),
                        group_offsets=t(np.arange(0, n + 1, cfg.group, dtype=np.int64)),
                        tok_offsets=t(toff), tokens=t(tok), logp_old=t(lpo),
                        assume_unique=cfg.assume_unique)

        while obuf.size() < cfg.capacity:
            push(1, 0)
        per = cfg.batch // cfg.shards
        lo, hi = rank * per, (rank + 1) * per
        debt = 0.0
        for step in range(STEPS):
            debt += cfg.per_step
            ng = int(debt // cfg.group)
            debt -= ng * cfg.group
            if ng:
                push(ng, step)
            grec = gbuf.sample(cfg.batch, grng)
            orec, _, _ = obuf.sample(cfg.batch, orng)
            if not same_records(grec, orec):
                diffs = [f for f in orec.dtype.names if not np.array_equal(grec[f], orec[f])]
                i = int(np.argmax(grec[diffs[0]] != orec[diffs[0]])) if diffs else -1
                raise AssertionError(f"rank {rank}: sampled records, step {step}: fields {diffs}, "
                                     f"first at {i}: got {grec[i]} want {orec[i]}")
            # owned selections: packed tokens
            ids = orec["rollout_id"][lo:hi]
            lens = np.array([lengths[int(i)] for i in ids], np.int64)
            off = np.zeros(per + 1, np.int64)
            np.cumsum(lens, out=off[1:])
            tot = int(off[-1])
            tok_want, lpo_want, _ = ora.synth_payload(cfg.seed, ids, lens)
            pad = (tot + 3) // 4 * 4 + 4
            gt = torch.zeros(pad, dtype=torch.int32, device=dev)
            go = torch.zeros(per + 1, dtype=torch.int64, device=dev)
            torch.cuda.synchronize()
            gbuf.gather(gt, None, go)
            gbuf.synchronize()
            assert np.array_equal(go.cpu().numpy(), off), f"rank {rank}: offsets, step {step}"
            assert np.array_equal(gt[:tot].cpu().numpy(), tok_want), f"rank {rank}: tokens, step {step}"
            # loss: the whole batch's token loss (oracle), this rank's slice of it
            all_ids = orec["rollout_id"]
            all_lens = np.array([lengths[int(i)] for i in all_ids], np.int64)
            aoff = np.zeros(cfg.batch + 1, np.int64)
            np.cumsum(all_lens, out=aoff[1:])
            lpn_all = ora.synth_logp_now(cfg.seed, step + 1, all_ids, aoff)
            if step % 2 == 1:  # the same excluded tokens on every rank (one per shard)
                for r0 in range(cfg.shards):
                    if aoff[(r0 + 1) * per] > aoff[r0 * per] + 1:
                        lpn_all[aoff[r0 * per] + 1] = np.float32(np.inf)
            _, lpo_all, _ = ora.synth_payload(cfg.seed, all_ids, all_lens)
            d_want, obj, inc, exc = ora.loss_grpo_tokens(lpn_all, lpo_all, orec["advantage"], aoff,
                                                         cfg.eps_low, cfg.eps_high)
            lpn = torch.zeros(pad, dtype=torch.float32, device=dev)
            lpn[:tot] = torch.from_numpy(lpn_all[aoff[lo]:aoff[hi]])
            dl = torch.zeros(pad, dtype=torch.float32, device=dev)
            stats = torch.zeros(5, dtype=torch.float64, device=dev)
            torch.cuda.synchronize()
            if one_collective:  # the registered reduce vector, one all-reduce
                gbuf.loss_set_reduce_vector(vec3)
                gbuf.loss_grpo(lpn, dl, cfg.eps_low, cfg.eps_high, stats=stats)
                gbuf.synchronize()
                red = vec3.cpu()
                dist.all_reduce(red)
                vec3.copy_(red.to(dev))
                torch.cuda.synchronize()
                gbuf.loss_finalize_vec(dl, vec3, stats)
                gbuf.synchronize()
                host = stats.cpu()
                s_obj = host[0:1].clone()
                s_cnt = host[2:4].clone().view(torch.int64)
            else:
                gbuf.loss_grpo(lpn, dl, cfg.eps_low, cfg.eps_high, stats=stats)
                gbuf.synchronize()
                host = stats.cpu()
                s_obj = host[0:1].clone()
                s_cnt = host[2:4].clone().view(torch.int64)
                dist.all_reduce(s_obj)
                dist.all_reduce(s_cnt)
                host[0:1] = s_obj
                host[2:4] = s_cnt.view(torch.float64)
                stats.copy_(host.to(dev))
                torch.cuda.synchronize()  # torch's stream wrote the reduced stats
                gbuf.loss_finalize(dl, stats)
                gbuf.synchronize()
            got = dl[:tot].cpu().numpy()
            np.testing.assert_allclose(got, d_want[aoff[lo]:aoff[hi]], rtol=1e-5, atol=1e-12,
                                       err_msg=f"rank {rank}: dlogp, step {step}")
            inc_got, exc_got = (int(x) for x in s_cnt)
            assert (inc_got, exc_got) == (inc, exc), (rank, step, inc_got, exc_got, inc, exc)
            assert abs(float(s_obj[0]) / max(inc_got, 1) - obj) <= 1e-5 * max(1.0, abs(obj))
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        import traceback

        q.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("one_collective", [False, True])
@pytest.mark.parametrize("side_lookahead", [False, True])
@pytest.mark.parametrize("case", sorted(CASES))
def test_two_ranks_one_shard_each(case, side_lookahead, one_collective, monkeypatch):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    if side_lookahead:  # every sampling call forks its ring lookahead (inherited by the ranks)
        monkeypatch.setenv("RB_LOOKAHEAD_MIN_DRAWS", "0")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, 2, port, case, q, one_collective))
             for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    bad = {r: m for r, m in res.items() if m != "ok"}
    assert not bad, "\n".join(f"rank {r}:\n{m}" for r, m in sorted(bad.items()))


# ---------------------------------------------------------------- owned metadata
def _run_owned(rank, world, port, q, seed):
    """Each rank holds one shard and receives ONLY the records the round robin
    routes to it (rb_insert_owned, with their advantages); it maps only its
    slice of the draws; the loss is normalised by the all-reduced count."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from oracle.pyoracle import Oracle, same_records
        from paper_2604_08706_b200 import Rng, ShardedReplayBuffer

        cfg = StepConfig(capacity=64 * world, shards=world, batch=16 * world, group=8, lmax=40,
                         ragged=True, seed=seed, assume_unique=True)
        ora = Oracle()
        obuf = ora.buffer(cfg.shards, cfg.capacity, cfg.strategy, cfg.retention, cfg.delta)
        orng = ora.rng(cfg.seed).stream("buffer_sampling")
        gbuf = ShardedReplayBuffer(cfg.shards, cfg.capacity, cfg.strategy, cfg.retention,
                                   cfg.delta, max_tokens=cfg.lmax, shard_range=(rank, rank + 1))
        gbuf.set_stream(torch.cuda.current_stream().cuda_stream)
        gbuf.set_owned_metadata()
        vec3 = torch.zeros(3, dtype=torch.float64, device="cuda:0")
        gbuf.loss_set_reduce_vector(vec3)
        grng = Rng(cfg.seed).stream("buffer_sampling")
        prod = Producer(cfg, ora)
        lengths = {}
        dev = "cuda:0"
        T = cfg.shards
        cursor = [0]

        def push(ng, step):
            rec, length, tok, lpo, toff, _ = prod.groups(ng, step)
            n = rec.shape[0]
            for r, L in zip(rec, length):
                lengths[int(r["rollout_id"])] = int(L)
                obuf.push(r)
            idx = np.array([j for j in range(n) if (cursor[0] + j) % T == rank], np.int64)
            sub = rec[idx]
            sl = length[idx].astype(np.int64)
            soff = np.zeros(len(idx) + 1, np.int64)
            np.cumsum(sl, out=soff[1:])
            stok = np.concatenate([tok[toff[j]:toff[j + 1]] for j in idx] + [np.zeros(0, tok.dtype)])
            slpo = np.concatenate([lpo[toff[j]:toff[j + 1]] for j in idx] + [np.zeros(0, lpo.dtype)])
            t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
            pad = lambda x: np.concatenate([x, np.zeros(4, x.dtype)])  # noqa: E731
            gbuf.insert(rollout_id=t(sub["rollout_id"].copy()), prompt_id=t(sub["prompt_id"].copy()),
                        group_id=t(sub["group_id"].copy()),
                        creation_step=t(sub["creation_step"].copy()),
                        policy_version=t(sub["policy_version"].copy()),
                        reward=t(sub["reward"].copy()),
                        behavior_logprob=t(sub["behavior_logprob"].copy()),
                        advantage=t(sub["advantage"].copy()), tok_offsets=t(soff),
                        tokens=t(pad(stok)), logp_old=t(pad(slpo)), assume_unique=True,
                        n_global=n)
            cursor[0] = (cursor[0] + n) % T

        while obuf.size() < cfg.capacity:
            push(1, 0)
        got, want = gbuf.shard_contents(rank), obuf.shard_contents(rank)
        assert same_records(got, want), (f"rank {rank}: own shard after the fill: "
                                         f"{got['rollout_id'][:8]} vs {want['rollout_id'][:8]}")
        per = cfg.batch // T
        lo, hi = rank * per, (rank + 1) * per
        debt = 0.0
        for step in range(STEPS):
            debt += cfg.per_step
            ng = int(debt // cfg.group)
            debt -= ng * cfg.group
            if ng:
                push(ng, step)
            gbuf.sample_device(cfg.batch, grng)
            orec, _, _ = obuf.sample(cfg.batch, orng)
            gids, glens, goff = gbuf.batch_ids()
            want_ids = orec["rollout_id"][lo:hi]
            bad_i = np.nonzero(gids != want_ids)[0] if gids.shape == want_ids.shape else [-1]
            assert np.array_equal(gids, want_ids), (
                f"rank {rank}: ids, step {step}: {gids.shape} {want_ids.shape} at {bad_i[:4]}: "
                f"{gids[bad_i[:4]] if len(bad_i) and bad_i[0] >= 0 else gids} vs "
                f"{want_ids[bad_i[:4]] if len(bad_i) and bad_i[0] >= 0 else want_ids}")
            ids = orec["rollout_id"][lo:hi]
            lens = np.array([lengths[int(i)] for i in ids], np.int64)
            off = np.zeros(per + 1, np.int64)
            np.cumsum(lens, out=off[1:])
            tot = int(off[-1])
            assert np.array_equal(goff, off), f"rank {rank}: offsets, step {step}"
            tok_want, _, _ = ora.synth_payload(cfg.seed, ids, lens)
            padn = (tot + 3) // 4 * 4 + 4
            gt = torch.zeros(padn, dtype=torch.int32, device=dev)
            torch.cuda.synchronize()
            gbuf.gather(gt, None, None)
            gbuf.synchronize()
            assert np.array_equal(gt[:tot].cpu().numpy(), tok_want), f"rank {rank}: tokens, step {step}"
            all_ids = orec["rollout_id"]
            all_lens = np.array([lengths[int(i)] for i in all_ids], np.int64)
            aoff = np.zeros(cfg.batch + 1, np.int64)
            np.cumsum(all_lens, out=aoff[1:])
            lpn_all = ora.synth_logp_now(cfg.seed, step + 1, all_ids, aoff)
            if step % 2 == 1 and aoff[lo + 1] > aoff[lo] + 1:  # an excluded token on this rank
                lpn_all[aoff[lo] + 1] = np.float32(np.inf)
            # both ranks must see the same exclusions: rank r excludes in its own slice only
            for r0 in range(T):
                if r0 != rank and step % 2 == 1 and aoff[r0 * per + 1] > aoff[r0 * per] + 1:
                    lpn_all[aoff[r0 * per] + 1] = np.float32(np.inf)
            _, lpo_all, _ = ora.synth_payload(cfg.seed, all_ids, all_lens)
            d_want, obj, inc, exc = ora.loss_grpo_tokens(lpn_all, lpo_all, orec["advantage"], aoff,
                                                         cfg.eps_low, cfg.eps_high)
            lpn = torch.zeros(padn, dtype=torch.float32, device=dev)
            lpn[:tot] = torch.from_numpy(lpn_all[aoff[lo]:aoff[hi]])
            dl = torch.zeros(padn, dtype=torch.float32, device=dev)
            stats = torch.zeros(5, dtype=torch.float64, device=dev)
            torch.cuda.synchronize()
            gbuf.loss_grpo(lpn, dl, cfg.eps_low, cfg.eps_high, stats=stats)
            gbuf.synchronize()
            red = vec3.cpu()
            dist.all_reduce(red)
            vec3.copy_(red.to(dev))
            torch.cuda.synchronize()
            gbuf.loss_finalize_vec(dl, vec3, stats)
            gbuf.synchronize()
            got = dl[:tot].cpu().numpy()
            np.testing.assert_allclose(got, d_want[aoff[lo]:aoff[hi]], rtol=1e-5, atol=1e-12,
                                       err_msg=f"rank {rank}: dlogp, step {step}")
            host = stats.cpu()
            inc_got, exc_got = (int(x) for x in host[2:4].clone().view(torch.int64))
            assert (inc_got, exc_got) == (inc, exc), (rank, step, inc_got, exc_got, inc, exc)
            assert abs(float(host[1]) - obj) <= 1e-5 * max(1.0, abs(obj))
        assert same_records(gbuf.shard_contents(rank), obuf.shard_contents(rank)), "own shard"
        q.put((rank, "ok"))
    except Exception:  # noqa: BLE001
        import traceback

        q.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("world,seed", [(2, 41), (3, 42)])
def test_owned_metadata_ranks(world, seed):
    """rb_set_owned_metadata + rb_insert_owned: every rank receives only its
    own records, maps only its slice, and still matches the oracle."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run_owned, args=(r, world, port, q, seed)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    bad = {r: m for r, m in res.items() if m != "ok"}
    assert not bad, "\n".join(f"rank {r}:\n{m}" for r, m in sorted(bad.items()))
