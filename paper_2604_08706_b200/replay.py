"""Python mirror of the reference's replay-path API over the C-ABI.

Names, argument meaning and error behaviour follow the reference's C++ API
(/root/reference/proj/include/replab): ``Rng`` (rng.hpp:22-69),
``ShardedReplayBuffer`` (replay_buffer.hpp:57-108), ``group_advantages``
(bandit.hpp:106) and the two losses (bandit.hpp:133-139, token-level form).
Invalid arguments raise ValueError (the reference's std::invalid_argument).

Arrays may be numpy (host) or torch tensors (host or CUDA); device tensors
stay on the device (the hot path), host arrays are staged by the library.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from ._lib import (GRPO_MODES, RB_INSERT_ASSUME_UNIQUE, RETENTIONS, STRATEGIES, STRATEGY_NAMES,
                   InsertBatch, LossStats, Record, check, lib)

RECORD_DTYPE = np.dtype(
    {
        "names": ["rollout_id", "prompt_id", "group_id", "creation_step", "policy_version",
                  "reward", "is_correct", "behavior_logprob", "advantage", "use_count"],
        "formats": ["<u8", "<u8", "<u8", "<i8", "<i8", "<f8", "u1", "<f8", "<f8", "<u4"],
        "offsets": [0, 8, 16, 24, 32, 40, 48, 56, 64, 72],
        "itemsize": 80,
    }
)
EVENT_DTYPE = np.dtype([("rollout_id", "<u8"), ("creation_step", "<i8"), ("use_step", "<i8"),
                        ("batch_id", "<i8"), ("within_batch_rank", "<i8")])
NONE_ID = np.iinfo(np.uint64).max


def _ptr(a) -> Optional[int]:
    """Raw address of a numpy array or torch tensor (None passes through)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("arrays must be contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensors must be contiguous")
        return a.data_ptr()
    raise TypeError(f"unsupported array type {type(a)}")


def _host(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _arr(a, dtype):
    """Keep torch tensors (any device) as they are; coerce the rest to numpy."""
    if a is None:
        return None
    if hasattr(a, "data_ptr") and not isinstance(a, np.ndarray):
        return a
    return _host(a, dtype)


# ---------------------------------------------------------------------------
class Rng:
    """replab::Rng — MT19937-64 with named sub-streams (rng.hpp:22-69)."""

    def __init__(self, seed: int = 0, _handle=None):
        if _handle is None:
            h = C.c_void_p()
            check(lib.rb_rng_create(int(seed) & (2**64 - 1), C.byref(h)))
            _handle = h
        self._h = _handle

    def __del__(self):
        if getattr(self, "_h", None):
            lib.rb_rng_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def stream(self, name: str, index: Optional[int] = None) -> "Rng":
        h = C.c_void_p()
        if index is None:
            check(lib.rb_rng_stream(self._h, name.encode(), C.byref(h)))
        else:
            check(lib.rb_rng_stream_index(self._h, name.encode(), int(index), C.byref(h)))
        return Rng(_handle=h)

    def copy(self) -> "Rng":
        h = C.c_void_p()
        check(lib.rb_rng_clone(self._h, C.byref(h)))
        return Rng(_handle=h)

    def seed(self) -> int:
        return lib.rb_rng_seed(self._h)

    @property
    def draws(self) -> int:
        return lib.rb_rng_draws(self._h)

    def get_state(self):
        """(312 uint64 words, next index, outputs consumed) — a checkpoint."""
        mt = np.zeros(312, np.uint64)
        idx, dr = C.c_uint32(), C.c_uint64()
        check(lib.rb_rng_get_state(self._h, mt.ctypes.data, C.byref(idx), C.byref(dr)))
        return mt, idx.value, dr.value

    def set_state(self, state) -> None:
        mt, idx, dr = state
        mt = np.ascontiguousarray(mt, np.uint64)
        check(lib.rb_rng_set_state(self._h, mt.ctypes.data, int(idx), int(dr)))

    def next_u64(self) -> int:
        v = C.c_uint64()
        check(lib.rb_rng_next_u64(self._h, C.byref(v)))
        return v.value

    def below(self, bound: int) -> int:
        v = C.c_uint64()
        check(lib.rb_rng_below(self._h, int(bound), C.byref(v)))
        return v.value

    def uniform01(self) -> float:
        v = C.c_double()
        check(lib.rb_rng_uniform01(self._h, C.byref(v)))
        return v.value

    def normal(self) -> float:
        v = C.c_double()
        check(lib.rb_rng_normal(self._h, C.byref(v)))
        return v.value

    def sample_without_replacement(self, n: int, k: int) -> np.ndarray:
        out = np.zeros(max(k, 1), np.uint64)
        check(lib.rb_rng_sample_without_replacement(self._h, n, k, out.ctypes.data))
        return out[:k]

    def fill_u64(self, n: int, out=None):
        """n raw engine outputs produced by the GPU generator."""
        if out is None:
            out = np.zeros(n, np.uint64)
        check(lib.rb_rng_fill_u64(self._h, n, _ptr(out)))
        return out


def hash_name(name: str) -> int:
    return lib.rb_hash_name(name.encode())


# ---------------------------------------------------------------------------
def _records_from(recs) -> np.ndarray:
    r = np.asarray(recs, RECORD_DTYPE)
    out = np.zeros(r.shape, RECORD_DTYPE)  # zero padding
    for f in RECORD_DTYPE.names:
        out[f] = r[f]
    return out


class ShardedReplayBuffer:
    """replab::ShardedReplayBuffer (replay_buffer.hpp:57-108) in HBM."""

    def __init__(self, num_shards: int, total_capacity: int,
                 strategy: str = "uniform_with_replacement", retention: str = "plain_fifo",
                 delta: float = 0.0, max_tokens: int = 0, device: int = -1,
                 shard_range: Optional[tuple] = None, _handle=None):
        if _handle is None:
            if strategy not in STRATEGIES:
                raise ValueError(f"unknown sampling strategy: '{strategy}'")
            if retention not in RETENTIONS:
                raise ValueError(f"unknown retention policy: '{retention}'")
            sb, se = shard_range if shard_range else (0, 0)
            h = C.c_void_p()
            check(lib.rb_create(num_shards, total_capacity, STRATEGIES[strategy],
                                RETENTIONS[retention], float(delta), int(max_tokens), int(device),
                                sb, se, C.byref(h)))
            _handle = h
        self._h = _handle
        self.max_tokens = int(max_tokens)
        # shards whose slice of the draws this buffer maps (None: every shard)
        self._owned_shards = (shard_range[1] - shard_range[0]) if shard_range else None

    def __del__(self):
        if getattr(self, "_h", None):
            lib.rb_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    # -- configuration (replay_buffer.hpp:74-84)
    def _sz(self, fn, *args) -> int:
        v = C.c_size_t()
        check(fn(self._h, *args, C.byref(v)))
        return v.value

    def num_shards(self) -> int:
        return self._sz(lib.rb_num_shards)

    def total_capacity(self) -> int:
        return self._sz(lib.rb_total_capacity)

    def shard_capacity(self) -> int:
        return self._sz(lib.rb_shard_capacity)

    def size(self) -> int:
        return self._sz(lib.rb_size)

    def shard_size(self, shard: int) -> int:
        return self._sz(lib.rb_shard_size, shard)

    def route_cursor(self) -> int:
        return self._sz(lib.rb_route_cursor)

    def strategy(self) -> str:
        v = C.c_int()
        check(lib.rb_strategy(self._h, C.byref(v)))
        return STRATEGY_NAMES[v.value]

    def retention(self):
        k, d = C.c_int(), C.c_double()
        check(lib.rb_retention(self._h, C.byref(k), C.byref(d)))
        return ("plain_fifo" if k.value == 0 else "positive_bias", d.value)

    def set_priority(self, base: int = 1, adv_scale: int = 0, pos_bonus: int = 0) -> None:
        """Weights of the priority_with_replacement strategy (builder extension,
        include/replay_b200.h rb_set_priority): w = base + floor(min(|A|, 2^15) *
        adv_scale) + pos_bonus * [reward > 0]; (1, 0, 0) draws exactly as
        uniform_with_replacement (replay_buffer.cpp:141-145)."""
        check(lib.rb_set_priority(self._h, int(base), int(adv_scale), int(pos_bonus)))

    def priority(self):
        b, a, p = C.c_uint32(), C.c_uint32(), C.c_uint32()
        check(lib.rb_get_priority(self._h, C.byref(b), C.byref(a), C.byref(p)))
        return b.value, a.value, p.value

    def priority_mass(self, out=None):
        """Per-shard priority mass (rb_priority_mass): W_s for the shards this
        buffer holds, 0 for the others.  out: a device uint64/int64 tensor of
        num_shards (asynchronous) or None (returns a numpy uint64 array)."""
        if out is None:
            host = np.zeros(self.num_shards(), np.uint64)
            check(lib.rb_priority_mass(self._h, host.ctypes.data))
            return host
        check(lib.rb_priority_mass(self._h, _ptr(out)))
        return out

    def allreduce_priority_mass(self, nccl_comm: int, masses) -> None:
        """rb_allreduce_priority_mass: masses (device, num_shards x 64-bit) <-
        the sum over the communicator's ranks of each rank's priority_mass."""
        check(lib.rb_allreduce_priority_mass(self._h, C.c_void_p(nccl_comm), _ptr(masses)))

    def set_stream(self, stream) -> None:
        """Enqueue on an external stream (int handle, e.g. torch.cuda.current_stream().cuda_stream)."""
        check(lib.rb_set_stream(self._h, C.c_void_p(stream)))

    def stream(self) -> int:
        return lib.rb_get_stream(self._h) or 0

    # -- push / insert
    def push(self, record, tokens=None, logp_old=None):
        """replay_buffer.cpp:83-96 — returns the evicted record or None."""
        rec = _records_from(np.asarray(record, RECORD_DTYPE).reshape(1))
        ev = np.zeros(1, RECORD_DTYPE)
        has = C.c_int(0)
        tk = _arr(tokens, np.int32)
        lp = _arr(logp_old, np.float32)
        n = 0 if tk is None and lp is None else int((tk if tk is not None else lp).shape[0])
        check(lib.rb_push(self._h, rec.ctypes.data, _ptr(tk), _ptr(lp), n, ev.ctypes.data,
                          C.byref(has)))
        return ev[0] if has.value else None

    def insert(self, *, rollout_id, reward, prompt_id=None, group_id=None, creation_step=None,
               policy_version=None, is_correct=None, behavior_logprob=None, advantage=None,
               group_mean=None, group_offsets=None, tok_offsets=None, tokens=None,
               logp_old=None, evicted=None, assume_unique: bool = False,
               n_global: Optional[int] = None) -> int:
        """Batched push of n trajectories (rb_insert).  Returns the number applied.
        n_global (owned-metadata buffers, rb_insert_owned): the batch holds only
        this buffer's shard's records out of a global batch of n_global."""
        keep = []

        def a(x, dt):
            y = _arr(x, dt)
            keep.append(y)
            return _ptr(y)

        rid = _arr(rollout_id, np.uint64)
        keep.append(rid)
        n = int(rid.shape[0])
        bt = InsertBatch()
        bt.n = n
        bt.rollout_id = _ptr(rid)
        bt.prompt_id = a(prompt_id, np.uint64)
        bt.group_id = a(group_id, np.uint64)
        bt.creation_step = a(creation_step, np.int64)
        bt.policy_version = a(policy_version, np.int64)
        bt.reward = a(reward, np.float64)
        bt.is_correct = a(is_correct, np.uint8)
        bt.behavior_logprob = a(behavior_logprob, np.float64)
        bt.advantage = a(advantage, np.float64)
        bt.group_mean = a(group_mean, np.float64)
        go = _arr(group_offsets, np.int64)
        keep.append(go)
        bt.group_offsets = _ptr(go)
        bt.n_groups = 0 if go is None else int(go.shape[0]) - 1
        bt.tok_offsets = a(tok_offsets, np.int64)
        bt.tokens = a(tokens, np.int32)
        bt.logp_old = a(logp_old, np.float32)
        applied = C.c_size_t(0)
        ev = _arr(evicted, np.uint64)
        flags = RB_INSERT_ASSUME_UNIQUE if assume_unique else 0
        if n_global is not None:
            check(lib.rb_insert_owned(self._h, C.byref(bt), int(n_global), flags))
            return n
        check(lib.rb_insert(self._h, C.byref(bt), _ptr(ev), C.byref(applied), flags))
        return applied.value

    def set_owned_metadata(self, on: bool = True) -> None:
        """Keep the metadata of the one owned shard only (rb_set_owned_metadata)."""
        check(lib.rb_set_owned_metadata(self._h, 1 if on else 0))

    # -- sample / gather / loss
    def sample(self, batch_size: int, rng: Rng, ledger: bool = False, batch_id: int = 0,
               use_step: int = 0, with_index: bool = False):
        """replay_buffer.cpp:184-217 — record copies in shard-major draw order."""
        out = np.zeros(batch_size, RECORD_DTYPE)
        ev = np.zeros(batch_size, EVENT_DTYPE) if ledger else None
        sh = np.zeros(batch_size, np.int64) if with_index else None
        ix = np.zeros(batch_size, np.int64) if with_index else None
        check(lib.rb_sample(self._h, batch_size, rng.handle, out.ctypes.data, _ptr(sh), _ptr(ix),
                            _ptr(ev), batch_id, use_step))
        res = [out]
        if ledger:
            res.append(ev)
        if with_index:
            res += [sh, ix]
        return res[0] if len(res) == 1 else tuple(res)

    def sample_device(self, batch_size: int, rng: Rng) -> None:
        """Hot path: select a batch, keep it on the device (no host outputs)."""
        check(lib.rb_sample(self._h, batch_size, rng.handle, None, None, None, None, 0, 0))

    def batch_size(self) -> int:
        return self._sz(lib.rb_batch_size)

    def batch_total_tokens(self) -> int:
        v = C.c_int64()
        check(lib.rb_batch_total_tokens(self._h, C.byref(v)))
        return v.value

    def batch_ids(self):
        """(ids, lengths, packed offsets) of the current batch's selections held here
        (a shard-range buffer: its own shards' slice of the draws)."""
        T = self.num_shards()
        n = self.batch_size() // max(1, T) * (self._owned_shards or T)
        ids = np.zeros(max(n, 1), np.uint64)
        lens = np.zeros(max(n, 1), np.int32)
        off = np.zeros(n + 1, np.int64)
        check(lib.rb_batch_ids(self._h, ids.ctypes.data, lens.ctypes.data, off.ctypes.data))
        return ids[:n], lens[:n], off

    def gather(self, out_tokens=None, out_logp_old=None, out_offsets=None) -> None:
        check(lib.rb_gather(self._h, _ptr(out_tokens), _ptr(out_logp_old), _ptr(out_offsets)))

    def set_async_outputs(self, on: bool = True) -> None:
        """rb_set_async_outputs: pinned host dlogp of a loss completes after
        synchronize() instead of before the call returns."""
        check(lib.rb_set_async_outputs(self._h, int(bool(on))))

    def gather_dlpack(self):
        """The packed batch as library-owned device arrays handed over through
        DLPack (rb_gather_dlpack): returns (tokens int32, logp_old float32,
        offsets int64) as PyCapsules any DLPack consumer takes without a copy,
        e.g. torch.from_dlpack(capsule)."""
        ptrs = [C.c_void_p() for _ in range(3)]
        check(lib.rb_gather_dlpack(self._h, *[C.byref(p) for p in ptrs]))
        return tuple(_dl_capsule(p.value) for p in ptrs)

    @staticmethod
    def _stats_arg(stats):
        """True -> host LossStats (synchronous); None/False -> no stats;
        a 40-byte device tensor -> device rb_loss_stats (asynchronous)."""
        if stats is True:
            st = LossStats()
            return st, C.byref(st)
        if stats is None or stats is False:
            return None, None
        return stats, _ptr(stats)

    def loss_grpo(self, logp_now, out_dlogp, eps_low=0.2, eps_high=0.2, norm_tokens=0,
                  stats=True, mode="token_mean"):
        """GRPO clipped surrogate (bandit.cpp:363-408) per token of the batch.
        mode: "token_mean" (default), "seq_mean" or "seq_ratio" (sequence-level
        ratio; norm_tokens is then the global sequence count, 0 = this batch)."""
        st, p = self._stats_arg(stats)
        if mode not in GRPO_MODES:
            raise ValueError(f"unknown GRPO normalisation mode: '{mode}'")
        check(lib.rb_loss_grpo_ex(self._h, _ptr(logp_now), _ptr(out_dlogp), eps_low, eps_high,
                                  GRPO_MODES[mode], int(norm_tokens), p))
        return st

    def loss_asymre(self, logp_now, out_dlogp, delta_v=-0.1, norm_batch=0, stats=True):
        st, p = self._stats_arg(stats)
        check(lib.rb_loss_asymre(self._h, _ptr(logp_now), _ptr(out_dlogp), delta_v,
                                 int(norm_batch), p))
        return st

    def loss_finalize(self, dlogp, stats):
        """Re-normalise after a cross-rank reduction of `stats` (LossStats or device tensor)."""
        p = C.byref(stats) if isinstance(stats, LossStats) else _ptr(stats)
        check(lib.rb_loss_finalize(self._h, _ptr(dlogp), p))
        return stats

    def loss_set_reduce_vector(self, vec3) -> None:
        """Register a device float64[3] that every loss call fills with
        {objective_sum, included, excluded} (one-collective multi-GPU path)."""
        check(lib.rb_loss_set_reduce_vector(self._h, _ptr(vec3)))

    def loss_finalize_vec(self, dlogp, vec3, stats=None):
        """After all-reducing the registered vector: global normalisation
        (one kernel); `stats` a LossStats, a device tensor or None."""
        p = C.byref(stats) if isinstance(stats, LossStats) else _ptr(stats)
        check(lib.rb_loss_finalize_vec(self._h, _ptr(dlogp), _ptr(vec3), p))
        return stats

    def allreduce_loss_stats(self, nccl_comm: int, dlogp, stats=None):
        """The one collective of a multi-GPU step inside the library: NCCL
        all-reduce (sum) of the registered vector on the buffer's stream, then
        the global normalisation.  `nccl_comm`: an ncclComm_t address of the
        NCCL loaded in this process, e.g. torch's
        ``dist.group.WORLD._get_backend(torch.device("cuda"))._comm_ptr()``."""
        p = C.byref(stats) if isinstance(stats, LossStats) else _ptr(stats)
        check(lib.rb_allreduce_loss_stats(self._h, C.c_void_p(int(nccl_comm)), _ptr(dlogp), p))
        return stats

    def batch_ids_device(self, out_ids, out_lengths=None, out_offsets=None) -> None:
        """Per-selection ids / lengths / packed offsets into device arrays (no sync)."""
        check(lib.rb_batch_ids(self._h, _ptr(out_ids), _ptr(out_lengths), _ptr(out_offsets)))

    # -- inspection / persistence
    def shard_contents(self, shard: int) -> np.ndarray:
        cap = self.shard_capacity()
        out = np.zeros(cap + 1, RECORD_DTYPE)
        cnt = C.c_size_t()
        check(lib.rb_shard_contents(self._h, shard, out.ctypes.data, cap + 1, C.byref(cnt)))
        return out[: cnt.value]

    def record_tokens(self, shard: int, index: int):
        cap = max(self.max_tokens, 1)
        tk = np.zeros(cap, np.int32)
        lp = np.zeros(cap, np.float32)
        n = C.c_int32()
        check(lib.rb_record_tokens(self._h, shard, index, tk.ctypes.data, lp.ctypes.data, cap,
                                   C.byref(n)))
        return tk[: n.value], lp[: n.value]

    def dump(self) -> str:
        n = C.c_size_t()
        check(lib.rb_dump(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(lib.rb_dump(self._h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    @staticmethod
    def load(text: str, max_tokens: int = 0, device: int = -1) -> "ShardedReplayBuffer":
        h = C.c_void_p()
        check(lib.rb_load(text.encode(), int(max_tokens), int(device), C.byref(h)))
        return ShardedReplayBuffer(0, 0, _handle=h, max_tokens=max_tokens)

    def staleness_hist(self, use_step: int, max_bin: int = 255):
        """Histogram (bins 0..max_bin, last = overflow) and sum of the current
        batch's staleness use_step - creation_step (metrics.cpp:37-39)."""
        h = np.zeros(max_bin + 1, np.uint64)
        sm = C.c_int64()
        check(lib.rb_batch_staleness_hist(self._h, int(use_step), int(max_bin), h.ctypes.data,
                                          C.byref(sm)))
        return h, sm.value

    def use_count_hist(self, max_bin: int = 255):
        """Histogram and sum of the resident records' use counts."""
        h = np.zeros(max_bin + 1, np.uint64)
        sm = C.c_uint64()
        check(lib.rb_use_count_hist(self._h, int(max_bin), h.ctypes.data, C.byref(sm)))
        return h, sm.value

    def snapshot(self, out=None):
        """Binary checkpoint of the device state (rb_snapshot) into a new
        numpy uint8 array, or into `out` (numpy or torch, host or device)."""
        n = C.c_size_t()
        check(lib.rb_snapshot(self._h, None, 0, C.byref(n)))
        if out is None:
            out = np.empty(n.value, np.uint8)
        cap = out.nbytes if hasattr(out, "nbytes") else out.numel() * out.element_size()
        check(lib.rb_snapshot(self._h, _ptr(out), cap, C.byref(n)))
        return out

    def restore(self, snap) -> None:
        """Restore a buffer of the same shape from rb_snapshot bytes."""
        cap = snap.nbytes if hasattr(snap, "nbytes") else snap.numel() * snap.element_size()
        check(lib.rb_restore(self._h, _ptr(snap), cap))

    def check(self) -> None:
        check(lib.rb_check(self._h))

    def synchronize(self) -> None:
        check(lib.rb_synchronize(self._h))


# ---------------------------------------------------------------------------
def group_advantages(rewards, offsets=None, out=None, out_mean=None):
    """bandit.cpp:276-294 (segmented when offsets are given)."""
    r = _arr(rewards, np.float64)
    if offsets is None:
        offsets = np.array([0, r.shape[0]], np.int64)
    off = _arr(offsets, np.int64)
    if out is None:
        out = np.zeros(r.shape[0], np.float64)
    check(lib.rb_group_advantages(_ptr(r), _ptr(off), int(off.shape[0]) - 1, _ptr(out),
                                  _ptr(out_mean)))
    return out


def grpo_tokens(logp_now, logp_old, adv, offsets, eps_low=0.2, eps_high=0.2, out=None,
                mode="token_mean", behavior_logprob=None):
    """grpo_loss_grad at the token level; mode as in ShardedReplayBuffer.loss_grpo
    (behavior_logprob: per-trajectory sequence log-prob for "seq_ratio",
    default sum_t logp_old)."""
    if mode not in GRPO_MODES:
        raise ValueError(f"unknown GRPO normalisation mode: '{mode}'")
    lpn, lpo = _arr(logp_now, np.float32), _arr(logp_old, np.float32)
    a, off = _arr(adv, np.float64), _arr(offsets, np.int64)
    blp = _arr(behavior_logprob, np.float64)
    if out is None:
        out = np.zeros(lpn.shape[0], np.float32)
    st = LossStats()
    check(lib.rb_grpo_tokens_ex(_ptr(lpn), _ptr(lpo), _ptr(a), _ptr(blp), _ptr(off),
                                int(off.shape[0]) - 1, eps_low, eps_high, GRPO_MODES[mode],
                                _ptr(out), C.byref(st)))
    return out, st


def grpo_records(logp_now, behavior_logprob, adv, eps_low=0.2, eps_high=0.2, out=None):
    lpn, blp, a = (_arr(x, np.float64) for x in (logp_now, behavior_logprob, adv))
    if out is None:
        out = np.zeros(lpn.shape[0], np.float64)
    st = LossStats()
    check(lib.rb_grpo_records(_ptr(lpn), _ptr(blp), _ptr(a), int(lpn.shape[0]), eps_low,
                              eps_high, _ptr(out), C.byref(st)))
    return out, st


def asymre_tokens(logp_now, reward, group_mean, offsets, delta_v=-0.1, out=None):
    lpn = _arr(logp_now, np.float32)
    r, g, off = _arr(reward, np.float64), _arr(group_mean, np.float64), _arr(offsets, np.int64)
    if out is None:
        out = np.zeros(lpn.shape[0], np.float32)
    st = LossStats()
    check(lib.rb_asymre_tokens(_ptr(lpn), _ptr(r), _ptr(g), _ptr(off), int(off.shape[0]) - 1,
                               delta_v, _ptr(out), C.byref(st)))
    return out, st


def asymre_records(logp_now, reward, group_mean, delta_v=-0.1, out=None):
    lpn, r, g = (_arr(x, np.float64) for x in (logp_now, reward, group_mean))
    if out is None:
        out = np.zeros(lpn.shape[0], np.float64)
    st = LossStats()
    check(lib.rb_asymre_records(_ptr(lpn), _ptr(r), _ptr(g), int(lpn.shape[0]), delta_v,
                                _ptr(out), C.byref(st)))
    return out, st


# ---------------------------------------------------------------------------
class MetricsLedger:
    """replab::MetricsLedger (metrics.hpp:36-93) on the device, with
    replay_counts / global_use_order / steps_since_last_use
    (metrics.cpp:123-170) computed by kernels (rb_ledger_*)."""

    def __init__(self, device: int = -1):
        h = C.c_void_p()
        check(lib.rb_ledger_create(device, C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.rb_ledger_destroy(h)
            self._h = None

    def note_generated(self, ids) -> None:
        a = _arr(ids, np.uint64)
        check(lib.rb_ledger_note_generated(self._h, _ptr(a), int(a.shape[0])))

    def record_batch(self, buffer: "ShardedReplayBuffer", batch_id: int, use_step: int) -> None:
        """The events of buffer's current batch (sample(..., &ledger, batch_id,
        use_step)), appended on the device."""
        check(lib.rb_ledger_record_batch(self._h, buffer._h, int(batch_id), int(use_step)))

    def record_use(self, events) -> None:
        ev = np.ascontiguousarray(events, EVENT_DTYPE).reshape(-1)
        check(lib.rb_ledger_record_uses(self._h, ev.ctypes.data, ev.shape[0]))

    def check(self) -> None:
        check(lib.rb_ledger_check(self._h))

    def __len__(self) -> int:
        n = C.c_size_t()
        check(lib.rb_ledger_sizes(self._h, C.byref(n), None))
        return n.value

    def events(self) -> np.ndarray:
        n = C.c_size_t()
        check(lib.rb_ledger_events(self._h, None, 0, C.byref(n)))
        out = np.zeros(n.value, EVENT_DTYPE)
        check(lib.rb_ledger_events(self._h, out.ctypes.data, n.value, C.byref(n)))
        return out

    def replay_counts(self, include_zero_use: bool = True):
        """(ids ascending, use counts) — replay_counts() as two arrays."""
        n = C.c_size_t()
        check(lib.rb_ledger_replay_counts(self._h, int(include_zero_use), None, None, 0, C.byref(n)))
        ids, cnt = np.zeros(n.value, np.uint64), np.zeros(n.value, np.uint64)
        check(lib.rb_ledger_replay_counts(self._h, int(include_zero_use), ids.ctypes.data,
                                          cnt.ctypes.data, n.value, C.byref(n)))
        return ids, cnt

    def global_use_order(self, rng: Rng) -> np.ndarray:
        m = len(self)
        out = np.zeros(m, np.uint64)
        n = C.c_size_t()
        check(lib.rb_ledger_global_use_order(self._h, rng.handle, out.ctypes.data, m, C.byref(n)))
        return out

    def steps_since_last_use(self, rng: Rng):
        """(event_index, gap, has_gap) in global use order; has_gap 0 = first use."""
        m = len(self)
        idx, gap, has = np.zeros(m, np.uint64), np.zeros(m, np.int64), np.zeros(m, np.uint8)
        n = C.c_size_t()
        check(lib.rb_ledger_steps_since_last_use(self._h, rng.handle, idx.ctypes.data,
                                                 gap.ctypes.data, has.ctypes.data, m, C.byref(n)))
        return idx, gap, has


class TransferQueue:
    """replab::TransferQueue (transfer_queue.hpp:12-35) on the GPU: a
    consume-once LIFO hand-off whose records and token payload stay in HBM.
    capacity=None is the reference's unbounded queue."""

    def __init__(self, capacity: Optional[int] = None, max_tokens: int = 0, device: int = -1):
        if capacity is not None and capacity <= 0:
            raise ValueError("TransferQueue: capacity must be positive")  # transfer_queue.cpp:8-10
        h = C.c_void_p()
        check(lib.rb_queue_create(int(capacity or 0), int(max_tokens), int(device), C.byref(h)))
        self._h = h
        self._cap = capacity
        self.max_tokens = max_tokens

    def __del__(self):
        if getattr(self, "_h", None):
            lib.rb_queue_destroy(self._h)
            self._h = None

    def capacity(self) -> Optional[int]:
        return self._cap

    def size(self) -> int:
        v = C.c_size_t()
        check(lib.rb_queue_size(self._h, C.byref(v)))
        return v.value

    def push_group(self, records, tok_offsets=None, tokens=None, logp_old=None,
                   group_offsets=None) -> bool:
        """All or nothing (transfer_queue.cpp:22-29).  `records`: RECORD_DTYPE
        array (advantages as given), or None with the SoA keyword form of
        ShardedReplayBuffer.insert passed through `group_offsets`."""
        recs = np.ascontiguousarray(np.atleast_1d(_records_from(records)))
        keep = []

        def col(name, dt):
            a = np.ascontiguousarray(recs[name].astype(dt))
            keep.append(a)
            return a.ctypes.data

        bt = InsertBatch()
        bt.n = recs.shape[0]
        bt.rollout_id = col("rollout_id", np.uint64)
        bt.prompt_id = col("prompt_id", np.uint64)
        bt.group_id = col("group_id", np.uint64)
        bt.creation_step = col("creation_step", np.int64)
        bt.policy_version = col("policy_version", np.int64)
        bt.reward = col("reward", np.float64)
        bt.is_correct = col("is_correct", np.uint8)
        bt.behavior_logprob = col("behavior_logprob", np.float64)
        if group_offsets is None:
            bt.advantage = col("advantage", np.float64)
        else:
            go = _arr(group_offsets, np.int64)
            keep.append(go)
            bt.group_offsets = _ptr(go)
            bt.n_groups = int(go.shape[0]) - 1
        for name, x, dt in (("tok_offsets", tok_offsets, np.int64), ("tokens", tokens, np.int32),
                            ("logp_old", logp_old, np.float32)):
            y = _arr(x, dt)
            keep.append(y)
            setattr(bt, name, _ptr(y))
        ok = C.c_int()
        check(lib.rb_queue_push_group(self._h, C.byref(bt), C.byref(ok)))
        return bool(ok.value)

    def push(self, record, tokens=None, logp_old=None) -> bool:
        """transfer_queue.cpp:13-20 (a group of one)."""
        toff = None
        if tokens is not None or logp_old is not None:
            n = len(tokens if tokens is not None else logp_old)
            toff = np.array([0, n], np.int64)
        return self.push_group(record, toff, tokens, logp_old)

    def pop(self):
        """transfer_queue.cpp:31-39: the most recent record, or None."""
        r = self.pop_batch(1)[0]
        return r[0] if len(r) else None

    def pop_batch(self, k: int, out_tokens=None, out_logp_old=None, out_offsets=None):
        """k pops, most recent first; optional packed payload (+ offsets)."""
        out = np.zeros(k, RECORD_DTYPE)
        n = C.c_size_t()
        check(lib.rb_queue_pop(self._h, k, out.ctypes.data, C.byref(n), _ptr(out_tokens),
                               _ptr(out_logp_old), _ptr(out_offsets)))
        return out[: n.value], n.value


def summarize_hist(hist, total_sum=None):
    """The reference's summarize() (metrics.cpp:185-202: mean, nearest-rank
    quartiles, histogram) from an integer-valued histogram — exact while the
    last (overflow) bin is empty."""
    hist = np.asarray(hist, np.uint64)
    n = int(hist.sum())
    if n == 0:
        raise ValueError("summarize requires at least one value")
    cdf = np.cumsum(hist)

    def rank(q):  # value at rank ceil(q * n), 1-indexed (metrics.cpp:174-181)
        r = min(max(int(np.ceil(q * n)), 1), n)
        return float(np.searchsorted(cdf, r))

    mean = (float(total_sum) if total_sum is not None
            else float((np.arange(hist.size) * hist).sum())) / n
    return {"count": n, "mean": mean, "q25": rank(0.25), "median": rank(0.5), "q75": rank(0.75),
            "histogram": {int(i): int(c) for i, c in enumerate(hist) if c}}


# DLPack capsules (the legacy "dltensor" protocol): a consumer renames the
# capsule "used_dltensor" and owns the tensor; an unconsumed capsule releases
# it through rb_dlpack_free when collected.
_capsule_new = C.pythonapi.PyCapsule_New
_capsule_new.restype = C.py_object
_capsule_new.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]
# (the destructor sees the dying capsule as a raw pointer: no refcounting)
_capsule_valid = C.pythonapi.PyCapsule_IsValid
_capsule_valid.restype = C.c_int
_capsule_valid.argtypes = [C.c_void_p, C.c_char_p]
_capsule_ptr = C.pythonapi.PyCapsule_GetPointer
_capsule_ptr.restype = C.c_void_p
_capsule_ptr.argtypes = [C.c_void_p, C.c_char_p]


@C.CFUNCTYPE(None, C.c_void_p)
def _dl_capsule_destructor(cap):
    if _capsule_valid(cap, b"dltensor"):
        lib.rb_dlpack_free(_capsule_ptr(cap, b"dltensor"))


def _dl_capsule(ptr):
    return _capsule_new(ptr, b"dltensor", C.cast(_dl_capsule_destructor, C.c_void_p))
