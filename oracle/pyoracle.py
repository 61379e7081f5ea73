"""ctypes bindings for the CHECKERS (test infrastructure only).

* ``Oracle``   — oracle/_build/liboracle.so, the C restatement (replay_oracle.c)
* ``Reference`` — oracle/_ref/libreplab_ref.so, the UNMODIFIED reference
  library compiled from /root/reference/proj/src plus ref_driver.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libreplab_ref.so")

# rollout.hpp:13-31 — 80-byte record; same layout as rb_record in include/replay_b200.h
RECORD_DTYPE = np.dtype(
    {
        "names": ["rollout_id", "prompt_id", "group_id", "creation_step", "policy_version",
                  "reward", "is_correct", "behavior_logprob", "advantage", "use_count"],
        "formats": ["<u8", "<u8", "<u8", "<i8", "<i8", "<f8", "u1", "<f8", "<f8", "<u4"],
        "offsets": [0, 8, 16, 24, 32, 40, 48, 56, 64, 72],
        "itemsize": 80,
    }
)

STRATEGIES = {"uniform_with_replacement": 0, "uniform_without_replacement": 1,
              "unused_first_without_replacement": 2,
              "priority_with_replacement": 3}  # builder extension: oracle only


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def build_oracle(with_ref: bool = True) -> None:
    """Compile the checkers (make -C oracle [ref])."""
    targets = ["all"]
    if with_ref and os.path.isdir(os.environ.get("REPLAB_REF", "/root/reference/proj")):
        targets += ["ref", "reftests"]
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def records(n: int) -> np.ndarray:
    return np.zeros(n, dtype=RECORD_DTYPE)


def canon(recs) -> np.ndarray:
    """Copy into a zero-initialised array so padding bytes compare equal."""
    recs = np.asarray(recs, RECORD_DTYPE)
    out = np.zeros(recs.shape, RECORD_DTYPE)
    for name in RECORD_DTYPE.names:
        out[name] = recs[name]
    return out


def same_records(a, b) -> bool:
    return canon(a).tobytes() == canon(b).tobytes()


class OracleError(ValueError):
    pass


# ---------------------------------------------------------------------------
class _OrRng(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_uint32), ("seed", C.c_uint64),
                ("draws", C.c_uint64)]


class Oracle:
    """The C restatement."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build_oracle(with_ref=False)
        L = self.lib = C.CDLL(path)
        u64, i64, sz, vp, dbl = C.c_uint64, C.c_int64, C.c_size_t, C.c_void_p, C.c_double
        L.or_last_error.restype = C.c_char_p
        L.or_hash_name.restype = u64
        L.or_hash_name.argtypes = [C.c_char_p, sz]
        L.or_rng_init.argtypes = [vp, u64]
        L.or_rng_stream.argtypes = [vp, C.c_char_p, sz, vp]
        L.or_rng_stream_idx.argtypes = [vp, C.c_char_p, sz, u64, vp]
        L.or_rng_next.restype = u64
        L.or_rng_next.argtypes = [vp]
        L.or_rng_below.argtypes = [vp, u64, vp]
        L.or_rng_uniform01.restype = dbl
        L.or_rng_uniform01.argtypes = [vp]
        L.or_rng_swor.argtypes = [vp, sz, sz, vp]
        L.or_rng_discard.argtypes = [vp, u64]
        L.or_buf_new.restype = vp
        L.or_buf_new.argtypes = [sz, sz, C.c_int, C.c_int, dbl]
        L.or_buf_free.argtypes = [vp]
        L.or_buf_push.argtypes = [vp, vp, vp, vp]
        L.or_buf_sample.argtypes = [vp, sz, vp, vp, vp, vp]
        L.or_buf_set_priority.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_uint32]
        L.or_buf_size.restype = sz
        L.or_buf_size.argtypes = [vp]
        L.or_buf_shard_size.restype = sz
        L.or_buf_shard_size.argtypes = [vp, sz]
        L.or_buf_shard_contents.restype = sz
        L.or_buf_shard_contents.argtypes = [vp, sz, vp]
        L.or_buf_route_cursor.restype = sz
        L.or_buf_route_cursor.argtypes = [vp]
        L.or_group_advantages.argtypes = [vp, sz, vp]
        L.or_loss_grpo_tokens.argtypes = [vp, vp, vp, vp, sz, dbl, dbl, vp, vp, vp, vp]
        L.or_loss_grpo_records.argtypes = [vp, vp, vp, sz, dbl, dbl, vp, vp, vp, vp]
        L.or_loss_grpo_tokens_mode.argtypes = [vp, vp, vp, vp, vp, sz, dbl, dbl, C.c_int, vp, vp,
                                               vp, vp]
        L.or_loss_asymre_tokens.argtypes = [vp, vp, vp, vp, sz, dbl, vp, vp]
        L.or_loss_asymre_records.argtypes = [vp, vp, vp, sz, dbl, vp, vp]
        L.or_production_groups.restype = i64
        L.or_production_groups.argtypes = [dbl, sz, vp]
        L.or_gather_tokens.argtypes = [vp, i64, vp, vp, sz, vp, vp]
        L.or_synth_payload.argtypes = [u64, vp, vp, sz, vp, vp]
        L.or_synth_logp_now.argtypes = [u64, u64, vp, vp, sz, vp]
        L.or_synth_meta.argtypes = [u64, vp, sz, C.c_int32, C.c_int, vp, vp, vp]

    # -- synthetic workload (include/replay_synth.h)
    def synth_meta(self, seed, ids, lmax, ragged):
        ids = np.ascontiguousarray(ids, np.uint64)
        r = np.zeros(ids.size, np.float64)
        ln = np.zeros(ids.size, np.int32)
        blp = np.zeros(ids.size, np.float64)
        self.lib.or_synth_meta(seed, _p(ids), ids.size, lmax, int(ragged), _p(r), _p(ln), _p(blp))
        return r, ln, blp

    def synth_payload(self, seed, ids, lengths):
        ids = np.ascontiguousarray(ids, np.uint64)
        off = np.zeros(ids.size + 1, np.int64)
        np.cumsum(np.asarray(lengths, np.int64), out=off[1:])
        tok = np.zeros(int(off[-1]), np.int32)
        lpo = np.zeros(int(off[-1]), np.float32)
        self.lib.or_synth_payload(seed, _p(ids), _p(off), ids.size, _p(tok), _p(lpo))
        return tok, lpo, off

    def synth_logp_now(self, seed, version, ids, offsets):
        ids = np.ascontiguousarray(ids, np.uint64)
        off = np.ascontiguousarray(offsets, np.int64)
        out = np.zeros(int(off[-1]), np.float32)
        self.lib.or_synth_logp_now(seed, version, _p(ids), _p(off), ids.size, _p(out))
        return out

    def err(self):
        return OracleError(self.lib.or_last_error().decode())

    # -- rng
    def rng(self, seed: int) -> "OracleRng":
        return OracleRng(self, seed)

    def hash_name(self, name: str) -> int:
        b = name.encode()
        return self.lib.or_hash_name(b, len(b))

    # -- buffer
    def buffer(self, shards, capacity, strategy="uniform_with_replacement",
               retention="plain_fifo", delta=0.0) -> "OracleBuffer":
        return OracleBuffer(self, shards, capacity, strategy, retention, delta)

    # -- advantage / losses
    def group_advantages(self, rewards):
        r = np.ascontiguousarray(rewards, dtype=np.float64)
        out = np.zeros_like(r)
        if self.lib.or_group_advantages(_p(r), r.size, _p(out)):
            raise self.err()
        return out

    def loss_grpo_tokens(self, logp_now, logp_old, adv, offsets, eps_low=0.2, eps_high=0.2):
        lpn = np.ascontiguousarray(logp_now, np.float32)
        lpo = np.ascontiguousarray(logp_old, np.float32)
        a = np.ascontiguousarray(adv, np.float64)
        off = np.ascontiguousarray(offsets, np.int64)
        d = np.zeros(lpn.size, np.float32)
        obj = np.zeros(1, np.float64)
        inc = np.zeros(1, np.int64)
        exc = np.zeros(1, np.int64)
        self.lib.or_loss_grpo_tokens(_p(lpn), _p(lpo), _p(a), _p(off), a.size, eps_low,
                                     eps_high, _p(d), _p(obj), _p(inc), _p(exc))
        return d, float(obj[0]), int(inc[0]), int(exc[0])

    def loss_grpo_tokens_mode(self, logp_now, logp_old, adv, offsets, mode, blp=None,
                              eps_low=0.2, eps_high=0.2):
        """mode 0 token mean, 1 per-sequence mean, 2 sequence ratio (replay_oracle.c)."""
        lpn = np.ascontiguousarray(logp_now, np.float32)
        lpo = np.ascontiguousarray(logp_old, np.float32)
        a = np.ascontiguousarray(adv, np.float64)
        b = None if blp is None else np.ascontiguousarray(blp, np.float64)
        off = np.ascontiguousarray(offsets, np.int64)
        d = np.zeros(lpn.size, np.float32)
        obj = np.zeros(1, np.float64)
        inc = np.zeros(1, np.int64)
        exc = np.zeros(1, np.int64)
        self.lib.or_loss_grpo_tokens_mode(_p(lpn), _p(lpo), _p(a), _p(b), _p(off), a.size,
                                          eps_low, eps_high, int(mode), _p(d), _p(obj), _p(inc),
                                          _p(exc))
        return d, float(obj[0]), int(inc[0]), int(exc[0])

    def loss_grpo_records(self, logp_now, blp, adv, eps_low=0.2, eps_high=0.2):
        lpn = np.ascontiguousarray(logp_now, np.float64)
        b = np.ascontiguousarray(blp, np.float64)
        a = np.ascontiguousarray(adv, np.float64)
        d = np.zeros(lpn.size, np.float64)
        obj = np.zeros(1, np.float64)
        inc = np.zeros(1, np.int64)
        exc = np.zeros(1, np.int64)
        self.lib.or_loss_grpo_records(_p(lpn), _p(b), _p(a), lpn.size, eps_low, eps_high,
                                      _p(d), _p(obj), _p(inc), _p(exc))
        return d, float(obj[0]), int(inc[0]), int(exc[0])

    def loss_asymre_tokens(self, logp_now, reward, group_mean, offsets, delta_v=-0.1):
        lpn = np.ascontiguousarray(logp_now, np.float32)
        r = np.ascontiguousarray(reward, np.float64)
        g = np.ascontiguousarray(group_mean, np.float64)
        off = np.ascontiguousarray(offsets, np.int64)
        d = np.zeros(lpn.size, np.float32)
        obj = np.zeros(1, np.float64)
        self.lib.or_loss_asymre_tokens(_p(lpn), _p(r), _p(g), _p(off), r.size, delta_v, _p(d),
                                       _p(obj))
        return d, float(obj[0])

    def loss_asymre_records(self, logp_now, reward, group_mean, delta_v=-0.1):
        lpn = np.ascontiguousarray(logp_now, np.float64)
        r = np.ascontiguousarray(reward, np.float64)
        g = np.ascontiguousarray(group_mean, np.float64)
        d = np.zeros(lpn.size, np.float64)
        obj = np.zeros(1, np.float64)
        self.lib.or_loss_asymre_records(_p(lpn), _p(r), _p(g), lpn.size, delta_v, _p(d), _p(obj))
        return d, float(obj[0])

    def production_groups(self, per_step, group, debt):
        d = C.c_double(debt)
        n = self.lib.or_production_groups(per_step, group, C.byref(d))
        return n, d.value


class OracleRng:
    def __init__(self, o: Oracle, seed: int | None, _state=None):
        self.o = o
        self.st = _OrRng() if _state is None else _state
        if _state is None:
            o.lib.or_rng_init(C.byref(self.st), seed)

    @property
    def seed(self):
        return self.st.seed

    @property
    def draws(self):
        return self.st.draws

    def stream(self, name: str, index: int | None = None) -> "OracleRng":
        out = _OrRng()
        b = name.encode()
        if index is None:
            self.o.lib.or_rng_stream(C.byref(self.st), b, len(b), C.byref(out))
        else:
            self.o.lib.or_rng_stream_idx(C.byref(self.st), b, len(b), index, C.byref(out))
        return OracleRng(self.o, None, out)

    def next_u64(self) -> int:
        return self.o.lib.or_rng_next(C.byref(self.st))

    def below(self, b: int) -> int:
        v = C.c_uint64()
        if self.o.lib.or_rng_below(C.byref(self.st), b, C.byref(v)):
            raise self.o.err()
        return v.value

    def uniform01(self) -> float:
        return self.o.lib.or_rng_uniform01(C.byref(self.st))

    def sample_without_replacement(self, n: int, k: int):
        out = np.zeros(max(k, 1), np.uint64)
        if self.o.lib.or_rng_swor(C.byref(self.st), n, k, _p(out)):
            raise self.o.err()
        return out[:k]

    def discard(self, n: int):
        self.o.lib.or_rng_discard(C.byref(self.st), n)


class OracleBuffer:
    def __init__(self, o: Oracle, shards, capacity, strategy, retention, delta):
        self.o = o
        kind = 1 if retention == "positive_bias" else 0
        self.h = o.lib.or_buf_new(shards, capacity, STRATEGIES[strategy], kind, delta)
        if not self.h:
            raise o.err()
        self.num_shards = shards
        self.shard_capacity = capacity // shards

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.or_buf_free(self.h)

    def push(self, rec):
        r = np.ascontiguousarray(np.asarray(rec, RECORD_DTYPE).reshape(1))
        ev = records(1)
        has = C.c_int(0)
        if self.o.lib.or_buf_push(self.h, _p(r), _p(ev), C.byref(has)):
            raise self.o.err()
        return ev[0] if has.value else None

    def set_priority(self, base=1, adv_scale=0, pos_bonus=0):
        if self.o.lib.or_buf_set_priority(self.h, int(base), int(adv_scale), int(pos_bonus)):
            raise self.o.err()

    def sample(self, batch, rng: OracleRng):
        out = records(batch)
        sh = np.zeros(batch, np.int64)
        ix = np.zeros(batch, np.int64)
        if self.o.lib.or_buf_sample(self.h, batch, C.byref(rng.st), _p(out), _p(sh), _p(ix)):
            raise self.o.err()
        return out, sh, ix

    def size(self):
        return self.o.lib.or_buf_size(self.h)

    def shard_size(self, s):
        return self.o.lib.or_buf_shard_size(self.h, s)

    def shard_contents(self, s):
        out = records(self.shard_capacity + 1)
        n = self.o.lib.or_buf_shard_contents(self.h, s, _p(out))
        return out[:n]

    def route_cursor(self):
        return self.o.lib.or_buf_route_cursor(self.h)


# ---------------------------------------------------------------------------
class Reference:
    """The unmodified reference library (oracle/_ref/libreplab_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        u64, vp, dbl, i64 = C.c_uint64, C.c_void_p, C.c_double, C.c_int64
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng_new.restype = vp
        L.ref_rng_new.argtypes = [u64]
        L.ref_rng_free.argtypes = [vp]
        L.ref_rng_stream.restype = vp
        L.ref_rng_stream.argtypes = [vp, C.c_char_p]
        L.ref_rng_stream_idx.restype = vp
        L.ref_rng_stream_idx.argtypes = [vp, C.c_char_p, u64]
        L.ref_rng_seed.restype = u64
        L.ref_rng_seed.argtypes = [vp]
        L.ref_rng_next.restype = u64
        L.ref_rng_next.argtypes = [vp]
        L.ref_rng_below.argtypes = [vp, u64, vp]
        L.ref_rng_uniform01.restype = dbl
        L.ref_rng_uniform01.argtypes = [vp]
        L.ref_rng_swor.argtypes = [vp, u64, u64, vp]
        L.ref_hash_name.restype = u64
        L.ref_hash_name.argtypes = [C.c_char_p]
        L.ref_summarize.argtypes = [vp, u64, vp, vp, vp, u64, vp]
        L.ref_buf_new.restype = vp
        L.ref_buf_new.argtypes = [u64, u64, C.c_int, C.c_int, dbl]
        L.ref_buf_free.argtypes = [vp]
        L.ref_buf_push.argtypes = [vp, vp, vp, vp]
        L.ref_buf_sample.argtypes = [vp, u64, vp, vp, vp, i64, i64]
        L.ref_buf_size.restype = u64
        L.ref_buf_size.argtypes = [vp]
        L.ref_buf_shard_size.restype = u64
        L.ref_buf_shard_size.argtypes = [vp, u64]
        L.ref_buf_shard_contents.restype = u64
        L.ref_buf_shard_contents.argtypes = [vp, u64, vp]
        L.ref_buf_dump.restype = u64
        L.ref_buf_dump.argtypes = [vp, C.c_char_p, u64]
        L.ref_buf_load.restype = vp
        L.ref_buf_load.argtypes = [C.c_char_p]
        L.ref_group_advantages.argtypes = [vp, u64, vp]
        L.ref_ledger_new.restype = vp
        L.ref_ledger_free.argtypes = [vp]
        L.ref_ledger_note_generated.argtypes = [vp, u64]
        L.ref_ledger_record_use.argtypes = [vp, vp]
        L.ref_ledger_events.restype = u64
        L.ref_ledger_events.argtypes = [vp, vp]
        L.ref_ledger_replay_counts.restype = u64
        L.ref_ledger_replay_counts.argtypes = [vp, C.c_int, vp, vp]
        L.ref_ledger_global_use_order.restype = u64
        L.ref_ledger_global_use_order.argtypes = [vp, vp, vp]
        L.ref_ledger_steps_since_last_use.restype = u64
        L.ref_ledger_steps_since_last_use.argtypes = [vp, vp, vp, vp, vp]
        L.ref_loss_records.argtypes = [C.c_int, vp, vp, vp, u64, dbl, dbl, dbl, vp, vp, vp, vp]

    def err(self):
        return OracleError(self.lib.ref_last_error().decode())

    def rng(self, seed):
        return RefRng(self, self.lib.ref_rng_new(seed))

    def buffer(self, shards, capacity, strategy="uniform_with_replacement",
               retention="plain_fifo", delta=0.0):
        return RefBuffer(self, shards, capacity, strategy, retention, delta)

    def group_advantages(self, rewards):
        r = np.ascontiguousarray(rewards, np.float64)
        out = np.zeros_like(r)
        if self.lib.ref_group_advantages(_p(r), r.size, _p(out)):
            raise self.err()
        return out

    def ledger(self):
        return RefLedger(self)

    def summarize(self, values):
        """The reference's summarize() (metrics.cpp:185-202) as a dict."""
        v = np.ascontiguousarray(values, np.float64)
        out = np.zeros(5)
        cap = 4096
        keys = np.zeros(cap, np.int64)
        cnt = np.zeros(cap, np.uint64)
        hn = C.c_uint64()
        if self.lib.ref_summarize(_p(v), v.size, _p(out), _p(keys), _p(cnt), cap, C.byref(hn)):
            raise self.err()
        n = min(hn.value, cap)
        return {"count": int(out[0]), "mean": out[1], "q25": out[2], "median": out[3],
                "q75": out[4], "histogram": {int(k): int(c) for k, c in zip(keys[:n], cnt[:n])}}

    def loss_records(self, kind, logp_want, recs, group_mean=None, eps_low=0.2, eps_high=0.2,
                     delta_v=-0.1):
        """kind 'grpo'|'asymre'. Returns (logp_used, dlogp, objective, excluded)."""
        lw = np.ascontiguousarray(logp_want, np.float64)
        r = np.ascontiguousarray(recs, RECORD_DTYPE)
        gm = None if group_mean is None else np.ascontiguousarray(group_mean, np.float64)
        used = np.zeros_like(lw)
        d = np.zeros_like(lw)
        obj = C.c_double()
        exc = C.c_uint64()
        if self.lib.ref_loss_records(0 if kind == "grpo" else 1, _p(lw), _p(r), _p(gm), lw.size,
                                     eps_low, eps_high, delta_v, _p(used), _p(d), C.byref(obj),
                                     C.byref(exc)):
            raise self.err()
        return used, d, obj.value, exc.value


class RefRng:
    def __init__(self, ref: Reference, h):
        self.ref, self.h = ref, h

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_rng_free(self.h)

    @property
    def seed(self):
        return self.ref.lib.ref_rng_seed(self.h)

    def stream(self, name, index=None):
        if index is None:
            return RefRng(self.ref, self.ref.lib.ref_rng_stream(self.h, name.encode()))
        return RefRng(self.ref, self.ref.lib.ref_rng_stream_idx(self.h, name.encode(), index))

    def next_u64(self):
        return self.ref.lib.ref_rng_next(self.h)

    def below(self, b):
        v = C.c_uint64()
        if self.ref.lib.ref_rng_below(self.h, b, C.byref(v)):
            raise self.ref.err()
        return v.value

    def uniform01(self):
        return self.ref.lib.ref_rng_uniform01(self.h)

    def sample_without_replacement(self, n, k):
        out = np.zeros(max(k, 1), np.uint64)
        if self.ref.lib.ref_rng_swor(self.h, n, k, _p(out)):
            raise self.ref.err()
        return out[:k]


class RefBuffer:
    def __init__(self, ref: Reference, shards, capacity, strategy, retention, delta, _h=None):
        self.ref = ref
        if _h is None:
            kind = 1 if retention == "positive_bias" else 0
            _h = ref.lib.ref_buf_new(shards, capacity, STRATEGIES[strategy], kind, delta)
            if not _h:
                raise ref.err()
        self.h = _h
        self.num_shards = shards
        self.shard_capacity = capacity // shards if shards else 0

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_buf_free(self.h)

    def push(self, rec):
        r = np.ascontiguousarray(np.asarray(rec, RECORD_DTYPE).reshape(1))
        ev = records(1)
        has = C.c_int(0)
        if self.ref.lib.ref_buf_push(self.h, _p(r), _p(ev), C.byref(has)):
            raise self.ref.err()
        return ev[0] if has.value else None

    def sample(self, batch, rng: RefRng, with_events=False, batch_id=0, use_step=0):
        out = records(batch)
        ev = np.zeros((batch, 5), np.int64) if with_events else None
        if self.ref.lib.ref_buf_sample(self.h, batch, rng.h, _p(out), _p(ev), batch_id, use_step):
            raise self.ref.err()
        return (out, ev) if with_events else out

    def size(self):
        return self.ref.lib.ref_buf_size(self.h)

    def shard_size(self, s):
        return self.ref.lib.ref_buf_shard_size(self.h, s)

    def shard_contents(self, s):
        out = records(self.shard_capacity + 1)
        n = self.ref.lib.ref_buf_shard_contents(self.h, s, _p(out))
        return out[:n]

    def dump(self) -> str:
        n = self.ref.lib.ref_buf_dump(self.h, None, 0)
        buf = C.create_string_buffer(n + 1)
        self.ref.lib.ref_buf_dump(self.h, buf, n + 1)
        return buf.value.decode()

    @staticmethod
    def load(ref: Reference, text: str) -> "RefBuffer":
        h = ref.lib.ref_buf_load(text.encode())
        if not h:
            raise ref.err()
        return RefBuffer(ref, 0, 0, None, None, 0.0, _h=h)


class RefLedger:
    """replab::MetricsLedger and its diagnostics (metrics.cpp:44-170)."""

    def __init__(self, ref: Reference):
        self.r, self.h = ref, ref.lib.ref_ledger_new()

    def __del__(self):
        try:
            self.r.lib.ref_ledger_free(self.h)
        except Exception:  # noqa: BLE001
            pass

    def note_generated(self, rid):
        if self.r.lib.ref_ledger_note_generated(self.h, int(rid)):
            raise self.r.err()

    def record_use(self, rid, creation_step, use_step, batch_id, rank):
        e = np.array([rid, creation_step, use_step, batch_id, rank], np.int64)
        if self.r.lib.ref_ledger_record_use(self.h, _p(e)):
            raise self.r.err()

    def events(self):
        n = self.r.lib.ref_ledger_events(self.h, None)
        out = np.zeros((n, 5), np.int64)
        self.r.lib.ref_ledger_events(self.h, _p(out))
        return out

    def replay_counts(self, include_zero_use=True):
        n = self.r.lib.ref_ledger_replay_counts(self.h, int(include_zero_use), None, None)
        ids, cnt = np.zeros(n, np.uint64), np.zeros(n, np.uint64)
        self.r.lib.ref_ledger_replay_counts(self.h, int(include_zero_use), _p(ids), _p(cnt))
        return ids, cnt

    def global_use_order(self, rng: "RefRng"):
        n = self.r.lib.ref_ledger_events(self.h, None)
        out = np.zeros(n, np.uint64)
        self.r.lib.ref_ledger_global_use_order(self.h, rng.h, _p(out))
        return out

    def steps_since_last_use(self, rng: "RefRng"):
        n = self.r.lib.ref_ledger_events(self.h, None)
        idx, gap, has = np.zeros(n, np.uint64), np.zeros(n, np.int64), np.zeros(n, np.uint8)
        self.r.lib.ref_ledger_steps_since_last_use(self.h, rng.h, _p(idx), _p(gap), _p(has))
        return idx, gap, has
