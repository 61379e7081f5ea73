"""ctypes loader for libreplay_b200.so (the C-ABI in include/replay_b200.h).

The library is the product: there is no CPU fallback.  Importing this module
fails loudly if the shared object is missing; every compute call fails with
RB_ECUDA when no sm_100 device is present.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("REPLAY_B200_LIB", os.path.join(HERE, "libreplay_b200.so"))

RB_OK, RB_EINVAL, RB_ELOGIC, RB_ECUDA, RB_ENOMEM = range(5)
RB_INSERT_ASSUME_UNIQUE = 1

STRATEGIES = {"uniform_with_replacement": 0, "uniform_without_replacement": 1,
              "unused_first_without_replacement": 2,
              # builder extension (include/replay_b200.h RB_PRIORITY_WITH_REPLACEMENT)
              "priority_with_replacement": 3}
STRATEGY_NAMES = {v: k for k, v in STRATEGIES.items()}
RETENTIONS = {"plain_fifo": 0, "positive_bias": 1}
# GRPO normalisation modes (include/replay_b200.h RB_GRPO_*)
GRPO_MODES = {"token_mean": 0, "seq_mean": 1, "seq_ratio": 2}


class Record(C.Structure):  # rb_record, rollout.hpp:13-31
    _fields_ = [("rollout_id", C.c_uint64), ("prompt_id", C.c_uint64), ("group_id", C.c_uint64),
                ("creation_step", C.c_int64), ("policy_version", C.c_int64),
                ("reward", C.c_double), ("is_correct", C.c_uint8),
                ("behavior_logprob", C.c_double), ("advantage", C.c_double),
                ("use_count", C.c_uint32)]


class InsertBatch(C.Structure):  # rb_insert_batch
    _fields_ = [("n", C.c_size_t), ("rollout_id", C.c_void_p), ("prompt_id", C.c_void_p),
                ("group_id", C.c_void_p), ("creation_step", C.c_void_p),
                ("policy_version", C.c_void_p), ("reward", C.c_void_p),
                ("is_correct", C.c_void_p), ("behavior_logprob", C.c_void_p),
                ("advantage", C.c_void_p), ("group_mean", C.c_void_p),
                ("group_offsets", C.c_void_p), ("n_groups", C.c_size_t),
                ("tok_offsets", C.c_void_p), ("tokens", C.c_void_p), ("logp_old", C.c_void_p)]


class LossStats(C.Structure):  # rb_loss_stats
    _fields_ = [("objective_sum", C.c_double), ("objective", C.c_double),
                ("included", C.c_int64), ("excluded", C.c_int64), ("total_tokens", C.c_int64)]


assert C.sizeof(Record) == 80


class ReplayError(Exception):
    """Raised for RB_ELOGIC / RB_ECUDA / RB_ENOMEM."""


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libreplay_b200.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    vp, sz, u64, i64, i32, dbl, ip = (C.c_void_p, C.c_size_t, C.c_uint64, C.c_int64, C.c_int32,
                                      C.c_double, C.c_int)
    sig = {
        "rb_last_error": (C.c_char_p, []),
        "rb_device_info": (ip, [vp, vp, vp, vp]),
        "rb_rng_create": (ip, [u64, vp]),
        "rb_rng_stream": (ip, [vp, C.c_char_p, vp]),
        "rb_rng_stream_index": (ip, [vp, C.c_char_p, u64, vp]),
        "rb_rng_clone": (ip, [vp, vp]),
        "rb_rng_destroy": (None, [vp]),
        "rb_rng_seed": (u64, [vp]),
        "rb_rng_draws": (u64, [vp]),
        "rb_rng_next_u64": (ip, [vp, vp]),
        "rb_rng_below": (ip, [vp, u64, vp]),
        "rb_rng_uniform01": (ip, [vp, vp]),
        "rb_rng_normal": (ip, [vp, vp]),
        "rb_rng_sample_without_replacement": (ip, [vp, u64, u64, vp]),
        "rb_rng_fill_u64": (ip, [vp, u64, vp]),
        "rb_hash_name": (u64, [C.c_char_p]),
        "rb_create": (ip, [sz, sz, ip, ip, dbl, i32, ip, sz, sz, vp]),
        "rb_destroy": (None, [vp]),
        "rb_set_stream": (ip, [vp, vp]),
        "rb_get_stream": (vp, [vp]),
        "rb_push": (ip, [vp, vp, vp, vp, i32, vp, vp]),
        "rb_insert": (ip, [vp, vp, vp, vp, ip]),
        "rb_insert_owned": (ip, [vp, vp, sz, ip]),
        "rb_set_owned_metadata": (ip, [vp, ip]),
        "rb_sample": (ip, [vp, sz, vp, vp, vp, vp, vp, i64, i64]),
        "rb_batch_size": (ip, [vp, vp]),
        "rb_batch_total_tokens": (ip, [vp, vp]),
        "rb_batch_ids": (ip, [vp, vp, vp, vp]),
        "rb_gather": (ip, [vp, vp, vp, vp]),
        "rb_gather_dlpack": (ip, [vp, vp, vp, vp]),
        "rb_dlpack_free": (None, [vp]),
        "rb_set_async_outputs": (ip, [vp, ip]),
        "rb_ledger_create": (ip, [ip, vp]),
        "rb_ledger_destroy": (None, [vp]),
        "rb_ledger_note_generated": (ip, [vp, vp, sz]),
        "rb_ledger_record_batch": (ip, [vp, vp, i64, i64]),
        "rb_ledger_record_uses": (ip, [vp, vp, sz]),
        "rb_ledger_check": (ip, [vp]),
        "rb_ledger_sizes": (ip, [vp, vp, vp]),
        "rb_ledger_events": (ip, [vp, vp, sz, vp]),
        "rb_ledger_replay_counts": (ip, [vp, ip, vp, vp, sz, vp]),
        "rb_ledger_global_use_order": (ip, [vp, vp, vp, sz, vp]),
        "rb_ledger_steps_since_last_use": (ip, [vp, vp, vp, vp, vp, sz, vp]),
        "rb_loss_grpo": (ip, [vp, vp, vp, dbl, dbl, i64, vp]),
        "rb_loss_grpo_ex": (ip, [vp, vp, vp, dbl, dbl, ip, i64, vp]),
        "rb_loss_asymre": (ip, [vp, vp, vp, dbl, i64, vp]),
        "rb_loss_finalize": (ip, [vp, vp, vp]),
        "rb_loss_set_reduce_vector": (ip, [vp, vp]),
        "rb_loss_finalize_vec": (ip, [vp, vp, vp, vp]),
        "rb_allreduce_loss_stats": (ip, [vp, vp, vp, vp]),
        "rb_num_shards": (ip, [vp, vp]),
        "rb_total_capacity": (ip, [vp, vp]),
        "rb_shard_capacity": (ip, [vp, vp]),
        "rb_size": (ip, [vp, vp]),
        "rb_shard_size": (ip, [vp, sz, vp]),
        "rb_shard_contents": (ip, [vp, sz, vp, sz, vp]),
        "rb_record_tokens": (ip, [vp, sz, sz, vp, vp, i32, vp]),
        "rb_strategy": (ip, [vp, vp]),
        "rb_retention": (ip, [vp, vp, vp]),
        "rb_set_priority": (ip, [vp, C.c_uint32, C.c_uint32, C.c_uint32]),
        "rb_get_priority": (ip, [vp, vp, vp, vp]),
        "rb_priority_mass": (ip, [vp, vp]),
        "rb_allreduce_priority_mass": (ip, [vp, vp, vp]),
        "rb_route_cursor": (ip, [vp, vp]),
        "rb_dump": (ip, [vp, C.c_char_p, sz, vp]),
        "rb_load": (ip, [C.c_char_p, i32, ip, vp]),
        "rb_batch_staleness_hist": (ip, [vp, i64, i32, vp, vp]),
        "rb_use_count_hist": (ip, [vp, i32, vp, vp]),
        "rb_snapshot": (ip, [vp, vp, sz, vp]),
        "rb_restore": (ip, [vp, vp, sz]),
        "rb_rng_get_state": (ip, [vp, vp, vp, vp]),
        "rb_rng_set_state": (ip, [vp, vp, C.c_uint32, u64]),
        "rb_queue_create": (ip, [sz, i32, ip, vp]),
        "rb_queue_destroy": (None, [vp]),
        "rb_queue_push_group": (ip, [vp, vp, vp]),
        "rb_queue_pop": (ip, [vp, sz, vp, vp, vp, vp, vp]),
        "rb_queue_size": (ip, [vp, vp]),
        "rb_queue_capacity": (ip, [vp, vp, vp]),
        "rb_check": (ip, [vp]),
        "rb_synchronize": (ip, [vp]),
        "rb_group_advantages": (ip, [vp, vp, sz, vp, vp]),
        "rb_grpo_tokens": (ip, [vp, vp, vp, vp, sz, dbl, dbl, vp, vp]),
        "rb_grpo_tokens_ex": (ip, [vp, vp, vp, vp, vp, sz, dbl, dbl, ip, vp, vp]),
        "rb_grpo_records": (ip, [vp, vp, vp, sz, dbl, dbl, vp, vp]),
        "rb_asymre_tokens": (ip, [vp, vp, vp, vp, sz, dbl, vp, vp]),
        "rb_asymre_records": (ip, [vp, vp, vp, sz, dbl, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()
EXPORTED = ("rb_last_error", "rb_device_info", "rb_rng_create", "rb_create", "rb_insert",
            "rb_sample", "rb_gather", "rb_loss_grpo", "rb_loss_asymre")


def check(status: int) -> None:
    if status == RB_OK:
        return
    msg = lib.rb_last_error().decode()
    if status == RB_EINVAL:
        raise ValueError(msg)  # std::invalid_argument in the reference
    raise ReplayError(f"[{status}] {msg}")
