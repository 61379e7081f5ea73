"""B200-native replay-step library (arXiv 2604.08706 experience replay).

The hot path — insert/evict, MT19937-64 sampling, ragged token gather, GRPO
group advantage and the clipped / AsymRE losses — runs in hand-written
sm_100a CUDA kernels behind the C-ABI of include/replay_b200.h
(libreplay_b200.so).  This package is a thin mirror of the reference's API
over that ABI; there is no CPU fallback.
"""
from ._lib import LossStats
from .replay import (EVENT_DTYPE, NONE_ID, RECORD_DTYPE, MetricsLedger, Rng, ShardedReplayBuffer,
                     TransferQueue,
                     asymre_records,
                     asymre_tokens, group_advantages, grpo_records, grpo_tokens, hash_name,
                     summarize_hist)

__all__ = ["Rng", "ShardedReplayBuffer", "TransferQueue", "MetricsLedger", "group_advantages", "grpo_tokens", "grpo_records",
           "asymre_tokens", "asymre_records", "hash_name", "RECORD_DTYPE", "EVENT_DTYPE",
           "NONE_ID", "summarize_hist", "LossStats"]
