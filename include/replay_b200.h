/* replay_b200.h — C-ABI of the B200 replay-step library (libreplay_b200.so).
 *
 * This is the drop-in boundary for the reference's replay path.  The
 * reference (/root/reference/proj, C++20, CPU only) has no FFI: its operator
 * API is the C++ headers.  Each entry point below names the reference
 * interface it replaces (file:line relative to /root/reference/proj); the
 * C++ facade in paper_2604_08706_b200/facade/replab/ (one .hpp per header) re-exposes the
 * reference's own class/function signatures on top of this ABI (see
 * INTEGRATION.md for the bindings a maintainer would add).
 *
 * Conventions
 *   - Plain pointers and sizes only.  Every status-returning call returns
 *     RB_OK (0) or an error code; rb_last_error() gives the thread-local
 *     message, identical to the reference's std::invalid_argument text where
 *     the reference throws (the facade re-throws it with the same type).
 *   - Array arguments may point to device memory (the hot path) or to host
 *     memory (staged through pinned buffers inside the call); the library
 *     classifies each pointer with cudaPointerGetAttributes.  Packed token
 *     arrays must be 16-byte aligned and readable up to the next 16-byte
 *     boundary (true of any cudaMalloc / torch allocation).
 *   - All work is enqueued on the buffer's CUDA stream (rb_set_stream); calls
 *     that return host-visible results synchronise that stream.
 *   - No CPU fallback: every compute entry point runs a CUDA kernel and fails
 *     with RB_ECUDA when no sm_100 device is present.
 */
#ifndef REPLAY_B200_H
#define REPLAY_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the ABI is exported; internals are hidden */
#endif
#ifdef __cplusplus
extern "C" {
#endif

/* ---- status ------------------------------------------------------------ */
enum {
    RB_OK = 0,
    RB_EINVAL = 1, /* std::invalid_argument in the reference */
    RB_ELOGIC = 2, /* std::logic_error in the reference */
    RB_ECUDA = 3,  /* CUDA runtime failure / no device */
    RB_ENOMEM = 4
};
const char* rb_last_error(void);
/* Library / device info: compiled arch and the device the library runs on. */
int rb_device_info(int* device, int* sm_count, int* cc_major, int* cc_minor);

/* ---- enums (replay_buffer.hpp:17-46) ------------------------------------ */
enum { RB_UNIFORM_WITH_REPLACEMENT = 0, RB_UNIFORM_WITHOUT_REPLACEMENT = 1,
       RB_UNUSED_FIRST_WITHOUT_REPLACEMENT = 2,
       /* builder extension (no reference counterpart): per
        * shard B/T draws with probability w_i / W, see rb_set_priority */
       RB_PRIORITY_WITH_REPLACEMENT = 3 };
enum { RB_PLAIN_FIFO = 0, RB_POSITIVE_BIAS = 1 };

/* ---- record (rollout.hpp:13-31; same 80-byte layout) -------------------- */
typedef struct rb_record {
    uint64_t rollout_id;
    uint64_t prompt_id;
    uint64_t group_id;
    int64_t creation_step;
    int64_t policy_version;
    double reward;
    uint8_t is_correct;
    double behavior_logprob;
    double advantage;
    uint32_t use_count;
} rb_record;

/* One selection of sample() with a ledger (metrics.hpp:22-34 UseEvent). */
typedef struct rb_use_event {
    uint64_t rollout_id;
    int64_t creation_step;
    int64_t use_step;
    int64_t batch_id;
    int64_t within_batch_rank;
} rb_use_event;

/* ======================================================================
 * Rng — replaces replab::Rng (rng.hpp:22-69, rng.cpp:25-121).
 * The engine is MT19937-64 reproduced bit-exactly; its 312-word state lives
 * on the GPU while the sampler consumes it and migrates to the host only
 * when a host-side draw is requested (rng.cpp:38-55 semantics).
 * ==================================================================== */
typedef struct rb_rng rb_rng;
int rb_rng_create(uint64_t seed, rb_rng** out);                         /* rng.hpp:24 */
int rb_rng_stream(const rb_rng* parent, const char* name, rb_rng** out); /* rng.hpp:30 */
int rb_rng_stream_index(const rb_rng* parent, const char* name, uint64_t index,
                        rb_rng** out);                                  /* rng.hpp:31 */
int rb_rng_clone(const rb_rng* r, rb_rng** out); /* value copy (Rng is copyable) */
void rb_rng_destroy(rb_rng* r);
uint64_t rb_rng_seed(const rb_rng* r);                                  /* rng.hpp:33 */
uint64_t rb_rng_draws(const rb_rng* r); /* raw engine outputs consumed so far */
int rb_rng_next_u64(rb_rng* r, uint64_t* out);                          /* rng.hpp:35 */
int rb_rng_below(rb_rng* r, uint64_t bound, uint64_t* out);             /* rng.hpp:38 */
int rb_rng_uniform01(rb_rng* r, double* out);                           /* rng.hpp:41 */
int rb_rng_normal(rb_rng* r, double* out);                              /* rng.hpp:46 */
int rb_rng_sample_without_replacement(rb_rng* r, uint64_t n, uint64_t k,
                                      uint64_t* out);                   /* rng.hpp:56 */
/* Engine position for checkpoints (the reference's Rng has none, rng.hpp:26-31):
 * the 312 state words, the index of the next word and the outputs consumed. */
int rb_rng_get_state(rb_rng* r, uint64_t* mt312, uint32_t* idx, uint64_t* draws);
int rb_rng_set_state(rb_rng* r, const uint64_t* mt312, uint32_t idx, uint64_t draws);
/* Device bulk generation: n raw engine outputs into out (device or host),
 * produced by the GPU generator (parity aid for the sampler's stream). */
int rb_rng_fill_u64(rb_rng* r, uint64_t n, uint64_t* out);
uint64_t rb_hash_name(const char* name);                                /* rng.hpp:11 */

/* ======================================================================
 * ShardedReplayBuffer — replaces replab::ShardedReplayBuffer
 * (replay_buffer.hpp:57-108, replay_buffer.cpp:67-324) with an HBM-resident
 * SoA store: per-slot metadata columns plus fixed-stride token payload
 * slots {int32 token, fp32 logp_old} of max_tokens per trajectory.
 * ==================================================================== */
typedef struct rb_buffer rb_buffer;

/* replay_buffer.cpp:67-81 (+ RetentionPolicy::positive_bias 38-46).
 * max_tokens: payload stride (>= the longest trajectory; 0 = metadata only).
 * device: CUDA ordinal; -1 = current device.
 * shard_begin/shard_end: shards whose token payload this process holds
 * (multi-GPU: one shard per rank; metadata is replicated on every rank).
 * Pass 0,0 for "all shards". */
int rb_create(size_t num_shards, size_t total_capacity, int strategy, int retention,
              double delta, int32_t max_tokens, int device, size_t shard_begin,
              size_t shard_end, rb_buffer** out);
void rb_destroy(rb_buffer* b);
/* Enqueue on the given CUDA stream (cudaStream_t as void*; NULL = the legacy
 * default stream).  Buffers start on a library-owned non-blocking stream. */
int rb_set_stream(rb_buffer* b, void* stream);
/* Asynchronous host outputs (off by default): a loss whose out_dlogp is
 * pinned host memory returns once its stats are final while the dlogp
 * download drains on a copy stream beside the caller's next call (e.g. the
 * next insert's upload, the other PCIe direction); a gather into pinned host
 * arrays returns once its offsets are on the host while the packed tokens /
 * logp_old drain the same way (beside the loss's logp_now upload).  The host
 * arrays are complete after rb_synchronize (or cudaDeviceSynchronize). */
int rb_set_async_outputs(rb_buffer* b, int on);
void* rb_get_stream(rb_buffer* b);

/* push (replay_buffer.cpp:83-96): one record, synchronous.  Rejects an id
 * present in any shard before mutating.  *has_evicted = 1 and *evicted set
 * when the shard's retention policy evicted a record.  Optional payload
 * (tokens/logp_old of n_tokens, host or device; NULL = no payload). */
int rb_push(rb_buffer* b, const rb_record* rec, const int32_t* tokens, const float* logp_old,
            int32_t n_tokens, rb_record* evicted, int* has_evicted);

/* Batched insert of whole trajectories — the hot path of the replay step.
 * Semantics are exactly n sequential push() calls (routing, eviction,
 * duplicate rejection).  If advantage == NULL the group-relative advantage
 * (bandit.cpp:276-294) and the group mean reward (bandit.cpp:316-318) are
 * computed on the device over the groups delimited by group_offsets
 * (n_groups+1 entries) and frozen into the stored records; otherwise the
 * given advantages are stored and group_mean (may be NULL) is taken as the
 * AsymRE baseline.  tok_offsets has n+1 entries into tokens/logp_old.
 * out_evicted_ids[j] = id evicted by push j or UINT64_MAX (may be NULL).
 * flags: RB_INSERT_ASSUME_UNIQUE promises ids are new and strictly
 * increasing (verified on the device; a violation is a sticky RB_EINVAL
 * reported by the next synchronising call).  Without it the call
 * synchronises and, on a duplicate at push j, applies pushes [0, j) and
 * returns RB_EINVAL with *out_applied = j. */
enum { RB_INSERT_ASSUME_UNIQUE = 1 };
typedef struct rb_insert_batch {
    size_t n;
    const uint64_t* rollout_id;
    const uint64_t* prompt_id;
    const uint64_t* group_id;
    const int64_t* creation_step;
    const int64_t* policy_version;
    const double* reward;
    const uint8_t* is_correct; /* NULL = (reward == 1.0) */
    const double* behavior_logprob;
    const double* advantage;   /* NULL = compute per group on the device */
    const double* group_mean;  /* used when advantage != NULL; may be NULL */
    const int64_t* group_offsets;
    size_t n_groups;
    const int64_t* tok_offsets; /* n+1; NULL = no payload */
    const int32_t* tokens;
    const float* logp_old;
} rb_insert_batch;
int rb_insert(rb_buffer* b, const rb_insert_batch* batch, uint64_t* out_evicted_ids,
              size_t* out_applied, int flags);

/* Owned metadata (multi-GPU): a buffer holding ONE shard of
 * 2..64 (shard_begin + 1 == shard_end; FIFO, uniform draws with
 * replacement) keeps the metadata of its own records only.  After
 * rb_set_owned_metadata(b, 1), rb_insert_owned(b, batch, n_global, flags)
 * takes only the records the reference's round robin (replay_buffer.cpp:
 * 89-90) routes to the owned shard out of a global batch of n_global — in
 * arrival order, with their advantages (a group spans every rank's shard),
 * ids promised unique — and advances every shard's push count; the sampler
 * still draws the whole MT19937-64 stream (an earlier shard's below()
 * rejection shifts this shard's draws; occupancies are closed-form) but maps
 * only the owned slice [s*B/T, (s+1)*B/T): use counts, lengths, packed
 * offsets.  The loss normalises by the rank's own tokens until the
 * all-reduced {objective_sum, included, excluded} arrives
 * (rb_allreduce_loss_stats / rb_loss_finalize_vec rescale dlogp to the
 * global count).  Inspection of other shards returns stale metadata. */
int rb_set_owned_metadata(rb_buffer* b, int on);
int rb_insert_owned(rb_buffer* b, const rb_insert_batch* batch, size_t n_global, int flags);

/* sample (replay_buffer.cpp:184-217): batch_size/num_shards draws per shard
 * in shard order 0..T-1 from rng (replay_buffer.cpp:135-182), use counts
 * incremented.  The selection is kept inside the buffer as the "current
 * batch" for rb_gather / rb_loss_* (device-resident).  Optional outputs
 * (host or device, may be NULL): record copies carrying the post-increment
 * use count, (shard, arrival index) pairs, UseEvents (metrics.hpp:22-34).
 * On an error the shards before the failing one are already mutated, as in
 * the reference.  Asynchronous unless a host output is requested. */
int rb_sample(rb_buffer* b, size_t batch_size, rb_rng* rng, rb_record* out_records,
              int64_t* out_shard, int64_t* out_index, rb_use_event* out_events,
              int64_t batch_id, int64_t use_step);

/* Current batch: number of selections, total tokens (sync), device views. */
int rb_batch_size(const rb_buffer* b, size_t* n);
int rb_batch_total_tokens(rb_buffer* b, int64_t* total);
/* Per-selection rollout ids / lengths / packed offsets (n+1) into caller arrays. */
int rb_batch_ids(rb_buffer* b, uint64_t* out_ids, int32_t* out_lengths, int64_t* out_offsets);

/* Ragged token gather of the current batch: packs the sampled trajectories'
 * tokens (and optionally logp_old) contiguously in selection order;
 * out_offsets (n+1, may be NULL) = exclusive scan of lengths.  No reference
 * counterpart (the reference has no tokens). */
int rb_gather(rb_buffer* b, int32_t* out_tokens, float* out_logp_old, int64_t* out_offsets);
/* Zero-copy hand-off of the packed batch (SURVEY.md §8f producer/consumer
 * edge): gathers this buffer's selections into library-owned device arrays
 * and returns them as DLPack tensors (DLManagedTensor*, DLPack ABI v0.8:
 * int32 tokens [total], float32 logp_old [total], int64 offsets [n+1]) that
 * any DLPack consumer (torch.from_dlpack, cupy, jax) takes over without a
 * copy; the consumer calls each tensor's deleter.  Synchronises the buffer's
 * stream (the shapes are device values).  Any output pointer may be NULL. */
int rb_gather_dlpack(rb_buffer* b, void** out_tokens, void** out_logp_old, void** out_offsets);
/* Releases an exported tensor nobody consumed (calls its deleter). */
void rb_dlpack_free(void* managed_tensor);

/* Loss statistics of one step (bandit.hpp:127-131 LossResult, token form). */
typedef struct rb_loss_stats {
    double objective_sum; /* sum of per-unit objective terms */
    double objective;     /* objective_sum / included (GRPO) or / B (AsymRE) */
    int64_t included;
    int64_t excluded;
    int64_t total_tokens;
} rb_loss_stats;

/* GRPO clipped surrogate over the current batch, per token
 * (grpo_loss_grad, bandit.cpp:363-408): ratio = exp(logp_now - logp_old),
 * non-finite ratios excluded, clip to [1-eps_low, 1+eps_high], ties take the
 * unclipped branch; out_dlogp = d(-objective)/d logp_now, normalised by the
 * included token count.  logp_now/out_dlogp are packed in gather order.
 * stats (host or device, may be NULL).  Multi-GPU: pass norm_tokens = the
 * global token count (0 = this buffer's batch) and reduce `stats` across
 * ranks, then call rb_loss_finalize with the reduced stats. */
int rb_loss_grpo(rb_buffer* b, const float* logp_now, float* out_dlogp, double eps_low,
                 double eps_high, int64_t norm_tokens, rb_loss_stats* stats);
/* GRPO normalisation modes (SURVEY.md §8c token generalisation; the
 * reference has no tokens):
 *   RB_GRPO_TOKEN_MEAN  per-token ratio, mean over the batch's included
 *                       tokens (rb_loss_grpo);
 *   RB_GRPO_SEQ_MEAN    per-token ratio, mean over each sequence's included
 *                       tokens, then over the sequences with one or more;
 *   RB_GRPO_SEQ_RATIO   sequence-level ratio pi(z|q)/pi_old(z|q) =
 *                       exp(sum_t logp_now_t - behavior_logprob) (PAPER.md
 *                       :1022-1025): the reference's record-level
 *                       grpo_loss_grad (bandit.cpp:363-408) per trajectory,
 *                       its dL/dlogp on every token.
 * In the sequence modes stats.included / excluded count sequences (mode 2)
 * or included sequences / excluded tokens (mode 1) and `norm` (0 = the batch
 * size) is the global sequence count used as the normaliser. */
enum { RB_GRPO_TOKEN_MEAN = 0, RB_GRPO_SEQ_MEAN = 1, RB_GRPO_SEQ_RATIO = 2 };
int rb_loss_grpo_ex(rb_buffer* b, const float* logp_now, float* out_dlogp, double eps_low,
                    double eps_high, int mode, int64_t norm, rb_loss_stats* stats);
/* AsymRE (asymre_loss_grad, bandit.cpp:410-438): coef = reward - (group
 * mean + delta_v); dlogp = -coef / norm_batch on every token; objective =
 * sum coef * sum_t logp_now / norm_batch.  norm_batch 0 = this batch size. */
int rb_loss_asymre(rb_buffer* b, const float* logp_now, float* out_dlogp, double delta_v,
                   int64_t norm_batch, rb_loss_stats* stats);
/* Re-normalise out_dlogp after a cross-rank reduction of stats (only does
 * work when excluded > 0; objective recomputed).  Device or host stats. */
int rb_loss_finalize(rb_buffer* b, float* dlogp, rb_loss_stats* stats);
/* The same reduction with ONE collective: once a device vector of three
 * doubles is registered, every loss call also writes {objective_sum,
 * included, excluded} into it (counts exact below 2^53); the caller
 * all-reduces it (sum) across ranks and calls rb_loss_finalize_vec, which
 * applies the global normalisation in one kernel and fills `stats` (host,
 * device or NULL).  vec3 = NULL unregisters. */
int rb_loss_set_reduce_vector(rb_buffer* b, double* vec3);
int rb_loss_finalize_vec(rb_buffer* b, float* dlogp, const double* vec3, rb_loss_stats* stats);
/* The collective itself (SURVEY.md §8b `rb_allreduce_loss_stats(comm, ...)`):
 * ncclAllReduce (sum, in place, on the buffer's stream) of the registered
 * vector across the communicator's ranks, then rb_loss_finalize_vec.
 * nccl_comm is an ncclComm_t of the NCCL library loaded in the process
 * (e.g. torch's ProcessGroupNCCL `_comm_ptr()`); libnccl.so.2 is resolved at
 * run time, never linked.  RB_ELOGIC without a registered vector.  The
 * reference runs its shards in one process and needs no collective
 * (async_sim.cpp:138-139, bandit.cpp:363-408 over the whole batch). */
int rb_allreduce_loss_stats(rb_buffer* b, void* nccl_comm, float* dlogp, rb_loss_stats* stats);

/* Inspection (replay_buffer.hpp:74-84). */
int rb_num_shards(const rb_buffer* b, size_t* out);
int rb_total_capacity(const rb_buffer* b, size_t* out);
int rb_shard_capacity(const rb_buffer* b, size_t* out);
int rb_size(rb_buffer* b, size_t* out);                      /* replay_buffer.cpp:219-226 */
int rb_shard_size(rb_buffer* b, size_t shard, size_t* out);  /* 228-231 */
/* shard_contents (233-236): arrival order, oldest first; returns count. */
int rb_shard_contents(rb_buffer* b, size_t shard, rb_record* out, size_t capacity,
                      size_t* count);
/* Token payload of one stored record (by shard + arrival index). */
int rb_record_tokens(rb_buffer* b, size_t shard, size_t index, int32_t* tokens,
                     float* logp_old, int32_t capacity, int32_t* n_tokens);
int rb_strategy(const rb_buffer* b, int* out);
int rb_retention(const rb_buffer* b, int* kind, double* delta);
/* priority_with_replacement (builder extension; the reference's sampler is
 * uniform, replay_buffer.cpp:135-182, and its "positive bias" is a retention
 * rule).  Record weight w = base + floor(min(|advantage|, 2^15) * adv_scale)
 * + pos_bonus * [reward > 0] (integers: the per-shard CDF is exact); each
 * draw is index = upper_bound(cdf, rng.below(W)) over the shard's arrival
 * order, shards in order, B/T draws each as rb_sample.  Defaults (1, 0, 0)
 * reproduce uniform_with_replacement draw for draw.  base >= 1 (every
 * record stays reachable), adv_scale <= 65536.  The weights are a setting
 * of the buffer object, not of its contents: rb_dump / rb_snapshot do not
 * carry them (set them again after rb_load / rb_restore). */
int rb_set_priority(rb_buffer* b, uint32_t base, uint32_t adv_scale, uint32_t pos_bonus);
int rb_get_priority(const rb_buffer* b, uint32_t* base, uint32_t* adv_scale, uint32_t* pos_bonus);
/* Priority mass per shard: out[s] = W_s = sum of the weights of shard s's
 * records for the shards this process holds ([shard_begin, shard_end) of
 * rb_create), 0 for the others (uint64, exact).  Host or device out[num_shards]. */
int rb_priority_mass(rb_buffer* b, uint64_t* out);
/* The priority-mass all-reduce (north star): rb_priority_mass into the
 * device vector masses[num_shards], then ncclAllReduce(sum, uint64) in place
 * on the buffer's stream through the caller's communicator (ncclComm_t, as
 * rb_allreduce_loss_stats), so every rank holds every shard's mass.  The
 * sampler itself needs no collective: it draws B/T per shard from the
 * shard's own CDF (replay_buffer.cpp:193-204). */
int rb_allreduce_priority_mass(rb_buffer* b, void* nccl_comm, uint64_t* masses);
int rb_route_cursor(rb_buffer* b, size_t* out);

/* dump/load (replay_buffer.cpp:238-324): byte-identical text format.
 * rb_dump writes at most cap bytes (NUL-terminated) and sets *len to the
 * full length; call with out=NULL to size. */
int rb_dump(rb_buffer* b, char* out, size_t cap, size_t* len);
int rb_load(const char* text, int32_t max_tokens, int device, rb_buffer** out);

/* Replay diagnostics on the device (the reference derives
 * them from the UseEvent ledger on the host, metrics.cpp:37-44, 123-131,
 * 185-202).  Integer-valued metrics as histograms of bins 0..max_bin (the last
 * bin counts every value >= max_bin), from which the reference's summarize()
 * (mean, nearest-rank quartiles) follows exactly while no value reaches
 * max_bin:
 *   rb_batch_staleness_hist — staleness(e) = use_step - creation_step of
 *     every selection of the current batch (metrics.cpp:37-39);
 *   rb_use_count_hist       — use counts of the resident records (replay
 *     counts so far, replay_buffer.cpp:201). */
int rb_batch_staleness_hist(rb_buffer* b, int64_t use_step, int32_t max_bin, uint64_t* hist,
                            int64_t* sum);
int rb_use_count_hist(rb_buffer* b, int32_t max_bin, uint64_t* hist, uint64_t* sum);

/* ---- the UseEvent ledger on the device (metrics.hpp:36-93) -------------
 * Replaces MetricsLedger + replay_counts / global_use_order /
 * steps_since_last_use (metrics.cpp:44-69, 123-170).  Events are SoA device
 * arrays; record_batch appends the buffer's current batch from a kernel on
 * the buffer's stream (call it after rb_sample*, before the next insert).
 * Generated twice / duplicate (batch, rank) fail at the call with the
 * reference's messages; a use before creation is detected on the device and
 * reported (RB_EINVAL) by the next rb_ledger_* call that synchronises, which
 * then holds the events recorded before the offending one — the reference's
 * state after its throw.  Output arrays may be host or device memory. */
typedef struct rb_ledger rb_ledger;
int rb_ledger_create(int device, rb_ledger** out);
void rb_ledger_destroy(rb_ledger* l);
int rb_ledger_note_generated(rb_ledger* l, const uint64_t* ids, size_t n);        /* metrics.cpp:44-53 */
int rb_ledger_record_batch(rb_ledger* l, rb_buffer* b, int64_t batch_id, int64_t use_step);
                                                             /* replay_buffer.cpp:205-215 */
int rb_ledger_record_uses(rb_ledger* l, const rb_use_event* events, size_t n);   /* metrics.cpp:56-69 */
int rb_ledger_check(rb_ledger* l);
int rb_ledger_sizes(rb_ledger* l, size_t* n_events, size_t* n_generated);
int rb_ledger_events(rb_ledger* l, rb_use_event* out, size_t cap, size_t* n);
/* metrics.cpp:123-131: ascending ids and their use counts (generated ids
 * never used at 0 when include_zero_use); call with NULL outputs to size. */
int rb_ledger_replay_counts(rb_ledger* l, int include_zero_use, uint64_t* out_ids,
                            uint64_t* out_counts, size_t cap, size_t* n);
/* metrics.cpp:133-151: event indices in global use order; consumes rng
 * exactly like Rng::shuffle of every batch (rng.hpp:59-64). */
int rb_ledger_global_use_order(rb_ledger* l, rb_rng* rng, uint64_t* out_order, size_t cap,
                               size_t* n);
/* metrics.cpp:153-170: per position of the global use order, the event
 * index and the gap to the rollout's previous use (has_gap 0 = first use). */
int rb_ledger_steps_since_last_use(rb_ledger* l, rb_rng* rng, uint64_t* out_event_index,
                                   int64_t* out_gap, uint8_t* out_has_gap, size_t cap, size_t* n);

/* Binary checkpoint of the whole device state — metadata columns, arrival
 * structures (positive-bias queues), owned token payload rows, route cursor,
 * per-shard push counts — for run resumption (the
 * reference persists only the text dump above, replay_buffer.cpp:238-324,
 * SPEC.md:113-114).  dst / src may be host or device memory.  rb_snapshot
 * with dst = NULL only sets *len.  rb_restore requires a buffer of the same
 * shape (shards, capacity, strategy, retention, max_tokens, owned shards). */
int rb_snapshot(rb_buffer* b, void* dst, size_t cap, size_t* len);
int rb_restore(rb_buffer* b, const void* src, size_t len);

/* ======================================================================
 * TransferQueue — replaces replab::TransferQueue (transfer_queue.hpp:12-35,
 * transfer_queue.cpp:1-50), the consume-once LIFO of the no-buffer
 * baseline, with the token payload kept in HBM next to the records.
 * ==================================================================== */
typedef struct rb_queue rb_queue;
/* capacity 0 = unbounded (the reference's nullopt; device storage grows). */
int rb_queue_create(size_t capacity, int32_t max_tokens, int device, rb_queue** out);
void rb_queue_destroy(rb_queue* q);
/* push_group (transfer_queue.cpp:22-29): all or nothing; *accepted = 0 when
 * the group does not fit (back-pressure, nothing enqueued).  A single push is
 * a group of one (13-20).  Advantages: given, or per group on the device. */
int rb_queue_push_group(rb_queue* q, const rb_insert_batch* batch, int* accepted);
/* k pops (31-39): up to k most recent records, most recent first; optional
 * packed payload + offsets (host or device).  *n_popped = 0: empty queue. */
int rb_queue_pop(rb_queue* q, size_t k, rb_record* out_records, size_t* n_popped,
                 int32_t* out_tokens, float* out_logp_old, int64_t* out_offsets);
int rb_queue_size(const rb_queue* q, size_t* out);                       /* 41-44 */
int rb_queue_capacity(const rb_queue* q, size_t* capacity, int* bounded); /* hpp:31 */

/* Sticky asynchronous error check (synchronises the stream). */
int rb_check(rb_buffer* b);
int rb_synchronize(rb_buffer* b);

/* ======================================================================
 * Stateless kernels over explicit arrays (host or device pointers).
 * ==================================================================== */
/* group_advantages (bandit.cpp:276-294), segmented: groups delimited by
 * offsets (n_groups+1).  Bit-exact fp64.  out_mean (may be NULL) = group
 * mean reward (bandit.cpp:316-318).  Every group needs >= 2 rewards. */
int rb_group_advantages(const double* rewards, const int64_t* offsets, size_t n_groups,
                        double* out_adv, double* out_mean);
/* grpo_loss_grad at the token level over explicit arrays (offsets n+1). */
int rb_grpo_tokens(const float* logp_now, const float* logp_old, const double* adv,
                   const int64_t* offsets, size_t n_traj, double eps_low, double eps_high,
                   float* out_dlogp, rb_loss_stats* stats);
/* The same with a normalisation mode; behavior_logprob (n_traj, may be NULL
 * = sum_t logp_old) is the record's sequence log-prob for RB_GRPO_SEQ_RATIO. */
int rb_grpo_tokens_ex(const float* logp_now, const float* logp_old, const double* adv,
                      const double* behavior_logprob, const int64_t* offsets, size_t n_traj,
                      double eps_low, double eps_high, int mode, float* out_dlogp,
                      rb_loss_stats* stats);
/* Record-level fp64 form (L = 1): the reference's grpo_loss_grad per record. */
int rb_grpo_records(const double* logp_now, const double* behavior_logprob,
                    const double* adv, size_t n, double eps_low, double eps_high,
                    double* out_dlogp, rb_loss_stats* stats);
int rb_asymre_tokens(const float* logp_now, const double* reward, const double* group_mean,
                     const int64_t* offsets, size_t n_traj, double delta_v,
                     float* out_dlogp, rb_loss_stats* stats);
int rb_asymre_records(const double* logp_now, const double* reward, const double* group_mean,
                      size_t n, double delta_v, double* out_dlogp, rb_loss_stats* stats);

#ifdef __cplusplus
}
#endif
#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif /* REPLAY_B200_H */
