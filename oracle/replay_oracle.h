/* replay_oracle.h — CPU restatement of the reference replay-step path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2604_08706_b200/,
 * include/replay_b200.h) links or calls this; only tests/, the smoke() check
 * in __graft_entry__.py and the cpu_baseline / --impl reference legs of
 * bench.py use it, and only as the checker / the CPU baseline.
 *
 * Parity is PINNED: every function below restates a reference function
 * (file:line under /root/reference/proj) and the restatement is checked
 *   (1) against the compiled, unmodified reference (oracle/_ref, built by
 *       oracle/Makefile from the reference's own sources), and
 *   (2) against committed golden fixtures (tests/golden/, generated from the
 *       compiled reference by tests/golden/make_golden.py) and the
 *       reference tests' own known answers.
 */
#ifndef REPLAY_ORACLE_H
#define REPLAY_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp / rng.cpp ------------------------------------------------- */
typedef struct or_rng {
    uint64_t mt[312];
    uint32_t idx;
    uint64_t seed;
    uint64_t draws; /* raw engine outputs consumed (debug / parity aid) */
} or_rng;

uint64_t or_hash_name(const char* name, size_t len);            /* rng.cpp:8-15  */
uint64_t or_splitmix64(uint64_t* state);                        /* rng.cpp:17-23 */
void or_rng_init(or_rng* r, uint64_t seed);                     /* rng.cpp:25    */
void or_rng_stream(const or_rng* p, const char* name, size_t len, or_rng* out);       /* 27-30 */
void or_rng_stream_idx(const or_rng* p, const char* name, size_t len, uint64_t index,
                       or_rng* out);                            /* rng.cpp:32-36 */
uint64_t or_rng_next(or_rng* r);                                /* rng.cpp:38    */
int or_rng_below(or_rng* r, uint64_t bound, uint64_t* out);     /* rng.cpp:40-51 */
double or_rng_uniform01(or_rng* r);                             /* rng.cpp:53-55 */
double or_rng_normal(or_rng* r);                                /* rng.cpp:59-70 */
int or_rng_swor(or_rng* r, size_t n, size_t k, uint64_t* out);  /* rng.cpp:108-121 */
void or_rng_discard(or_rng* r, uint64_t n);

/* ---- rollout.hpp:13-31 (80-byte record, same layout as rb_record) ------- */
typedef struct or_record {
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
} or_record;

/* ---- replay_buffer.hpp / replay_buffer.cpp ------------------------------ */
enum { OR_UNIFORM_WITH = 0, OR_UNIFORM_WITHOUT = 1, OR_UNUSED_FIRST = 2, OR_PRIORITY_WITH = 3 };
enum { OR_FIFO = 0, OR_POSITIVE_BIAS = 1 };
enum { OR_OK = 0, OR_INVALID = 1 };

typedef struct or_buffer or_buffer;

/* replay_buffer.cpp:67-81; NULL on invalid config (message via or_last_error) */
or_buffer* or_buf_new(size_t num_shards, size_t total_capacity, int strategy, int retention,
                      double delta);
void or_buf_free(or_buffer* b);
/* replay_buffer.cpp:83-133 */
int or_buf_push(or_buffer* b, const or_record* rec, or_record* evicted, int* has_evicted);
/* replay_buffer.cpp:135-217.  out_shard/out_index may be NULL.  On error the
 * shards before the failing one are already mutated (as in the reference).  */
/* priority_with_replacement weights (builder extension; rb_set_priority) */
int or_buf_set_priority(or_buffer* b, uint32_t base, uint32_t adv_scale, uint32_t pos_bonus);
int or_buf_sample(or_buffer* b, size_t batch, or_rng* rng, or_record* out, int64_t* out_shard,
                  int64_t* out_index);
size_t or_buf_size(const or_buffer* b);
size_t or_buf_shard_size(const or_buffer* b, size_t shard);
size_t or_buf_shard_contents(const or_buffer* b, size_t shard, or_record* out);
size_t or_buf_route_cursor(const or_buffer* b);
const char* or_last_error(void);

/* ---- bandit.cpp --------------------------------------------------------- */
/* bandit.cpp:276-294 */
int or_group_advantages(const double* rewards, size_t n, double* out);

/* Token-level generalisation of grpo_loss_grad (bandit.cpp:363-408): one
 * importance ratio per token, computed in fp64 from the fp32 inputs;
 * excluded/included counted per token; normalisation = mean over included
 * tokens; dlogp = dL/dlogp_now of the NEGATED objective, rounded to fp32.
 * `adv` is per trajectory; offsets has n_traj+1 entries.  At L=1 this is
 * exactly the reference's per-record loss.  */
void or_loss_grpo_tokens(const float* logp_now, const float* logp_old, const double* adv,
                         const int64_t* offsets, size_t n_traj, double eps_low,
                         double eps_high, float* dlogp, double* objective, int64_t* included,
                         int64_t* excluded);
/* GRPO normalisation modes (0 token mean, 1 per-sequence mean, 2 sequence
 * ratio); see replay_oracle.c.  blp may be NULL (sum of logp_old). */
void or_loss_grpo_tokens_mode(const float* logp_now, const float* logp_old, const double* adv,
                              const double* blp, const int64_t* offsets, size_t n_traj,
                              double eps_low, double eps_high, int mode, float* dlogp,
                              double* objective, int64_t* included, int64_t* excluded);
/* Same over fp64 per-record inputs with fp64 output (the L=1 record form). */
void or_loss_grpo_records(const double* logp_now, const double* behavior_logprob,
                          const double* adv, size_t n, double eps_low, double eps_high,
                          double* dlogp, double* objective, int64_t* included,
                          int64_t* excluded);
/* Token-level asymre_loss_grad (bandit.cpp:410-438): coef_i = reward_i -
 * (group_mean_i + delta_v); objective = sum_i coef_i * sum_t logp_now / B;
 * dlogp = -coef_i / B on every token of trajectory i.  */
void or_loss_asymre_tokens(const float* logp_now, const double* reward,
                           const double* group_mean, const int64_t* offsets, size_t n_traj,
                           double delta_v, float* dlogp, double* objective);
void or_loss_asymre_records(const double* logp_now, const double* reward,
                            const double* group_mean, size_t n, double delta_v, double* dlogp,
                            double* objective);

/* train()'s production schedule (bandit.cpp:617-640): returns the number of
 * whole groups pushed this step and updates *debt. */
int64_t or_production_groups(double per_step_production, size_t group, double* debt);

/* Ragged gather: pack tokens of the sampled trajectories (row-major slots of
 * stride `stride`) into out, offsets = exclusive scan of lengths. */
void or_gather_tokens(const int32_t* slot_tokens, int64_t stride, const int64_t* slots,
                      const int32_t* lengths, size_t n, int32_t* out, int64_t* offsets);

#ifdef __cplusplus
}
#endif
#endif

#ifdef __cplusplus
extern "C" {
#endif
/* Synthetic workload (include/replay_synth.h), exported for tests. */
void or_synth_payload(uint64_t seed, const uint64_t* ids, const int64_t* offsets, size_t n,
                      int32_t* tokens, float* logp_old);
void or_synth_logp_now(uint64_t seed, uint64_t version, const uint64_t* ids,
                       const int64_t* offsets, size_t n, float* out);
void or_synth_meta(uint64_t seed, const uint64_t* ids, size_t n, int32_t lmax, int ragged,
                   double* reward, int32_t* length, double* behavior_logprob);
#ifdef __cplusplus
}
#endif
