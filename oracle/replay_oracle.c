/* replay_oracle.c — CPU restatement of the reference replay-step path.
 *
 * TEST INFRASTRUCTURE ONLY (see replay_oracle.h).  Each function cites the
 * reference function it restates (paths relative to /root/reference/proj).
 * Plain C99, single-threaded, written for clarity rather than speed.
 */
#include "replay_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];
const char* or_last_error(void) { return g_err; }
static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return OR_INVALID;
}

/* ======================================================================
 * rng.hpp:68 — std::mt19937_64, as fixed by [rand.predef]:
 * w=64 n=312 m=156 r=31 a=0xB5026F5AA96619E9, tempering (29,0x5555..),
 * (17,0x71D67FFFEDA60000), (37,0xFFF7EEE000000000), 43; f=6364136223846793005.
 * ==================================================================== */
#define MT_N 312
#define MT_M 156
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x000000007FFFFFFFULL
#define MT_A 0xB5026F5AA96619E9ULL

void or_rng_init(or_rng* r, uint64_t seed) {
    r->seed = seed;
    r->mt[0] = seed;
    for (uint32_t i = 1; i < MT_N; ++i) {
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + i;
    }
    r->idx = MT_N; /* libstdc++ twists lazily on the first draw */
    r->draws = 0;
}

static void mt_twist(uint64_t* mt) {
    for (uint32_t i = 0; i < MT_N; ++i) {
        const uint64_t x = (mt[i] & MT_UM) | (mt[(i + 1) % MT_N] & MT_LM);
        uint64_t xa = x >> 1;
        if (x & 1ULL) xa ^= MT_A;
        mt[i] = mt[(i + MT_M) % MT_N] ^ xa;
    }
}

static uint64_t mt_temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

uint64_t or_rng_next(or_rng* r) { /* rng.cpp:38 next_u64 = engine_() */
    if (r->idx >= MT_N) {
        mt_twist(r->mt);
        r->idx = 0;
    }
    r->draws++;
    return mt_temper(r->mt[r->idx++]);
}

void or_rng_discard(or_rng* r, uint64_t n) {
    while (n--) (void)or_rng_next(r);
}

uint64_t or_hash_name(const char* name, size_t len) { /* rng.cpp:8-15 FNV-1a 64 */
    uint64_t h = 1469598103934665603ULL;
    for (size_t i = 0; i < len; ++i) {
        h ^= (unsigned char)name[i];
        h *= 1099511628211ULL;
    }
    return h;
}

uint64_t or_splitmix64(uint64_t* state) { /* rng.cpp:17-23 */
    *state += 0x9e3779b97f4a7c15ULL;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

void or_rng_stream(const or_rng* p, const char* name, size_t len, or_rng* out) {
    uint64_t state = p->seed ^ or_hash_name(name, len); /* rng.cpp:27-30 */
    or_rng_init(out, or_splitmix64(&state));
}

void or_rng_stream_idx(const or_rng* p, const char* name, size_t len, uint64_t index,
                       or_rng* out) {
    uint64_t state = p->seed ^ or_hash_name(name, len); /* rng.cpp:32-36 */
    state = or_splitmix64(&state) ^ (index * 0x9e3779b97f4a7c15ULL);
    or_rng_init(out, or_splitmix64(&state));
}

int or_rng_below(or_rng* r, uint64_t bound, uint64_t* out) { /* rng.cpp:40-51 */
    if (bound == 0) return fail("Rng::below: bound must be positive");
    const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
    uint64_t v;
    do {
        v = or_rng_next(r);
    } while (v >= limit);
    *out = v % bound;
    return OR_OK;
}

double or_rng_uniform01(or_rng* r) { /* rng.cpp:53-55 */
    return (double)(or_rng_next(r) >> 11) * 0x1.0p-53;
}

double or_rng_normal(or_rng* r) { /* rng.cpp:59-70, polar method, spare dropped */
    for (;;) {
        const double u = 2.0 * or_rng_uniform01(r) - 1.0;
        const double v = 2.0 * or_rng_uniform01(r) - 1.0;
        const double s = u * u + v * v;
        if (s > 0.0 && s < 1.0) return u * sqrt(-2.0 * log(s) / s);
    }
}

int or_rng_swor(or_rng* r, size_t n, size_t k, uint64_t* out) { /* rng.cpp:108-121 */
    if (k > n) return fail("Rng::sample_without_replacement: k exceeds population");
    uint64_t* idx = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    for (size_t i = 0; i < n; ++i) idx[i] = i;
    for (size_t i = 0; i < k; ++i) {
        uint64_t j;
        or_rng_below(r, n - i, &j);
        const uint64_t t = idx[i];
        idx[i] = idx[i + j];
        idx[i + j] = t;
    }
    memcpy(out, idx, k * sizeof(uint64_t));
    free(idx);
    return OR_OK;
}

/* ======================================================================
 * replay_buffer.cpp — ShardedReplayBuffer
 * ==================================================================== */
typedef struct {
    or_record* rec; /* arrival order, oldest first (replay_buffer.hpp:93) */
    size_t size;
} or_shard;

/* open-addressing u64 set standing in for present_ids_ (replay_buffer.hpp:104) */
typedef struct {
    uint64_t* keys;
    uint8_t* state; /* 0 empty, 1 full, 2 tombstone */
    size_t cap;
} or_idset;

struct or_buffer {
    size_t total_capacity, shard_capacity, num_shards, route_cursor;
    int strategy, retention;
    double delta;
    uint32_t prio_base, prio_adv_scale, prio_pos_bonus; /* priority_with_replacement */
    or_shard* shards;
    or_idset ids;
};

static size_t idset_slot(const or_idset* s, uint64_t key, int* found) {
    size_t i = (size_t)((key * 0x9E3779B97F4A7C15ULL) >> 20) & (s->cap - 1);
    size_t tomb = (size_t)-1;
    for (;;) {
        if (s->state[i] == 0) {
            *found = 0;
            return tomb != (size_t)-1 ? tomb : i;
        }
        if (s->state[i] == 1 && s->keys[i] == key) {
            *found = 1;
            return i;
        }
        if (s->state[i] == 2 && tomb == (size_t)-1) tomb = i;
        i = (i + 1) & (s->cap - 1);
    }
}
static int idset_insert(or_idset* s, uint64_t key) { /* 1 if newly inserted */
    int found;
    size_t i = idset_slot(s, key, &found);
    if (found) return 0;
    s->keys[i] = key;
    s->state[i] = 1;
    return 1;
}
static void idset_erase(or_idset* s, uint64_t key) {
    int found;
    size_t i = idset_slot(s, key, &found);
    if (found) s->state[i] = 2;
}

or_buffer* or_buf_new(size_t num_shards, size_t total_capacity, int strategy, int retention,
                      double delta) {
    if (num_shards == 0) { /* replay_buffer.cpp:73-75 */
        fail("ShardedReplayBuffer: need at least one shard");
        return NULL;
    }
    if (total_capacity == 0 || total_capacity % num_shards != 0) { /* 76-79 */
        fail("ShardedReplayBuffer: capacity must be a positive multiple of the shard count");
        return NULL;
    }
    if (retention == OR_POSITIVE_BIAS && !(delta >= 0.0 && delta <= 1.0)) { /* 38-41 */
        fail("RetentionPolicy: delta must be in [0, 1]");
        return NULL;
    }
    or_buffer* b = (or_buffer*)calloc(1, sizeof *b);
    b->num_shards = num_shards;
    b->total_capacity = total_capacity;
    b->shard_capacity = total_capacity / num_shards;
    b->strategy = strategy;
    b->prio_base = 1;
    b->retention = retention;
    b->delta = retention == OR_POSITIVE_BIAS ? delta : 0.0;
    b->shards = (or_shard*)calloc(num_shards, sizeof(or_shard));
    for (size_t s = 0; s < num_shards; ++s) {
        b->shards[s].rec = (or_record*)calloc(b->shard_capacity + 1, sizeof(or_record));
    }
    size_t cap = 16;
    while (cap < 4 * total_capacity + 16) cap <<= 1;
    b->ids.cap = cap;
    b->ids.keys = (uint64_t*)calloc(cap, sizeof(uint64_t));
    b->ids.state = (uint8_t*)calloc(cap, 1);
    return b;
}

void or_buf_free(or_buffer* b) {
    if (!b) return;
    for (size_t s = 0; s < b->num_shards; ++s) free(b->shards[s].rec);
    free(b->shards);
    free(b->ids.keys);
    free(b->ids.state);
    free(b);
}

static void idset_rehash_if_needed(or_idset* s) {
    size_t used = 0;
    for (size_t i = 0; i < s->cap; ++i) used += s->state[i] != 0;
    if (used * 2 < s->cap) return;
    or_idset n = {(uint64_t*)calloc(s->cap, 8), (uint8_t*)calloc(s->cap, 1), s->cap};
    for (size_t i = 0; i < s->cap; ++i)
        if (s->state[i] == 1) idset_insert(&n, s->keys[i]);
    free(s->keys);
    free(s->state);
    *s = n;
}

/* replay_buffer.cpp:98-133 shard_push */
static int shard_push(or_buffer* b, or_shard* sh, const or_record* rec, or_record* evicted) {
    sh->rec[sh->size++] = *rec;
    if (sh->size <= b->shard_capacity) return 0;
    size_t victim = 0;
    if (b->retention == OR_POSITIVE_BIAS) {
        const size_t n = b->shard_capacity;
        /* 110-111: floor(delta*n + 1e-9) correctness-reserved slots */
        const size_t correct_slots = (size_t)floor(b->delta * (double)n + 1e-9);
        const size_t fresh_slots = n - correct_slots;
        const size_t outside = sh->size - fresh_slots; /* 116 */
        for (size_t i = 0; i < outside; ++i) {          /* 117-127 */
            if (!sh->rec[i].is_correct) {
                victim = i;
                break;
            }
        }
    }
    *evicted = sh->rec[victim]; /* 130-131: erase keeps arrival order */
    memmove(&sh->rec[victim], &sh->rec[victim + 1], (sh->size - victim - 1) * sizeof(or_record));
    sh->size--;
    return 1;
}

int or_buf_push(or_buffer* b, const or_record* rec, or_record* evicted, int* has_evicted) {
    *has_evicted = 0;
    idset_rehash_if_needed(&b->ids);
    if (!idset_insert(&b->ids, rec->rollout_id)) { /* replay_buffer.cpp:85-88 */
        snprintf(g_err, sizeof g_err, "ShardedReplayBuffer: rollout id %llu is already stored",
                 (unsigned long long)rec->rollout_id);
        return OR_INVALID;
    }
    or_shard* sh = &b->shards[b->route_cursor]; /* 89-90 round-robin */
    b->route_cursor = (b->route_cursor + 1) % b->num_shards;
    or_record ev;
    if (shard_push(b, sh, rec, &ev)) {
        idset_erase(&b->ids, ev.rollout_id); /* 92-94 */
        *evicted = ev;
        *has_evicted = 1;
    }
    return OR_OK;
}

/* priority_with_replacement (builder extension, no reference counterpart;
 * include/replay_b200.h rb_set_priority): integer weight of one record. */
static uint64_t prio_weight(const or_buffer* b, const or_record* r) {
    double a = fabs(r->advantage);
    if (!(a <= 32768.0)) a = a > 32768.0 ? 32768.0 : 0.0; /* clamp; NaN -> 0 */
    uint64_t w = (uint64_t)b->prio_base + (uint64_t)(a * (double)b->prio_adv_scale);
    if (b->prio_pos_bonus != 0 && r->reward > 0.0) w += b->prio_pos_bonus;
    return w;
}

int or_buf_set_priority(or_buffer* b, uint32_t base, uint32_t adv_scale, uint32_t pos_bonus) {
    if (base == 0) return fail("rb_set_priority: base weight must be >= 1");
    if (adv_scale > 65536u) return fail("rb_set_priority: adv_scale must be <= 65536");
    b->prio_base = base;
    b->prio_adv_scale = adv_scale;
    b->prio_pos_bonus = pos_bonus;
    return OR_OK;
}

/* replay_buffer.cpp:135-182 pick_indices; returns count written */
static int pick_indices(const or_buffer* b, const or_shard* sh, size_t k, or_rng* rng,
                        uint64_t* picks) {
    const size_t n = sh->size;
    if (b->strategy == OR_UNIFORM_WITH) {
        for (size_t i = 0; i < k; ++i) {
            int st = or_rng_below(rng, n, &picks[i]);
            if (st) return st;
        }
        return OR_OK;
    }
    if (b->strategy == OR_PRIORITY_WITH) { /* the 141-145 loop over a weighted CDF */
        uint64_t* cdf = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
        uint64_t W = 0;
        for (size_t i = 0; i < n; ++i) cdf[i] = (W += prio_weight(b, &sh->rec[i]));
        for (size_t i = 0; i < k; ++i) {
            uint64_t x;
            int st = or_rng_below(rng, W, &x);
            if (st) {
                free(cdf);
                return st;
            }
            size_t lo = 0, hi = n; /* upper_bound: first i with cdf[i] > x */
            while (lo < hi) {
                const size_t mid = (lo + hi) / 2;
                if (cdf[mid] > x) hi = mid;
                else lo = mid + 1;
            }
            picks[i] = lo;
        }
        free(cdf);
        return OR_OK;
    }
    if (k > n) {
        return fail(
            "ShardedReplayBuffer: batch exceeds shard occupancy for sampling without "
            "replacement");
    }
    if (b->strategy == OR_UNIFORM_WITHOUT) return or_rng_swor(rng, n, k, picks);
    /* unused_first_without_replacement, 155-179 */
    size_t got = 0;
    for (size_t i = n; i-- > 0 && got < k;) {
        if (sh->rec[i].use_count == 0) picks[got++] = i;
    }
    if (got < k) {
        uint64_t* used = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
        size_t nu = 0;
        for (size_t i = 0; i < n; ++i)
            if (sh->rec[i].use_count != 0) used[nu++] = i;
        uint64_t* sel = (uint64_t*)malloc((k - got) * sizeof(uint64_t) + 8);
        int st = or_rng_swor(rng, nu, k - got, sel);
        if (st) {
            free(used);
            free(sel);
            return st;
        }
        for (size_t j = 0; j < k - got; ++j) picks[got + j] = used[sel[j]];
        free(used);
        free(sel);
    }
    return OR_OK;
}

int or_buf_sample(or_buffer* b, size_t batch, or_rng* rng, or_record* out, int64_t* out_shard,
                  int64_t* out_index) {
    if (batch == 0 || batch % b->num_shards != 0) { /* replay_buffer.cpp:189-192 */
        return fail(
            "ShardedReplayBuffer: batch size must be a positive multiple of the shard count");
    }
    const size_t per = batch / b->num_shards;
    uint64_t* picks = (uint64_t*)malloc(per * sizeof(uint64_t));
    size_t pos = 0;
    for (size_t s = 0; s < b->num_shards; ++s) { /* 196-204, shard order 0..T-1 */
        or_shard* sh = &b->shards[s];
        if (sh->size == 0) {
            free(picks);
            return fail("ShardedReplayBuffer: cannot sample from an empty shard");
        }
        int st = pick_indices(b, sh, per, rng, picks);
        if (st) {
            free(picks);
            return st;
        }
        for (size_t i = 0; i < per; ++i) {
            sh->rec[picks[i]].use_count += 1; /* 201-202: copy after increment */
            out[pos] = sh->rec[picks[i]];
            if (out_shard) out_shard[pos] = (int64_t)s;
            if (out_index) out_index[pos] = (int64_t)picks[i];
            ++pos;
        }
    }
    free(picks);
    return OR_OK;
}

size_t or_buf_size(const or_buffer* b) {
    size_t t = 0;
    for (size_t s = 0; s < b->num_shards; ++s) t += b->shards[s].size;
    return t;
}
size_t or_buf_shard_size(const or_buffer* b, size_t s) { return b->shards[s].size; }
size_t or_buf_shard_contents(const or_buffer* b, size_t s, or_record* out) {
    memcpy(out, b->shards[s].rec, b->shards[s].size * sizeof(or_record));
    return b->shards[s].size;
}
size_t or_buf_route_cursor(const or_buffer* b) { return b->route_cursor; }

/* ======================================================================
 * bandit.cpp
 * ==================================================================== */
int or_group_advantages(const double* r, size_t n, double* out) { /* bandit.cpp:276-294 */
    if (n < 2) return fail("group advantages need >= 2 rewards");
    const double dn = (double)n;
    double mean = 0.0;
    for (size_t i = 0; i < n; ++i) mean += r[i];
    mean /= dn;
    double var = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double d = r[i] - mean;
        const double sq = d * d; /* separate statement: no FMA contraction */
        var += sq;
    }
    var /= dn;
    const double sd = sqrt(var);
    for (size_t i = 0; i < n; ++i) out[i] = 0.0;
    if (sd < 1e-8) return OR_OK;
    for (size_t i = 0; i < n; ++i) out[i] = (r[i] - mean) / sd;
    return OR_OK;
}

/* One GRPO unit (bandit.cpp:380-400).  Returns 0 if excluded (non-finite
 * ratio), else 1 with the objective term and the un-normalised coefficient
 * (A*ratio on the unclipped branch, 0 on the clipped one). */
static int grpo_unit(double lp_now, double lp_old, double a, double eps_low, double eps_high,
                     double* obj_term, double* coef) {
    const double ratio = exp(lp_now - lp_old);
    if (!isfinite(ratio)) return 0;
    double clipped = ratio;
    if (clipped < 1.0 - eps_low) clipped = 1.0 - eps_low; /* std::clamp */
    if (clipped > 1.0 + eps_high) clipped = 1.0 + eps_high;
    volatile double uv = ratio * a; /* volatile: keep the two products rounded */
    volatile double cv = clipped * a;
    if (uv <= cv) { /* ties resolve to the unclipped branch */
        *obj_term = uv;
        *coef = a * ratio;
    } else {
        *obj_term = cv;
        *coef = 0.0;
    }
    return 1;
}

void or_loss_grpo_tokens(const float* logp_now, const float* logp_old, const double* adv,
                         const int64_t* offsets, size_t n_traj, double eps_low,
                         double eps_high, float* dlogp, double* objective, int64_t* included,
                         int64_t* excluded) {
    double obj = 0.0;
    int64_t inc = 0, exc = 0;
    const int64_t total = offsets[n_traj];
    double* coef = (double*)malloc((size_t)(total ? total : 1) * sizeof(double));
    for (size_t i = 0; i < n_traj; ++i) {
        for (int64_t t = offsets[i]; t < offsets[i + 1]; ++t) {
            double term, c;
            if (grpo_unit((double)logp_now[t], (double)logp_old[t], adv[i], eps_low, eps_high,
                          &term, &c)) {
                ++inc;
                obj += term;
                coef[t] = c;
            } else {
                ++exc;
                coef[t] = 0.0;
            }
        }
    }
    const double scale = inc > 0 ? 1.0 / (double)inc : 0.0; /* bandit.cpp:402-406 */
    for (int64_t t = 0; t < total; ++t) dlogp[t] = (float)(-coef[t] * scale);
    *objective = inc > 0 ? obj * scale : 0.0;
    *included = inc;
    *excluded = exc;
    free(coef);
}

/* GRPO normalisation modes at the token level (SURVEY.md §8c "token
 * generalisation"; the reference has no tokens):
 *   mode 0  per-token ratio, mean over the batch's included tokens
 *           (or_loss_grpo_tokens above);
 *   mode 1  per-token ratio, mean over each sequence's included tokens, then
 *           mean over the sequences with at least one included token:
 *           objective = (1/S) sum_i (1/n_i) sum_t term_t,
 *           dL/dlogp_t = -coef_t / (n_i * S); included = S;
 *   mode 2  sequence-level ratio pi(z|q)/pi_old(z|q):
 *           the reference's record-level grpo_loss_grad (bandit.cpp:363-408)
 *           with logp_now(record) = sum_t logp_now_t (fp64, token order) and
 *           behavior_logprob = blp[i] (the record field, bandit.cpp:380; NULL:
 *           sum_t logp_old_t); every token of sequence i gets the record's
 *           dL/dlogp = -coef_i / included; included/excluded count sequences.
 * dlogp is rounded to fp32 once from the fp64 value. */
void or_loss_grpo_tokens_mode(const float* logp_now, const float* logp_old, const double* adv,
                              const double* blp, const int64_t* offsets, size_t n_traj,
                              double eps_low, double eps_high, int mode, float* dlogp,
                              double* objective, int64_t* included, int64_t* excluded) {
    if (mode == 0) {
        or_loss_grpo_tokens(logp_now, logp_old, adv, offsets, n_traj, eps_low, eps_high, dlogp,
                            objective, included, excluded);
        return;
    }
    double obj = 0.0;
    int64_t inc = 0, exc = 0;
    const int64_t total = offsets[n_traj];
    double* coef = (double*)malloc((size_t)(total ? total : 1) * sizeof(double));
    double* seqn = (double*)malloc((n_traj ? n_traj : 1) * sizeof(double)); /* mode 1: n_i */
    for (size_t i = 0; i < n_traj; ++i) {
        const int64_t o0 = offsets[i], o1 = offsets[i + 1];
        if (mode == 2) {
            double lp = 0.0, lo = 0.0;
            for (int64_t t = o0; t < o1; ++t) {
                lp += (double)logp_now[t];
                lo += (double)logp_old[t];
            }
            double term, c;
            if (grpo_unit(lp, blp ? blp[i] : lo, adv[i], eps_low, eps_high, &term, &c)) {
                ++inc;
                obj += term;
            } else {
                ++exc;
                c = 0.0;
            }
            for (int64_t t = o0; t < o1; ++t) coef[t] = c;
        } else {
            double sum = 0.0;
            int64_t n = 0;
            for (int64_t t = o0; t < o1; ++t) {
                double term, c;
                if (grpo_unit((double)logp_now[t], (double)logp_old[t], adv[i], eps_low, eps_high,
                              &term, &c)) {
                    ++n;
                    sum += term;
                    coef[t] = c;
                } else {
                    ++exc;
                    coef[t] = 0.0;
                }
            }
            seqn[i] = (double)n;
            if (n > 0) {
                ++inc;
                obj += sum / (double)n;
            }
        }
    }
    const double scale = inc > 0 ? 1.0 / (double)inc : 0.0;
    for (size_t i = 0; i < n_traj; ++i) {
        const double ni = mode == 1 ? seqn[i] : 1.0;
        for (int64_t t = offsets[i]; t < offsets[i + 1]; ++t)
            dlogp[t] = (inc > 0 && ni > 0) ? (float)(-coef[t] / (ni * (double)inc)) : 0.0f;
    }
    *objective = inc > 0 ? obj * scale : 0.0;
    *included = inc;
    *excluded = exc;
    free(coef);
    free(seqn);
}

void or_loss_grpo_records(const double* logp_now, const double* behavior_logprob,
                          const double* adv, size_t n, double eps_low, double eps_high,
                          double* dlogp, double* objective, int64_t* included,
                          int64_t* excluded) {
    double obj = 0.0;
    int64_t inc = 0, exc = 0;
    for (size_t i = 0; i < n; ++i) {
        double term, c;
        if (grpo_unit(logp_now[i], behavior_logprob[i], adv[i], eps_low, eps_high, &term, &c)) {
            ++inc;
            obj += term;
            dlogp[i] = c;
        } else {
            ++exc;
            dlogp[i] = 0.0;
        }
    }
    const double scale = inc > 0 ? 1.0 / (double)inc : 0.0;
    for (size_t i = 0; i < n; ++i) dlogp[i] = inc > 0 ? dlogp[i] * -scale : 0.0;
    *objective = inc > 0 ? obj * scale : 0.0;
    *included = inc;
    *excluded = exc;
}

void or_loss_asymre_tokens(const float* logp_now, const double* reward,
                           const double* group_mean, const int64_t* offsets, size_t n_traj,
                           double delta_v, float* dlogp, double* objective) {
    double obj = 0.0;
    const double scale = 1.0 / (double)n_traj; /* bandit.cpp:434 */
    for (size_t i = 0; i < n_traj; ++i) {
        const double coef = reward[i] - (group_mean[i] + delta_v); /* 429 */
        double seq_logp = 0.0;
        for (int64_t t = offsets[i]; t < offsets[i + 1]; ++t) {
            seq_logp += (double)logp_now[t];
            dlogp[t] = (float)(coef * -scale);
        }
        obj += coef * seq_logp; /* 431 */
    }
    *objective = obj * scale;
}

void or_loss_asymre_records(const double* logp_now, const double* reward,
                            const double* group_mean, size_t n, double delta_v, double* dlogp,
                            double* objective) {
    double obj = 0.0;
    const double scale = 1.0 / (double)n;
    for (size_t i = 0; i < n; ++i) {
        const double coef = reward[i] - (group_mean[i] + delta_v);
        obj += coef * logp_now[i];
        dlogp[i] = coef * -scale;
    }
    *objective = obj * scale;
}

int64_t or_production_groups(double per_step_production, size_t group, double* debt) {
    int64_t groups = 0; /* bandit.cpp:636-640 */
    *debt += per_step_production;
    while (*debt >= (double)group) {
        ++groups;
        *debt -= (double)group;
    }
    return groups;
}

void or_gather_tokens(const int32_t* slot_tokens, int64_t stride, const int64_t* slots,
                      const int32_t* lengths, size_t n, int32_t* out, int64_t* offsets) {
    int64_t pos = 0;
    for (size_t i = 0; i < n; ++i) {
        offsets[i] = pos;
        memcpy(out + pos, slot_tokens + slots[i] * stride, (size_t)lengths[i] * sizeof(int32_t));
        pos += lengths[i];
    }
    offsets[n] = pos;
}

/* ======================================================================
 * Synthetic workload (include/replay_synth.h) exported for the tests.
 * ==================================================================== */
#include "../include/replay_synth.h"

void or_synth_payload(uint64_t seed, const uint64_t* ids, const int64_t* offsets, size_t n,
                      int32_t* tokens, float* logp_old) {
    for (size_t i = 0; i < n; ++i) {
        for (int64_t t = offsets[i]; t < offsets[i + 1]; ++t) {
            const uint64_t tt = (uint64_t)(t - offsets[i]);
            if (tokens) tokens[t] = rs_token(seed, ids[i], tt);
            if (logp_old) logp_old[t] = rs_logp_old(seed, ids[i], tt);
        }
    }
}

void or_synth_logp_now(uint64_t seed, uint64_t version, const uint64_t* ids,
                       const int64_t* offsets, size_t n, float* out) {
    for (size_t i = 0; i < n; ++i)
        for (int64_t t = offsets[i]; t < offsets[i + 1]; ++t)
            out[t] = rs_logp_now(seed, ids[i], (uint64_t)(t - offsets[i]), version);
}

void or_synth_meta(uint64_t seed, const uint64_t* ids, size_t n, int32_t lmax, int ragged,
                   double* reward, int32_t* length, double* behavior_logprob) {
    for (size_t i = 0; i < n; ++i) {
        reward[i] = rs_reward(seed, ids[i]);
        length[i] = rs_length(seed, ids[i], lmax, ragged);
        double s = 0.0;
        for (int32_t t = 0; t < length[i]; ++t) s += (double)rs_logp_old(seed, ids[i], (uint64_t)t);
        behavior_logprob[i] = s;
    }
}
