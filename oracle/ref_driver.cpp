// ref_driver.cpp — extern "C" shim over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together
// with the reference's own sources (/root/reference/proj/src/*.cpp, read in
// place, never copied) into oracle/_ref/libreplab_ref.so.  Python tests use
// it to pin the C restatement (oracle/replay_oracle.c) and to generate the
// golden fixtures under tests/golden/; bench.py uses it as the CPU
// reference arm.  Every call below goes straight into the reference API:
//   replab::Rng                 rng.hpp:22-69
//   replab::ShardedReplayBuffer replay_buffer.hpp:57-108
//   replab::group_advantages    bandit.hpp:106
//   replab::grpo_loss_grad / asymre_loss_grad  bandit.hpp:133-139
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <algorithm>
#include <vector>

#include "replab/bandit.hpp"
#include "replab/metrics.hpp"
#include "replab/replay_buffer.hpp"
#include "replab/rng.hpp"
#include "replab/rollout.hpp"

using namespace replab;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

RetentionPolicy retention_of(int kind, double delta) {
    return kind == 1 ? RetentionPolicy::positive_bias(delta) : RetentionPolicy::plain_fifo();
}
SamplingStrategy strategy_of(int s) {
    switch (s) {
        case 1: return SamplingStrategy::uniform_without_replacement;
        case 2: return SamplingStrategy::unused_first_without_replacement;
        default: return SamplingStrategy::uniform_with_replacement;
    }
}
static_assert(sizeof(RolloutRecord) == 80, "record layout must match rb_record");
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- Rng ---------------------------------------------------------------
void* ref_rng_new(uint64_t seed) { return new Rng(seed); }
void ref_rng_free(void* r) { delete static_cast<Rng*>(r); }
void* ref_rng_stream(void* r, const char* name) {
    return new Rng(static_cast<Rng*>(r)->stream(name));
}
void* ref_rng_stream_idx(void* r, const char* name, uint64_t idx) {
    return new Rng(static_cast<Rng*>(r)->stream(name, idx));
}
uint64_t ref_rng_seed(void* r) { return static_cast<Rng*>(r)->seed(); }
uint64_t ref_rng_next(void* r) { return static_cast<Rng*>(r)->next_u64(); }
int ref_rng_below(void* r, uint64_t b, uint64_t* out) {
    return guard([&] { *out = static_cast<Rng*>(r)->below(b); });
}
double ref_rng_uniform01(void* r) { return static_cast<Rng*>(r)->uniform01(); }
double ref_rng_normal(void* r) { return static_cast<Rng*>(r)->normal(); }
int ref_rng_swor(void* r, uint64_t n, uint64_t k, uint64_t* out) {
    return guard([&] {
        auto v = static_cast<Rng*>(r)->sample_without_replacement(n, k);
        for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
    });
}
uint64_t ref_hash_name(const char* name) { return hash_name(name); }

// ---- ShardedReplayBuffer -----------------------------------------------
void* ref_buf_new(uint64_t shards, uint64_t cap, int strategy, int retention, double delta) {
    ShardedReplayBuffer* out = nullptr;
    int st = guard([&] {
        out = new ShardedReplayBuffer(shards, cap, strategy_of(strategy),
                                      retention_of(retention, delta));
    });
    return st == 0 ? out : nullptr;
}
void ref_buf_free(void* b) { delete static_cast<ShardedReplayBuffer*>(b); }
int ref_buf_push(void* b, const RolloutRecord* rec, RolloutRecord* evicted, int* has_evicted) {
    return guard([&] {
        *has_evicted = 0;
        auto ev = static_cast<ShardedReplayBuffer*>(b)->push(*rec);
        if (ev) {
            *evicted = *ev;
            *has_evicted = 1;
        }
    });
}
// events (optional): 5 int64 per selection {id, creation_step, use_step, batch_id, rank}
int ref_buf_sample(void* b, uint64_t batch, void* rng, RolloutRecord* out, int64_t* events,
                   int64_t batch_id, int64_t use_step) {
    return guard([&] {
        MetricsLedger ledger;
        auto v = static_cast<ShardedReplayBuffer*>(b)->sample(
            batch, *static_cast<Rng*>(rng), events ? &ledger : nullptr, batch_id, use_step);
        for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
        if (events) {
            const auto& ev = ledger.events();
            for (size_t i = 0; i < ev.size(); ++i) {
                events[5 * i + 0] = static_cast<int64_t>(ev[i].rollout_id);
                events[5 * i + 1] = ev[i].creation_step;
                events[5 * i + 2] = ev[i].use_step;
                events[5 * i + 3] = ev[i].batch_id;
                events[5 * i + 4] = ev[i].within_batch_rank;
            }
        }
    });
}
uint64_t ref_buf_size(void* b) { return static_cast<ShardedReplayBuffer*>(b)->size(); }
uint64_t ref_buf_shard_size(void* b, uint64_t s) {
    return static_cast<ShardedReplayBuffer*>(b)->shard_size(s);
}
uint64_t ref_buf_shard_contents(void* b, uint64_t s, RolloutRecord* out) {
    auto v = static_cast<ShardedReplayBuffer*>(b)->shard_contents(s);
    for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
    return v.size();
}
// Writes the dump into out (capacity cap incl. NUL); returns the full length.
uint64_t ref_buf_dump(void* b, char* out, uint64_t cap) {
    std::string d = static_cast<ShardedReplayBuffer*>(b)->dump();
    if (out && cap) {
        size_t n = d.size() < cap - 1 ? d.size() : cap - 1;
        std::memcpy(out, d.data(), n);
        out[n] = 0;
    }
    return d.size();
}
void* ref_buf_load(const char* text) {
    ShardedReplayBuffer* out = nullptr;
    int st = guard([&] { out = new ShardedReplayBuffer(ShardedReplayBuffer::load(text)); });
    return st == 0 ? out : nullptr;
}

// ---- metrics ------------------------------------------------------------
// The reference's summarize() (metrics.cpp:185-202): out = {count, mean,
// q25, median, q75}; the histogram goes to (hist_keys, hist_counts), up to
// hist_cap entries, *hist_n = its size.
int ref_summarize(const double* v, uint64_t n, double* out, int64_t* hist_keys,
                  uint64_t* hist_counts, uint64_t hist_cap, uint64_t* hist_n) {
    return guard([&] {
        const MetricSummary s = summarize(std::vector<double>(v, v + n));
        out[0] = (double)s.count;
        out[1] = s.mean;
        out[2] = s.q25;
        out[3] = s.median;
        out[4] = s.q75;
        *hist_n = s.histogram.size();
        uint64_t i = 0;
        for (const auto& kv : s.histogram) {
            if (i == hist_cap) break;
            hist_keys[i] = kv.first;
            hist_counts[i++] = kv.second;
        }
    });
}

// ---- advantages and losses ---------------------------------------------
// MetricsLedger + its diagnostics (metrics.hpp:36-93, metrics.cpp:44-170).
// Events as 5 int64 words: rollout_id, creation_step, use_step, batch_id, rank.
void* ref_ledger_new() { return new MetricsLedger(); }
void ref_ledger_free(void* l) { delete static_cast<MetricsLedger*>(l); }
int ref_ledger_note_generated(void* l, uint64_t id) {
    return guard([&] { static_cast<MetricsLedger*>(l)->note_generated(id); });
}
int ref_ledger_record_use(void* l, const int64_t* e) {
    return guard([&] {
        UseEvent u;
        u.rollout_id = (uint64_t)e[0];
        u.creation_step = e[1];
        u.use_step = e[2];
        u.batch_id = e[3];
        u.within_batch_rank = e[4];
        static_cast<MetricsLedger*>(l)->record_use(u);
    });
}
uint64_t ref_ledger_events(void* l, int64_t* out) {
    const auto& ev = static_cast<MetricsLedger*>(l)->events();
    if (out)
        for (size_t i = 0; i < ev.size(); ++i) {
            out[5 * i] = (int64_t)ev[i].rollout_id;
            out[5 * i + 1] = ev[i].creation_step;
            out[5 * i + 2] = ev[i].use_step;
            out[5 * i + 3] = ev[i].batch_id;
            out[5 * i + 4] = ev[i].within_batch_rank;
        }
    return ev.size();
}
uint64_t ref_ledger_replay_counts(void* l, int include_zero, uint64_t* ids, uint64_t* counts) {
    const auto m = replay_counts(*static_cast<MetricsLedger*>(l), include_zero != 0);
    size_t i = 0;
    for (const auto& [k, v] : m) {
        if (ids) ids[i] = k;
        if (counts) counts[i] = v;
        ++i;
    }
    return m.size();
}
uint64_t ref_ledger_global_use_order(void* l, void* rng, uint64_t* order) {
    const auto o = global_use_order(static_cast<MetricsLedger*>(l)->events(), *static_cast<Rng*>(rng));
    for (size_t i = 0; i < o.size(); ++i) order[i] = o[i];
    return o.size();
}
uint64_t ref_ledger_steps_since_last_use(void* l, void* rng, uint64_t* idx, int64_t* gap,
                                         uint8_t* has) {
    const auto lab = steps_since_last_use(*static_cast<MetricsLedger*>(l), *static_cast<Rng*>(rng));
    for (size_t i = 0; i < lab.size(); ++i) {
        idx[i] = lab[i].event_index;
        has[i] = lab[i].gap.has_value();
        gap[i] = lab[i].gap.value_or(0);
    }
    return lab.size();
}

int ref_group_advantages(const double* r, uint64_t n, double* out) {
    return guard([&] {
        auto v = group_advantages(std::vector<double>(r, r + n));
        for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
    });
}

// Record-level losses through the reference's own grpo_loss_grad /
// asymre_loss_grad.  Each record i gets its own prompt row with two arms and
// logits (log(p/(1-p)), 0), p = exp(logp_want[i]), so the reference's
// logprob(i, arm 0) ~= logp_want[i]; the value the reference actually used
// is returned in logp_used.  Per-record dL/dlogp is recovered from the logit
// gradient: grad[i,0] = dL/dlogp * (1 - p_i) / tau with tau = 1.
int ref_loss_records(int kind, const double* logp_want, const RolloutRecord* recs,
                     const double* group_mean, uint64_t n, double eps_low, double eps_high,
                     double delta_v, double* logp_used, double* dlogp, double* objective,
                     uint64_t* excluded) {
    return guard([&] {
        SoftmaxPolicy pol = SoftmaxPolicy::uniform(n, 2);
        RolloutSideTables tables;
        std::vector<RolloutRecord> batch(recs, recs + n);
        for (uint64_t i = 0; i < n; ++i) {
            const double p = std::exp(logp_want[i]);
            pol.logit(i, 0) = std::log(p / (1.0 - p));
            pol.logit(i, 1) = 0.0;
            batch[i].prompt_id = i;
            batch[i].rollout_id = i;  // side tables are keyed by our row index
            batch[i].group_id = i;
            tables.arm_of[i] = 0;
            tables.group_mean_reward[i] = group_mean ? group_mean[i] : 0.0;
            logp_used[i] = pol.logprob(i, 0, 1.0);
        }
        LossSpec spec = kind == 0 ? LossSpec::grpo(eps_low, eps_high, 2)
                                  : LossSpec::asymre(delta_v, 2);
        LossResult res = loss_grad(pol, batch, tables, spec);
        for (uint64_t i = 0; i < n; ++i) {
            const double p0 = pol.probs(i, 1.0)[0];
            dlogp[i] = res.grad[2 * i] / (1.0 - p0);
        }
        *objective = res.objective;
        *excluded = res.excluded;
    });
}

}  // extern "C"

// =========================================================================
// CPU reference arm of bench.py: the replay step on the host.
//
// Record-level work goes through the unmodified reference library:
// group_advantages (bandit.cpp:276-294) for every inserted group,
// ShardedReplayBuffer::push (replay_buffer.cpp:83-133) for every record and
// ShardedReplayBuffer::sample (184-217) with the "buffer_sampling" stream.
// The reference has no tokens, so the token payload store,
// the ragged gather and the per-token GRPO loss are the C restatement of
// bandit.cpp:363-408 (same arithmetic as oracle/replay_oracle.c), spread
// over all host threads.
namespace {

struct RefBench {
    ShardedReplayBuffer buf;
    Rng sampling;
    int lmax;
    int threads;
    std::vector<int32_t> tok;  // [rows][lmax]
    std::vector<float> lpo;
    std::unordered_map<uint64_t, std::pair<int, int>> row_of;  // id -> (row, len)
    std::vector<int> free_rows;
    std::vector<RolloutRecord> batch;
    std::vector<int64_t> off;
    RefBench(size_t T, size_t N, int strategy, int retention, double delta, int lmax_, uint64_t seed,
             int threads_)
        : buf(T, N, strategy_of(strategy), retention_of(retention, delta)),
          sampling(Rng(seed).stream("buffer_sampling")),
          lmax(lmax_),
          threads(threads_ > 0 ? threads_ : (int)std::max(1u, std::thread::hardware_concurrency())),
          tok(N * (size_t)lmax_),
          lpo(N * (size_t)lmax_) {
        for (int r = (int)N - 1; r >= 0; --r) free_rows.push_back(r);
    }
};

template <class F>
void parallel_for(int threads, int64_t n, F&& f) {
    if (threads <= 1 || n < 2) {
        f(0, n, 0);
        return;
    }
    const int t = (int)std::min<int64_t>(threads, n);
    std::vector<std::thread> pool;
    for (int k = 0; k < t; ++k) {
        const int64_t a = n * k / t, b = n * (k + 1) / t;
        pool.emplace_back([&, a, b, k] { f(a, b, k); });
    }
    for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

void* ref_bench_new(uint64_t T, uint64_t N, int strategy, int retention, double delta, int lmax,
                    uint64_t seed, int threads) {
    RefBench* out = nullptr;
    int st = guard([&] { out = new RefBench(T, N, strategy, retention, delta, lmax, seed, threads); });
    return st == 0 ? out : nullptr;
}
void ref_bench_free(void* h) { delete static_cast<RefBench*>(h); }
int ref_bench_threads(void* h) { return static_cast<RefBench*>(h)->threads; }

// Phase A: insert n records (groups of `group`, advantages computed here by
// the reference), evict, sample `batch`, gather tokens.  recs carry
// everything but the advantage; toff (n+1) indexes tokens/logp_old.
int ref_bench_phase_a(void* hv, uint64_t n, uint64_t group, const RolloutRecord* recs,
                      const int64_t* toff, const int32_t* tokens, const float* logp_old,
                      uint64_t batch, uint64_t* out_ids, int32_t* out_tokens, int64_t* out_off) {
    RefBench& h = *static_cast<RefBench*>(hv);
    return guard([&] {
        std::vector<RolloutRecord> rs(recs, recs + n);
        for (uint64_t g = 0; g + group <= n; g += group) {
            std::vector<double> rewards(group);
            for (uint64_t i = 0; i < group; ++i) rewards[i] = rs[g + i].reward;
            const auto adv = group_advantages(rewards);  // bandit.cpp:315
            for (uint64_t i = 0; i < group; ++i) rs[g + i].advantage = adv[i];
        }
        std::vector<int64_t> rec_row(n, -1);
        std::unordered_map<uint64_t, uint64_t> pending;  // id -> index in this batch
        for (uint64_t j = 0; j < n; ++j) {
            auto ev = h.buf.push(rs[j]);
            pending[rs[j].rollout_id] = j;
            if (ev) {
                auto it = h.row_of.find(ev->rollout_id);
                if (it != h.row_of.end()) {
                    h.free_rows.push_back(it->second.first);
                    h.row_of.erase(it);
                }
                pending.erase(ev->rollout_id);
            }
        }
        std::vector<std::pair<uint64_t, int>> copies;  // (batch index, row)
        for (auto& [id, j] : pending) {
            const int row = h.free_rows.back();
            h.free_rows.pop_back();
            h.row_of[id] = {row, (int)(toff[j + 1] - toff[j])};
            copies.push_back({j, row});
        }
        parallel_for(h.threads, (int64_t)copies.size(), [&](int64_t a, int64_t b, int) {
            for (int64_t c = a; c < b; ++c) {
                const uint64_t j = copies[c].first;
                const size_t row = (size_t)copies[c].second * h.lmax;
                const int64_t len = toff[j + 1] - toff[j];
                std::memcpy(&h.tok[row], tokens + toff[j], len * 4);
                std::memcpy(&h.lpo[row], logp_old + toff[j], len * 4);
            }
        });
        h.batch = h.buf.sample(batch, h.sampling);
        h.off.assign(batch + 1, 0);
        for (uint64_t i = 0; i < batch; ++i) {
            out_ids[i] = h.batch[i].rollout_id;
            h.off[i + 1] = h.off[i] + h.row_of.at(h.batch[i].rollout_id).second;
        }
        std::memcpy(out_off, h.off.data(), (batch + 1) * 8);
        parallel_for(h.threads, (int64_t)batch, [&](int64_t a, int64_t b, int) {
            for (int64_t i = a; i < b; ++i) {
                const auto& ro = h.row_of.at(h.batch[i].rollout_id);
                std::memcpy(out_tokens + h.off[i], &h.tok[(size_t)ro.first * h.lmax],
                            (size_t)ro.second * 4);
            }
        });
    });
}

// Phase B: per-token GRPO (bandit.cpp:363-408 restated) over the batch.
int ref_bench_phase_b(void* hv, const float* logp_now, double eps_low, double eps_high,
                      float* out_dlogp, double* objective, int64_t* included, int64_t* excluded) {
    RefBench& h = *static_cast<RefBench*>(hv);
    return guard([&] {
        const int64_t nb = (int64_t)h.batch.size();
        std::vector<double> obj(h.threads, 0.0);
        std::vector<int64_t> inc(h.threads, 0), exc(h.threads, 0);
        parallel_for(h.threads, nb, [&](int64_t a, int64_t b, int k) {
            for (int64_t i = a; i < b; ++i) {
                const auto& ro = h.row_of.at(h.batch[i].rollout_id);
                const float* lo = &h.lpo[(size_t)ro.first * h.lmax];
                const double A = h.batch[i].advantage;
                for (int64_t t = h.off[i]; t < h.off[i + 1]; ++t) {
                    const double ratio = std::exp((double)logp_now[t] - (double)lo[t - h.off[i]]);
                    if (!std::isfinite(ratio)) {
                        ++exc[k];
                        out_dlogp[t] = 0.f;
                        continue;
                    }
                    ++inc[k];
                    const double c = std::clamp(ratio, 1.0 - eps_low, 1.0 + eps_high);
                    const double uv = ratio * A, cv = c * A;
                    if (uv <= cv) {
                        obj[k] += uv;
                        out_dlogp[t] = (float)(A * ratio);
                    } else {
                        obj[k] += cv;
                        out_dlogp[t] = 0.f;
                    }
                }
            }
        });
        double o = 0.0;
        int64_t ni = 0, ne = 0;
        for (int k = 0; k < h.threads; ++k) {
            o += obj[k];
            ni += inc[k];
            ne += exc[k];
        }
        const double scale = ni ? 1.0 / (double)ni : 0.0;
        parallel_for(h.threads, h.off[nb], [&](int64_t a, int64_t b, int) {
            for (int64_t t = a; t < b; ++t) out_dlogp[t] = (float)((double)out_dlogp[t] * -scale);
        });
        *objective = ni ? o * scale : 0.0;
        *included = ni;
        *excluded = ne;
    });
}

}  // extern "C"

// =========================================================================
// CPU reference arm of the C5 sweep (record level): the
// (W,T) schedule of train()/simulate() through the unmodified reference
// buffer — warm-up fill (bandit.cpp:609-615), then per step the production
// debt W*B/(mu*T) in whole groups (617-640, records pushed one by one,
// replay_buffer.cpp:83-133) and sample(B) with the "buffer_sampling" stream
// (replay_buffer.cpp:184-217).  Returns the seconds spent in the timed
// steps and the records processed (inserted + sampled).
extern "C" int ref_c5_run(uint64_t T, uint64_t N, int W, int Ttr, double mu, uint64_t B,
                          uint64_t G, int retention, double delta, uint64_t seed, int steps,
                          double* seconds, uint64_t* records) {
    return guard([&] {
        ShardedReplayBuffer buf(T, N, SamplingStrategy::uniform_with_replacement,
                                retention_of(retention, delta));
        Rng sampling = Rng(seed).stream("buffer_sampling");
        Rng gen = Rng(seed).stream("generation");
        uint64_t next_id = 0;
        auto push_group = [&](int64_t step) {
            for (uint64_t i = 0; i < G; ++i) {
                RolloutRecord r{};
                r.rollout_id = next_id++;
                r.group_id = r.rollout_id / G;
                r.creation_step = step;
                r.policy_version = step;
                r.reward = gen.uniform01() < 0.5 ? 1.0 : 0.0;
                r.is_correct = r.reward == 1.0;
                buf.push(r);
            }
        };
        while (buf.size() < N) push_group(0);
        const double per = (double)W * (double)B / (mu * (double)Ttr);
        double debt = 0.0;
        uint64_t recs = 0;
        const auto t0 = std::chrono::steady_clock::now();
        for (int step = 0; step < steps; ++step) {
            debt += per;
            while (debt >= (double)G) {
                push_group(step);
                debt -= (double)G;
                recs += G;
            }
            auto batch = buf.sample(B, sampling);
            recs += batch.size();
        }
        const auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
        *records = recs;
    });
}

