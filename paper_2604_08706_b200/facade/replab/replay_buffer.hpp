// replab/replay_buffer.hpp — drop-in C++ facade of replab::ShardedReplayBuffer
// (replay_buffer.hpp:14-110) over the libreplay_b200 C-ABI.  Same enums,
// string codecs, class, methods and exceptions; the store is the HBM-resident
// SoA buffer of the library (metadata-only here: max_tokens = 0 keeps the
// reference's record-level semantics; payload-carrying buffers use the C-ABI
// or the Python mirror directly).
#pragma once

#include <memory>
#include <optional>
#include <string>
#include <string_view>
#include <vector>

#include "replab/metrics.hpp"
#include "replab/rng.hpp"
#include "replab/rollout.hpp"

namespace replab {

enum class SamplingStrategy {
    uniform_with_replacement,
    uniform_without_replacement,
    unused_first_without_replacement,
    // builder extension (include/replay_b200.h RB_PRIORITY_WITH_REPLACEMENT):
    // weighted draws over an integer CDF; set_priority() sets the weights
    priority_with_replacement,
};

inline std::string to_string(SamplingStrategy s) {  // replay_buffer.cpp:11-21
    switch (s) {
        case SamplingStrategy::uniform_with_replacement: return "uniform_with_replacement";
        case SamplingStrategy::uniform_without_replacement: return "uniform_without_replacement";
        case SamplingStrategy::unused_first_without_replacement:
            return "unused_first_without_replacement";
        case SamplingStrategy::priority_with_replacement: return "priority_with_replacement";
    }
    throw std::logic_error("bad SamplingStrategy");
}

inline SamplingStrategy sampling_strategy_from_string(std::string_view s) {  // 23-34
    if (s == "uniform_with_replacement") return SamplingStrategy::uniform_with_replacement;
    if (s == "uniform_without_replacement") return SamplingStrategy::uniform_without_replacement;
    if (s == "unused_first_without_replacement")
        return SamplingStrategy::unused_first_without_replacement;
    if (s == "priority_with_replacement") return SamplingStrategy::priority_with_replacement;
    throw std::invalid_argument("unknown sampling strategy: '" + std::string(s) + "'");
}

struct RetentionPolicy {
    enum class Kind { plain_fifo, positive_bias };
    static RetentionPolicy plain_fifo() { return RetentionPolicy{}; }
    static RetentionPolicy positive_bias(double delta) {  // replay_buffer.cpp:38-46
        if (!(delta >= 0.0) || !(delta <= 1.0))
            throw std::invalid_argument("RetentionPolicy: delta must be in [0, 1]");
        RetentionPolicy r;
        r.kind = Kind::positive_bias;
        r.delta = delta;
        return r;
    }
    Kind kind = Kind::plain_fifo;
    double delta = 0.0;
};

inline std::string to_string(const RetentionPolicy& r) {  // 48-53
    if (r.kind == RetentionPolicy::Kind::plain_fifo) return "plain_fifo";
    return "positive_bias delta=" + format_double(r.delta);
}

inline RetentionPolicy retention_policy_from_string(std::string_view s) {  // 55-65
    auto trim = [](std::string_view x) {
        std::size_t b = 0, e = x.size();
        while (b < e && (x[b] == ' ' || x[b] == '\t' || x[b] == '\r' || x[b] == '\n')) ++b;
        while (e > b && (x[e - 1] == ' ' || x[e - 1] == '\t' || x[e - 1] == '\r' || x[e - 1] == '\n'))
            --e;
        return x.substr(b, e - b);
    };
    const std::string_view t = trim(s);
    if (t == "plain_fifo") return RetentionPolicy::plain_fifo();
    constexpr std::string_view kPrefix = "positive_bias delta=";
    if (t.substr(0, kPrefix.size()) == kPrefix) {
        const std::string_view num = trim(t.substr(kPrefix.size()));
        double v = 0.0;
        auto res = std::from_chars(num.data(), num.data() + num.size(), v);
        if (res.ec != std::errc() || res.ptr != num.data() + num.size() || num.empty())
            throw std::invalid_argument("not a number: '" + std::string(t.substr(kPrefix.size())) + "'");
        return RetentionPolicy::positive_bias(v);
    }
    throw std::invalid_argument("unknown retention policy: '" + std::string(s) + "'");
}

class ShardedReplayBuffer {
public:
    ShardedReplayBuffer(std::size_t num_shards, std::size_t total_capacity,
                        SamplingStrategy strategy, RetentionPolicy retention) {
        rb_buffer* h = nullptr;
        detail::rb_check(rb_create(num_shards, total_capacity, static_cast<int>(strategy),
                                   static_cast<int>(retention.kind), retention.delta,
                                   /*max_tokens=*/0, /*device=*/-1, 0, 0, &h));
        h_.reset(h);
    }

    // replay_buffer.cpp:83-96
    std::optional<RolloutRecord> push(const RolloutRecord& record) {
        const rb_record r = record.to_rb();
        rb_record ev{};
        int has = 0;
        detail::rb_check(rb_push(h_.get(), &r, nullptr, nullptr, 0, &ev, &has));
        if (!has) return std::nullopt;
        return RolloutRecord::from_rb(ev);
    }

    // replay_buffer.cpp:184-217
    std::vector<RolloutRecord> sample(std::size_t batch_size, Rng& rng,
                                      MetricsLedger* ledger = nullptr, std::int64_t batch_id = 0,
                                      std::int64_t use_step = 0) {
        std::vector<rb_record> out(batch_size ? batch_size : 1);
        std::vector<rb_use_event> ev(ledger ? (batch_size ? batch_size : 1) : 0);
        detail::rb_check(rb_sample(h_.get(), batch_size, rng.handle(), out.data(), nullptr, nullptr,
                                   ledger ? ev.data() : nullptr, batch_id, use_step));
        std::vector<RolloutRecord> batch;
        batch.reserve(batch_size);
        for (std::size_t i = 0; i < batch_size; ++i) batch.push_back(RolloutRecord::from_rb(out[i]));
        if (ledger) {
            for (std::size_t i = 0; i < batch_size; ++i) {
                UseEvent e;
                e.rollout_id = ev[i].rollout_id;
                e.creation_step = ev[i].creation_step;
                e.use_step = ev[i].use_step;
                e.batch_id = ev[i].batch_id;
                e.within_batch_rank = ev[i].within_batch_rank;
                ledger->record_use(e);
            }
        }
        return batch;
    }

    std::size_t num_shards() const { return get(rb_num_shards); }
    std::size_t total_capacity() const { return get(rb_total_capacity); }
    std::size_t shard_capacity() const { return get(rb_shard_capacity); }
    std::size_t size() const {
        std::size_t v = 0;
        detail::rb_check(rb_size(h_.get(), &v));
        return v;
    }
    std::size_t shard_size(std::size_t shard) const {
        std::size_t v = 0;
        detail::rb_check(rb_shard_size(h_.get(), shard, &v));
        return v;
    }
    std::vector<RolloutRecord> shard_contents(std::size_t shard) const {
        std::size_t n = 0;
        detail::rb_check(rb_shard_contents(h_.get(), shard, nullptr, 0, &n));
        std::vector<rb_record> out(n ? n : 1);
        detail::rb_check(rb_shard_contents(h_.get(), shard, out.data(), out.size(), &n));
        std::vector<RolloutRecord> v;
        v.reserve(n);
        for (std::size_t i = 0; i < n; ++i) v.push_back(RolloutRecord::from_rb(out[i]));
        return v;
    }

    // priority_with_replacement weights: w = base + floor(min(|advantage|, 2^15)
    // * adv_scale) + pos_bonus * [reward > 0] (rb_set_priority)
    void set_priority(std::uint32_t base, std::uint32_t adv_scale, std::uint32_t pos_bonus) {
        detail::rb_check(rb_set_priority(h_.get(), base, adv_scale, pos_bonus));
    }
    // per-shard priority mass of the shards this process holds (rb_priority_mass)
    std::vector<std::uint64_t> priority_mass() const {
        std::vector<std::uint64_t> m(num_shards());
        detail::rb_check(rb_priority_mass(h_.get(), m.data()));
        return m;
    }

    SamplingStrategy strategy() const {
        int s = 0;
        detail::rb_check(rb_strategy(h_.get(), &s));
        return static_cast<SamplingStrategy>(s);
    }
    const RetentionPolicy& retention() const {
        int k = 0;
        double d = 0.0;
        detail::rb_check(rb_retention(h_.get(), &k, &d));
        retention_.kind = static_cast<RetentionPolicy::Kind>(k);
        retention_.delta = d;
        return retention_;
    }

    // replay_buffer.cpp:238-324 (byte-identical text)
    std::string dump() const {
        std::size_t len = 0;
        detail::rb_check(rb_dump(h_.get(), nullptr, 0, &len));
        std::string s(len + 1, '\0');
        detail::rb_check(rb_dump(h_.get(), s.data(), s.size(), &len));
        s.resize(len);
        return s;
    }
    static ShardedReplayBuffer load(std::string_view text) {
        rb_buffer* h = nullptr;
        detail::rb_check(rb_load(std::string(text).c_str(), 0, -1, &h));
        return ShardedReplayBuffer(h);
    }

    rb_buffer* handle() const { return h_.get(); }

private:
    explicit ShardedReplayBuffer(rb_buffer* h) { h_.reset(h); }
    std::size_t get(int (*fn)(const rb_buffer*, std::size_t*)) const {
        std::size_t v = 0;
        detail::rb_check(fn(h_.get(), &v));
        return v;
    }
    struct Del {
        void operator()(rb_buffer* b) const { rb_destroy(b); }
    };
    std::unique_ptr<rb_buffer, Del> h_;
    mutable RetentionPolicy retention_;
};

}  // namespace replab
