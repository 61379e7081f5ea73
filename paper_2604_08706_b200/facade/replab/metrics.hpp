// replab/metrics.hpp — the part of the use ledger (metrics.hpp:22-70) that the
// replay path touches: UseEvent and MetricsLedger::record_use / events().
// The ledger diagnostics (staleness, replay counts, summaries) are SURVEY.md
// §8f row 1 ("next") and not part of this facade.
#pragma once

#include <cstdint>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "replab/rng.hpp"

namespace replab {

struct UseEvent {
    std::uint64_t rollout_id = 0;
    std::int64_t creation_step = 0;
    std::int64_t use_step = 0;
    std::int64_t batch_id = 0;
    std::int64_t within_batch_rank = 0;
    bool operator==(const UseEvent&) const = default;
};

class MetricsLedger {
public:
    // metrics.cpp:56-69: use_step >= creation_step, (batch, rank) unique.
    void record_use(const UseEvent& e) {
        std::lock_guard<std::mutex> lock(mu_);
        if (e.use_step < e.creation_step)
            throw std::invalid_argument("use event for rollout " + std::to_string(e.rollout_id) +
                                        " precedes its creation step");
        if (!slots_.insert({e.batch_id, e.within_batch_rank}).second)
            throw std::invalid_argument("duplicate batch slot (batch " +
                                        std::to_string(e.batch_id) + ", rank " +
                                        std::to_string(e.within_batch_rank) + ")");
        events_.push_back(e);
    }
    const std::vector<UseEvent>& events() const { return events_; }

private:
    std::vector<UseEvent> events_;
    std::set<std::pair<std::int64_t, std::int64_t>> slots_;
    std::mutex mu_;
};

}  // namespace replab
