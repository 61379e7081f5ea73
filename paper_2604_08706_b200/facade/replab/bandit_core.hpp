// replab/bandit_core.hpp — array-level calls shared by the two bandit
// drop-ins over the libreplay_b200 C-ABI:
//   * replab/bandit.hpp      standalone header of the in-scope bandit surface
//                            (LossSpec, LossResult, group_advantages, losses);
//   * facade/bandit_b200.cpp the translation unit a maintainer compiles INSIDE
//                            the reference project, against its own
//                            replab/bandit.hpp, in place of bandit.cpp's hot
//                            functions (bandit.cpp:276-294, 363-447).
// Every computation here is a GPU kernel of the library; this header only
// moves arrays and turns status codes into the reference's exceptions.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <vector>

#include "replay_b200.h"

namespace replab::b200 {

inline void check(int st) {
    if (st == RB_OK) return;
    if (st == RB_EINVAL) throw std::invalid_argument(rb_last_error());
    if (st == RB_ELOGIC) throw std::logic_error(rb_last_error());
    throw std::runtime_error(rb_last_error());
}

// bandit.cpp:276-294 — one group; throws std::invalid_argument("group
// advantages need >= 2 rewards") like the reference.
inline std::vector<double> group_advantages(const std::vector<double>& rewards) {
    if (rewards.size() < 2) throw std::invalid_argument("group advantages need >= 2 rewards");
    std::vector<double> adv(rewards.size());
    const int64_t off[2] = {0, static_cast<int64_t>(rewards.size())};
    double mean = 0.0;
    check(rb_group_advantages(rewards.data(), off, 1, adv.data(), &mean));
    return adv;
}

// Record level (L = 1), fp64: dL/dlogp_now per record and the batch stats.
struct RecordLoss {
    std::vector<double> dlogp;  // d(-objective)/d logp_now_i, already normalised
    rb_loss_stats stats{};
};

// bandit.cpp:363-408 per record.
inline RecordLoss grpo_records(const std::vector<double>& logp_now,
                               const std::vector<double>& behavior_logprob,
                               const std::vector<double>& advantage, double eps_low,
                               double eps_high) {
    RecordLoss r;
    r.dlogp.resize(logp_now.size());
    check(rb_grpo_records(logp_now.data(), behavior_logprob.data(), advantage.data(),
                          logp_now.size(), eps_low, eps_high, r.dlogp.data(), &r.stats));
    return r;
}

// bandit.cpp:410-438 per record.
inline RecordLoss asymre_records(const std::vector<double>& logp_now,
                                 const std::vector<double>& reward,
                                 const std::vector<double>& group_mean, double delta_v) {
    RecordLoss r;
    r.dlogp.resize(logp_now.size());
    check(rb_asymre_records(logp_now.data(), reward.data(), group_mean.data(), logp_now.size(),
                            delta_v, r.dlogp.data(), &r.stats));
    return r;
}

}  // namespace replab::b200
