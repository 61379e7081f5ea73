// replab/rollout.hpp — RolloutRecord (rollout.hpp:13-31) for the facade.
// Layout-identical to rb_record (80 bytes); to_line/from_line follow
// rollout.cpp:9-35 and text_io.cpp (shortest round-trip doubles).
#pragma once

#include <charconv>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "replay_b200.h"

namespace replab {

inline std::string format_double(double v) {  // text_io.cpp:10-14
    char buf[64];
    auto res = std::to_chars(buf, buf + sizeof(buf), v);
    return std::string(buf, res.ptr);
}

struct RolloutRecord {
    uint64_t rollout_id = 0;
    uint64_t prompt_id = 0;
    uint64_t group_id = 0;
    int64_t creation_step = 0;
    int64_t policy_version = 0;
    double reward = 0.0;
    bool is_correct = false;
    double behavior_logprob = 0.0;
    double advantage = 0.0;
    uint32_t use_count = 0;

    std::string to_line() const {
        return std::to_string(rollout_id) + "," + std::to_string(prompt_id) + "," +
               std::to_string(group_id) + "," + std::to_string(creation_step) + "," +
               std::to_string(policy_version) + "," + format_double(reward) + "," +
               (is_correct ? "1" : "0") + "," + format_double(behavior_logprob) + "," +
               format_double(advantage) + "," + std::to_string(use_count);
    }
    bool operator==(const RolloutRecord&) const = default;

    rb_record to_rb() const {
        rb_record r{};
        r.rollout_id = rollout_id;
        r.prompt_id = prompt_id;
        r.group_id = group_id;
        r.creation_step = creation_step;
        r.policy_version = policy_version;
        r.reward = reward;
        r.is_correct = is_correct ? 1 : 0;
        r.behavior_logprob = behavior_logprob;
        r.advantage = advantage;
        r.use_count = use_count;
        return r;
    }
    static RolloutRecord from_rb(const rb_record& r) {
        RolloutRecord o;
        o.rollout_id = r.rollout_id;
        o.prompt_id = r.prompt_id;
        o.group_id = r.group_id;
        o.creation_step = r.creation_step;
        o.policy_version = r.policy_version;
        o.reward = r.reward;
        o.is_correct = r.is_correct != 0;
        o.behavior_logprob = r.behavior_logprob;
        o.advantage = r.advantage;
        o.use_count = r.use_count;
        return o;
    }
};
static_assert(sizeof(RolloutRecord) == sizeof(rb_record), "record layout");

}  // namespace replab
