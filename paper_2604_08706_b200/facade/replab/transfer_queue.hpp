// replab/transfer_queue.hpp — drop-in C++ facade of replab::TransferQueue
// (transfer_queue.hpp:12-35) over the libreplay_b200 C-ABI: the consume-once
// LIFO hand-off of the no-buffer baseline, stored in HBM (records only here;
// payload-carrying queues use the C-ABI or the Python mirror directly).
#pragma once

#include <memory>
#include <optional>
#include <stdexcept>
#include <vector>

#include "replab/rng.hpp"
#include "replab/rollout.hpp"

namespace replab {

class TransferQueue {
public:
    explicit TransferQueue(std::optional<std::size_t> capacity = std::nullopt)
        : capacity_(capacity) {
        if (capacity_ && *capacity_ == 0)  // transfer_queue.cpp:8-10
            throw std::invalid_argument("TransferQueue: capacity must be positive");
        rb_queue* q = nullptr;
        detail::rb_check(rb_queue_create(capacity_ ? *capacity_ : 0, 0, -1, &q));
        q_.reset(q);
    }

    // false = queue full (record not enqueued) — transfer_queue.cpp:13-20
    bool push(const RolloutRecord& record) { return push_group({record}); }

    // all or nothing — transfer_queue.cpp:22-29
    bool push_group(const std::vector<RolloutRecord>& records) {
        const std::size_t n = records.size();
        std::vector<uint64_t> id(n), prompt(n), group(n);
        std::vector<int64_t> cstep(n), pver(n);
        std::vector<double> reward(n), blp(n), adv(n);
        std::vector<uint8_t> correct(n);
        for (std::size_t i = 0; i < n; ++i) {
            const RolloutRecord& r = records[i];
            id[i] = r.rollout_id;
            prompt[i] = r.prompt_id;
            group[i] = r.group_id;
            cstep[i] = r.creation_step;
            pver[i] = r.policy_version;
            reward[i] = r.reward;
            correct[i] = r.is_correct ? 1 : 0;
            blp[i] = r.behavior_logprob;
            adv[i] = r.advantage;
        }
        rb_insert_batch b{};
        b.n = n;
        b.rollout_id = id.data();
        b.prompt_id = prompt.data();
        b.group_id = group.data();
        b.creation_step = cstep.data();
        b.policy_version = pver.data();
        b.reward = reward.data();
        b.is_correct = correct.data();
        b.behavior_logprob = blp.data();
        b.advantage = adv.data();
        int ok = 0;
        detail::rb_check(rb_queue_push_group(q_.get(), &b, &ok));
        return ok != 0;
    }

    // nullopt = queue empty — transfer_queue.cpp:31-39
    std::optional<RolloutRecord> pop() {
        rb_record r{};
        std::size_t n = 0;
        detail::rb_check(rb_queue_pop(q_.get(), 1, &r, &n, nullptr, nullptr, nullptr));
        if (!n) return std::nullopt;
        return RolloutRecord::from_rb(r);
    }

    std::size_t size() const {
        std::size_t v = 0;
        detail::rb_check(rb_queue_size(q_.get(), &v));
        return v;
    }
    std::optional<std::size_t> capacity() const { return capacity_; }

private:
    struct Del {
        void operator()(rb_queue* q) const { rb_queue_destroy(q); }
    };
    std::optional<std::size_t> capacity_;
    std::unique_ptr<rb_queue, Del> q_;
};

}  // namespace replab
