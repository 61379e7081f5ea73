// replab/bandit.hpp — drop-in C++ facade of the replay-step part of
// replab's bandit.hpp (bandit.hpp:66-144) over the libreplay_b200 C-ABI:
// LossSpec (+ validate, factories, name codecs), RolloutSideTables,
// group_advantages, LossResult and the two off-policy losses.
//
// The reference's losses take the toy SoftmaxPolicy (bandit.hpp:48-64) and
// return the gradient over its logit table.  That policy is the LLM's
// stand-in and is out of scope here: these overloads
// take what the policy contributes — each record's log-probability under the
// current policy, logp_now — and return dL/dlogp_now per record (the
// quantity the trainer back-propagates).  A project that keeps the toy
// policy compiles facade/bandit_b200.cpp instead, which provides the
// reference's exact signatures on top of the same kernels.  Token-level
// (LLM) forms are below; the hot path inside a buffer is rb_loss_grpo_ex /
// rb_loss_asymre (include/replay_b200.h).
#pragma once

#include <cmath>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "replab/bandit_core.hpp"
#include "replab/rollout.hpp"

namespace replab {

// bandit.hpp:73-90, bandit.cpp:229-259
struct LossSpec {
    enum class Kind { grpo, asymre };

    Kind kind = Kind::grpo;
    double eps_low = 0.2;
    double eps_high = 0.2;
    double delta_v = -0.1;
    std::size_t group_size = 16;

    static LossSpec grpo(double eps_low = 0.2, double eps_high = 0.2, std::size_t group_size = 16) {
        LossSpec s;
        s.kind = Kind::grpo;
        s.eps_low = eps_low;
        s.eps_high = eps_high;
        s.group_size = group_size;
        s.validate();
        return s;
    }
    static LossSpec asymre(double delta_v = -0.1, std::size_t group_size = 16) {
        LossSpec s;
        s.kind = Kind::asymre;
        s.delta_v = delta_v;
        s.group_size = group_size;
        s.validate();
        return s;
    }
    // Same checks, order and messages as bandit.cpp:246-258.
    void validate() const {
        if (eps_low < 0.0 || eps_high < 0.0)
            throw std::invalid_argument("loss spec: clip bounds must be >= 0");
        if (!std::isfinite(eps_low) || !std::isfinite(eps_high) || !std::isfinite(delta_v))
            throw std::invalid_argument("loss spec: parameters must be finite");
        if (group_size < 2)
            throw std::invalid_argument("loss spec: group_size must be >= 2, got " +
                                        std::to_string(group_size));
    }
};

inline std::string to_string(LossSpec::Kind k) {  // bandit.cpp:261-267
    switch (k) {
        case LossSpec::Kind::grpo: return "grpo";
        case LossSpec::Kind::asymre: return "asymre";
    }
    throw std::logic_error("unknown loss kind");
}

inline LossSpec::Kind loss_kind_from_string(std::string_view s) {  // bandit.cpp:269-274
    if (s == "grpo") return LossSpec::Kind::grpo;
    if (s == "asymre") return LossSpec::Kind::asymre;
    throw std::invalid_argument("unknown loss kind '" + std::string(s) +
                                "' (expected grpo or asymre)");
}

// bandit.hpp:98-101: the AsymRE baseline V-hat per group, frozen at
// generation (the arm table belongs to the toy policy and is not needed
// when logp_now is given).
struct RolloutSideTables {
    std::map<uint64_t, std::size_t> arm_of;
    std::map<uint64_t, double> group_mean_reward;
};

// bandit.cpp:276-294 on the GPU (k_group_adv, bit-exact fp64).
inline std::vector<double> group_advantages(const std::vector<double>& rewards) {
    return b200::group_advantages(rewards);
}

// bandit.hpp:124-131, with the gradient w.r.t. each record's logp_now in
// place of the logit-table gradient: grad[i] = d(-objective)/d logp_now_i.
struct LossResult {
    double objective = 0.0;
    std::vector<double> grad;
    std::size_t excluded = 0;
};

namespace detail {
inline void check_batch(const std::vector<RolloutRecord>& batch, const std::vector<double>& lpn) {
    if (batch.empty()) throw std::invalid_argument("loss gradient needs a non-empty batch");
    if (lpn.size() != batch.size())
        throw std::invalid_argument("loss gradient: one logp_now per record required");
}
}  // namespace detail

// bandit.cpp:363-408: ratio exp(logp_now - behavior_logprob), non-finite
// ratios excluded, clip to [1-eps_low, 1+eps_high], ties unclipped, mean
// over the included records.
inline LossResult grpo_loss_grad(const std::vector<double>& logp_now,
                                 const std::vector<RolloutRecord>& batch, const LossSpec& spec) {
    spec.validate();
    detail::check_batch(batch, logp_now);
    std::vector<double> blp(batch.size()), adv(batch.size());
    for (std::size_t i = 0; i < batch.size(); ++i) {
        blp[i] = batch[i].behavior_logprob;
        adv[i] = batch[i].advantage;
    }
    auto r = b200::grpo_records(logp_now, blp, adv, spec.eps_low, spec.eps_high);
    LossResult out;
    out.objective = r.stats.objective;
    out.grad = std::move(r.dlogp);
    out.excluded = static_cast<std::size_t>(r.stats.excluded);
    return out;
}

// bandit.cpp:410-438: coef = reward - (group mean + delta_v), objective =
// mean coef * logp_now.  Throws like the reference when a group's mean is
// missing from the side table.
inline LossResult asymre_loss_grad(const std::vector<double>& logp_now,
                                   const std::vector<RolloutRecord>& batch,
                                   const RolloutSideTables& tables, const LossSpec& spec) {
    spec.validate();
    detail::check_batch(batch, logp_now);
    std::vector<double> reward(batch.size()), gmean(batch.size());
    for (std::size_t i = 0; i < batch.size(); ++i) {
        const auto it = tables.group_mean_reward.find(batch[i].group_id);
        if (it == tables.group_mean_reward.end())
            throw std::invalid_argument("group " + std::to_string(batch[i].group_id) +
                                        " missing from the mean-reward side table");
        reward[i] = batch[i].reward;
        gmean[i] = it->second;
    }
    auto r = b200::asymre_records(logp_now, reward, gmean, spec.delta_v);
    LossResult out;
    out.objective = r.stats.objective;
    out.grad = std::move(r.dlogp);
    return out;
}

// bandit.cpp:440-447
inline LossResult loss_grad(const std::vector<double>& logp_now,
                            const std::vector<RolloutRecord>& batch,
                            const RolloutSideTables& tables, const LossSpec& spec) {
    switch (spec.kind) {
        case LossSpec::Kind::grpo: return grpo_loss_grad(logp_now, batch, spec);
        case LossSpec::Kind::asymre: return asymre_loss_grad(logp_now, batch, tables, spec);
    }
    throw std::logic_error("unknown loss kind");
}

// ---- token level (the LLM form) ---------------------------
enum class GrpoMode { token_mean = RB_GRPO_TOKEN_MEAN, seq_mean = RB_GRPO_SEQ_MEAN,
                      seq_ratio = RB_GRPO_SEQ_RATIO };

struct TokenLossResult {
    double objective = 0.0;
    std::vector<float> dlogp;  // d(-objective)/d logp_now per token, packed like the input
    std::size_t included = 0;  // tokens (token_mean / seq_mean) or trajectories (seq_ratio)
    std::size_t excluded = 0;
};

// offsets: n_traj + 1 packed token offsets; advantage per trajectory;
// behavior_logprob per trajectory (seq_ratio; empty = sum_t logp_old).
inline TokenLossResult grpo_loss_grad_tokens(const std::vector<float>& logp_now,
                                             const std::vector<float>& logp_old,
                                             const std::vector<double>& advantage,
                                             const std::vector<int64_t>& offsets,
                                             const LossSpec& spec,
                                             GrpoMode mode = GrpoMode::token_mean,
                                             const std::vector<double>& behavior_logprob = {}) {
    spec.validate();
    if (offsets.size() < 2 || advantage.size() + 1 != offsets.size())
        throw std::invalid_argument("loss gradient needs a non-empty batch");
    const std::size_t ntok = static_cast<std::size_t>(offsets.back());
    if (logp_now.size() < ntok || logp_old.size() < ntok)
        throw std::invalid_argument("loss gradient: token arrays shorter than offsets.back()");
    TokenLossResult out;
    out.dlogp.resize(ntok + 4);
    rb_loss_stats st{};
    b200::check(rb_grpo_tokens_ex(logp_now.data(), logp_old.data(), advantage.data(),
                                  behavior_logprob.empty() ? nullptr : behavior_logprob.data(),
                                  offsets.data(), advantage.size(), spec.eps_low, spec.eps_high,
                                  static_cast<int>(mode), out.dlogp.data(), &st));
    out.dlogp.resize(ntok);
    out.objective = st.objective;
    out.included = static_cast<std::size_t>(st.included);
    out.excluded = static_cast<std::size_t>(st.excluded);
    return out;
}

inline TokenLossResult asymre_loss_grad_tokens(const std::vector<float>& logp_now,
                                               const std::vector<double>& reward,
                                               const std::vector<double>& group_mean,
                                               const std::vector<int64_t>& offsets,
                                               const LossSpec& spec) {
    spec.validate();
    if (offsets.size() < 2 || reward.size() + 1 != offsets.size() ||
        group_mean.size() != reward.size())
        throw std::invalid_argument("loss gradient needs a non-empty batch");
    const std::size_t ntok = static_cast<std::size_t>(offsets.back());
    if (logp_now.size() < ntok)
        throw std::invalid_argument("loss gradient: token arrays shorter than offsets.back()");
    TokenLossResult out;
    out.dlogp.resize(ntok + 4);
    rb_loss_stats st{};
    b200::check(rb_asymre_tokens(logp_now.data(), reward.data(), group_mean.data(), offsets.data(),
                                 reward.size(), spec.delta_v, out.dlogp.data(), &st));
    out.dlogp.resize(ntok);
    out.objective = st.objective;
    out.included = static_cast<std::size_t>(st.included);
    return out;
}

}  // namespace replab
