// bandit_b200.cpp — the replay-step functions of replab's bandit.cpp with the
// reference's exact signatures, computed by libreplay_b200's kernels.
//
// A maintainer compiles this file INSIDE the reference project, against the
// project's own include/replab/bandit.hpp, and drops the four definitions
// below from bandit.cpp (or, as tests/test_reference_suites.py does, links
// this object ahead of the unmodified library: an executable's definitions
// interpose on the shared library's, so train() in the library calls these
// too).  Replaced:
//   group_advantages   bandit.cpp:276-294
//   grpo_loss_grad     bandit.cpp:363-408
//   asymre_loss_grad   bandit.cpp:410-438
//   loss_grad          bandit.cpp:440-447
// The toy policy stays the project's: its logprob() supplies each record's
// logp_now, and the chain rule into its logit table,
// d logprob(arm)/d logit_j = (1[j == arm] - p_j) / temperature
// (bandit.cpp:342-350), is applied to the per-record dL/dlogp the GPU returns.
#include <cmath>
#include <cstdlib>
#include <iostream>
#include <stdexcept>
#include <string>
#include <vector>

#include <replab/bandit.hpp>       // the PROJECT's header (reference API; -I order)
#include "replab/bandit_core.hpp"  // libreplay_b200 array calls

namespace replab {

namespace {

// Count of replaced calls (RB_FACADE_TRACE=1 prints it at exit), so a test
// can show these definitions, not the library's, ran.
struct Trace {
    long calls = 0;
    ~Trace() {
        const char* e = std::getenv("RB_FACADE_TRACE");
        if (e && e[0] == '1') std::cout << "[b200-bandit] " << calls << " calls\n";
    }
} g_trace;

std::size_t arm_of(const RolloutSideTables& tables, const RolloutRecord& rec) {
    const auto it = tables.arm_of.find(rec.rollout_id);
    if (it == tables.arm_of.end())
        throw std::invalid_argument("rollout " + std::to_string(rec.rollout_id) +
                                    " missing from the arm side table");
    return it->second;
}

// grad[prompt row] += g * d logprob(arm) / d logits, g = dL/dlogp_now.
void chain_into_logits(const SoftmaxPolicy& policy, const std::vector<RolloutRecord>& batch,
                       const std::vector<std::size_t>& arms, const std::vector<double>& dlogp,
                       std::vector<double>& grad) {
    const double tau = policy.temperature_train;
    for (std::size_t i = 0; i < batch.size(); ++i) {
        if (dlogp[i] == 0.0) continue;
        const std::size_t prompt = batch[i].prompt_id;
        const std::vector<double> p = policy.probs(prompt, tau);
        double* row = grad.data() + prompt * policy.num_arms;
        for (std::size_t j = 0; j < policy.num_arms; ++j)
            row[j] += dlogp[i] * ((j == arms[i] ? 1.0 : 0.0) - p[j]) / tau;
    }
}

}  // namespace

std::vector<double> group_advantages(const std::vector<double>& rewards) {
    ++g_trace.calls;
    return b200::group_advantages(rewards);
}

LossResult grpo_loss_grad(const SoftmaxPolicy& policy, const std::vector<RolloutRecord>& batch,
                          const RolloutSideTables& tables, const LossSpec& spec) {
    ++g_trace.calls;
    spec.validate();
    if (batch.empty()) throw std::invalid_argument("loss gradient needs a non-empty batch");
    const double tau = policy.temperature_train;
    const std::size_t n = batch.size();
    std::vector<std::size_t> arms(n);
    std::vector<double> lpn(n), blp(n), adv(n);
    for (std::size_t i = 0; i < n; ++i) {
        arms[i] = arm_of(tables, batch[i]);
        lpn[i] = policy.logprob(batch[i].prompt_id, arms[i], tau);
        blp[i] = batch[i].behavior_logprob;
        adv[i] = batch[i].advantage;
    }
    auto r = b200::grpo_records(lpn, blp, adv, spec.eps_low, spec.eps_high);
    LossResult result;
    result.grad.assign(policy.logits.size(), 0.0);
    result.excluded = static_cast<std::size_t>(r.stats.excluded);
    if (result.excluded) {  // the reference's per-record warning (bandit.cpp:381-384)
        for (std::size_t i = 0; i < n; ++i)
            if (!std::isfinite(std::exp(lpn[i] - blp[i])))
                std::cerr << "warning: rollout " << batch[i].rollout_id
                          << " has non-finite importance ratio; excluded from the update\n";
    }
    if (r.stats.included > 0) {
        result.objective = r.stats.objective;
        chain_into_logits(policy, batch, arms, r.dlogp, result.grad);
    }
    return result;
}

LossResult asymre_loss_grad(const SoftmaxPolicy& policy, const std::vector<RolloutRecord>& batch,
                            const RolloutSideTables& tables, const LossSpec& spec) {
    ++g_trace.calls;
    spec.validate();
    if (batch.empty()) throw std::invalid_argument("loss gradient needs a non-empty batch");
    const double tau = policy.temperature_train;
    const std::size_t n = batch.size();
    std::vector<std::size_t> arms(n);
    std::vector<double> lpn(n), reward(n), gmean(n);
    for (std::size_t i = 0; i < n; ++i) {
        arms[i] = arm_of(tables, batch[i]);
        const auto it = tables.group_mean_reward.find(batch[i].group_id);
        if (it == tables.group_mean_reward.end())
            throw std::invalid_argument("group " + std::to_string(batch[i].group_id) +
                                        " missing from the mean-reward side table");
        gmean[i] = it->second;
        reward[i] = batch[i].reward;
        lpn[i] = policy.logprob(batch[i].prompt_id, arms[i], tau);
    }
    auto r = b200::asymre_records(lpn, reward, gmean, spec.delta_v);
    LossResult result;
    result.grad.assign(policy.logits.size(), 0.0);
    result.objective = r.stats.objective;
    chain_into_logits(policy, batch, arms, r.dlogp, result.grad);
    return result;
}

LossResult loss_grad(const SoftmaxPolicy& policy, const std::vector<RolloutRecord>& batch,
                     const RolloutSideTables& tables, const LossSpec& spec) {
    switch (spec.kind) {
        case LossSpec::Kind::grpo: return grpo_loss_grad(policy, batch, tables, spec);
        case LossSpec::Kind::asymre: return asymre_loss_grad(policy, batch, tables, spec);
    }
    throw std::logic_error("unknown loss kind");
}

}  // namespace replab
