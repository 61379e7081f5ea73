// Suite for the standalone facade header replab/bandit.hpp (GPU): the
// reference's known answers for group advantages, LossSpec validation and the
// record-level losses (test_bandit.cpp:169-214, 301-470, restated over
// logp_now instead of the toy policy), and the token form at L = 1 agreeing
// with the record form.  Built by oracle/Makefile (reftests), run by
// tests/test_reference_suites.py.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"

#include <cmath>
#include <limits>
#include <stdexcept>
#include <vector>

#include "replab/bandit.hpp"

using replab::LossSpec;
using replab::RolloutRecord;
using replab::RolloutSideTables;

namespace {
RolloutRecord rec(uint64_t id, uint64_t group, double reward, double blp, double adv) {
    RolloutRecord r;
    r.rollout_id = id;
    r.group_id = group;
    r.reward = reward;
    r.is_correct = reward == 1.0;
    r.behavior_logprob = blp;
    r.advantage = adv;
    return r;
}
}  // namespace

TEST_CASE("group advantages: worked example, constant groups, too-small groups") {
    const auto a = replab::group_advantages({1.0, 0.0, 1.0, 0.0});
    REQUIRE(a.size() == 4);
    CHECK(a[0] == doctest::Approx(1.0).epsilon(1e-12));
    CHECK(a[1] == doctest::Approx(-1.0).epsilon(1e-12));
    for (double v : replab::group_advantages({1.0, 1.0, 1.0})) CHECK(v == 0.0);
    CHECK_THROWS_AS(replab::group_advantages({1.0}), std::invalid_argument);
    // population std, exactly as bandit.cpp:276-294
    const std::vector<double> r = {0.0, 1.0, 1.0, 0.5, 0.25};
    double m = 0.0;
    for (double x : r) m += x;
    m /= 5.0;
    double v = 0.0;
    for (double x : r) v += (x - m) * (x - m);
    v /= 5.0;
    const auto g = replab::group_advantages(r);
    for (int i = 0; i < 5; ++i) CHECK(g[i] == (r[i] - m) / std::sqrt(v));
}

TEST_CASE("loss specs validate and names round trip") {
    CHECK_NOTHROW(LossSpec::grpo(0.2, 0.2, 16).validate());
    CHECK_THROWS_AS(LossSpec::grpo(-0.1, 0.2, 16), std::invalid_argument);
    CHECK_THROWS_AS(LossSpec::grpo(0.2, -0.1, 16), std::invalid_argument);
    CHECK_THROWS_AS(LossSpec::grpo(0.2, 0.2, 1), std::invalid_argument);
    CHECK_THROWS_AS(LossSpec::asymre(-0.1, 1), std::invalid_argument);
    LossSpec nan_spec;
    nan_spec.delta_v = std::numeric_limits<double>::quiet_NaN();
    CHECK_THROWS_AS(nan_spec.validate(), std::invalid_argument);
    CHECK(replab::to_string(LossSpec::Kind::grpo) == "grpo");
    CHECK(replab::loss_kind_from_string("asymre") == LossSpec::Kind::asymre);
    CHECK_THROWS_AS(replab::loss_kind_from_string("ppo"), std::invalid_argument);
}

TEST_CASE("clipped surrogate: saturated ratio gives the clipped value and zero gradient") {
    // ratio = exp(log 2) = 2 > 1.2 with A = 1: clipped branch, value 1.2
    const auto spec = LossSpec::grpo(0.2, 0.2, 2);
    std::vector<RolloutRecord> b = {rec(1, 0, 1.0, std::log(0.25), 1.0)};
    const auto r = replab::grpo_loss_grad({std::log(0.5)}, b, spec);
    CHECK(r.objective == doctest::Approx(1.2).epsilon(1e-12));
    CHECK(r.grad[0] == 0.0);
    CHECK(r.excluded == 0);
    // negative advantage, ratio 0.5 < 0.8: min(0.5 * -1, 0.8 * -1) = -0.8 (clipped)
    b[0].advantage = -1.0;
    b[0].behavior_logprob = std::log(1.0);
    const auto c = replab::grpo_loss_grad({std::log(0.5)}, b, spec);
    CHECK(c.objective == doctest::Approx(-0.8).epsilon(1e-12));
    CHECK(c.grad[0] == 0.0);
    CHECK_THROWS_AS(replab::grpo_loss_grad({}, {}, spec), std::invalid_argument);
}

TEST_CASE("on-policy batches reduce to advantage-weighted ascent") {
    const auto spec = LossSpec::grpo(0.2, 0.2, 2);
    std::vector<RolloutRecord> b;
    std::vector<double> lpn;
    double mean_adv = 0.0;
    for (int i = 0; i < 6; ++i) {
        const double a = (i % 3) - 1.0 + 0.25 * i;
        b.push_back(rec(i, 0, 0.0, -0.5 - 0.1 * i, a));
        lpn.push_back(-0.5 - 0.1 * i);
        mean_adv += a;
    }
    const auto r = replab::grpo_loss_grad(lpn, b, spec);
    CHECK(r.objective == doctest::Approx(mean_adv / 6.0).epsilon(1e-12));
    for (int i = 0; i < 6; ++i) CHECK(r.grad[i] == doctest::Approx(-b[i].advantage / 6.0).epsilon(1e-12));
}

TEST_CASE("non-finite importance ratios are excluded with the rest averaged") {
    const auto spec = LossSpec::grpo(0.2, 0.2, 2);
    std::vector<RolloutRecord> b = {rec(1, 0, 1.0, -1.0, 1.0), rec(2, 0, 0.0, -1000.0, -1.0)};
    const auto r = replab::grpo_loss_grad({-1.0, 0.0}, b, spec);  // exp(1000) = inf
    CHECK(r.excluded == 1);
    CHECK(r.objective == doctest::Approx(1.0).epsilon(1e-12));
    CHECK(r.grad[0] == doctest::Approx(-1.0).epsilon(1e-12));
    CHECK(r.grad[1] == 0.0);
}

TEST_CASE("ratio-free loss: zero coefficient freezes, single record scales the score") {
    const auto spec = LossSpec::asymre(0.0, 2);
    RolloutSideTables t;
    t.group_mean_reward[7] = 1.0;
    std::vector<RolloutRecord> b = {rec(1, 7, 1.0, 0.0, 0.0)};
    const auto frozen = replab::asymre_loss_grad({std::log(0.5)}, b, t, spec);
    CHECK(frozen.objective == 0.0);
    CHECK(frozen.grad[0] == 0.0);
    t.group_mean_reward[7] = 0.5;
    const auto scaled = replab::asymre_loss_grad({std::log(0.5)}, b, t, spec);
    CHECK(scaled.objective == doctest::Approx(0.5 * std::log(0.5)).epsilon(1e-12));
    CHECK(scaled.grad[0] == doctest::Approx(-0.5).epsilon(1e-12));
    RolloutSideTables missing;
    CHECK_THROWS_AS(replab::asymre_loss_grad({0.0}, b, missing, spec), std::invalid_argument);
    // dispatch
    const auto d = replab::loss_grad({std::log(0.5)}, b, t, spec);
    CHECK(d.objective == scaled.objective);
}

TEST_CASE("token form at L = 1 equals the record form; sequence ratio mode") {
    const auto spec = LossSpec::grpo(0.2, 0.3, 2);
    std::vector<RolloutRecord> b;
    std::vector<double> lpn_d;
    std::vector<float> lpn, lpo;
    std::vector<double> adv;
    std::vector<int64_t> off = {0};
    for (int i = 0; i < 64; ++i) {
        const float now = -1.0f + 0.01f * (i % 17), old = -1.0f + 0.013f * (i % 11);
        lpn.push_back(now);
        lpo.push_back(old);
        lpn_d.push_back(now);
        adv.push_back((i % 5) - 2.0);
        b.push_back(rec(i, 0, 0.0, old, adv.back()));
        off.push_back(i + 1);
    }
    const auto rr = replab::grpo_loss_grad(lpn_d, b, spec);
    const auto tr = replab::grpo_loss_grad_tokens(lpn, lpo, adv, off, spec);
    REQUIRE(tr.dlogp.size() == 64);
    CHECK(tr.included == 64);
    CHECK(tr.objective == doctest::Approx(rr.objective).epsilon(1e-6));
    for (int i = 0; i < 64; ++i)
        CHECK(tr.dlogp[i] == doctest::Approx(rr.grad[i]).epsilon(1e-5));
    const auto sr = replab::grpo_loss_grad_tokens(lpn, lpo, adv, off, spec,
                                                  replab::GrpoMode::seq_ratio);
    CHECK(sr.objective == doctest::Approx(rr.objective).epsilon(1e-6));
    // AsymRE token form: every token of trajectory i gets -coef_i / B
    std::vector<double> reward(64, 1.0), gm(64, 0.25);
    const auto at = replab::asymre_loss_grad_tokens(lpn, reward, gm, off, LossSpec::asymre(-0.1, 2));
    for (int i = 0; i < 64; ++i)
        CHECK(at.dlogp[i] == doctest::Approx(-(1.0 - (0.25 - 0.1)) / 64.0).epsilon(1e-6));
}
