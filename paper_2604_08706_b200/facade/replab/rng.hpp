// replab/rng.hpp — drop-in C++ facade of replab::Rng (rng.hpp:22-69) over the
// libreplay_b200 C-ABI.  Same class, methods, semantics and exceptions; the
// MT19937-64 state lives in rb_rng (host or GPU, migrating on demand), so a
// stream consumed by ShardedReplayBuffer::sample on the GPU continues
// seamlessly with host draws, exactly as in the reference.
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "replay_b200.h"

namespace replab {

namespace detail {
inline void rb_check(int st) {
    if (st == RB_OK) return;
    if (st == RB_EINVAL) throw std::invalid_argument(rb_last_error());
    if (st == RB_ELOGIC) throw std::logic_error(rb_last_error());
    throw std::runtime_error(rb_last_error());
}
}  // namespace detail

// rng.cpp:8-15 (FNV-1a 64)
inline uint64_t hash_name(std::string_view name) {
    return rb_hash_name(std::string(name).c_str());
}

// rng.cpp:17-23
inline uint64_t splitmix64(uint64_t& state) {
    state += 0x9e3779b97f4a7c15ULL;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

class Rng {
public:
    explicit Rng(uint64_t seed) { detail::rb_check(rb_rng_create(seed, &h_)); }
    Rng(const Rng& o) { detail::rb_check(rb_rng_clone(o.h_, &h_)); }
    Rng(Rng&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    Rng& operator=(const Rng& o) {
        if (this != &o) {
            rb_rng* c = nullptr;
            detail::rb_check(rb_rng_clone(o.h_, &c));
            rb_rng_destroy(h_);
            h_ = c;
        }
        return *this;
    }
    Rng& operator=(Rng&& o) noexcept {
        std::swap(h_, o.h_);
        return *this;
    }
    ~Rng() {
        if (h_) rb_rng_destroy(h_);
    }

    Rng stream(std::string_view name) const {
        rb_rng* s = nullptr;
        detail::rb_check(rb_rng_stream(h_, std::string(name).c_str(), &s));
        return Rng(s);
    }
    Rng stream(std::string_view name, uint64_t index) const {
        rb_rng* s = nullptr;
        detail::rb_check(rb_rng_stream_index(h_, std::string(name).c_str(), index, &s));
        return Rng(s);
    }

    uint64_t seed() const { return rb_rng_seed(h_); }

    uint64_t next_u64() {
        uint64_t v;
        detail::rb_check(rb_rng_next_u64(h_, &v));
        return v;
    }
    uint64_t below(uint64_t bound) {
        uint64_t v;
        detail::rb_check(rb_rng_below(h_, bound, &v));
        return v;
    }
    double uniform01() {
        double v;
        detail::rb_check(rb_rng_uniform01(h_, &v));
        return v;
    }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
    double normal() {
        double v;
        detail::rb_check(rb_rng_normal(h_, &v));
        return v;
    }
    double normal(double mean, double stddev) { return mean + stddev * normal(); }

    // rng.cpp:72-85
    double lognormal_mean_cv(double mean, double cv) {
        if (mean <= 0.0) throw std::invalid_argument("Rng::lognormal_mean_cv: mean must be positive");
        if (cv < 0.0) throw std::invalid_argument("Rng::lognormal_mean_cv: cv must be non-negative");
        if (cv == 0.0) return mean;
        const double sigma_sq = std::log1p(cv * cv);
        const double mu_log = std::log(mean) - 0.5 * sigma_sq;
        return std::exp(mu_log + std::sqrt(sigma_sq) * normal());
    }

    // rng.cpp:87-104
    std::vector<double> unit_vector(std::size_t dim) {
        if (dim == 0) throw std::invalid_argument("Rng::unit_vector: dim must be positive");
        std::vector<double> v(dim);
        double norm_sq = 0.0;
        do {
            norm_sq = 0.0;
            for (auto& x : v) {
                x = normal();
                norm_sq += x * x;
            }
        } while (norm_sq == 0.0);
        const double inv = 1.0 / std::sqrt(norm_sq);
        for (auto& x : v) x *= inv;
        return v;
    }

    std::vector<std::size_t> sample_without_replacement(std::size_t n, std::size_t k) {
        std::vector<uint64_t> out(k ? k : 1);
        detail::rb_check(rb_rng_sample_without_replacement(h_, n, k, out.data()));
        return std::vector<std::size_t>(out.begin(), out.begin() + static_cast<std::ptrdiff_t>(k));
    }

    template <class T>
    void shuffle(std::vector<T>& v) {  // rng.hpp:59-64
        for (std::size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[below(i)]);
    }

    rb_rng* handle() const { return h_; }

private:
    explicit Rng(rb_rng* h) : h_(h) {}
    rb_rng* h_ = nullptr;
};

}  // namespace replab
