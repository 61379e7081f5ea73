// doctest.h — minimal doctest-compatible shim (test infrastructure).
//
// The reference's test suites include "doctest.h" from vendor/, which is
// absent from the mount (proj/.gitignore:2).  This shim
// implements exactly the subset those suites use — TEST_CASE, SUBCASE
// (sibling subcases, re-running the case once per subcase as doctest does),
// CHECK/REQUIRE (+_FALSE/_MESSAGE), CHECK_THROWS/_AS/_WITH_AS,
// CHECK_NOTHROW, FAIL, doctest::Approx(.epsilon), doctest::Contains — so the
// reference's own test_buffer_core.cpp / test_rng.cpp compile unchanged,
// against the reference library and against the libreplay_b200 facade.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <iostream>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.v_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.v_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

private:
    double v_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
    double scale_ = 1.0;
};

struct Contains {
    explicit Contains(const char* s) : str(s) {}
    bool check(const std::string& m) const { return m.find(str) != std::string::npos; }
    std::string str;
};

namespace detail {

struct TestCase {
    const char* name;
    void (*fn)();
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
struct Reg {
    Reg(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};

struct State {
    int failures = 0, checks = 0;
    int subcase_target = 0, subcase_seen = 0;
    bool case_failed = false;
};
inline State& st() {
    static State s;
    return s;
}

inline bool enter_subcase() {
    State& s = st();
    return s.subcase_seen++ == s.subcase_target;
}

inline void report(const char* kind, const char* expr, const char* file, int line,
                   const std::string& msg) {
    std::cerr << file << ":" << line << ": FAILED " << kind << "( " << expr << " )";
    if (!msg.empty()) std::cerr << " with message: " << msg;
    std::cerr << "\n";
}

inline bool check(bool ok, const char* expr, const char* file, int line, bool require,
                  const std::string& msg = std::string()) {
    State& s = st();
    ++s.checks;
    if (!ok) {
        ++s.failures;
        s.case_failed = true;
        report(require ? "REQUIRE" : "CHECK", expr, file, line, msg);
        if (require) throw RequireFailed{};
    }
    return ok;
}

template <class... A>
std::string cat(const A&... a) {
    std::ostringstream os;
    (os << ... << a);
    return os.str();
}

inline int run_all() {
    int failed_cases = 0;
    for (const TestCase& tc : registry()) {
        State& s = st();
        s.case_failed = false;
        s.subcase_target = 0;
        for (;;) {
            s.subcase_seen = 0;
            try {
                tc.fn();
            } catch (RequireFailed&) {
            } catch (const std::exception& e) {
                ++s.failures;
                s.case_failed = true;
                std::cerr << "TEST CASE '" << tc.name << "' threw: " << e.what() << "\n";
            }
            if (s.subcase_seen <= s.subcase_target + 1) break;
            ++s.subcase_target;
        }
        if (s.case_failed) {
            ++failed_cases;
            std::cerr << "TEST CASE FAILED: " << tc.name << "\n";
        }
    }
    std::cout << "[doctest-shim] test cases: " << registry().size() << " | "
              << registry().size() - failed_cases << " passed | " << failed_cases
              << " failed | assertions: " << st().checks << " | " << st().failures
              << " failed\n";
    return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                    \
    static void fn();                                            \
    static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, &fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __LINE__), name)
#define SUBCASE(name) if (::doctest::detail::enter_subcase())

#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE_FALSE(...) ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_MESSAGE(cond, ...) \
    ::doctest::detail::check(static_cast<bool>(cond), #cond, __FILE__, __LINE__, false, ::doctest::detail::cat(__VA_ARGS__))
#define REQUIRE_MESSAGE(cond, ...) \
    ::doctest::detail::check(static_cast<bool>(cond), #cond, __FILE__, __LINE__, true, ::doctest::detail::cat(__VA_ARGS__))
#define FAIL(...) ::doctest::detail::check(false, "FAIL", __FILE__, __LINE__, true, ::doctest::detail::cat(__VA_ARGS__))

#define CHECK_THROWS(expr)                                                                   \
    do {                                                                                     \
        bool _thrown = false;                                                                \
        try {                                                                                \
            (void)(expr);                                                                    \
        } catch (...) {                                                                      \
            _thrown = true;                                                                  \
        }                                                                                    \
        ::doctest::detail::check(_thrown, "CHECK_THROWS(" #expr ")", __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                               \
    do {                                                                                          \
        bool _ok = false;                                                                         \
        try {                                                                                     \
            (void)(expr);                                                                         \
        } catch (const type&) {                                                                   \
            _ok = true;                                                                           \
        } catch (...) {                                                                           \
        }                                                                                         \
        ::doctest::detail::check(_ok, "CHECK_THROWS_AS(" #expr ", " #type ")", __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, type)                                                 \
    do {                                                                                          \
        bool _ok = false;                                                                         \
        try {                                                                                     \
            (void)(expr);                                                                         \
        } catch (const type& _e) {                                                                \
            _ok = (matcher).check(_e.what());                                                     \
        } catch (...) {                                                                           \
        }                                                                                         \
        ::doctest::detail::check(_ok, "CHECK_THROWS_WITH_AS(" #expr ")", __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                  \
    do {                                                                                     \
        bool _ok = true;                                                                     \
        try {                                                                                \
            (void)(expr);                                                                    \
        } catch (...) {                                                                      \
            _ok = false;                                                                     \
        }                                                                                    \
        ::doctest::detail::check(_ok, "CHECK_NOTHROW(" #expr ")", __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
