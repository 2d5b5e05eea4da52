// doctest.h — minimal self-written stand-in for the subset of the doctest
// 2.4 API the reference's unit tests use (TEST_CASE, CHECK, CHECK_FALSE,
// REQUIRE, CHECK_THROWS_AS, doctest::Approx(...).epsilon(...)), so the
// reference's UNMODIFIED tests/test_objectives.cpp, test_solvers.cpp and
// test_multigrid.cpp compile against the B200 drop-in headers
// (paper_1810_05628_b200/cpp/include/ptycho).  Not doctest itself: the real
// header is not vendored by the reference and there is no network.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    // doctest's rule: |lhs - rhs| < eps * (scale + max(|lhs|, |rhs|))
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator<=(double lhs, const Approx& a) { return lhs < a.value_ || lhs == a; }
    friend bool operator>=(double lhs, const Approx& a) { return lhs > a.value_ || lhs == a; }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

namespace detail {
struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Register {
    Register(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct Stats {
    long checks = 0, failed = 0;
    bool case_failed = false;
};
inline Stats& stats() {
    static Stats s;
    return s;
}
struct RequireFailed {};
inline void report(bool ok, const char* file, int line, const char* expr, bool require) {
    ++stats().checks;
    if (ok) return;
    ++stats().failed;
    stats().case_failed = true;
    std::printf("  %s:%d: %s FAILED: %s\n", file, line, require ? "REQUIRE" : "CHECK", expr);
    if (require) throw RequireFailed{};
}
}  // namespace detail

inline int run_all() {
    int failed_cases = 0;
    for (const auto& c : detail::registry()) {
        detail::stats().case_failed = false;
        try {
            c.fn();
        } catch (const detail::RequireFailed&) {
        } catch (const std::exception& e) {
            ++detail::stats().failed;
            detail::stats().case_failed = true;
            std::printf("  uncaught exception: %s\n", e.what());
        }
        if (detail::stats().case_failed) {
            ++failed_cases;
            std::printf("[FAILED] %s\n", c.name);
        } else {
            std::printf("[ok] %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu, failed: %d; checks: %ld, failed: %ld\n", detail::registry().size(),
                failed_cases, detail::stats().checks, detail::stats().failed);
    return failed_cases ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC(fn, name)                                                     \
    static void fn();                                                            \
    static ::doctest::detail::Register DOCTEST_CAT(fn, _reg)(name, &fn);         \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define CHECK_FALSE(...) ::doctest::detail::report(!(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define CHECK_THROWS_AS(expr, ...)                                                            \
    do {                                                                                      \
        bool doctest_ok_ = false;                                                             \
        try {                                                                                 \
            static_cast<void>(expr);                                                          \
        } catch (const __VA_ARGS__&) {                                                        \
            doctest_ok_ = true;                                                               \
        } catch (...) {                                                                       \
        }                                                                                     \
        ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, #expr " throws " #__VA_ARGS__, false); \
    } while (0)
