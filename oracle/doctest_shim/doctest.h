// Minimal doctest-compatible test shim (TEST INFRASTRUCTURE).
//
// The reference's unit tests (proj/tests/unit/*.cpp) are written against
// doctest, which is not vendored here.  This header implements the subset
// they use -- TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS and
// doctest::Approx(..).epsilon(..) -- so those test files compile UNCHANGED
// against this repo's drop-in headers (oracle/Makefile target `reftests`).
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
    bool matches(double lhs) const {
        return std::fabs(lhs - value_) <
               eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
    }
    friend bool operator==(double lhs, const Approx& r) { return r.matches(lhs); }
    friend bool operator==(const Approx& r, double rhs) { return r.matches(rhs); }
    friend bool operator!=(double lhs, const Approx& r) { return !r.matches(lhs); }
    friend bool operator!=(const Approx& r, double rhs) { return !r.matches(rhs); }

private:
    double value_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
    double scale_ = 1.0;
};

namespace shim {

struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Stats {
    long checks = 0, failed_checks = 0;
    bool case_failed = false;
};

inline Stats& stats() {
    static Stats s;
    return s;
}

struct RequireFailed {};

inline int add(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
    return 0;
}

inline void check(bool ok, const char* expr, const char* file, int line, bool require) {
    ++stats().checks;
    if (ok) return;
    ++stats().failed_checks;
    stats().case_failed = true;
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
    if (require) throw RequireFailed{};
}

inline int run_all() {
    int failedCases = 0;
    for (const Case& c : registry()) {
        stats().case_failed = false;
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw: %s\n", c.file, c.line, c.name,
                         e.what());
            stats().case_failed = true;
        }
        if (stats().case_failed) {
            ++failedCases;
            std::fprintf(stderr, "FAILED: %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n",
                registry().size(), registry().size() - failedCases, failedCases);
    std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", stats().checks,
                stats().checks - stats().failed_checks, stats().failed_checks);
    return failedCases ? 1 : 0;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_TC(fn, name)                                                       \
    static void fn();                                                                   \
    static const int DOCTEST_SHIM_CAT(fn, _reg) =                                       \
        doctest::shim::add(name, __FILE__, __LINE__, &fn);                              \
    static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TC(DOCTEST_SHIM_CAT(doctest_shim_case_, __COUNTER__), name)

#define CHECK(...) doctest::shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::shim::check(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                     \
    do {                                                                                \
        bool thrown_ = false;                                                           \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (const type&) {                                                         \
            thrown_ = true;                                                             \
        } catch (...) {                                                                 \
        }                                                                               \
        doctest::shim::check(thrown_, "throws " #type ": " #expr, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::shim::run_all(); }
#endif
