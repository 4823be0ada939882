// Minimal doctest-compatible test runner -- TEST INFRASTRUCTURE ONLY.
//
// The reference's unit tests (proj/tests/test_*.cpp) are written against
// doctest, which is not installed in this image.  This header implements the
// small subset of doctest's interface they use (TEST_CASE, CHECK, CHECK_FALSE,
// CHECK_THROWS_AS, REQUIRE, FAIL, doctest::Approx and the
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN entry point) so those test files compile
// unchanged; oracle/Makefile links them against the drop-in headers and
// libpafft_b200.so (oracle/_ref/unit_dropin), run on the GPU by
// tests/test_gpu_dropin_ref.py.  Every failed assertion prints one line
// "FAILED <file>:<line>: <expression>" so a test can compare the failures with
// the list of intended behaviour changes.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

// approximate floating-point comparison, doctest's default relative epsilon
class Approx {
public:
    explicit Approx(double value) : value_(value) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& rhs) {
        const double scale = std::max(std::fabs(lhs), std::fabs(rhs.value_));
        return std::fabs(lhs - rhs.value_) <= rhs.eps_ * (1.0 + scale);
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

private:
    double value_;
    double eps_ = 1.1920929e-05;  // float epsilon * 100, as doctest
};

namespace shim {
struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};
inline std::vector<Case>& cases() {
    static std::vector<Case> v;
    return v;
}
struct Stats {
    long checks = 0, failed_checks = 0;
    bool case_failed = false;
};
inline Stats& stats() {
    static Stats s;
    return s;
}
struct Abort {};  // a failed REQUIRE / FAIL ends the test case
inline bool report(bool ok, const char* what, const char* file, int line) {
    ++stats().checks;
    if (!ok) {
        ++stats().failed_checks;
        stats().case_failed = true;
        std::printf("FAILED %s:%d: %s\n", file, line, what);
    }
    return ok;
}
struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) { cases().push_back({name, file, line, fn}); }
};
inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : cases()) {
        stats().case_failed = false;
        try {
            c.fn();
        } catch (const Abort&) {
        } catch (const std::exception& e) {
            report(false, (std::string("unexpected exception: ") + e.what()).c_str(), c.file, c.line);
        } catch (...) {
            report(false, "unexpected exception", c.file, c.line);
        }
        if (stats().case_failed) {
            ++failed_cases;
            std::printf("TEST CASE FAILED: \"%s\" (%s:%d)\n", c.name, c.file, c.line);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", cases().size(),
                cases().size() - (size_t)failed_cases, failed_cases);
    std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", stats().checks,
                stats().checks - stats().failed_checks, stats().failed_checks);
    return failed_cases ? 1 : 0;
}
}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_TEST(fn, name)                                                                    \
    static void fn();                                                                                  \
    static const ::doctest::shim::Registrar DOCTEST_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TEST(DOCTEST_SHIM_CAT(doctest_shim_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
    ::doctest::shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                                    \
    do {                                                                                                \
        if (!::doctest::shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)) \
            throw ::doctest::shim::Abort{};                                                             \
    } while (0)
#define FAIL(msg)                                                      \
    do {                                                               \
        ::doctest::shim::report(false, "FAIL: " msg, __FILE__, __LINE__); \
        throw ::doctest::shim::Abort{};                                \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                          \
    do {                                                                                    \
        bool doctest_shim_ok = false;                                                       \
        try {                                                                               \
            static_cast<void>(expr);                                                        \
        } catch (const __VA_ARGS__&) {                                                      \
            doctest_shim_ok = true;                                                         \
        } catch (...) {                                                                     \
        }                                                                                   \
        ::doctest::shim::report(doctest_shim_ok, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::shim::run_all(); }
#endif
