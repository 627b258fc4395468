// Minimal doctest-compatible shim (the real doctest is not vendored in the
// reference tree).  Enough for the reference's suites
// (/root/reference/proj/tests/test_*.cpp): TEST_CASE, SUBCASE (run inline,
// in order), CHECK/REQUIRE and friends, CHECK_THROWS_AS / CHECK_NOTHROW /
// REQUIRE_NOTHROW, doctest::Approx, and a main().
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <limits>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    double v, eps = 1e-5;  // doctest's default epsilon is float-ish; tests set it
    explicit Approx(double x) : v(x), eps(std::numeric_limits<float>::epsilon() * 100) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v) <= b.eps * (1.0 + std::max(std::fabs(a), std::fabs(b.v)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }
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
inline int& failures() {
    static int f = 0;
    return f;
}
inline int& checks() {
    static int c = 0;
    return c;
}
struct Reg {
    Reg(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct RequireFailed {};
inline void fail(const char* file, int line, const char* expr, bool fatal) {
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
    if (fatal) throw RequireFailed{};
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                            \
    static void DOCTEST_CAT(dt_case_, __LINE__)();                                                 \
    static doctest::detail::Reg DOCTEST_CAT(dt_reg_, __LINE__)(name, &DOCTEST_CAT(dt_case_, __LINE__)); \
    static void DOCTEST_CAT(dt_case_, __LINE__)()
#define SUBCASE(name) if (true)
#define DT_CHECK_IMPL(expr, fatal)                                                            \
    do {                                                                                      \
        ++doctest::detail::checks();                                                          \
        if (!(expr)) doctest::detail::fail(__FILE__, __LINE__, #expr, fatal);                 \
    } while (0)
#define CHECK(...) DT_CHECK_IMPL((__VA_ARGS__), false)
#define REQUIRE(...) DT_CHECK_IMPL((__VA_ARGS__), true)
#define CHECK_FALSE(...) DT_CHECK_IMPL(!(__VA_ARGS__), false)
#define CHECK_MESSAGE(cond, ...) DT_CHECK_IMPL((cond), false)
#define FAIL(...) doctest::detail::fail(__FILE__, __LINE__, "FAIL", true)
#define DT_THROWS_IMPL(expr, T, fatal)                                                        \
    do {                                                                                      \
        ++doctest::detail::checks();                                                          \
        bool dt_ok = false;                                                                   \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (const T&) {                                                                  \
            dt_ok = true;                                                                     \
        } catch (...) {                                                                       \
        }                                                                                     \
        if (!dt_ok) doctest::detail::fail(__FILE__, __LINE__, #expr " throws " #T, fatal);    \
    } while (0)
#define CHECK_THROWS_AS(expr, ...) DT_THROWS_IMPL(expr, __VA_ARGS__, false)
#define REQUIRE_THROWS_AS(expr, ...) DT_THROWS_IMPL(expr, __VA_ARGS__, true)
#define DT_NOTHROW_IMPL(expr, fatal)                                                          \
    do {                                                                                      \
        ++doctest::detail::checks();                                                          \
        bool dt_ok = true;                                                                    \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (const std::exception& e) {                                                   \
            dt_ok = false;                                                                    \
            std::fprintf(stderr, "  threw: %s\n", e.what());                                  \
        } catch (...) {                                                                       \
            dt_ok = false;                                                                    \
        }                                                                                     \
        if (!dt_ok) doctest::detail::fail(__FILE__, __LINE__, #expr " does not throw", fatal); \
    } while (0)
#define CHECK_NOTHROW(expr) DT_NOTHROW_IMPL(expr, false)
#define REQUIRE_NOTHROW(expr) DT_NOTHROW_IMPL(expr, true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int cases = 0, failed_cases = 0;
    for (const auto& c : doctest::detail::registry()) {
        ++cases;
        const int before = doctest::detail::failures();
        try {
            c.fn();
        } catch (const doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            ++doctest::detail::failures();
            std::fprintf(stderr, "test case '%s' threw: %s\n", c.name, e.what());
        }
        if (doctest::detail::failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "test case FAILED: %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %d | %d failed\n", cases,
                cases - failed_cases, failed_cases, doctest::detail::checks(), doctest::detail::failures());
    return failed_cases ? 1 : 0;
}
#endif
