// TEST INFRASTRUCTURE ONLY — a minimal stand-in for doctest (absent from this
// image; the reference vendors it under proj/vendor/, which is gitignored and
// missing).  Implements the subset the reference's unit tests use so that
// proj/tests/test_{tensor,matvec,io,aca,compress,scene}.cpp compile unchanged
// against oracle/_ref: TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, CHECK_NOTHROW, FAIL, doctest::Approx (doctest's
// published comparison rule: |a - b| < eps * (scale + max(|a|, |b|)), default
// eps = 100 * float epsilon, scale 1) and doctest::Contains.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    double value, eps = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100, scale = 1.0;
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
    Approx& scale_(double s) {
        scale = s;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.value) < b.eps * (b.scale + std::max(std::fabs(a), std::fabs(b.value)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }
    friend bool operator!=(const Approx& b, double a) { return !(a == b); }
    friend bool operator<=(double a, const Approx& b) { return a < b.value || a == b; }
    friend bool operator>=(double a, const Approx& b) { return a > b.value || a == b; }
};

struct Contains {
    std::string s;
    explicit Contains(const char* x) : s(x) {}
    bool check(const std::string& what) const { return what.find(s) != std::string::npos; }
};

namespace detail {
struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& cases() {
    static std::vector<Case> v;
    return v;
}
inline int& failures() {
    static int f = 0;
    return f;
}
inline int& checks() {
    static int c = 0;
    return c;
}
struct Abort {};
inline int reg(const char* name, void (*fn)()) {
    cases().push_back({name, fn});
    return 0;
}
inline void fail(const char* file, int line, const char* what) {
    ++failures();
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, what);
}
inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : cases()) {
        const int before = failures();
        try {
            c.fn();
        } catch (const Abort&) {
        } catch (const std::exception& e) {
            ++failures();
            std::fprintf(stderr, "TEST CASE \"%s\": uncaught exception: %s\n", c.name, e.what());
        } catch (...) {
            ++failures();
            std::fprintf(stderr, "TEST CASE \"%s\": uncaught unknown exception\n", c.name);
        }
        if (failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "TEST CASE FAILED: %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
                cases().size(), cases().size() - size_t(failed_cases), failed_cases, checks(), failures());
    return failed_cases == 0 ? 0 : 1;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(f, v, name)                                         \
    static void f();                                                    \
    [[maybe_unused]] static const int v = doctest::detail::reg(name, &f); \
    static void f()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_fn_, __COUNTER__), DOCTEST_CAT(doctest_tc_reg_, __COUNTER__), name)

#define CHECK(...)                                                                  \
    do {                                                                            \
        ++doctest::detail::checks();                                                \
        if (!(__VA_ARGS__)) doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__); \
    } while (0)
#define REQUIRE(...)                                                      \
    do {                                                                  \
        ++doctest::detail::checks();                                      \
        if (!(__VA_ARGS__)) {                                             \
            doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__);      \
            throw doctest::detail::Abort{};                               \
        }                                                                 \
    } while (0)
#define FAIL(msg)                                                         \
    do {                                                                  \
        ++doctest::detail::checks();                                      \
        doctest::detail::fail(__FILE__, __LINE__, "FAIL");                \
        throw doctest::detail::Abort{};                                   \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                   \
    do {                                                                                             \
        ++doctest::detail::checks();                                                                 \
        bool doctest_ok_ = false;                                                                    \
        try {                                                                                        \
            (void)(expr);                                                                            \
        } catch (const __VA_ARGS__&) {                                                               \
            doctest_ok_ = true;                                                                      \
        } catch (...) {                                                                              \
        }                                                                                            \
        if (!doctest_ok_) doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ")");   \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                                       \
    do {                                                                                               \
        ++doctest::detail::checks();                                                                   \
        bool doctest_ok_ = false;                                                                      \
        try {                                                                                          \
            (void)(expr);                                                                              \
        } catch (const __VA_ARGS__& e) {                                                               \
            doctest_ok_ = (matcher).check(e.what());                                                   \
        } catch (...) {                                                                                \
        }                                                                                              \
        if (!doctest_ok_) doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_WITH_AS(" #expr ")"); \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                      \
    do {                                                                                         \
        ++doctest::detail::checks();                                                             \
        try {                                                                                    \
            (void)(expr);                                                                        \
        } catch (...) {                                                                          \
            doctest::detail::fail(__FILE__, __LINE__, "CHECK_NOTHROW(" #expr ")");               \
        }                                                                                        \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
