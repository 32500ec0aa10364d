// Minimal doctest-compatible shim (doctest itself is not in this image).
// Implements exactly the macros the reference tests use:
// TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS, CHECK_NOTHROW,
// CAPTURE, FAIL, doctest::Approx(x).epsilon(e). Test infrastructure only.
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) { eps = e; return *this; }
    double value;
    double eps = 1e-5;
};
inline bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value) <= a.eps * (1.0 + std::fmax(std::fabs(lhs), std::fabs(a.value)));
}
inline bool operator==(const Approx& a, double rhs) { return rhs == a; }
inline bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

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
inline int& case_failed() {
    static int f = 0;
    return f;
}
struct RequireAbort {};
struct Registrar {
    Registrar(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
inline void fail(const char* file, int line, const char* what) {
    std::printf("  %s:%d: FAILED: %s\n", file, line, what);
    ++case_failed();
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                             \
    static void fn();                                                                     \
    static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);                   \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...)                                                                        \
    do {                                                                                  \
        if (!(__VA_ARGS__)) doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__);     \
    } while (0)
#define REQUIRE(...)                                                                      \
    do {                                                                                  \
        if (!(__VA_ARGS__)) {                                                             \
            doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__);                      \
            throw doctest::detail::RequireAbort{};                                        \
        }                                                                                 \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                       \
    do {                                                                                  \
        bool ok_ = false;                                                                 \
        try { (void)(expr); } catch (const type&) { ok_ = true; } catch (...) {}          \
        if (!ok_) doctest::detail::fail(__FILE__, __LINE__, "throws " #type ": " #expr);  \
    } while (0)
#define CHECK_THROWS(expr)                                                                \
    do {                                                                                  \
        bool ok_ = false;                                                                 \
        try { (void)(expr); } catch (...) { ok_ = true; }                                 \
        if (!ok_) doctest::detail::fail(__FILE__, __LINE__, "throws: " #expr);            \
    } while (0)
#define CHECK_NOTHROW(expr)                                                               \
    do {                                                                                  \
        try { (void)(expr); } catch (...) {                                               \
            doctest::detail::fail(__FILE__, __LINE__, "nothrow: " #expr);                 \
        }                                                                                 \
    } while (0)
#define CAPTURE(x) (void)(x)
#define FAIL(msg)                                                                         \
    do {                                                                                  \
        doctest::detail::fail(__FILE__, __LINE__, "FAIL");                                \
        throw doctest::detail::RequireAbort{};                                            \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int cases_failed = 0;
    for (auto& c : doctest::detail::registry()) {
        doctest::detail::case_failed() = 0;
        try {
            c.fn();
        } catch (doctest::detail::RequireAbort&) {
        } catch (const std::exception& e) {
            std::printf("  exception: %s\n", e.what());
            ++doctest::detail::case_failed();
        }
        const bool ok = doctest::detail::case_failed() == 0;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
        cases_failed += ok ? 0 : 1;
    }
    std::printf("%zu test cases, %d failed\n", doctest::detail::registry().size(), cases_failed);
    return cases_failed;
}
#endif
