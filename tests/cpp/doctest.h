// tests/cpp/doctest.h — a minimal doctest-compatible harness (the vendored doctest is absent
// from the reference checkout, proj/.gitignore:2).  Supports exactly what the reference's
// solver suites use: TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, FAIL and
// doctest::Approx(..).epsilon(..).  Test infrastructure only.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
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
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) <
               a.eps_ * (1.0 + std::max(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
};

namespace detail {

struct TestCase {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, void (*fn)(), const char* file, int line) {
        registry().push_back({name, fn, file, line});
    }
};

struct RequireFailed {};

inline int& assertion_failures() {
    static int n = 0;
    return n;
}

inline void report(const char* file, int line, const char* what) {
    ++assertion_failures();
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what);
}

} // namespace detail
} // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define TEST_CASE(name)                                                                         \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                           \
    static ::doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(                    \
        name, &DOCTEST_CAT(doctest_fn_, __LINE__), __FILE__, __LINE__);                         \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define CHECK(...)                                                                              \
    do {                                                                                        \
        if (!(__VA_ARGS__)) ::doctest::detail::report(__FILE__, __LINE__, "CHECK(" #__VA_ARGS__ ")"); \
    } while (0)

#define CHECK_FALSE(...)                                                                        \
    do {                                                                                        \
        if ((__VA_ARGS__))                                                                      \
            ::doctest::detail::report(__FILE__, __LINE__, "CHECK_FALSE(" #__VA_ARGS__ ")");     \
    } while (0)

#define REQUIRE(...)                                                                            \
    do {                                                                                        \
        if (!(__VA_ARGS__)) {                                                                   \
            ::doctest::detail::report(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")");         \
            throw ::doctest::detail::RequireFailed{};                                           \
        }                                                                                       \
    } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                              \
    do {                                                                                        \
        bool doctest_threw_ = false;                                                            \
        try {                                                                                   \
            (void)(expr);                                                                       \
        } catch (const __VA_ARGS__&) {                                                          \
            doctest_threw_ = true;                                                              \
        } catch (...) {                                                                         \
        }                                                                                       \
        if (!doctest_threw_)                                                                    \
            ::doctest::detail::report(__FILE__, __LINE__,                                       \
                                      "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")");          \
    } while (0)

#define FAIL(msg)                                                                               \
    do {                                                                                        \
        ::doctest::detail::report(__FILE__, __LINE__, msg);                                     \
        throw ::doctest::detail::RequireFailed{};                                               \
    } while (0)
