// doctest-API shim -- TEST INFRASTRUCTURE ONLY.
//
// The reference tests (/root/reference/proj/tests/*.cpp) are written against doctest,
// which the reference expects under vendor/ (tests/CMakeLists.txt:2) but which is
// git-ignored there and absent here. This header provides the subset they use:
// TEST_CASE, SUBCASE, CHECK, CHECK_THROWS_AS, doctest::Approx{epsilon,scale}.
//
// SUBCASEs run sequentially inside one execution of their TEST_CASE (the reference's
// subcases are independent blocks, so the doctest re-entry model is not needed).
// The runner (doctest_main.cpp) prints one line per failed CHECK and exits 1 on any
// failure, 0 otherwise.
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
    explicit Approx(double v)
        : m_value(v)
    {
    }
    Approx& epsilon(double e)
    {
        m_epsilon = e;
        return *this;
    }
    Approx& scale(double s)
    {
        m_scale = s;
        return *this;
    }
    // doctest's comparison: |lhs - v| < eps * (scale + max(|lhs|, |v|))
    friend bool operator==(double lhs, const Approx& rhs)
    {
        return std::fabs(lhs - rhs.m_value)
            < rhs.m_epsilon * (rhs.m_scale + std::max(std::fabs(lhs), std::fabs(rhs.m_value)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

private:
    double m_value;
    double m_epsilon = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double m_scale = 1.0;
};

namespace detail {
struct TestCase {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};
inline std::vector<TestCase>& registry()
{
    static std::vector<TestCase> r;
    return r;
}
struct Stats {
    long checks = 0;
    long failures = 0;
    const char* current = "";
};
inline Stats& stats()
{
    static Stats s;
    return s;
}
struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)())
    {
        registry().push_back({name, file, line, fn});
    }
};
inline void report(bool ok, const char* expr, const char* file, int line)
{
    auto& s = stats();
    ++s.checks;
    if (!ok) {
        ++s.failures;
        std::printf("%s:%d: CHECK FAILED in \"%s\": %s\n", file, line, s.current, expr);
    }
}
} // namespace detail
} // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                          \
    static void fn();                                                                             \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);      \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_test_fn_, __COUNTER__), name)
#define SUBCASE(name) if (const char* doctest_subcase_name_ = name; doctest_subcase_name_)
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...) CHECK(__VA_ARGS__)
#define CHECK_THROWS_AS(expr, ...)                                                                \
    do {                                                                                          \
        bool doctest_ok_ = false;                                                                 \
        try {                                                                                     \
            (void)(expr);                                                                         \
        } catch (const __VA_ARGS__&) {                                                            \
            doctest_ok_ = true;                                                                   \
        } catch (...) {                                                                           \
        }                                                                                         \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")",      \
                                  __FILE__, __LINE__);                                            \
    } while (0)
