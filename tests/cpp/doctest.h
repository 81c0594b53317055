// doctest.h — minimal stand-in for the doctest macros the reference unit
// suite uses (the real doctest is not vendored in this image).
//
// TEST INFRASTRUCTURE ONLY: lets tests/test_reference_unit_suite.py compile
// the reference's own unit tests (/root/reference/proj/tests/*_test.cpp)
// against this repository's include/specsim headers, as an API- and
// semantics-compatibility check.  Supports TEST_CASE, CHECK/REQUIRE (and
// _FALSE), CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, CHECK_NOTHROW, FAIL,
// doctest::Approx (epsilon/scale) and doctest::Contains.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
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
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
    friend bool operator<=(double lhs, const Approx& a) { return lhs < a.value_ || lhs == a; }
    friend bool operator>=(double lhs, const Approx& a) { return lhs > a.value_ || lhs == a; }
    friend bool operator<(double lhs, const Approx& a) { return lhs < a.value_ && lhs != a; }
    friend bool operator>(double lhs, const Approx& a) { return lhs > a.value_ && lhs != a; }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

struct Contains {
    explicit Contains(const char* s) : text(s) {}
    std::string text;
    bool matches(const std::string& what) const { return what.find(text) != std::string::npos; }
};

namespace detail {

struct TestCase {
    const char* name;
    const char* file;
    int line;
    std::function<void()> fn;
};

struct Abort {};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

inline int& failures() {
    static int f = 0;
    return f;
}

inline int& current_failures() {
    static int f = 0;
    return f;
}

inline void report(const char* file, int line, const char* what) {
    ++failures();
    ++current_failures();
    std::printf("%s:%d: FAILED: %s\n", file, line, what);
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

inline bool matches(const char* expected, const std::string& what) { return what == expected; }
inline bool matches(const std::string& expected, const std::string& what) { return what == expected; }
inline bool matches(const Contains& c, const std::string& what) { return c.matches(what); }

inline int run_all() {
    int cases_failed = 0;
    for (const TestCase& tc : registry()) {
        current_failures() = 0;
        try {
            tc.fn();
        } catch (const Abort&) {
        } catch (const std::exception& e) {
            report(tc.file, tc.line, (std::string("unexpected exception: ") + e.what()).c_str());
        }
        if (current_failures()) {
            ++cases_failed;
            std::printf("test case FAILED: %s\n", tc.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | passed: %zu | failed: %d | assertion failures: %d\n",
                registry().size(), registry().size() - cases_failed, cases_failed, failures());
    return failures() ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                                   \
    static void fn();                                                                               \
    static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);          \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define DOCTEST_ASSERT_(cond, text, fatal)                                       \
    do {                                                                         \
        bool ok_ = false;                                                        \
        try {                                                                    \
            ok_ = static_cast<bool>(cond);                                       \
        } catch (...) {                                                          \
        }                                                                        \
        if (!ok_) {                                                              \
            doctest::detail::report(__FILE__, __LINE__, text);                   \
            if (fatal) throw doctest::detail::Abort{};                           \
        }                                                                        \
    } while (0)

#define CHECK(...) DOCTEST_ASSERT_((__VA_ARGS__), #__VA_ARGS__, false)
#define REQUIRE(...) DOCTEST_ASSERT_((__VA_ARGS__), #__VA_ARGS__, true)
#define CHECK_FALSE(...) DOCTEST_ASSERT_(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", false)
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", true)
#define FAIL(msg)                                                                 \
    do {                                                                          \
        doctest::detail::report(__FILE__, __LINE__, "FAIL");                      \
        throw doctest::detail::Abort{};                                           \
    } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                 \
    do {                                                                           \
        bool got_ = false;                                                         \
        try {                                                                      \
            (void)(expr);                                                          \
        } catch (const __VA_ARGS__&) {                                             \
            got_ = true;                                                           \
        } catch (...) {                                                            \
        }                                                                          \
        if (!got_) doctest::detail::report(__FILE__, __LINE__, "throws " #__VA_ARGS__ ": " #expr); \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                   \
    do {                                                                           \
        bool got_ = false;                                                         \
        try {                                                                      \
            (void)(expr);                                                          \
        } catch (const __VA_ARGS__& e_) {                                          \
            got_ = doctest::detail::matches(matcher, std::string(e_.what()));      \
        } catch (...) {                                                            \
        }                                                                          \
        if (!got_) doctest::detail::report(__FILE__, __LINE__, "throws-with " #expr); \
    } while (0)

#define CHECK_NOTHROW(expr)                                                        \
    do {                                                                           \
        try {                                                                      \
            (void)(expr);                                                          \
        } catch (...) {                                                            \
            doctest::detail::report(__FILE__, __LINE__, "nothrow " #expr);         \
        }                                                                          \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
