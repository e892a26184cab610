// doctest-lite -- TEST INFRASTRUCTURE ONLY (oracle/_ref build).
//
// The reference's unit tests include a vendored <doctest.h>
// (CMakeLists.txt:10, proj/vendor/, absent).  This header implements the
// subset they use: TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, FAIL, doctest::Approx (epsilon, scale; the
// comparison |a-b| < eps*(scale + max(|a|,|b|)), default eps = 100*FLT_EPSILON)
// and doctest::Contains.  main() (DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN) runs
// every registered case, or those matching -tc=<glob>[,<glob>] (also
// --test-case=), -tce=<glob> excludes, -ltc lists; exit code 1 on any
// failure, in doctest's summary format.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v)
        : value_(v), eps_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100), scale_(1.0) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool eq(double lhs) const {
        return std::fabs(lhs - value_) < eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
    }
    friend bool operator==(double lhs, const Approx& r) { return r.eq(lhs); }
    friend bool operator==(const Approx& r, double rhs) { return r.eq(rhs); }
    friend bool operator!=(double lhs, const Approx& r) { return !r.eq(lhs); }
    friend bool operator!=(const Approx& r, double rhs) { return !r.eq(rhs); }
    friend bool operator<=(double lhs, const Approx& r) { return lhs < r.value_ || r.eq(lhs); }
    friend bool operator>=(double lhs, const Approx& r) { return lhs > r.value_ || r.eq(lhs); }
    friend bool operator<(double lhs, const Approx& r) { return lhs < r.value_ && !r.eq(lhs); }
    friend bool operator>(double lhs, const Approx& r) { return lhs > r.value_ && !r.eq(lhs); }
    double value() const { return value_; }

private:
    double value_, eps_, scale_;
};

class Contains {
public:
    explicit Contains(const char* s) : s_(s) {}
    bool checkWith(const std::string& what) const { return what.find(s_) != std::string::npos; }
    const std::string& str() const { return s_; }

private:
    std::string s_;
};

namespace detail {

struct TestCase {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};
struct RequireFailed {};
struct State {
    long asserts = 0, failed_asserts = 0;
    bool current_failed = false;
    const char* current = "";
};
inline State& state() {
    static State s;
    return s;
}
inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   const std::string& extra = std::string()) {
    State& s = state();
    ++s.asserts;
    if (ok) return;
    ++s.failed_asserts;
    s.current_failed = true;
    std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct!  [test case: %s]%s%s\n", file, line,
                 kind, expr, s.current, extra.empty() ? "" : "\n  ", extra.c_str());
}
inline bool matches(const std::string& pat, const std::string& s) {
    // glob with '*' and '?'
    size_t p = 0, t = 0, star = std::string::npos, mark = 0;
    while (t < s.size()) {
        if (p < pat.size() && (pat[p] == '?' || pat[p] == s[t])) {
            ++p;
            ++t;
        } else if (p < pat.size() && pat[p] == '*') {
            star = p++;
            mark = t;
        } else if (star != std::string::npos) {
            p = star + 1;
            t = ++mark;
        } else {
            return false;
        }
    }
    while (p < pat.size() && pat[p] == '*') ++p;
    return p == pat.size();
}
inline std::vector<std::string> split(const std::string& v) {
    std::vector<std::string> out;
    std::stringstream ss(v);
    std::string item;
    while (std::getline(ss, item, ',')) out.push_back(item);
    return out;
}
inline bool msg_matches(const std::string& what, const Contains& c) { return c.checkWith(what); }
inline bool msg_matches(const std::string& what, const char* exact) { return what == exact; }
inline bool msg_matches(const std::string& what, const std::string& exact) { return what == exact; }

inline int run(int argc, char** argv) {
    std::vector<std::string> inc, exc;
    bool list = false;
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        auto val = [&](const char* key) -> const char* {
            const size_t n = std::strlen(key);
            return a.compare(0, n, key) == 0 ? argv[i] + n : nullptr;
        };
        if (const char* v = val("-tc=")) inc = split(v);
        else if (const char* v2 = val("--test-case=")) inc = split(v2);
        else if (const char* v3 = val("-tce=")) exc = split(v3);
        else if (const char* v4 = val("--test-case-exclude=")) exc = split(v4);
        else if (a == "-ltc" || a == "--list-test-cases") list = true;
    }
    State& s = state();
    int run_cases = 0, failed_cases = 0, skipped = 0;
    for (const TestCase& tc : registry()) {
        bool take = inc.empty();
        for (const auto& p : inc) take = take || matches(p, tc.name);
        for (const auto& p : exc) take = take && !matches(p, tc.name);
        if (!take) {
            ++skipped;
            continue;
        }
        if (list) {
            std::printf("%s\n", tc.name);
            continue;
        }
        ++run_cases;
        s.current = tc.name;
        s.current_failed = false;
        try {
            tc.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            report(false, "TEST CASE", "threw exception", tc.file, tc.line, e.what());
        } catch (...) {
            report(false, "TEST CASE", "threw unknown exception", tc.file, tc.line);
        }
        if (s.current_failed) {
            ++failed_cases;
            std::fprintf(stderr, "[doctest-lite] FAILED: %s\n", tc.name);
        }
    }
    if (list) return 0;
    std::printf("[doctest] test cases: %d | %d passed | %d failed | %d skipped\n", run_cases,
                run_cases - failed_cases, failed_cases, skipped);
    std::printf("[doctest] assertions: %ld | %ld passed | %ld failed |\n", s.asserts,
                s.asserts - s.failed_asserts, s.failed_asserts);
    std::printf("[doctest] Status: %s!\n", failed_cases ? "FAILURE" : "SUCCESS");
    return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                   \
    static void fn();                                                                      \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_lite_tc_, __COUNTER__), name)

#define CHECK(...) \
    ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
    ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                              \
    do {                                                                                          \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                 \
        ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);     \
        if (!doctest_ok_) throw ::doctest::detail::RequireFailed();                               \
    } while (0)
#define FAIL(msg)                                                                  \
    do {                                                                           \
        std::ostringstream doctest_os_;                                            \
        doctest_os_ << msg;                                                        \
        ::doctest::detail::report(false, "FAIL", "", __FILE__, __LINE__, doctest_os_.str()); \
        throw ::doctest::detail::RequireFailed();                                  \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                          \
    do {                                                                                    \
        bool doctest_ok_ = false;                                                           \
        std::string doctest_what_ = "did not throw";                                        \
        try {                                                                               \
            (void)(expr);                                                                   \
        } catch (const __VA_ARGS__&) {                                                      \
            doctest_ok_ = true;                                                             \
        } catch (const std::exception& e) {                                                 \
            doctest_what_ = std::string("threw another type: ") + e.what();                 \
        } catch (...) {                                                                     \
            doctest_what_ = "threw another type";                                           \
        }                                                                                   \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, \
                                  __LINE__, doctest_ok_ ? "" : doctest_what_);              \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                               \
    do {                                                                                    \
        bool doctest_ok_ = false;                                                           \
        std::string doctest_what_ = "did not throw";                                        \
        try {                                                                               \
            (void)(expr);                                                                   \
        } catch (const __VA_ARGS__& e) {                                                    \
            doctest_ok_ = ::doctest::detail::msg_matches(e.what(), with);                   \
            doctest_what_ = std::string("message: ") + e.what();                            \
        } catch (const std::exception& e) {                                                 \
            doctest_what_ = std::string("threw another type: ") + e.what();                 \
        } catch (...) {                                                                     \
            doctest_what_ = "threw another type";                                           \
        }                                                                                   \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr ", " #with,   \
                                  __FILE__, __LINE__, doctest_ok_ ? "" : doctest_what_);    \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                 \
    do {                                                                                    \
        bool doctest_ok_ = true;                                                            \
        std::string doctest_what_;                                                          \
        try {                                                                               \
            (void)(expr);                                                                   \
        } catch (const std::exception& e) {                                                 \
            doctest_ok_ = false;                                                            \
            doctest_what_ = e.what();                                                       \
        }                                                                                   \
        ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__, doctest_what_); \
    } while (0)
#define MESSAGE(msg) ((void)0)
#define INFO(msg) ((void)0)
#define CAPTURE(x) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
