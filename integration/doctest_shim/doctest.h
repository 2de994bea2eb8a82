// doctest.h -- a minimal, self-written stand-in for the subset of the doctest
// API the reference's unit tests use (TEST_CASE, CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, CHECK_NOTHROW,
// doctest::Approx(x).epsilon(e), doctest::Contains, and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN).  The reference does not vendor doctest
// (proj/.gitignore:2); this header lets its test files compile unchanged so
// they can run against the GPU drop-in.  Not doctest's source.
//
// Approx semantics follow doctest: |a - b| < eps * (scale + max(|a|, |b|)),
// scale = 1, default eps = 100 * FLT_EPSILON.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
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
    bool matches(double other) const {
        return std::fabs(other - value_) < eps_ * (1.0 + std::fmax(std::fabs(other), std::fabs(value_)));
    }
    double value() const { return value_; }

private:
    double value_;
    double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
};
inline bool operator==(double a, const Approx& b) { return b.matches(a); }
inline bool operator==(const Approx& a, double b) { return a.matches(b); }
inline bool operator!=(double a, const Approx& b) { return !b.matches(a); }
inline bool operator!=(const Approx& a, double b) { return !a.matches(b); }

struct Contains {
    explicit Contains(const char* s) : text(s) {}
    std::string text;
    bool matches(const char* what) const { return std::strstr(what, text.c_str()) != nullptr; }
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
    int failed_checks = 0;
    int checks = 0;
    bool case_failed = false;
};
inline State& state() {
    static State s;
    return s;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line, bool fatal,
                   const std::string& extra = "") {
    State& s = state();
    ++s.checks;
    if (ok) return;
    ++s.failed_checks;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED%s%s\n", file, line, kind, expr, extra.empty() ? "" : " -- ",
                 extra.c_str());
    if (fatal) throw RequireFailed{};
}

}  // namespace detail

// Filters: "-tc=<substring>" runs matching cases, "-tce=<substring>" excludes.
inline int run_all(int argc, char** argv) {
    std::vector<std::string> inc, exc;
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        if (a.rfind("-tc=", 0) == 0) inc.push_back(a.substr(4));
        if (a.rfind("-tce=", 0) == 0) exc.push_back(a.substr(5));
    }
    int cases = 0, failed_cases = 0;
    for (const auto& tc : detail::registry()) {
        const std::string name = tc.name;
        bool take = inc.empty();
        for (auto& f : inc) take = take || name.find(f) != std::string::npos;
        for (auto& f : exc) take = take && name.find(f) == std::string::npos;
        if (!take) continue;
        ++cases;
        if (std::getenv("DOCTEST_SHIM_VERBOSE")) std::fprintf(stderr, "[run] %s\n", tc.name);
        detail::state().case_failed = false;
        try {
            tc.fn();
        } catch (const detail::RequireFailed&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw: %s\n", tc.file, tc.line, tc.name, e.what());
            detail::state().case_failed = true;
        }
        if (detail::state().case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "[FAILED] %s\n", tc.name);
        }
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed; assertions: %d | %d failed\n", cases,
                cases - failed_cases, failed_cases, detail::state().checks, detail::state().failed_checks);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                             \
    static void fn();                                                                         \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)

#define CHECK_THROWS_AS(expr, ...)                                                                        \
    do {                                                                                                   \
        bool ok_ = false;                                                                                  \
        std::string why_ = "did not throw";                                                                \
        try {                                                                                              \
            (void)(expr);                                                                                  \
        } catch (const __VA_ARGS__&) {                                                                     \
            ok_ = true;                                                                                    \
        } catch (const std::exception& e_) {                                                               \
            why_ = std::string("threw a different type: ") + e_.what();                                    \
        } catch (...) {                                                                                    \
            why_ = "threw a different type";                                                               \
        }                                                                                                  \
        ::doctest::detail::report(ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__, false, ok_ ? "" : why_); \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                                          \
    do {                                                                                                   \
        bool ok_ = false;                                                                                  \
        std::string why_ = "did not throw";                                                                \
        try {                                                                                              \
            (void)(expr);                                                                                  \
        } catch (const __VA_ARGS__& e_) {                                                                  \
            ok_ = (matcher).matches(e_.what());                                                            \
            if (!ok_) why_ = std::string("message mismatch: ") + e_.what();                                \
        } catch (const std::exception& e_) {                                                               \
            why_ = std::string("threw a different type: ") + e_.what();                                    \
        } catch (...) {                                                                                    \
            why_ = "threw a different type";                                                               \
        }                                                                                                  \
        ::doctest::detail::report(ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__, false, ok_ ? "" : why_); \
    } while (0)

#define CHECK_NOTHROW(expr)                                                                               \
    do {                                                                                                   \
        bool ok_ = true;                                                                                   \
        std::string why_;                                                                                  \
        try {                                                                                              \
            (void)(expr);                                                                                  \
        } catch (const std::exception& e_) {                                                               \
            ok_ = false;                                                                                   \
            why_ = e_.what();                                                                              \
        } catch (...) {                                                                                    \
            ok_ = false;                                                                                   \
        }                                                                                                  \
        ::doctest::detail::report(ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__, false, why_);          \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::run_all(argc, argv); }
#endif
