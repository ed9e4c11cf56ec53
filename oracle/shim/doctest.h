// Minimal doctest stand-in.
//
// TEST INFRASTRUCTURE (oracle/): the reference's unit tests include
// <doctest.h> from proj/vendor/, which is git-ignored and absent
// (proj/.gitignore:2).  This header implements only the subset those tests
// use: TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, FAIL, INFO, CAPTURE, doctest::Approx (epsilon/scale)
// and doctest::Contains, with DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN providing a
// main() that runs every case and exits non-zero on any failure.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    Approx& scale(double s) { scale_ = s; return *this; }
    friend bool operator==(double lhs, const Approx& r) {
        return std::fabs(lhs - r.value_) < r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.value_)));
    }
    friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
    friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
    friend bool operator!=(const Approx& r, double rhs) { return !(rhs == r); }
    friend bool operator<=(double lhs, const Approx& r) { return lhs < r.value_ || lhs == r; }
    friend bool operator>=(double lhs, const Approx& r) { return lhs > r.value_ || lhs == r; }
    friend bool operator<(double lhs, const Approx& r) { return lhs < r.value_ && lhs != r; }
    friend bool operator>(double lhs, const Approx& r) { return lhs > r.value_ && lhs != r; }
    double value() const { return value_; }

private:
    double value_;
    double eps_ = 1.1920928955078125e-07 * 100;  // float epsilon * 100, doctest's default
    double scale_ = 1.0;
};

struct Contains {
    explicit Contains(std::string s) : needle(std::move(s)) {}
    std::string needle;
    bool matches(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
};

namespace detail {

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

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct RequireAbort {};

struct State {
    long long checks = 0;
    long long failed_checks = 0;
    bool case_failed = false;
    std::vector<std::string> context;
};

inline State& state() {
    static State s;
    return s;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    State& s = state();
    ++s.checks;
    if (ok) return;
    ++s.failed_checks;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
    for (const auto& c : s.context) std::fprintf(stderr, "  with context: %s\n", c.c_str());
}

struct ContextScope {
    explicit ContextScope(std::string s) { state().context.push_back(std::move(s)); }
    ~ContextScope() { state().context.pop_back(); }
};

template <class T>
std::string to_string_any(const T& v) {
    std::ostringstream os;
    if constexpr (requires(std::ostream& o, const T& x) { o << x; }) {
        os << v;
    } else {
        os << "{?}";
    }
    return os.str();
}

inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : registry()) {
        state().case_failed = false;
        try {
            c.fn();
        } catch (const RequireAbort&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
            state().case_failed = true;
        } catch (...) {
            std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw an unknown exception\n", c.file, c.line, c.name);
            state().case_failed = true;
        }
        if (state().case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "  -> test case FAILED: %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | passed: %zu | failed: %d; assertions: %lld | failed: %lld\n",
                registry().size(), registry().size() - static_cast<size_t>(failed_cases), failed_cases,
                state().checks, state().failed_checks);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                   \
    static void fn();                                                                    \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
    ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                  \
    do {                                                                                              \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                      \
        ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);          \
        if (!doctest_ok_) throw ::doctest::detail::RequireAbort{};                                    \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                    \
    do {                                                                                              \
        bool doctest_thrown_ = false;                                                                 \
        try {                                                                                         \
            (void)(expr);                                                                             \
        } catch (const __VA_ARGS__&) {                                                                \
            doctest_thrown_ = true;                                                                   \
        } catch (...) {                                                                               \
        }                                                                                             \
        ::doctest::detail::report(doctest_thrown_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);     \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                         \
    do {                                                                                              \
        bool doctest_ok_ = false;                                                                     \
        try {                                                                                         \
            (void)(expr);                                                                             \
        } catch (const __VA_ARGS__& e_) {                                                             \
            doctest_ok_ = ::doctest::Contains(with).matches(e_.what());                               \
        } catch (...) {                                                                               \
        }                                                                                             \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__);    \
    } while (0)
#define FAIL(msg)                                                                 \
    do {                                                                          \
        ::doctest::detail::report(false, "FAIL", #msg, __FILE__, __LINE__);       \
        throw ::doctest::detail::RequireAbort{};                                  \
    } while (0)
#define INFO(...)                                                                  \
    ::doctest::detail::ContextScope DOCTEST_CAT(doctest_info_, __LINE__)([&] {     \
        std::ostringstream doctest_os_;                                            \
        doctest_os_ << __VA_ARGS__;                                                \
        return doctest_os_.str();                                                  \
    }())
#define CAPTURE(x) \
    ::doctest::detail::ContextScope DOCTEST_CAT(doctest_cap_, __LINE__)(std::string(#x " := ") + ::doctest::detail::to_string_any(x))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
