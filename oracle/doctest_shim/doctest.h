// TEST INFRASTRUCTURE ONLY.  A minimal stand-in for the doctest single
// header (absent from the reference's vendor/ directory) implementing exactly
// the macro subset the reference suites use: TEST_CASE, CHECK, REQUIRE,
// REQUIRE_MESSAGE, CAPTURE, CHECK_NOTHROW, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, doctest::Approx(..).epsilon(..), doctest::Contains.
// oracle/Makefile builds the reference's own test files against it so the
// compiled reference (oracle/_ref) is checked by its own known-answer tests.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    double value;
    double eps = 1e-5;  // doctest's default: float epsilon * 100
    explicit Approx(double v) : value(v), eps(static_cast<double>(1.1920929e-7f) * 100) {}
    Approx& epsilon(double e) { eps = e; return *this; }
    bool matches(double other) const {
        return std::fabs(other - value) <
               eps * (1.0 + std::fmax(std::fabs(other), std::fabs(value)));
    }
};
inline bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
inline bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
inline bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }

struct Contains {
    std::string needle;
    explicit Contains(const char* s) : needle(s) {}
};

namespace detail {
struct Registry {
    std::vector<std::pair<const char*, void (*)()>> cases;
    int checks = 0;
    int failures = 0;
    const char* current = "";
    static Registry& get() {
        static Registry r;
        return r;
    }
};
struct Reg {
    Reg(const char* name, void (*fn)()) { Registry::get().cases.emplace_back(name, fn); }
};
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool hard) {
    Registry& r = Registry::get();
    ++r.checks;
    if (!ok) {
        ++r.failures;
        std::fprintf(stderr, "%s:%d: FAILED in [%s]: %s\n", file, line, r.current, expr);
        if (hard) throw RequireFailed{};
    }
}
inline bool matches(const std::string& what, const Contains& c) {
    return what.find(c.needle) != std::string::npos;
}
inline bool matches(const std::string& what, const char* s) { return what == s; }
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                              \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                \
    static doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(                 \
        name, &DOCTEST_CAT(doctest_fn_, __LINE__));                                  \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_MESSAGE(cond, msg) doctest::detail::report(static_cast<bool>(cond), #cond, __FILE__, __LINE__, true)
#define CAPTURE(x) (void)(x)
#define CHECK_NOTHROW(...)                                                           \
    do {                                                                             \
        bool ok_ = true;                                                             \
        try { (void)(__VA_ARGS__); } catch (...) { ok_ = false; }                    \
        doctest::detail::report(ok_, "NOTHROW " #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                   \
    do {                                                                             \
        bool ok_ = false;                                                            \
        try { (void)(expr); } catch (const __VA_ARGS__&) { ok_ = true; } catch (...) {} \
        doctest::detail::report(ok_, "THROWS_AS " #expr, __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                        \
    do {                                                                             \
        bool ok_ = false;                                                            \
        try { (void)(expr); } catch (const __VA_ARGS__& e_) {                        \
            ok_ = doctest::detail::matches(std::string(e_.what()), with);            \
        } catch (...) {}                                                             \
        doctest::detail::report(ok_, "THROWS_WITH_AS " #expr, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    auto& r = doctest::detail::Registry::get();
    int failed_cases = 0;
    for (auto& [name, fn] : r.cases) {
        r.current = name;
        const int before = r.failures;
        try {
            fn();
        } catch (const doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            ++r.failures;
            std::fprintf(stderr, "[%s] threw: %s\n", name, e.what());
        }
        if (r.failures != before) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks %d | failures %d\n",
                r.cases.size(), r.cases.size() - failed_cases, failed_cases, r.checks, r.failures);
    return r.failures == 0 ? 0 : 1;
}
#endif
