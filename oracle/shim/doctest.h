// oracle/shim/doctest.h — TEST INFRASTRUCTURE ONLY.
//
// A tiny self-written stand-in for the doctest macros the reference unit tests
// use (proj/tests/test_*.cpp): TEST_CASE, CHECK, REQUIRE, CHECK_THROWS,
// CHECK_THROWS_AS and doctest::Approx(...).epsilon(...).  The real doctest is
// vendored by the reference under vendor/, which is absent, so
// this shim lets the reference's own tests run unchanged against the oracle
// build.  Differences from upstream doctest: no subcases/sections, no
// expression decomposition in failure messages (the stringified expression is
// printed), and Approx uses an inclusive bound (so `.epsilon(0)` means exact).
//
// Runner flags: `--list`, `--skip=<substring>` (repeatable), `--only=<substring>`.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    Approx& scale(double s) { scale_ = s; return *this; }
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) <=
               rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }

private:
    double value_;
    double eps_ = double(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
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

struct RequireFailed {};

inline int& failures() { static int f = 0; return f; }
inline int& checks() { static int c = 0; return c; }

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line, bool fatal) {
    ++checks();
    if (ok) return;
    ++failures();
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
    if (fatal) throw RequireFailed{};
}

} // namespace detail
} // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                                   \
    static void fn();                                                                              \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);      \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __LINE__), name)

#define CHECK(...) ::doctest::detail::report(bool(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(bool(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                                  \
    do {                                                                                            \
        bool doctest_ok_ = false;                                                                   \
        try { (void)(expr); } catch (const __VA_ARGS__&) { doctest_ok_ = true; } catch (...) {}      \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_THROWS(...)                                                                           \
    do {                                                                                            \
        bool doctest_ok_ = false;                                                                   \
        try { (void)(__VA_ARGS__); } catch (...) { doctest_ok_ = true; }                            \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS", #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    std::vector<std::string> skips;
    std::string only;
    bool list = false;
    for (int a = 1; a < argc; ++a) {
        if (std::strncmp(argv[a], "--skip=", 7) == 0) skips.emplace_back(argv[a] + 7);
        else if (std::strncmp(argv[a], "--only=", 7) == 0) only = argv[a] + 7;
        else if (std::strcmp(argv[a], "--list") == 0) list = true;
    }
    int ran = 0, failed_cases = 0, skipped = 0;
    for (const auto& c : ::doctest::detail::registry()) {
        const std::string name(c.name);
        bool skip = !only.empty() && name.find(only) == std::string::npos;
        for (const auto& s : skips) skip = skip || name.find(s) != std::string::npos;
        if (list) { std::printf("%s\n", c.name); continue; }
        if (skip) { ++skipped; continue; }
        const int before = ::doctest::detail::failures();
        try {
            c.fn();
        } catch (const ::doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            ++::doctest::detail::failures();
            std::fprintf(stderr, "%s:%d: unexpected exception in \"%s\": %s\n", c.file, c.line, c.name, e.what());
        } catch (...) {
            ++::doctest::detail::failures();
            std::fprintf(stderr, "%s:%d: unexpected non-std exception in \"%s\"\n", c.file, c.line, c.name);
        }
        ++ran;
        const bool bad = ::doctest::detail::failures() != before;
        failed_cases += bad;
        std::printf("[%s] %s\n", bad ? "FAIL" : " ok ", c.name);
    }
    if (list) return 0;
    std::printf("test cases: %d ran, %d failed, %d skipped; assertions: %d, %d failed\n", ran, failed_cases,
                skipped, ::doctest::detail::checks(), ::doctest::detail::failures());
    return failed_cases == 0 ? 0 : 1;
}
#endif
