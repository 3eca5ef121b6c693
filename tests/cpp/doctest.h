// Minimal doctest-compatible harness (test infrastructure, not product code).
// Enough of the doctest API to compile the reference's unit tests unmodified
// against libipt_b200: TEST_CASE, SUBCASE (run inline, in order), CHECK,
// CHECK_FALSE, REQUIRE, REQUIRE_FALSE, CHECK_THROWS_AS, FAIL, doctest::Approx.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
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

private:
    double value_;
    double eps_ = static_cast<double>(FLT_EPSILON) * 100;
    double scale_ = 1.0;
};

namespace shim {
struct Case {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(const char* n, void (*f)(), const char* file, int line) { registry().push_back({n, f, file, line}); }
};
struct RequireFailed {};
inline int& failures() { static int f = 0; return f; }
inline int& checks() { static int c = 0; return c; }
inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    ++checks();
    if (!ok) {
        ++failures();
        std::printf("%s:%d: FAILED %s( %s )\n", file, line, kind, expr);
    }
}
}  // namespace shim
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                            \
    static void DOCTEST_CAT(doctest_case_, __LINE__)();                                           \
    static ::doctest::shim::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(                        \
        name, &DOCTEST_CAT(doctest_case_, __LINE__), __FILE__, __LINE__);                         \
    static void DOCTEST_CAT(doctest_case_, __LINE__)()
#define SUBCASE(name) if (true)
#define CHECK(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::shim::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                               \
    do {                                                                                           \
        const bool ok_ = static_cast<bool>(__VA_ARGS__);                                           \
        ::doctest::shim::report(ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                 \
        if (!ok_) throw ::doctest::shim::RequireFailed{};                                          \
    } while (0)
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, type)                                                                \
    do {                                                                                           \
        bool thrown_ = false;                                                                      \
        try { (void)(expr); } catch (const type&) { thrown_ = true; } catch (...) {}               \
        ::doctest::shim::report(thrown_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);            \
    } while (0)
#define FAIL(msg)                                                                                  \
    do {                                                                                           \
        ::doctest::shim::report(false, "FAIL", "explicit failure", __FILE__, __LINE__);            \
        throw ::doctest::shim::RequireFailed{};                                                    \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0;
    for (const auto& c : ::doctest::shim::registry()) {
        const int before = ::doctest::shim::failures();
        try {
            c.fn();
        } catch (const ::doctest::shim::RequireFailed&) {
        } catch (const std::exception& e) {
            ++::doctest::shim::failures();
            std::printf("%s:%d: test case \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
        }
        const bool ok = ::doctest::shim::failures() == before;
        if (!ok) ++failed_cases;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("test cases: %zu | %d failed | checks: %d | %d failed\n", ::doctest::shim::registry().size(),
                failed_cases, ::doctest::shim::checks(), ::doctest::shim::failures());
    return failed_cases == 0 ? 0 : 1;
}
#endif
