// doctest.h -- a minimal stand-in for the doctest macros the reference's unit
// tests use (TEST_CASE, SUBCASE, CHECK*, REQUIRE*, CHECK_THROWS*, FAIL,
// doctest::Approx with .epsilon()), so those test sources compile UNCHANGED
// against this repository's C++ API (tests/cpp/Makefile).  The reference
// vendors the real doctest (proj/CMakeLists.txt vendor/), absent here.
// Test infrastructure only.
#pragma once
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
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v_) < b.eps_ * (b.scale_ + std::fmax(std::fabs(a), std::fabs(b.v_)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }
    friend bool operator!=(const Approx& b, double a) { return !(a == b); }
    friend bool operator<(double a, const Approx& b) { return a < b.v_ && a != b; }
    friend bool operator>(double a, const Approx& b) { return a > b.v_ && a != b; }
    friend bool operator<=(double a, const Approx& b) { return a < b.v_ || a == b; }
    friend bool operator>=(double a, const Approx& b) { return a > b.v_ || a == b; }
    double value() const { return v_; }

private:
    double v_;
    double eps_ = 1.1920928955078125e-07 * 100;  // doctest's default epsilon
    double scale_ = 1.0;
};

namespace detail {
struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& cases() {
    static std::vector<Case> c;
    return c;
}
struct Reg {
    Reg(const char* n, void (*f)()) { cases().push_back({n, f}); }
};
struct RequireFailed {};
inline int& failures() {
    static int f = 0;
    return f;
}
inline int& checks() {
    static int c = 0;
    return c;
}
inline void report(bool ok, const char* file, int line, const char* expr, bool require) {
    ++checks();
    if (ok) return;
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
    if (require) throw RequireFailed{};
}
// SUBCASE: every subcase of a test case runs once, each in a fresh pass
// through the case body (doctest semantics for one nesting level).
struct SubcaseState {
    int target = 0, seen = 0, total = 0;
};
inline SubcaseState& sub() {
    static SubcaseState s;
    return s;
}
struct Subcase {
    bool run;
    explicit Subcase(const char*) {
        SubcaseState& s = sub();
        run = s.seen++ == s.target;
    }
    explicit operator bool() const { return run; }
};
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                               \
    static void DOCTEST_CAT(doctest_case_, __LINE__)();                                               \
    static ::doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_case_, __LINE__)); \
    static void DOCTEST_CAT(doctest_case_, __LINE__)()
#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_CAT(doctest_sub_, __LINE__){name})

#define DOCTEST_CHECK_IMPL(expr, req) ::doctest::detail::report(static_cast<bool>(expr), __FILE__, __LINE__, #expr, req)
#define CHECK(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), false)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL(!(__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), true)
#define REQUIRE_FALSE(...) DOCTEST_CHECK_IMPL(!(__VA_ARGS__), true)
#define DOCTEST_THROWS_IMPL(expr, cond, text)                                                        \
    do {                                                                                             \
        bool doctest_ok = false;                                                                     \
        try {                                                                                        \
            (void)(expr);                                                                            \
        } catch (cond) {                                                                             \
            doctest_ok = true;                                                                       \
        } catch (...) {                                                                              \
        }                                                                                            \
        ::doctest::detail::report(doctest_ok, __FILE__, __LINE__, text, false);                      \
    } while (0)
#define CHECK_THROWS_AS(expr, ...) DOCTEST_THROWS_IMPL(expr, const __VA_ARGS__&, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")")
#define CHECK_THROWS(expr)                                                                           \
    do {                                                                                             \
        bool doctest_ok = false;                                                                     \
        try {                                                                                        \
            (void)(expr);                                                                            \
        } catch (...) {                                                                              \
            doctest_ok = true;                                                                       \
        }                                                                                            \
        ::doctest::detail::report(doctest_ok, __FILE__, __LINE__, "CHECK_THROWS(" #expr ")", false); \
    } while (0)
#define FAIL(msg)                                                                                    \
    do {                                                                                             \
        std::ostringstream doctest_os;                                                               \
        doctest_os << msg;                                                                           \
        ::doctest::detail::report(false, __FILE__, __LINE__, doctest_os.str().c_str(), true);        \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
// --test-case-exclude=<name> (repeatable) skips a test case by exact name
int main(int argc, char** argv) {
    using namespace doctest::detail;
    std::vector<std::string> skip;
    const std::string opt = "--test-case-exclude=";
    for (int i = 1; i < argc; ++i)
        if (std::string(argv[i]).rfind(opt, 0) == 0) skip.push_back(std::string(argv[i]).substr(opt.size()));
    int failed_cases = 0;
    for (const Case& c : cases()) {
        bool skipped = false;
        for (const std::string& n : skip) skipped |= n == c.name;
        if (skipped) {
            std::printf("[skipped] %s\n", c.name);
            continue;
        }
        const int before = failures();
        SubcaseState& s = sub();
        s = SubcaseState{};
        for (;;) {
            s.seen = 0;
            try {
                c.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                ++failures();
                std::fprintf(stderr, "test case '%s': unexpected exception: %s\n", c.name, e.what());
            }
            if (s.target + 1 >= s.seen) break;  // no further subcase to visit
            ++s.target;
        }
        const bool ok = failures() == before;
        failed_cases += ok ? 0 : 1;
        std::printf("[%s] %s\n", ok ? "ok" : "FAILED", c.name);
    }
    std::printf("%zu test cases, %d failed; %d checks, %d failed\n", cases().size(), failed_cases, checks(),
                failures());
    return failed_cases == 0 ? 0 : 1;
}
#endif
