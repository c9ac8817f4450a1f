// doctest.h — the subset of the doctest API the reference's suites use
// (/root/reference/proj/tests/test_*.cpp: TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// REQUIRE_FALSE, CHECK_THROWS_AS, doctest::Approx with .epsilon()), written for this repo
// because doctest itself is not vendored in the image. It lets the reference's own test
// files compile UNMODIFIED against the B200 drop-in (include/ssbh + libssbh.so); see
// tests/refsuite/Makefile. With DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN defined, main() runs every
// registered case and prints "[refsuite] N cases, M checks, F failed cases".
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <stdexcept>
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
        // doctest's rule: |lhs - v| < eps * (scale + max(|lhs|, |v|))
        return std::fabs(lhs - a.value_) <
               a.eps_ * (a.scale_ + std::fmax(std::fabs(lhs), std::fabs(a.value_)));
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
    double eps_ = 1.19209290e-07 * 100;  // doctest's default: 100 float epsilons
    double scale_ = 1.0;
};

namespace shim {

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
struct State {
    int checks = 0;
    int failed_checks = 0;
    bool case_failed = false;
};
inline State& state() {
    static State s;
    return s;
}
struct RequireFailed {};
struct Reg {
    Reg(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};
inline void fail(const char* file, int line, const char* kind, const char* expr) {
    ++state().failed_checks;
    state().case_failed = true;
    std::fprintf(stderr, "%s:%d: %s( %s ) failed\n", file, line, kind, expr);
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define TEST_CASE(name)                                                                    \
    static void DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__)();                          \
    static doctest::shim::Reg DOCTEST_SHIM_CAT(doctest_shim_reg_, __LINE__)(               \
        name, __FILE__, __LINE__, DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__));         \
    static void DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__)()

#define DOCTEST_SHIM_ASSERT(kind, cond, text, fatal)                                       \
    do {                                                                                   \
        ++doctest::shim::state().checks;                                                   \
        bool ok_ = false;                                                                  \
        try {                                                                              \
            ok_ = static_cast<bool>(cond);                                                 \
        } catch (const std::exception& e_) {                                               \
            std::fprintf(stderr, "  threw: %s\n", e_.what());                              \
        }                                                                                  \
        if (!ok_) {                                                                        \
            doctest::shim::fail(__FILE__, __LINE__, kind, text);                           \
            if (fatal) throw doctest::shim::RequireFailed{};                               \
        }                                                                                  \
    } while (0)
#define CHECK(...) DOCTEST_SHIM_ASSERT("CHECK", (__VA_ARGS__), #__VA_ARGS__, false)
#define CHECK_FALSE(...) DOCTEST_SHIM_ASSERT("CHECK_FALSE", !(__VA_ARGS__), #__VA_ARGS__, false)
#define REQUIRE(...) DOCTEST_SHIM_ASSERT("REQUIRE", (__VA_ARGS__), #__VA_ARGS__, true)
#define REQUIRE_FALSE(...) DOCTEST_SHIM_ASSERT("REQUIRE_FALSE", !(__VA_ARGS__), #__VA_ARGS__, true)
#define CHECK_THROWS_AS(expr, ...)                                                         \
    do {                                                                                   \
        ++doctest::shim::state().checks;                                                   \
        bool right_ = false;                                                               \
        try {                                                                              \
            (void)(expr);                                                                  \
        } catch (const __VA_ARGS__&) {                                                     \
            right_ = true;                                                                 \
        } catch (...) {                                                                    \
        }                                                                                  \
        if (!right_)                                                                       \
            doctest::shim::fail(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    using namespace doctest::shim;
    int failed_cases = 0;
    for (const Case& c : registry()) {
        state().case_failed = false;
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: TEST_CASE(\"%s\") threw: %s\n", c.file, c.line, c.name,
                         e.what());
            state().case_failed = true;
        }
        if (state().case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "FAILED: %s\n", c.name);
        }
    }
    std::printf("[refsuite] %zu cases, %d checks, %d failed cases\n", registry().size(),
                state().checks, failed_cases);
    return failed_cases ? 1 : 0;
}
#endif
