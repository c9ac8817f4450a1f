// mini_test.hpp — tiny self-registering test harness (the reference's doctest is not
// vendored in this image). TEST_CASE / CHECK / CHECK_FALSE / REQUIRE / CHECK_THROWS_AS;
// main() runs every case, prints failures, exits non-zero if any check failed.
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace mini {

struct Case {
    const char* name;
    std::function<void()> fn;
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
inline int& failures() {
    static int f = 0;
    return f;
}
inline int& checks() {
    static int c = 0;
    return c;
}
struct RequireFailed {};

struct Reg {
    Reg(const char* name, std::function<void()> fn) { registry().push_back({name, std::move(fn)}); }
};

inline void fail(const char* file, int line, const char* expr) {
    ++failures();
    std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", file, line, expr);
}

}  // namespace mini

#define MINI_CAT2(a, b) a##b
#define MINI_CAT(a, b) MINI_CAT2(a, b)
#define TEST_CASE(name)                                                                  \
    static void MINI_CAT(mini_case_, __LINE__)();                                        \
    static mini::Reg MINI_CAT(mini_reg_, __LINE__)(name, MINI_CAT(mini_case_, __LINE__)); \
    static void MINI_CAT(mini_case_, __LINE__)()

#define CHECK(expr)                                              \
    do {                                                         \
        ++mini::checks();                                        \
        if (!(expr)) mini::fail(__FILE__, __LINE__, #expr);      \
    } while (0)
#define CHECK_FALSE(expr) CHECK(!(expr))
#define REQUIRE(expr)                                            \
    do {                                                         \
        ++mini::checks();                                        \
        if (!(expr)) {                                           \
            mini::fail(__FILE__, __LINE__, #expr);               \
            throw mini::RequireFailed{};                         \
        }                                                        \
    } while (0)
#define REQUIRE_FALSE(expr) REQUIRE(!(expr))
#define CHECK_THROWS_AS(expr, type)                                                  \
    do {                                                                              \
        ++mini::checks();                                                             \
        bool mini_ok_ = false;                                                        \
        try {                                                                         \
            (void)(expr);                                                             \
        } catch (const type&) {                                                       \
            mini_ok_ = true;                                                          \
        } catch (...) {                                                               \
        }                                                                             \
        if (!mini_ok_) mini::fail(__FILE__, __LINE__, "throws " #type ": " #expr);    \
    } while (0)

int main() {
    int failed_cases = 0;
    for (const auto& c : mini::registry()) {
        const int before = mini::failures();
        try {
            c.fn();
        } catch (const mini::RequireFailed&) {
        } catch (const std::exception& e) {
            ++mini::failures();
            std::fprintf(stderr, "case '%s' threw: %s\n", c.name, e.what());
        }
        if (mini::failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "FAILED: %s\n", c.name);
        }
    }
    std::printf("%zu cases, %d checks, %d failed cases\n", mini::registry().size(),
                mini::checks(), failed_cases);
    return failed_cases ? 1 : 0;
}
