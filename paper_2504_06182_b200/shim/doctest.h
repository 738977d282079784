// Minimal doctest-compatible harness (the reference's tests include
// <doctest.h> from a vendor/ directory that is not shipped).  Supports the
// macros those tests use: TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// REQUIRE_FALSE, CHECK_THROWS_AS, CHECK_NOTHROW, INFO, MESSAGE.
#pragma once

#include <cstdio>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

namespace dtshim {

struct Case {
    const char *name;
    void (*fn)();
};

inline std::vector<Case> &registry() {
    static std::vector<Case> r;
    return r;
}
inline long long &checks() {
    static long long n = 0;
    return n;
}
inline long long &failed_checks() {
    static long long n = 0;
    return n;
}
inline std::vector<std::string> &infos() {
    static std::vector<std::string> s;
    return s;
}

struct Reg {
    Reg(const char *n, void (*f)()) { registry().push_back({n, f}); }
};
struct RequireFailure {};

template <typename... A>
std::string cat(const A &...a) {
    std::ostringstream os;
    (os << ... << a);
    return os.str();
}

struct InfoScope {
    explicit InfoScope(std::string s) { infos().push_back(std::move(s)); }
    ~InfoScope() { infos().pop_back(); }
};

inline void fail(const char *kind, const char *expr, const char *file, int line) {
    ++failed_checks();
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
    for (const auto &i : infos()) std::fprintf(stderr, "  with: %s\n", i.c_str());
}

inline void message(const std::string &m) { std::fprintf(stderr, "  message: %s\n", m.c_str()); }

}  // namespace dtshim

#define DTSHIM_CAT_(a, b) a##b
#define DTSHIM_CAT(a, b) DTSHIM_CAT_(a, b)
#define TEST_CASE(name)                                                                              \
    static void DTSHIM_CAT(dtshim_fn_, __LINE__)();                                                  \
    static dtshim::Reg DTSHIM_CAT(dtshim_reg_, __LINE__)(name, &DTSHIM_CAT(dtshim_fn_, __LINE__));   \
    static void DTSHIM_CAT(dtshim_fn_, __LINE__)()
#define CHECK(...)                                                                  \
    do {                                                                            \
        ++dtshim::checks();                                                         \
        if (!(__VA_ARGS__)) dtshim::fail("CHECK", #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                       \
    do {                                                                   \
        ++dtshim::checks();                                                \
        if (!(__VA_ARGS__)) {                                              \
            dtshim::fail("REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);     \
            throw dtshim::RequireFailure{};                                \
        }                                                                  \
    } while (0)
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, ...)                                                       \
    do {                                                                                 \
        ++dtshim::checks();                                                              \
        bool dtshim_ok = false;                                                          \
        try {                                                                            \
            (void)(expr);                                                                \
        } catch (const __VA_ARGS__ &) {                                                  \
            dtshim_ok = true;                                                            \
        } catch (...) {                                                                  \
        }                                                                                \
        if (!dtshim_ok) dtshim::fail("CHECK_THROWS_AS", #expr, __FILE__, __LINE__);      \
    } while (0)
#define CHECK_NOTHROW(expr)                                                   \
    do {                                                                      \
        ++dtshim::checks();                                                   \
        try {                                                                 \
            (void)(expr);                                                     \
        } catch (...) {                                                       \
            dtshim::fail("CHECK_NOTHROW", #expr, __FILE__, __LINE__);         \
        }                                                                     \
    } while (0)
#define INFO(...) dtshim::InfoScope DTSHIM_CAT(dtshim_info_, __LINE__)(dtshim::cat(__VA_ARGS__))
#define MESSAGE(...) dtshim::message(dtshim::cat(__VA_ARGS__))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0;
    for (const auto &c : dtshim::registry()) {
        const long long before = dtshim::failed_checks();
        try {
            c.fn();
        } catch (const dtshim::RequireFailure &) {
        } catch (const std::exception &e) {
            ++dtshim::failed_checks();
            std::fprintf(stderr, "TEST CASE \"%s\": unexpected exception: %s\n", c.name, e.what());
        }
        if (dtshim::failed_checks() != before) {
            ++failed_cases;
            std::fprintf(stderr, "TEST CASE FAILED: %s\n", c.name);
        }
    }
    std::printf("[doctest] test cases: %zu | %zu passed | %d failed | checks: %lld | %lld failed\n",
                dtshim::registry().size(), dtshim::registry().size() - (size_t)failed_cases, failed_cases,
                dtshim::checks(), dtshim::failed_checks());
    return failed_cases ? 1 : 0;
}
#endif
