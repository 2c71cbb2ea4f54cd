// Minimal doctest-compatible test shim — TEST INFRASTRUCTURE ONLY.
//
// The reference's unit tests (/root/reference/proj/tests/test_*.cpp) include
// <doctest.h>, which is gitignored/absent upstream (proj/.gitignore:2).  This
// header provides the subset they use — TEST_CASE, SUBCASE (the case is
// re-run once per subcase), CHECK / CHECK_FALSE / REQUIRE (variadic),
// CHECK_THROWS_AS and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN — so the reference's
// own tests can be compiled unmodified, either against the reference library
// (pinning oracle/_ref) or against the B200 drop-in plz:: API.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest_shim {

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
    int target = 0;      // which subcase this run executes
    int seen = 0;        // subcases encountered in this run
    long checks = 0;
    long failures = 0;
    bool case_failed = false;
};

inline State& state() {
    static State s;
    return s;
}

struct Register {
    Register(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct RequireFailed {};

inline void record(bool ok, const char* expr, const char* file, int line, bool fatal) {
    State& s = state();
    ++s.checks;
    if (ok) return;
    ++s.failures;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
    if (fatal) throw RequireFailed{};
}

inline bool enter_subcase() {
    State& s = state();
    return s.seen++ == s.target;
}

inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : registry()) {
        State& s = state();
        s.case_failed = false;
        for (s.target = 0;; ++s.target) {
            s.seen = 0;
            try {
                c.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                ++s.failures;
                s.case_failed = true;
                std::fprintf(stderr, "%s:%d: exception in \"%s\": %s\n", c.file, c.line, c.name,
                             e.what());
            }
            if (s.target + 1 >= s.seen) break;  // every subcase has had its run
        }
        if (s.case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "[FAIL] %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | failed: %d | checks: %ld | failed checks: %ld\n",
                registry().size(), failed_cases, state().checks, state().failures);
    return failed_cases ? 1 : 0;
}

}  // namespace doctest_shim

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_CASE(fn, name)                                                    \
    static void fn();                                                                  \
    static doctest_shim::Register DOCTEST_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, \
                                                             &fn);                     \
    static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_CASE(DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__), name)
#define SUBCASE(name) if (doctest_shim::enter_subcase())
#define CHECK(...) \
    doctest_shim::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) \
    doctest_shim::record(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) \
    doctest_shim::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                        \
    do {                                                                                   \
        bool doctest_shim_ok = false;                                                      \
        try {                                                                              \
            (void)(expr);                                                                  \
        } catch (const type&) {                                                            \
            doctest_shim_ok = true;                                                        \
        } catch (...) {                                                                    \
        }                                                                                  \
        doctest_shim::record(doctest_shim_ok, "throws " #type ": " #expr, __FILE__, __LINE__, \
                             false);                                                       \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest_shim::run_all(); }
#endif
