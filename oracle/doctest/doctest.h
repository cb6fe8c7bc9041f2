// TEST INFRASTRUCTURE ONLY — a minimal doctest-compatible header.
//
// The reference's unit tests (/root/reference/proj/tests/test_*.cpp) include
// "doctest.h", which lives in the reference's git-ignored vendor/ directory
// and is absent. This header implements exactly the subset they use
// (TEST_CASE, SUBCASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, FAIL,
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN) so those files compile unmodified
// against either the reference library or the GPU-backed shim.
//
// SUBCASE semantics follow doctest for one nesting level: a test case is run
// once per subcase, each run entering the next not-yet-run subcase and
// re-executing the surrounding code.
#pragma once
#include <cstdio>
#include <exception>
#include <functional>
#include <set>
#include <string>
#include <vector>

namespace doctest_shim {

struct Case {
    const char* name;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct State {
    long checks = 0, failures = 0;
    std::set<std::string> done;  // subcases completed in the current case
    std::string entered;         // subcase entered in the current run
};
inline State& state() {
    static State s;
    return s;
}

struct Abort {};

inline void report(bool ok, const char* file, int line, const char* what) {
    ++state().checks;
    if (!ok) {
        ++state().failures;
        std::fprintf(stderr, "%s:%d: FAILED: %s%s%s\n", file, line, what,
                     state().entered.empty() ? "" : "  [subcase ",
                     state().entered.empty() ? "" : (state().entered + "]").c_str());
    }
}

inline bool enter_subcase(const char* name) {
    State& s = state();
    if (!s.entered.empty() || s.done.count(name)) return false;
    s.entered = name;
    return true;
}

struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

inline int run_all() {
    long cases = 0, failed_cases = 0;
    for (const Case& c : registry()) {
        ++cases;
        State& s = state();
        const long before = s.failures;
        s.done.clear();
        for (;;) {
            s.entered.clear();
            try {
                c.fn();
            } catch (const Abort&) {
            } catch (const std::exception& e) {
                ++s.failures;
                std::fprintf(stderr, "test case \"%s\": uncaught exception: %s\n", c.name, e.what());
            } catch (...) {
                ++s.failures;
                std::fprintf(stderr, "test case \"%s\": uncaught unknown exception\n", c.name);
            }
            if (s.entered.empty()) break;
            s.done.insert(s.entered);
        }
        if (s.failures != before) {
            ++failed_cases;
            std::fprintf(stderr, "test case FAILED: %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %ld | %ld passed | %ld failed | checks: %ld | "
                "failed checks: %ld\n",
                cases, cases - failed_cases, failed_cases, state().checks, state().failures);
    return state().failures == 0 ? 0 : 1;
}

}  // namespace doctest_shim

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_TEST(fn, name)                                             \
    static void fn();                                                           \
    static doctest_shim::Registrar DOCTEST_SHIM_CAT(fn, _reg)(name, &fn);       \
    static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TEST(DOCTEST_SHIM_CAT(doctest_case_, __LINE__), name)
#define SUBCASE(name) if (doctest_shim::enter_subcase(name))
#define CHECK(...) doctest_shim::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define CHECK_FALSE(...) doctest_shim::report(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")")
#define REQUIRE(...)                                                                    \
    do {                                                                                \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                        \
        doctest_shim::report(doctest_ok_, __FILE__, __LINE__, #__VA_ARGS__);            \
        if (!doctest_ok_) throw doctest_shim::Abort{};                                  \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                     \
    do {                                                                                \
        bool doctest_ok_ = false;                                                       \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (const type&) {                                                         \
            doctest_ok_ = true;                                                         \
        } catch (...) {                                                                 \
        }                                                                               \
        doctest_shim::report(doctest_ok_, __FILE__, __LINE__, #expr " throws " #type);  \
    } while (0)
#define FAIL(msg)                                                                       \
    do {                                                                                \
        doctest_shim::report(false, __FILE__, __LINE__, "FAIL");                        \
        throw doctest_shim::Abort{};                                                    \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest_shim::run_all(); }
#endif
