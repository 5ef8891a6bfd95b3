// doctest.h -- a minimal stand-in for the doctest macros the reference's unit
// tests use (TEST_CASE, TEST_SUITE_BEGIN/END, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS).  TEST INFRASTRUCTURE ONLY: doctest itself is not
// installed in this image, and this lets oracle/Makefile compile the
// reference's own tests/test_{formats,spmm,conv}.cpp, unmodified, against
// this repo's headers and libshflbw_b200.so (the drop-in check).
#pragma once
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

namespace doctest_shim {

struct Case {
    const char* suite;
    const char* name;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
inline const char*& current_suite() {
    static const char* s = "";
    return s;
}
inline int set_suite(const char* s) {
    current_suite() = s;
    return 0;
}
inline int add(const char* name, void (*fn)()) {
    registry().push_back({current_suite(), name, fn});
    return 0;
}
struct State {
    int failed_checks = 0;
    int checks = 0;
};
inline State& state() {
    static State s;
    return s;
}
struct RequireFailed {};

inline void report(bool ok, const char* what, const char* expr, const char* file, int line) {
    ++state().checks;
    if (!ok) {
        ++state().failed_checks;
        std::printf("    %s:%d: %s( %s ) FAILED\n", file, line, what, expr);
    }
}

}  // namespace doctest_shim

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                          \
    static void fn();                                                                      \
    static int DOCTEST_CAT(fn, _reg) = ::doctest_shim::add(name, &fn);                     \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define TEST_SUITE_BEGIN(name) static int DOCTEST_CAT(doctest_suite_, __COUNTER__) = ::doctest_shim::set_suite(name)
#define TEST_SUITE_END() static int DOCTEST_CAT(doctest_suite_, __COUNTER__) = ::doctest_shim::set_suite("")
#define CHECK(...) ::doctest_shim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
    ::doctest_shim::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                       \
    do {                                                                                                   \
        const bool doctest_ok = static_cast<bool>(__VA_ARGS__);                                            \
        ::doctest_shim::report(doctest_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                   \
        if (!doctest_ok) throw ::doctest_shim::RequireFailed{};                                            \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                        \
    do {                                                                                                   \
        bool doctest_ok = false;                                                                           \
        try {                                                                                              \
            (void)(expr);                                                                                  \
        } catch (const __VA_ARGS__&) {                                                                     \
            doctest_ok = true;                                                                             \
        } catch (...) {                                                                                    \
        }                                                                                                  \
        ::doctest_shim::report(doctest_ok, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    const char* only = nullptr;
    for (int i = 1; i < argc; ++i)
        if (!std::strncmp(argv[i], "-ts=", 4)) only = argv[i] + 4;
    int failed_cases = 0, ran = 0;
    for (const auto& c : ::doctest_shim::registry()) {
        if (only && std::strcmp(only, c.suite)) continue;
        const int before = ::doctest_shim::state().failed_checks;
        bool threw = false;
        std::string what;
        try {
            c.fn();
        } catch (const ::doctest_shim::RequireFailed&) {
        } catch (const std::exception& e) {
            threw = true;
            what = e.what();
        }
        const bool ok = !threw && ::doctest_shim::state().failed_checks == before;
        ++ran;
        if (!ok) ++failed_cases;
        std::printf("[%s] %s :: %s%s%s\n", ok ? "PASS" : "FAIL", c.suite, c.name, threw ? " -- exception: " : "",
                    what.c_str());
    }
    std::printf("test cases: %d | %d passed | %d failed; checks: %d | %d failed\n", ran, ran - failed_cases,
                failed_cases, ::doctest_shim::state().checks, ::doctest_shim::state().failed_checks);
    return failed_cases;
}
#endif
