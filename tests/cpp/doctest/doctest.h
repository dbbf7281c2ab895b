// doctest.h — a minimal subset of the doctest API (TEST_CASE, CHECK, REQUIRE,
// CHECK_THROWS, doctest::Approx, the implement-with-main runner) so the
// reference's own suites (/root/reference/proj/tests/*.cpp; the vendored
// doctest is absent there, proj/.gitignore) compile UNCHANGED against
// libspike_b200.so.  Test infrastructure, written here; semantics follow the
// public doctest documentation: a failed CHECK marks the test case failed and
// continues, a failed REQUIRE (or an exception) ends the test case, Approx
// compares |a - b| < eps * (scale + max(|a|, |b|)).
//
// Runner options: --test-case=<name>[,<name>...] runs only those cases,
// --test-case-exclude=<name>[,...] skips them (exact names).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
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
    friend bool operator==(double lhs, const Approx& r) {
        return std::fabs(lhs - r.value_) < r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.value_)));
    }
    friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
    friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
    friend bool operator!=(const Approx& r, double rhs) { return !(rhs == r); }

private:
    double value_;
    double eps_ = 1.1920928955078125e-07 * 100;  // float epsilon * 100 (doctest's default)
    double scale_ = 1.0;
};

namespace detail {
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
    Registrar(const char* name, void (*fn)(), const char* file, int line) {
        registry().push_back({name, fn, file, line});
    }
};
struct RequireFailed {};
inline int& failures() {
    static int f = 0;
    return f;
}
inline int& assertions() {
    static int a = 0;
    return a;
}
inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    ++assertions();
    if (ok) return;
    ++failures();
    std::printf("%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, kind, expr);
    std::fflush(stdout);
}
inline std::vector<std::string> split(const char* s) {
    std::vector<std::string> out;
    std::string cur;
    for (const char* p = s; *p; ++p) {
        if (*p == ',') {
            out.push_back(cur);
            cur.clear();
        } else {
            cur += *p;
        }
    }
    if (!cur.empty()) out.push_back(cur);
    return out;
}
inline int run(int argc, char** argv) {
    std::vector<std::string> only, skip;
    for (int i = 1; i < argc; ++i) {
        if (!std::strncmp(argv[i], "--test-case=", 12)) only = split(argv[i] + 12);
        if (!std::strncmp(argv[i], "--test-case-exclude=", 20)) skip = split(argv[i] + 20);
    }
    int ran = 0, failed = 0, skipped = 0;
    for (const Case& c : registry()) {
        const std::string nm = c.name;
        if ((!only.empty() && std::find(only.begin(), only.end(), nm) == only.end()) ||
            std::find(skip.begin(), skip.end(), nm) != skip.end()) {
            ++skipped;
            continue;
        }
        ++ran;
        const int before = failures();
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++failures();
            std::printf("%s:%d: ERROR: test case THREW exception: %s\n", c.file, c.line, e.what());
        } catch (...) {
            ++failures();
            std::printf("%s:%d: ERROR: test case THREW an unknown exception\n", c.file, c.line);
        }
        const bool ok = failures() == before;
        failed += ok ? 0 : 1;
        std::printf("[doctest] %s: %s\n", ok ? "PASS" : "FAIL", c.name);
        std::fflush(stdout);
    }
    std::printf("[doctest] test cases: %d | %d passed | %d failed | %d skipped\n", ran, ran - failed, failed,
                skipped);
    std::printf("[doctest] assertions: %d | %d failed\n", assertions(), failures());
    return failed ? 1 : 0;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_(fn, name)                                                                  \
    static void fn();                                                                                 \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, fn, __FILE__, __LINE__);         \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                  \
    do {                                                                                              \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                     \
        ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);          \
        if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                                   \
    } while (0)
#define CHECK_THROWS(...)                                                                             \
    do {                                                                                              \
        bool doctest_threw_ = false;                                                                  \
        try {                                                                                         \
            (void)(__VA_ARGS__);                                                                      \
        } catch (...) {                                                                               \
            doctest_threw_ = true;                                                                    \
        }                                                                                             \
        ::doctest::detail::report(doctest_threw_, "CHECK_THROWS", #__VA_ARGS__, __FILE__, __LINE__);  \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
