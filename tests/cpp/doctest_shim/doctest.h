// TEST INFRASTRUCTURE ONLY — a small stand-in for doctest (the reference's unit tests
// include <doctest.h>, which proj/.gitignore:2 keeps out of the reference tree), enough to
// compile the reference's own test files UNMODIFIED against the drop-in headers
// (tests/cpp/Makefile.reftests, tests/test_reference_unit_tests.py).
//
// Supported: TEST_CASE, SUBCASE (one level, each leaf re-runs the test case), CHECK,
// CHECK_FALSE, REQUIRE (a failure ends the test case), CHECK_THROWS_AS, CAPTURE, and
// doctest::Approx with epsilon() / scale() (doctest's own comparison rule). The runner
// main() takes --exclude=<test case name> (repeatable) and --list; it prints one line per
// test case and exits non-zero if any check failed.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <sstream>
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
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

namespace detail {

struct RequireFailed {};

struct TestCase {
    const char* name;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct State {
    int failures = 0;
    int checks = 0;
    // subcase traversal of the running test case
    int target = 0;    // which leaf runs in this pass
    int seen = 0;      // SUBCASEs met so far in this pass
    std::vector<std::string> captures;
    std::string current;
};

inline State& state() {
    static State s;
    return s;
}

inline int reg(const char* name, void (*fn)()) {
    registry().push_back({name, fn});
    return 0;
}

inline void report(bool ok, const char* file, int line, const char* expr) {
    State& s = state();
    ++s.checks;
    if (ok) return;
    ++s.failures;
    std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, s.current.c_str(), expr);
    for (const auto& c : s.captures) std::fprintf(stderr, "    with %s\n", c.c_str());
}

struct Subcase {
    bool run;
    explicit Subcase(const char*) {
        State& s = state();
        run = s.seen++ == s.target;
    }
    explicit operator bool() const { return run; }
};

struct Capture {
    template <class T>
    Capture(const char* name, const T& v) {
        std::ostringstream o;
        o << name << " := " << v;
        state().captures.push_back(o.str());
    }
    ~Capture() { state().captures.pop_back(); }
};

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                                  \
    static void fn();                                                                          \
    static const int DOCTEST_CAT(fn, _reg) = doctest::detail::reg(name, &fn);                  \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) if (const doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name})
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define CHECK_FALSE(...) doctest::detail::report(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")")
#define REQUIRE(...)                                                                           \
    do {                                                                                       \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                               \
        doctest::detail::report(doctest_ok_, __FILE__, __LINE__, #__VA_ARGS__);                \
        if (!doctest_ok_) throw doctest::detail::RequireFailed{};                              \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                             \
    do {                                                                                       \
        bool doctest_thrown_ = false;                                                          \
        try {                                                                                  \
            static_cast<void>(expr);                                                           \
        } catch (const __VA_ARGS__&) {                                                         \
            doctest_thrown_ = true;                                                            \
        } catch (...) {                                                                        \
        }                                                                                      \
        doctest::detail::report(doctest_thrown_, __FILE__, __LINE__, #expr " throws " #__VA_ARGS__); \
    } while (0)
#define CAPTURE(x) const doctest::detail::Capture DOCTEST_CAT(doctest_cap_, __LINE__)(#x, x)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    using namespace doctest::detail;
    std::set<std::string> excluded;
    bool list = false;
    for (int i = 1; i < argc; ++i) {
        if (std::strncmp(argv[i], "--exclude=", 10) == 0) excluded.insert(argv[i] + 10);
        if (std::strcmp(argv[i], "--list") == 0) list = true;
    }
    State& s = state();
    int cases = 0, failed_cases = 0, skipped = 0;
    for (const TestCase& tc : registry()) {
        if (list) {
            std::printf("%s\n", tc.name);
            continue;
        }
        if (excluded.count(tc.name)) {
            ++skipped;
            std::printf("[skip] %s\n", tc.name);
            continue;
        }
        ++cases;
        const int before = s.failures;
        s.current = tc.name;
        for (s.target = 0;; ++s.target) {  // one pass per leaf SUBCASE (one pass if none)
            s.seen = 0;
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                report(false, "<exception>", 0, e.what());
            } catch (...) {
                report(false, "<exception>", 0, "unknown exception");
            }
            if (s.target + 1 >= s.seen) break;
        }
        const bool ok = s.failures == before;
        if (!ok) ++failed_cases;
        std::printf("[%s] %s\n", ok ? "pass" : "FAIL", tc.name);
    }
    if (!list)
        std::printf("test cases: %d run, %d failed, %d excluded; checks: %d, failed %d\n", cases, failed_cases, skipped,
                    s.checks, s.failures);
    return failed_cases ? 1 : 0;
}
#endif
