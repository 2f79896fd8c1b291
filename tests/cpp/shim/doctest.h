// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE).
//
// The reference's unit tests (/root/reference/proj/tests/test_*.cpp) include
// "doctest.h", which the reference does not ship (proj/.gitignore:2). This
// shim implements the subset they use — TEST_CASE, SUBCASE (doctest's
// re-run-per-leaf semantics), CHECK / CHECK_FALSE / REQUIRE, CHECK_THROWS,
// CHECK_THROWS_AS, CHECK_NOTHROW, FAIL and doctest::Approx with doctest's
// comparison rule |a - b| < eps * (scale + max(|a|, |b|)) — so those test
// files compile UNMODIFIED against the drop-in headers (include/cbct/*.hpp)
// and run against libcbct_b200.so (the GPU). Output: one line per test case
// ("TEST <name>: N checks, M failed") and a summary; exit status = failed cases.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
  public:
    template <typename T> explicit Approx(T v) : value_(static_cast<double>(v)) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.value_) < b.eps_ * (b.scale_ + std::max(std::fabs(a), std::fabs(b.value_)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }
    friend bool operator!=(const Approx& b, double a) { return !(a == b); }
    friend bool operator<=(double a, const Approx& b) { return a < b.value_ || a == b; }
    friend bool operator>=(double a, const Approx& b) { return a > b.value_ || a == b; }
    friend bool operator<(double a, const Approx& b) { return a < b.value_ && a != b; }
    friend bool operator>(double a, const Approx& b) { return a > b.value_ && a != b; }

  private:
    double value_;
    double eps_ = double(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

namespace detail {

struct Abort {};  // REQUIRE / FAIL: leave the current run of the test case

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

struct Reg {
    Reg(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};

// SUBCASE bookkeeping: each run of a test case enters at most one not yet
// finished subcase per nesting level; a subcase is finished once a run
// entered it and found no unfinished child. The case re-runs while work
// remains (doctest semantics).
struct State {
    std::set<std::string> done;
    std::vector<std::string> path;        // entered subcases of this run
    std::vector<bool> entered_at_depth;   // a subcase was entered at depth d this run
    std::vector<bool> pending_below;      // unfinished child seen under path[d]
    bool more = false;
    long checks = 0, failed = 0;
    const char* current = "";
};

inline State& st() {
    static State s;
    return s;
}

inline std::string key_of(const std::vector<std::string>& p) {
    std::string k;
    for (const auto& s : p) k += s + "\x1f";
    return k;
}

class Subcase {
  public:
    Subcase(const char* name, int line) {
        State& s = st();
        const size_t d = s.path.size();
        if (s.entered_at_depth.size() <= d) s.entered_at_depth.resize(d + 1, false);
        std::vector<std::string> p = s.path;
        p.push_back(std::string(name) + "@" + std::to_string(line));
        const bool finished = s.done.count(key_of(p)) != 0;
        if (!finished && !s.entered_at_depth[d]) {
            s.entered_at_depth[d] = true;
            s.path = p;
            s.pending_below.resize(s.path.size() + 1, false);
            s.pending_below[s.path.size()] = false;
            entered_ = true;
        } else if (!finished) {
            // a sibling runs this time: come back for this one
            s.more = true;
            if (d < s.pending_below.size()) s.pending_below[d] = true;
        }
    }
    ~Subcase() {
        if (!entered_) return;
        State& s = st();
        const size_t d = s.path.size();
        const bool children_left = d < s.pending_below.size() && s.pending_below[d];
        if (!children_left) s.done.insert(key_of(s.path));
        else s.more = true;
        s.path.pop_back();
        if (s.entered_at_depth.size() > d) s.entered_at_depth.resize(d);
        if (d - 1 < s.pending_below.size() && children_left) s.pending_below[d - 1] = true;
        s.pending_below.resize(d);
    }
    explicit operator bool() const { return entered_; }

  private:
    bool entered_ = false;
};

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
    State& s = st();
    ++s.checks;
    if (ok) return;
    ++s.failed;
    std::string where;
    for (const auto& p : s.path) where += " / " + p;
    std::printf("  FAILED %s:%d [%s%s]: %s\n", file, line, s.current, where.c_str(), expr);
    if (fatal) throw Abort{};
}

inline int run_all() {
    int failed_cases = 0;
    long total_checks = 0, total_failed = 0;
    for (const Case& c : registry()) {
        State& s = st();
        s = State{};
        s.current = c.name;
        int runs = 0;
        do {
            s.more = false;
            s.path.clear();
            s.entered_at_depth.assign(1, false);
            s.pending_below.assign(1, false);
            try {
                c.fn();
            } catch (const Abort&) {
            } catch (const std::exception& e) {
                ++s.failed;
                std::printf("  FAILED [%s]: unexpected exception: %s\n", c.name, e.what());
            } catch (...) {
                ++s.failed;
                std::printf("  FAILED [%s]: unexpected exception\n", c.name);
            }
            // a run that aborted inside subcases: mark them finished
            while (!s.path.empty()) {
                s.done.insert(key_of(s.path));
                s.path.pop_back();
            }
        } while (s.more && ++runs < 10000);
        std::printf("TEST %s: %ld checks, %ld failed\n", c.name, s.checks, s.failed);
        std::fflush(stdout);
        total_checks += s.checks;
        total_failed += s.failed;
        if (s.failed) ++failed_cases;
    }
    std::printf("SUMMARY: %zu test cases, %d failed; %ld checks, %ld failed\n", registry().size(),
                failed_cases, total_checks, total_failed);
    return failed_cases;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC(name, fn)                                                                   \
    static void fn();                                                                          \
    static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn);         \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC(name, DOCTEST_CAT(doctest_case_, __COUNTER__))
#define SUBCASE(name) if (const ::doctest::detail::Subcase& DOCTEST_CAT(doctest_sc_, __COUNTER__) = \
                              ::doctest::detail::Subcase(name, __LINE__))
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_FALSE(...) ::doctest::detail::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, true)
#define DOCTEST_THROWS_AS_IMPL(expr, type, fatal)                                              \
    do {                                                                                       \
        bool doctest_ok_ = false;                                                              \
        try {                                                                                  \
            static_cast<void>(expr);                                                           \
        } catch (const type&) {                                                                \
            doctest_ok_ = true;                                                                \
        } catch (...) {                                                                        \
        }                                                                                      \
        ::doctest::detail::report(doctest_ok_, "throws " #type ": " #expr, __FILE__, __LINE__, fatal); \
    } while (0)
#define CHECK_THROWS_AS(expr, ...) DOCTEST_THROWS_AS_IMPL(expr, __VA_ARGS__, false)
#define REQUIRE_THROWS_AS(expr, ...) DOCTEST_THROWS_AS_IMPL(expr, __VA_ARGS__, true)
#define CHECK_THROWS(...)                                                                      \
    do {                                                                                       \
        bool doctest_ok_ = false;                                                              \
        try {                                                                                  \
            static_cast<void>(__VA_ARGS__);                                                    \
        } catch (...) {                                                                        \
            doctest_ok_ = true;                                                                \
        }                                                                                      \
        ::doctest::detail::report(doctest_ok_, "throws: " #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_NOTHROW(...)                                                                     \
    do {                                                                                       \
        bool doctest_ok_ = true;                                                               \
        try {                                                                                  \
            static_cast<void>(__VA_ARGS__);                                                    \
        } catch (...) {                                                                        \
            doctest_ok_ = false;                                                               \
        }                                                                                      \
        ::doctest::detail::report(doctest_ok_, "nothrow: " #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)
#define FAIL(...) ::doctest::detail::report(false, "FAIL: " #__VA_ARGS__, __FILE__, __LINE__, true)
#define MESSAGE(...) static_cast<void>(0)
#define INFO(...) static_cast<void>(0)
#define CAPTURE(...) static_cast<void>(0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all() ? 1 : 0; }
#endif
