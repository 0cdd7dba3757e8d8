// oracle/doctest_mini/doctest.h — TEST INFRASTRUCTURE ONLY.
//
// The reference's unit tests include "doctest.h" from a vendor/ directory that is not
// shipped (proj/CMakeLists.txt:5, proj/.gitignore:2). This is a minimal, independent
// implementation of the doctest surface those tests use — TEST_CASE, SUBCASE (one level
// deep, re-running the case once per leaf like doctest), CHECK, REQUIRE, CHECK_THROWS_AS,
// FAIL and doctest::Approx(..).epsilon() — so the reference tests compile unchanged and can
// be run against the shim-FFT oracle build.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double value) : value_(value) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    Approx& scale(double s) { scale_ = s; return *this; }
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) <
               rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

private:
    double value_;
    double eps_ = 1.1920929e-05; // float epsilon * 100, doctest's default
    double scale_ = 1.0;
};

namespace detail {

struct RequireAbort {};

struct TestCase {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct State {
    int checks = 0;
    int failures = 0;
    bool case_failed = false;
    const char* case_name = "";
    // subcase bookkeeping (single nesting level is all the reference uses, but nested
    // subcases work as long as leaves are unique by line)
    std::set<std::string> done;
    std::string path;
    std::set<std::string> entered_parent; // parents that already entered a child this run
    int skipped = 0;
};

inline State& state() {
    static State s;
    return s;
}

inline void report(bool ok, const char* expr, const char* file, int line) {
    State& s = state();
    ++s.checks;
    if (!ok) {
        ++s.failures;
        s.case_failed = true;
        std::printf("%s:%d: FAILED in \"%s\" [%s]: %s\n", file, line, s.case_name, s.path.c_str(),
                    expr);
    }
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

class Subcase {
public:
    Subcase(const char* name, int line) {
        State& s = state();
        key_ = s.path + "/" + std::to_string(line) + ":" + name;
        if (s.done.count(key_)) return;
        if (s.entered_parent.count(s.path)) { ++s.skipped; return; }
        s.entered_parent.insert(s.path);
        entered_ = true;
        saved_ = s.path;
        skipped_at_entry_ = s.skipped;
        s.path = key_;
    }
    ~Subcase() {
        if (!entered_) return;
        State& s = state();
        if (s.skipped == skipped_at_entry_) s.done.insert(key_);
        s.path = saved_;
    }
    explicit operator bool() const { return entered_; }

private:
    bool entered_ = false;
    int skipped_at_entry_ = 0;
    std::string key_, saved_;
};

inline int run_all() {
    State& s = state();
    int failed_cases = 0;
    for (const TestCase& tc : registry()) {
        s.case_failed = false;
        s.case_name = tc.name;
        s.done.clear();
        for (int pass = 0; pass < 10000; ++pass) {
            s.path.clear();
            s.entered_parent.clear();
            s.skipped = 0;
            try {
                tc.fn();
            } catch (const RequireAbort&) {
            } catch (const std::exception& e) {
                std::printf("%s:%d: FAILED \"%s\": unexpected exception: %s\n", tc.file, tc.line,
                            tc.name, e.what());
                ++s.failures;
                s.case_failed = true;
            } catch (...) {
                std::printf("%s:%d: FAILED \"%s\": unknown exception\n", tc.file, tc.line, tc.name);
                ++s.failures;
                s.case_failed = true;
            }
            if (s.skipped == 0) break;
        }
        if (s.case_failed) ++failed_cases;
    }
    std::printf("[doctest-mini] test cases: %zu | %zu passed | %d failed\n", registry().size(),
                registry().size() - failed_cases, failed_cases);
    std::printf("[doctest-mini] assertions: %d | %d passed | %d failed\n", s.checks,
                s.checks - s.failures, s.failures);
    return failed_cases == 0 ? 0 : 1;
}

} // namespace detail
} // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                     \
    static void DOCTEST_ANON(doctest_fn_)();                                                \
    static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__, \
                                                                   &DOCTEST_ANON(doctest_fn_)); \
    static void DOCTEST_ANON(doctest_fn_)()

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_ANON(doctest_sc_){name, __LINE__})

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)

#define REQUIRE(...)                                                                        \
    do {                                                                                    \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                            \
        ::doctest::detail::report(doctest_ok_, #__VA_ARGS__, __FILE__, __LINE__);           \
        if (!doctest_ok_) throw ::doctest::detail::RequireAbort{};                          \
    } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                          \
    do {                                                                                    \
        bool doctest_ok_ = false;                                                           \
        try {                                                                               \
            (void)(expr);                                                                   \
        } catch (const __VA_ARGS__&) {                                                      \
            doctest_ok_ = true;                                                             \
        } catch (...) {                                                                     \
        }                                                                                   \
        ::doctest::detail::report(doctest_ok_, "throws " #__VA_ARGS__ ": " #expr, __FILE__, \
                                  __LINE__);                                                \
    } while (0)

#define FAIL(msg)                                                                           \
    do {                                                                                    \
        std::ostringstream doctest_os_;                                                     \
        doctest_os_ << msg;                                                                 \
        ::doctest::detail::report(false, doctest_os_.str().c_str(), __FILE__, __LINE__);    \
        throw ::doctest::detail::RequireAbort{};                                            \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
