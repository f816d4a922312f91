// Minimal doctest-compatible test harness — TEST INFRASTRUCTURE (oracle only).
//
// The reference's unit tests (/root/reference/proj/tests/*.cpp) include
// "doctest.h", which is not vendored (CMakeLists.txt:5 points at an absent
// vendor/). They use only TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_NOTHROW, CAPTURE, FAIL and doctest::Approx(v).epsilon(e) (SURVEY
// §8(c)). This header implements exactly that surface with doctest's
// published semantics so the reference tests compile and run unmodified:
//   * Approx: |a-b| < eps * (scale + max(|a|,|b|)), scale = 1, default
//     eps = 100 * FLT_EPSILON.
//   * REQUIRE aborts the current test case; CHECK records and continues.
//   * command line: -tc=<substring>[,<substring>...] selects test cases,
//     -tce=<substring> excludes, -s prints every case name.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
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
    bool eq(double lhs) const {
        return std::fabs(lhs - value_) <
               eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
    }
    double value() const { return value_; }

private:
    double value_;
    double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
    double scale_ = 1.0;
};

template <typename T>
bool operator==(const T& lhs, const Approx& rhs) { return rhs.eq(double(lhs)); }
template <typename T>
bool operator==(const Approx& lhs, const T& rhs) { return lhs.eq(double(rhs)); }
template <typename T>
bool operator!=(const T& lhs, const Approx& rhs) { return !rhs.eq(double(lhs)); }
template <typename T>
bool operator!=(const Approx& lhs, const T& rhs) { return !lhs.eq(double(rhs)); }
template <typename T>
bool operator<=(const T& lhs, const Approx& rhs) { return double(lhs) < rhs.value() || rhs.eq(double(lhs)); }
template <typename T>
bool operator>=(const T& lhs, const Approx& rhs) { return double(lhs) > rhs.value() || rhs.eq(double(lhs)); }

namespace detail {

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
    long checks = 0;
    long failed_checks = 0;
    bool case_failed = false;
    std::vector<std::string> captures;
};

inline State& state() {
    static State s;
    return s;
}

struct RequireAbort {};

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   bool fatal) {
    State& s = state();
    ++s.checks;
    if (ok) return;
    ++s.failed_checks;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s )\n", file, line, kind, expr);
    for (const std::string& c : s.captures) std::fprintf(stderr, "  with %s\n", c.c_str());
    if (fatal) throw RequireAbort{};
}

struct CaptureGuard {
    explicit CaptureGuard(std::string s) { state().captures.push_back(std::move(s)); }
    ~CaptureGuard() { state().captures.pop_back(); }
};

template <typename T>
std::string stringify(const char* name, const T& v) {
    std::ostringstream os;
    os << name << " := " << v;
    return os.str();
}

inline bool match_any(const std::string& name, const std::string& csv) {
    size_t start = 0;
    while (start <= csv.size()) {
        size_t end = csv.find(',', start);
        if (end == std::string::npos) end = csv.size();
        std::string tok = csv.substr(start, end - start);
        if (!tok.empty() && name.find(tok) != std::string::npos) return true;
        start = end + 1;
    }
    return false;
}

inline int run_all(int argc, char** argv) {
    std::string include, exclude;
    bool verbose = false;
    for (int i = 1; i < argc; ++i) {
        if (std::strncmp(argv[i], "-tc=", 4) == 0) include = argv[i] + 4;
        else if (std::strncmp(argv[i], "--test-case=", 12) == 0) include = argv[i] + 12;
        else if (std::strncmp(argv[i], "-tce=", 5) == 0) exclude = argv[i] + 5;
        else if (std::strcmp(argv[i], "-s") == 0) verbose = true;
    }
    State& s = state();
    int cases = 0, failed_cases = 0;
    for (const TestCase& tc : registry()) {
        std::string name = tc.name;
        if (!include.empty() && !match_any(name, include)) continue;
        if (!exclude.empty() && match_any(name, exclude)) continue;
        ++cases;
        s.case_failed = false;
        s.captures.clear();
        if (verbose) std::fprintf(stderr, "[case] %s\n", tc.name);
        try {
            tc.fn();
        } catch (const RequireAbort&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", tc.file, tc.line, tc.name,
                         e.what());
            s.case_failed = true;
            ++s.failed_checks;
        }
        if (s.case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "[FAILED] %s\n", tc.name);
        }
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n", cases,
                cases - failed_cases, failed_cases);
    std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", s.checks,
                s.checks - s.failed_checks, s.failed_checks);
    return failed_cases == 0 ? 0 : 1;
}

} // namespace detail
} // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)

#define DOCTEST_TEST_CASE_IMPL(fn, name)                                               \
    static void fn();                                                                  \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, \
                                                              &fn);                    \
    static void fn()

#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define DOCTEST_CHECK_IMPL(kind, expr, fatal)                                               \
    do {                                                                                    \
        bool doctest_ok_ = false;                                                           \
        try {                                                                               \
            doctest_ok_ = static_cast<bool>(expr);                                          \
        } catch (const ::doctest::detail::RequireAbort&) {                                  \
            throw;                                                                          \
        } catch (...) {                                                                     \
            doctest_ok_ = false;                                                            \
        }                                                                                   \
        ::doctest::detail::report(doctest_ok_, kind, #expr, __FILE__, __LINE__, fatal);     \
    } while (0)

#define CHECK(...) DOCTEST_CHECK_IMPL("CHECK", (__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL("REQUIRE", (__VA_ARGS__), true)

#define CHECK_THROWS_AS(expr, ...)                                                      \
    do {                                                                                \
        bool doctest_ok_ = false;                                                       \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (const __VA_ARGS__&) {                                                  \
            doctest_ok_ = true;                                                         \
        } catch (...) {                                                                 \
        }                                                                               \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, \
                                  __FILE__, __LINE__, false);                           \
    } while (0)

#define CHECK_NOTHROW(expr)                                                                  \
    do {                                                                                     \
        bool doctest_ok_ = true;                                                             \
        try {                                                                                \
            (void)(expr);                                                                    \
        } catch (...) {                                                                      \
            doctest_ok_ = false;                                                             \
        }                                                                                    \
        ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__,   \
                                  false);                                                    \
    } while (0)

#define CAPTURE(x)                                                        \
    ::doctest::detail::CaptureGuard DOCTEST_CAT(doctest_capture_, __LINE__)( \
        ::doctest::detail::stringify(#x, (x)))

#define FAIL(msg) ::doctest::detail::report(false, "FAIL", msg, __FILE__, __LINE__, true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run_all(argc, argv); }
#endif
