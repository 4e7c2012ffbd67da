// Minimal doctest-compatible test harness (original code, not doctest's).
//
// Enough of doctest's surface to compile and run the reference's own test
// sources unchanged (/root/reference/proj/tests/*.cpp):
// TEST_CASE, SUBCASE (re-entry: a test case is re-run until every leaf
// subcase has run once, the code outside subcases running every time),
// CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_MESSAGE, FAIL, MESSAGE,
// doctest::Approx(...).epsilon(...), and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
// main() accepts an optional "-tc=<substring>" filter and prints one line
// per test case plus a summary; the exit code is 1 on any failure.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
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
    // |a - b| < eps * (scale + max(|a|, |b|))
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.value_) <
               b.eps_ * (b.scale_ + std::fmax(std::fabs(a), std::fabs(b.value_)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }
    friend bool operator!=(const Approx& b, double a) { return !(a == b); }

private:
    double value_;
    double eps_ = 1.1920929e-7 * 100;  // float epsilon * 100
    double scale_ = 1.0;
};

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

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

// Per-test-case run state.  Each run of a test case enters at most one
// not-yet-finished subcase per nesting level; a subcase is finished once it
// ran with no unfinished children.  `more` asks for another run.
struct Runner {
    std::vector<std::string> path;      // names of the entered subcases
    std::set<std::string> finished;
    std::vector<bool> taken;            // a subcase was entered at depth d this run
    std::vector<bool> pending;          // depth d has unfinished children
    bool more = false;
    int failures = 0;
    int checks = 0;
    const TestCase* current = nullptr;

    std::string key(const char* name) const {
        std::string k;
        for (const std::string& p : path) k += p + '\x1f';
        return k + name;
    }
    void begin_run() {
        path.clear();
        taken.assign(1, false);
        pending.assign(1, false);
        more = false;
    }
};

inline Runner& runner() {
    static Runner r;
    return r;
}

struct AbortTest {};  // REQUIRE / FAIL: leave the test case

class Subcase {
public:
    Subcase(const char* name) {
        Runner& r = runner();
        const size_t d = r.path.size();
        key_ = r.key(name);
        if (r.taken.size() <= d) {
            r.taken.resize(d + 1, false);
            r.pending.resize(d + 1, false);
        }
        if (r.finished.count(key_)) return;
        if (r.taken[d]) {  // a sibling ran this time; come back on a later run
            r.more = true;
            if (d > 0) r.pending[d - 1] = true;
            return;
        }
        entered_ = true;
        r.taken[d] = true;
        r.path.push_back(name);
        if (r.taken.size() <= d + 1) {
            r.taken.resize(d + 2, false);
            r.pending.resize(d + 2, false);
        }
        r.taken[d + 1] = false;
        r.pending[d] = false;
    }
    ~Subcase() {
        if (!entered_) return;
        Runner& r = runner();
        const size_t d = r.path.size() - 1;
        r.path.pop_back();
        if (r.pending[d]) {
            if (d > 0) r.pending[d - 1] = true;
        } else {
            r.finished.insert(key_);
        }
    }
    explicit operator bool() const { return entered_; }

private:
    std::string key_;
    bool entered_ = false;
};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   const std::string& msg = "") {
    Runner& r = runner();
    ++r.checks;
    if (ok) return;
    ++r.failures;
    std::string where;
    for (const std::string& p : r.path) where += " / " + p;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s )%s%s  [in \"%s\"%s]\n", file, line, kind, expr,
                 msg.empty() ? "" : " : ", msg.c_str(), r.current ? r.current->name : "?",
                 where.c_str());
}

template <class T>
std::string to_text(const T& v) {
    std::ostringstream os;
    if constexpr (requires { os << v; }) {
        os.precision(17);
        os << v;
        return os.str();
    } else {
        return std::string();
    }
}

inline int run_all(int argc, char** argv) {
    std::string filter;
    for (int i = 1; i < argc; ++i) {
        const char* a = argv[i];
        if (std::strncmp(a, "-tc=", 4) == 0) filter = a + 4;
        if (std::strncmp(a, "--test-case=", 12) == 0) filter = a + 12;
    }
    int failed_cases = 0, ran = 0, total_checks = 0, total_failures = 0;
    for (const TestCase& tc : registry()) {
        if (!filter.empty() && std::string(tc.name).find(filter) == std::string::npos) continue;
        ++ran;
        Runner& r = runner();
        r.finished.clear();
        r.failures = 0;
        r.checks = 0;
        r.current = &tc;
        int runs = 0;
        do {
            r.begin_run();
            try {
                tc.fn();
            } catch (const AbortTest&) {
            } catch (const std::exception& e) {
                ++r.failures;
                std::fprintf(stderr, "%s:%d: FAILED: uncaught exception in \"%s\": %s\n", tc.file,
                             tc.line, tc.name, e.what());
            } catch (...) {
                ++r.failures;
                std::fprintf(stderr, "%s:%d: FAILED: unknown exception in \"%s\"\n", tc.file,
                             tc.line, tc.name);
            }
        } while (r.more && ++runs < 10000);
        total_checks += r.checks;
        total_failures += r.failures;
        if (r.failures) ++failed_cases;
        std::printf("[%s] %s (%d checks)\n", r.failures ? "FAIL" : " ok ", tc.name, r.checks);
        std::fflush(stdout);
    }
    std::printf("test cases: %d | %d passed | %d failed; assertions: %d | %d failed\n", ran,
                ran - failed_cases, failed_cases, total_checks, total_failures);
    return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_UNIQUE(base) DOCTEST_CAT(base, __COUNTER__)

#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                      \
    static void fn();                                                                          \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_UNIQUE(doctest_tc_), name)

#define SUBCASE(name) \
    if (const ::doctest::detail::Subcase DOCTEST_UNIQUE(doctest_sc_){name})

#define CHECK(...)                                                                          \
    do {                                                                                    \
        bool doctest_ok_ = false;                                                           \
        try {                                                                               \
            doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                   \
        } catch (const ::doctest::detail::AbortTest&) {                                     \
            throw;                                                                          \
        } catch (...) {                                                                     \
            ::doctest::detail::report(false, "CHECK", #__VA_ARGS__, __FILE__, __LINE__,     \
                                      "threw");                                             \
            break;                                                                          \
        }                                                                                   \
        ::doctest::detail::report(doctest_ok_, "CHECK", #__VA_ARGS__, __FILE__, __LINE__);  \
    } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define CHECK_MESSAGE(cond, msg)                                                             \
    ::doctest::detail::report(static_cast<bool>(cond), "CHECK_MESSAGE", #cond, __FILE__,     \
                              __LINE__, ::doctest::detail::to_text(msg))
#define REQUIRE(...)                                                                        \
    do {                                                                                    \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                            \
        ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__); \
        if (!doctest_ok_) throw ::doctest::detail::AbortTest{};                             \
    } while (0)
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, ...)                                                           \
    do {                                                                                     \
        bool doctest_right_ = false;                                                         \
        const char* doctest_what_ = "did not throw";                                         \
        try {                                                                                \
            static_cast<void>(expr);                                                         \
        } catch (const __VA_ARGS__&) {                                                       \
            doctest_right_ = true;                                                           \
        } catch (...) {                                                                      \
            doctest_what_ = "threw a different type";                                        \
        }                                                                                    \
        ::doctest::detail::report(doctest_right_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, \
                                  __FILE__, __LINE__, doctest_right_ ? "" : doctest_what_);  \
    } while (0)
#define FAIL(msg)                                                                             \
    do {                                                                                      \
        ::doctest::detail::report(false, "FAIL", "", __FILE__, __LINE__,                      \
                                  ::doctest::detail::to_text(msg));                           \
        throw ::doctest::detail::AbortTest{};                                                 \
    } while (0)
#define MESSAGE(msg) \
    std::printf("%s:%d: MESSAGE: %s\n", __FILE__, __LINE__, ::doctest::detail::to_text(msg).c_str())

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run_all(argc, argv); }
#endif
