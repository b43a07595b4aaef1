// Minimal doctest-compatible shim (test infrastructure only): enough of the
// doctest API for the reference's hot-path suites (proj/tests/test_packing.cpp,
// test_model.cpp, test_grpo.cpp, test_pipeline.cpp) to compile unmodified
// against the drop-in headers (include/parl/*.hpp) and run on the GPU.
//
// Supported: TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS,
// CHECK_NOTHROW, INFO, doctest::Approx(x).epsilon(e) (doctest's scale rule),
// doctest::Contains.  main() (DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN) runs every
// case, or the cases named by -tc=<a,b,...>, and prints one line per case:
//   CASE <PASS|FAIL> <asserts> <failed> <name>
// followed by one "FAILED_AT <file>:<line> x<count>" line per failing assertion
// site and the first failure messages.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <map>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : v_(v), eps_(1.19209290e-07 * 100) {}  // doctest's default epsilon
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& r) {
        // doctest: |lhs - v| < eps * (scale + max(|lhs|, |v|)), scale 1
        return std::fabs(lhs - r.v_) < r.eps_ * (1.0 + std::fmax(std::fabs(lhs), std::fabs(r.v_)));
    }
    friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
    friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
    double value() const { return v_; }

private:
    double v_, eps_;
};

struct Contains {
    explicit Contains(const char* s) : s_(s) {}
    bool check(const std::string& what) const { return what.find(s_) != std::string::npos; }
    std::string s_;
};

namespace detail {
struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Reg {
    Reg(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct State {
    long asserts = 0, failed = 0;
    std::vector<std::string> msgs;
    std::vector<std::string> info;
    std::map<std::string, long> sites;
};
inline State& state() {
    static State s;
    return s;
}
struct RequireAbort {};
inline void record(bool ok, const char* file, int line, const char* what, bool require) {
    auto& s = state();
    ++s.asserts;
    if (ok) return;
    ++s.failed;
    ++s.sites[std::string(file) + ":" + std::to_string(line)];
    if (s.msgs.size() < 8) {
        std::string m = std::string(file) + ":" + std::to_string(line) + ": " + what;
        for (const auto& i : s.info) m += "  [" + i + "]";
        s.msgs.push_back(m);
    }
    if (require) throw RequireAbort{};
}
struct InfoScope {
    template <class... A>
    explicit InfoScope(A&&... a) {
        std::ostringstream os;
        (os << ... << a);
        state().info.push_back(os.str());
    }
    ~InfoScope() { state().info.pop_back(); }
};
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                      \
    static void fn();                                                  \
    static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, fn);     \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __LINE__), name)

#define DOCTEST_ASSERT_(expr, req)                                                              \
    do {                                                                                        \
        bool ok_ = false;                                                                       \
        try {                                                                                   \
            ok_ = static_cast<bool>(expr);                                                      \
        } catch (const ::doctest::detail::RequireAbort&) {                                      \
            throw;                                                                              \
        } catch (const std::exception& e_) {                                                    \
            ::doctest::detail::record(false, __FILE__, __LINE__,                                \
                                      (std::string(#expr " threw ") + e_.what()).c_str(), req); \
            break;                                                                              \
        }                                                                                       \
        ::doctest::detail::record(ok_, __FILE__, __LINE__, #expr, req);                         \
    } while (0)
#define CHECK(...) DOCTEST_ASSERT_((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_ASSERT_((__VA_ARGS__), true)

#define CHECK_THROWS_AS(expr, T)                                                              \
    do {                                                                                      \
        bool ok_ = false;                                                                     \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (const T&) {                                                                  \
            ok_ = true;                                                                       \
        } catch (...) {                                                                       \
        }                                                                                     \
        ::doctest::detail::record(ok_, __FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #T ")", false); \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, T)                                                   \
    do {                                                                                      \
        bool ok_ = false;                                                                     \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (const T& e_) {                                                               \
            ok_ = (with).check(e_.what());                                                    \
        } catch (...) {                                                                       \
        }                                                                                     \
        ::doctest::detail::record(ok_, __FILE__, __LINE__, "CHECK_THROWS_WITH_AS(" #expr ")", false); \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                   \
    do {                                                                                      \
        bool ok_ = true;                                                                      \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (...) {                                                                       \
            ok_ = false;                                                                      \
        }                                                                                     \
        ::doctest::detail::record(ok_, __FILE__, __LINE__, "CHECK_NOTHROW(" #expr ")", false); \
    } while (0)
#define INFO(...) ::doctest::detail::InfoScope DOCTEST_CAT(doctest_info_, __LINE__)(__VA_ARGS__)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    std::vector<std::string> only;
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "-tc=", 4) == 0) {
            std::string s = argv[i] + 4;
            for (size_t p = 0; p <= s.size();) {
                size_t q = s.find(',', p);
                if (q == std::string::npos) q = s.size();
                only.push_back(s.substr(p, q - p));
                p = q + 1;
            }
        }
    int n_fail = 0, n_run = 0;
    for (const auto& c : ::doctest::detail::registry()) {
        if (!only.empty()) {
            bool hit = false;
            for (const auto& o : only) hit |= o == c.name;
            if (!hit) continue;
        }
        auto& s = ::doctest::detail::state();
        s = {};
        ++n_run;
        try {
            c.fn();
        } catch (const ::doctest::detail::RequireAbort&) {
        } catch (const std::exception& e) {
            ++s.failed;
            s.msgs.push_back(std::string("unexpected exception: ") + e.what());
        } catch (...) {
            ++s.failed;
            s.msgs.push_back("unexpected exception");
        }
        std::printf("CASE %s %ld %ld %s\n", s.failed ? "FAIL" : "PASS", s.asserts, s.failed, c.name);
        for (const auto& [site, n] : s.sites) std::printf("    FAILED_AT %s x%ld\n", site.c_str(), n);
        for (const auto& m : s.msgs) std::printf("    %s\n", m.c_str());
        std::fflush(stdout);
        n_fail += s.failed ? 1 : 0;
    }
    std::printf("[doctest-shim] %d test cases, %d failed\n", n_run, n_fail);
    return n_fail ? 1 : 0;
}
#endif
