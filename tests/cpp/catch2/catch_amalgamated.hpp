// Minimal Catch2-compatible test shim (our own, ~100 lines) so the reference's unit-test
// sources — and our own C++ tests written in the same style — compile and run against the
// drop-in headers without the Catch2 library.  Supports TEST_CASE, flat SECTIONs (each
// section runs in its own pass of the test case, as in Catch2), CHECK / CHECK_FALSE /
// REQUIRE / CHECK_NOTHROW / CHECK_THROWS_AS / REQUIRE_THROWS_AS and a relative Approx.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace shim {

struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct State {
    long checks = 0, failures = 0;
    int run_index = 0;      // which section this pass enters
    int seen = 0;           // sections met in this pass
    bool in_case_failed = false;
};
inline State& st() {
    static State s;
    return s;
}

struct RequireAbort {};

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
    ++st().checks;
    if (ok) return;
    ++st().failures;
    st().in_case_failed = true;
    std::printf("  FAILED %s:%d: %s\n", file, line, expr);
    if (fatal) throw RequireAbort{};
}

struct SectionGuard {
    bool enter;
    explicit SectionGuard(const char*) { enter = (st().seen++ == st().run_index); }
    explicit operator bool() const { return enter; }
};

class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    Approx& margin(double m) { margin_ = m; return *this; }
    friend bool operator==(double x, const Approx& a) {
        return std::fabs(x - a.v_) <= std::max(a.margin_, a.eps_ * (std::fabs(a.v_) + std::fabs(x)) * 0.5 + 1e-300);
    }
    friend bool operator==(const Approx& a, double x) { return x == a; }
    friend bool operator!=(double x, const Approx& a) { return !(x == a); }

private:
    double v_, eps_ = 1e-5 * 100, margin_ = 0.0;
};

inline int run_all(int argc, char** argv) {
    int cases = 0, failed_cases = 0;
    for (const Case& c : registry()) {
        if (argc > 1 && std::string(c.name).find(argv[1]) == std::string::npos) continue;
        ++cases;
        st().in_case_failed = false;
        for (st().run_index = 0;; ++st().run_index) {
            st().seen = 0;
            try {
                c.fn();
            } catch (const RequireAbort&) {
            } catch (const std::exception& e) {
                ++st().failures;
                st().in_case_failed = true;
                std::printf("  FAILED %s: unexpected exception: %s\n", c.name, e.what());
            }
            if (st().seen <= st().run_index + 1) break;
        }
        if (st().in_case_failed) {
            ++failed_cases;
            std::printf("test case FAILED: %s\n", c.name);
        }
    }
    std::printf("%d test cases, %d failed; %ld checks, %ld failures\n", cases, failed_cases, st().checks,
                st().failures);
    return failed_cases ? 1 : 0;
}

}  // namespace shim

namespace Catch { using shim::Approx; }
using shim::Approx;

#define SHIM_CAT2(a, b) a##b
#define SHIM_CAT(a, b) SHIM_CAT2(a, b)
#define TEST_CASE(name, ...)                                                          \
    static void SHIM_CAT(shim_case_, __LINE__)();                                    \
    static shim::Registrar SHIM_CAT(shim_reg_, __LINE__)(name, &SHIM_CAT(shim_case_, __LINE__)); \
    static void SHIM_CAT(shim_case_, __LINE__)()
#define SECTION(name) if (shim::SectionGuard SHIM_CAT(shim_sec_, __LINE__){name})
#define CHECK(...) shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define SHIM_THROWS(expr, type, fatal)                                                 \
    do {                                                                              \
        bool shim_ok = false;                                                         \
        try { (void)(expr); } catch (const type&) { shim_ok = true; } catch (...) {}  \
        shim::report(shim_ok, #expr " throws " #type, __FILE__, __LINE__, fatal);     \
    } while (0)
#define CHECK_THROWS_AS(expr, type) SHIM_THROWS(expr, type, false)
#define REQUIRE_THROWS_AS(expr, type) SHIM_THROWS(expr, type, true)
#define CHECK_NOTHROW(expr)                                                           \
    do {                                                                              \
        bool shim_ok = true;                                                          \
        try { (void)(expr); } catch (...) { shim_ok = false; }                        \
        shim::report(shim_ok, #expr " does not throw", __FILE__, __LINE__, false);     \
    } while (0)
