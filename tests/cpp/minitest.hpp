// Minimal GTest-compatible shim (GTest is not installed): TEST,
// EXPECT_*/ASSERT_* with the same names so the ported cases read like the
// reference's proj/tests/test_kernels.cpp.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace minitest {
struct Case {
    const char* suite;
    const char* name;
    std::function<void()> fn;
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
inline int& failures() {
    static int f = 0;
    return f;
}
struct Reg {
    Reg(const char* s, const char* n, std::function<void()> f) { registry().push_back({s, n, std::move(f)}); }
};
struct Abort {};
inline int run_all() {
    int failed_cases = 0;
    for (auto& c : registry()) {
        const int before = failures();
        try {
            c.fn();
        } catch (const Abort&) {
        } catch (const std::exception& e) {
            std::printf("  exception: %s\n", e.what());
            ++failures();
        }
        const bool ok = failures() == before;
        if (!ok) ++failed_cases;
        std::printf("[%s] %s.%s\n", ok ? "  OK  " : "FAILED", c.suite, c.name);
    }
    std::printf("%zu cases, %d failed\n", registry().size(), failed_cases);
    return failed_cases ? 1 : 0;
}
}  // namespace minitest

#define TEST(s, n)                                                  \
    static void s##_##n();                                          \
    static minitest::Reg s##_##n##_reg(#s, #n, s##_##n);            \
    static void s##_##n()
#define MT_FAIL(msg)                                                                 \
    do {                                                                             \
        std::printf("  %s:%d: %s\n", __FILE__, __LINE__, std::string(msg).c_str()); \
        ++minitest::failures();                                                      \
    } while (0)
#define EXPECT_TRUE(c) do { if (!(c)) MT_FAIL("EXPECT_TRUE(" #c ")"); } while (0)
#define ASSERT_TRUE(c) do { if (!(c)) { MT_FAIL("ASSERT_TRUE(" #c ")"); throw minitest::Abort{}; } } while (0)
#define EXPECT_EQ(a, b) do { if (!((a) == (b))) MT_FAIL("EXPECT_EQ(" #a ", " #b ")"); } while (0)
#define ASSERT_EQ(a, b) do { if (!((a) == (b))) { MT_FAIL("ASSERT_EQ(" #a ", " #b ")"); throw minitest::Abort{}; } } while (0)
#define EXPECT_DOUBLE_EQ(a, b) EXPECT_TRUE(std::abs((a) - (b)) <= 4 * 2.2e-16 * std::max(std::abs(a), std::abs(b)))
#define EXPECT_NEAR(a, b, tol) do { if (!(std::abs((a) - (b)) <= (tol))) MT_FAIL("EXPECT_NEAR(" #a ", " #b ", " #tol ") got " + std::to_string(a) + " vs " + std::to_string(b)); } while (0)
#define EXPECT_LT(a, b) do { if (!((a) < (b))) MT_FAIL("EXPECT_LT(" #a ", " #b ") got " + std::to_string(a) + " vs " + std::to_string(b)); } while (0)
#define EXPECT_LE(a, b) do { if (!((a) <= (b))) MT_FAIL("EXPECT_LE(" #a ", " #b ") got " + std::to_string(a) + " vs " + std::to_string(b)); } while (0)
#define EXPECT_GE(a, b) do { if (!((a) >= (b))) MT_FAIL("EXPECT_GE(" #a ", " #b ")"); } while (0)
#define EXPECT_THROW(stmt, ex) do { bool t_ = false; try { stmt; } catch (const ex&) { t_ = true; } catch (...) {} if (!t_) MT_FAIL("EXPECT_THROW(" #stmt ", " #ex ")"); } while (0)
