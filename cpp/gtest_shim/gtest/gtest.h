// Minimal GoogleTest-compatible harness (no gtest in this image). Covers the
// macro subset the reference's solver/grid/geometry suites use so those
// suites compile unmodified against the drop-in headers in include/porediff.
// Semantics follow gtest: EXPECT_* records and continues, ASSERT_* records
// and returns from the test body, EXPECT_DOUBLE_EQ is "within 4 ULPs".
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <filesystem>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <type_traits>
#include <vector>

namespace testing {

namespace internal {

struct Case {
    std::string suite, name;
    std::function<void()> body;
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct State {
    bool failed = false;
    bool fatal = false;
};
inline State& state() {
    static State s;
    return s;
}

struct Message {
    std::ostringstream os;
    template <class V>
    Message& operator<<(const V& v) {
        os << v;
        return *this;
    }
};

struct Failure {
    const char* file;
    int line;
    bool fatal;
    std::string text;
    void operator=(const Message& m) const {
        state().failed = true;
        state().fatal = state().fatal || fatal;
        std::printf("%s:%d: Failure\n  %s\n", file, line, text.c_str());
        const std::string extra = m.os.str();
        if (!extra.empty()) std::printf("  %s\n", extra.c_str());
    }
};

struct Registrar {
    Registrar(const char* s, const char* n, void (*f)()) { registry().push_back({s, n, f}); }
};

template <class V>
void print(std::ostream& os, const V& v) {
    if constexpr (requires { os << v; })
        os << v;
    else
        os << "<" << sizeof(V) << "-byte value>";
}

template <class A, class B>
std::string show(const char* ea, const char* eb, const A& a, const B& b) {
    std::ostringstream os;
    os.precision(17);
    os << ea << " vs " << eb << " (";
    print(os, a);
    os << " vs ";
    print(os, b);
    os << ")";
    return os.str();
}

template <class F>
bool ulps_equal(F a, F b) {
    if (std::isnan(a) || std::isnan(b)) return false;
    using U = std::conditional_t<sizeof(F) == 8, std::uint64_t, std::uint32_t>;
    auto biased = [](F v) {
        U bits;
        std::memcpy(&bits, &v, sizeof bits);
        const U sign = U{1} << (sizeof(U) * 8 - 1);
        return (bits & sign) ? ~bits + 1 : (bits | sign);
    };
    const U x = biased(a), y = biased(b);
    return (x >= y ? x - y : y - x) <= 4;
}

inline bool match_filter(const std::string& full, const std::string& filter) {
    if (filter.empty() || filter == "*") return true;
    // '*'-glob over the whole "Suite.Name", ':'-separated alternatives
    std::size_t start = 0;
    while (start <= filter.size()) {
        const std::size_t end = std::min(filter.find(':', start), filter.size());
        const std::string pat = filter.substr(start, end - start);
        std::function<bool(std::size_t, std::size_t)> m = [&](std::size_t i, std::size_t j) -> bool {
            if (j == pat.size()) return i == full.size();
            if (pat[j] == '*') return m(i, j + 1) || (i < full.size() && m(i + 1, j));
            return i < full.size() && (pat[j] == '?' || pat[j] == full[i]) && m(i + 1, j + 1);
        };
        if (m(0, 0)) return true;
        start = end + 1;
    }
    return false;
}

}  // namespace internal

struct Test {
    static bool HasFailure() { return internal::state().failed; }
    static bool HasFatalFailure() { return internal::state().fatal; }
};

inline std::string TempDir() { return std::filesystem::temp_directory_path().string() + "/"; }

inline int RunAllTests(int argc, char** argv) {
    std::string filter;
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "--gtest_filter=", 15) == 0) filter = argv[i] + 15;
    int ran = 0, failed = 0;
    std::vector<std::string> failures;
    for (const auto& c : internal::registry()) {
        const std::string full = c.suite + "." + c.name;
        if (!internal::match_filter(full, filter)) continue;
        internal::state() = {};
        std::printf("[ RUN      ] %s\n", full.c_str());
        std::fflush(stdout);
        try {
            c.body();
        } catch (const std::exception& e) {
            std::printf("  uncaught exception: %s\n", e.what());
            internal::state().failed = true;
        } catch (...) {
            std::printf("  uncaught non-standard exception\n");
            internal::state().failed = true;
        }
        ++ran;
        if (internal::state().failed) {
            ++failed;
            failures.push_back(full);
            std::printf("[  FAILED  ] %s\n", full.c_str());
        } else {
            std::printf("[       OK ] %s\n", full.c_str());
        }
        std::fflush(stdout);
    }
    std::printf("[==========] %d tests ran.\n[  PASSED  ] %d tests.\n", ran, ran - failed);
    for (const auto& f : failures) std::printf("[  FAILED  ] %s\n", f.c_str());
    return failed == 0 && ran > 0 ? 0 : 1;
}

}  // namespace testing

#define TEST(suite, name)                                                                             \
    static void pdgt_##suite##_##name();                                                              \
    static const ::testing::internal::Registrar pdgt_reg_##suite##_##name(#suite, #name,             \
                                                                          &pdgt_##suite##_##name);   \
    static void pdgt_##suite##_##name()

#define PDGT_CHECK_(ok, fatal, text)                                                                  \
    if (ok) {                                                                                         \
    } else                                                                                            \
        ::testing::internal::Failure{__FILE__, __LINE__, fatal, text} = ::testing::internal::Message()
#define PDGT_ASSERT_(ok, text)                                                                        \
    if (ok) {                                                                                         \
    } else                                                                                            \
        return ::testing::internal::Failure{__FILE__, __LINE__, true, text} = ::testing::internal::Message()

#define PDGT_CMP_(a, b, op, chk)                                                                      \
    chk(((a)op(b)), ::testing::internal::show(#a, #b, (a), (b)) + " expected " #op)

#define PDGT_EXPECT_(ok, text) PDGT_CHECK_(ok, false, text)

#define EXPECT_TRUE(c) PDGT_EXPECT_(static_cast<bool>(c), "expected true: " #c)
#define EXPECT_FALSE(c) PDGT_EXPECT_(!static_cast<bool>(c), "expected false: " #c)
#define ASSERT_TRUE(c) PDGT_ASSERT_(static_cast<bool>(c), "expected true: " #c)
#define ASSERT_FALSE(c) PDGT_ASSERT_(!static_cast<bool>(c), "expected false: " #c)

#define EXPECT_EQ(a, b) PDGT_CMP_(a, b, ==, PDGT_EXPECT_)
#define EXPECT_NE(a, b) PDGT_CMP_(a, b, !=, PDGT_EXPECT_)
#define EXPECT_LT(a, b) PDGT_CMP_(a, b, <, PDGT_EXPECT_)
#define EXPECT_LE(a, b) PDGT_CMP_(a, b, <=, PDGT_EXPECT_)
#define EXPECT_GT(a, b) PDGT_CMP_(a, b, >, PDGT_EXPECT_)
#define EXPECT_GE(a, b) PDGT_CMP_(a, b, >=, PDGT_EXPECT_)
#define ASSERT_EQ(a, b) PDGT_CMP_(a, b, ==, PDGT_ASSERT_)
#define ASSERT_NE(a, b) PDGT_CMP_(a, b, !=, PDGT_ASSERT_)
#define ASSERT_LT(a, b) PDGT_CMP_(a, b, <, PDGT_ASSERT_)
#define ASSERT_LE(a, b) PDGT_CMP_(a, b, <=, PDGT_ASSERT_)
#define ASSERT_GT(a, b) PDGT_CMP_(a, b, >, PDGT_ASSERT_)
#define ASSERT_GE(a, b) PDGT_CMP_(a, b, >=, PDGT_ASSERT_)

#define EXPECT_NEAR(a, b, tol)                                                                        \
    PDGT_EXPECT_(std::fabs(static_cast<double>(a) - static_cast<double>(b)) <= (tol),                 \
                 ::testing::internal::show(#a, #b, (a), (b)) + " tol " #tol)
#define ASSERT_NEAR(a, b, tol)                                                                        \
    PDGT_ASSERT_(std::fabs(static_cast<double>(a) - static_cast<double>(b)) <= (tol),                 \
                 ::testing::internal::show(#a, #b, (a), (b)) + " tol " #tol)
#define EXPECT_DOUBLE_EQ(a, b)                                                                        \
    PDGT_EXPECT_(::testing::internal::ulps_equal<double>((a), (b)),                                   \
                 ::testing::internal::show(#a, #b, (a), (b)) + " (4 ulps)")
#define EXPECT_FLOAT_EQ(a, b)                                                                         \
    PDGT_EXPECT_(::testing::internal::ulps_equal<float>((a), (b)),                                    \
                 ::testing::internal::show(#a, #b, (a), (b)) + " (4 ulps)")

#define PDGT_THROWS_(stmt, ex, chk)                                                                   \
    chk(([&]() -> bool {                                                                              \
            try {                                                                                     \
                stmt;                                                                                 \
            } catch (const ex&) {                                                                     \
                return true;                                                                          \
            } catch (...) {                                                                           \
                return false;                                                                         \
            }                                                                                         \
            return false;                                                                             \
        }()),                                                                                         \
        "expected " #stmt " to throw " #ex)
#define EXPECT_THROW(stmt, ex) PDGT_THROWS_(stmt, ex, PDGT_EXPECT_)
#define ASSERT_THROW(stmt, ex) PDGT_THROWS_(stmt, ex, PDGT_ASSERT_)
#define EXPECT_NO_THROW(stmt)                                                                         \
    PDGT_EXPECT_(([&]() -> bool {                                                                     \
                     try {                                                                            \
                         stmt;                                                                        \
                     } catch (...) {                                                                  \
                         return false;                                                                \
                     }                                                                                \
                     return true;                                                                     \
                 }()),                                                                                \
                 "expected " #stmt " not to throw")

#define FAIL() return ::testing::internal::Failure{__FILE__, __LINE__, true, "FAIL()"} = ::testing::internal::Message()
#define ADD_FAILURE() ::testing::internal::Failure{__FILE__, __LINE__, false, "ADD_FAILURE()"} = ::testing::internal::Message()
#define SUCCEED() static_cast<void>(0)
