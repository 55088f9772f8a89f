// Minimal GoogleTest-compatible shim (GoogleTest is not installable here) so
// the reference's own test suites (/root/reference/proj/tests/*_test.cpp)
// compile unchanged — against the reference headers and against the GPU
// drop-in (include/ppf_dropin). Supports the macros those suites use:
// TEST, EXPECT_/ASSERT_{TRUE,FALSE,EQ,NE,LT,LE,GT,GE}, EXPECT_NEAR,
// EXPECT_DOUBLE_EQ, EXPECT_THROW, EXPECT_NO_THROW, FAIL(), GTEST_SKIP(), with
// `<< message` streaming. main() runs every registered test; argv filters:
// a leading '-' excludes "Suite.Name" substrings, anything else includes.
#pragma once

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <limits>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace gshim {

struct Case {
    const char* suite;
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(const char* s, const char* n, void (*f)()) { registry().push_back({s, n, f}); }
};
inline int& current_failures() {
    static int n = 0;
    return n;
}
inline bool& current_skipped() {
    static bool s = false;
    return s;
}

template <class T, class = void>
struct printable : std::false_type {};
template <class T>
struct printable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};
template <class T>
std::string show(const T& v) {
    if constexpr (printable<T>::value) {
        std::ostringstream o;
        o.precision(17);
        o << v;
        return o.str();
    } else {
        return "<value>";
    }
}

struct Msg {
    std::ostringstream os;
    template <class T>
    Msg& operator<<(const T& v) {
        os << v;
        return *this;
    }
};

struct Sink {
    const char* file;
    int line;
    std::string what;
    void operator=(const Msg& m) const {
        ++current_failures();
        std::cout << file << ":" << line << ": Failure\n  " << what;
        const std::string extra = m.os.str();
        if (!extra.empty())
            std::cout << "\n  " << extra;
        std::cout << "\n";
    }
};
struct Skip {
    void operator=(const Msg& m) const {
        current_skipped() = true;
        std::cout << "  skipped: " << m.os.str() << "\n";
    }
};

template <class A, class B>
std::string binmsg(const char* ea, const char* op, const char* eb, const A& a, const B& b) {
    return std::string("Expected: ") + ea + " " + op + " " + eb + "\n  actual: " + show(a) + " vs " +
           show(b);
}

#if defined(__GNUC__)
#pragma GCC diagnostic push
#pragma GCC diagnostic ignored "-Wsign-compare"
#endif
template <class A, class B> bool eq(const A& a, const B& b) { return a == b; }
template <class A, class B> bool ne(const A& a, const B& b) { return a != b; }
template <class A, class B> bool lt(const A& a, const B& b) { return a < b; }
template <class A, class B> bool le(const A& a, const B& b) { return a <= b; }
template <class A, class B> bool gt(const A& a, const B& b) { return a > b; }
template <class A, class B> bool ge(const A& a, const B& b) { return a >= b; }
#if defined(__GNUC__)
#pragma GCC diagnostic pop
#endif

inline bool near(double a, double b, double tol) { return std::fabs(a - b) <= tol; }
inline bool double_eq(double a, double b) {
    if (a == b)
        return true;
    return std::fabs(a - b) <= 4 * std::numeric_limits<double>::epsilon() *
                                   std::max(std::fabs(a), std::fabs(b));
}

template <class E, class F>
bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}
template <class F>
bool no_throw(F&& f) {
    try {
        f();
    } catch (...) {
        return false;
    }
    return true;
}

inline int run_all(int argc, char** argv) {
    int failed = 0, passed = 0, skipped = 0;
    for (const auto& c : registry()) {
        const std::string full = std::string(c.suite) + "." + c.name;
        bool take = true;
        bool any_include = false;
        for (int i = 1; i < argc; ++i) {
            const char* a = argv[i];
            if (a[0] == '-') {
                if (full.find(a + 1) != std::string::npos)
                    take = false;
            } else {
                any_include = true;
            }
        }
        if (any_include) {
            bool hit = false;
            for (int i = 1; i < argc; ++i)
                if (argv[i][0] != '-' && full.find(argv[i]) != std::string::npos)
                    hit = true;
            take = take && hit;
        }
        if (!take)
            continue;
        current_failures() = 0;
        current_skipped() = false;
        std::cout << "[ RUN      ] " << full << "\n" << std::flush;
        try {
            c.fn();
        } catch (const std::exception& e) {
            ++current_failures();
            std::cout << "  uncaught exception: " << e.what() << "\n";
        } catch (...) {
            ++current_failures();
            std::cout << "  uncaught non-std exception\n";
        }
        if (current_skipped()) {
            ++skipped;
            std::cout << "[  SKIPPED ] " << full << "\n";
        } else if (current_failures()) {
            ++failed;
            std::cout << "[  FAILED  ] " << full << "\n";
        } else {
            ++passed;
            std::cout << "[       OK ] " << full << "\n";
        }
    }
    std::cout << "[==========] " << passed << " passed, " << failed << " failed, " << skipped
              << " skipped\n";
    return failed ? 1 : 0;
}

} // namespace gshim

namespace testing {
inline void InitGoogleTest(int*, char**) {}
} // namespace testing

#define TEST(suite, name)                                                                         \
    static void gshim_##suite##_##name();                                                         \
    static ::gshim::Registrar gshim_reg_##suite##_##name(#suite, #name, &gshim_##suite##_##name); \
    static void gshim_##suite##_##name()

#define GSHIM_FAIL_AT(what) ::gshim::Sink{__FILE__, __LINE__, (what)} = ::gshim::Msg()

#define GSHIM_BIN(fn, op, a, b, on_fail)                                                          \
    if (::gshim::fn((a), (b)))                                                                    \
        ;                                                                                         \
    else                                                                                          \
        on_fail GSHIM_FAIL_AT(::gshim::binmsg(#a, op, #b, (a), (b)))

#define EXPECT_EQ(a, b) GSHIM_BIN(eq, "==", a, b, )
#define EXPECT_NE(a, b) GSHIM_BIN(ne, "!=", a, b, )
#define EXPECT_LT(a, b) GSHIM_BIN(lt, "<", a, b, )
#define EXPECT_LE(a, b) GSHIM_BIN(le, "<=", a, b, )
#define EXPECT_GT(a, b) GSHIM_BIN(gt, ">", a, b, )
#define EXPECT_GE(a, b) GSHIM_BIN(ge, ">=", a, b, )
#define ASSERT_EQ(a, b) GSHIM_BIN(eq, "==", a, b, return)
#define ASSERT_NE(a, b) GSHIM_BIN(ne, "!=", a, b, return)
#define ASSERT_LT(a, b) GSHIM_BIN(lt, "<", a, b, return)
#define ASSERT_LE(a, b) GSHIM_BIN(le, "<=", a, b, return)
#define ASSERT_GT(a, b) GSHIM_BIN(gt, ">", a, b, return)
#define ASSERT_GE(a, b) GSHIM_BIN(ge, ">=", a, b, return)

#define EXPECT_TRUE(c)                                                                            \
    if (static_cast<bool>(c))                                                                     \
        ;                                                                                         \
    else                                                                                          \
        GSHIM_FAIL_AT(std::string("Expected true: ") + #c)
#define EXPECT_FALSE(c)                                                                           \
    if (!static_cast<bool>(c))                                                                    \
        ;                                                                                         \
    else                                                                                          \
        GSHIM_FAIL_AT(std::string("Expected false: ") + #c)
#define ASSERT_TRUE(c)                                                                            \
    if (static_cast<bool>(c))                                                                     \
        ;                                                                                         \
    else                                                                                          \
        return GSHIM_FAIL_AT(std::string("Expected true: ") + #c)
#define ASSERT_FALSE(c)                                                                           \
    if (!static_cast<bool>(c))                                                                    \
        ;                                                                                         \
    else                                                                                          \
        return GSHIM_FAIL_AT(std::string("Expected false: ") + #c)

#define EXPECT_NEAR(a, b, tol)                                                                    \
    if (::gshim::near((a), (b), (tol)))                                                           \
        ;                                                                                         \
    else                                                                                          \
        GSHIM_FAIL_AT(::gshim::binmsg(#a, "~=", #b, (a), (b)))
#define EXPECT_DOUBLE_EQ(a, b)                                                                    \
    if (::gshim::double_eq((a), (b)))                                                             \
        ;                                                                                         \
    else                                                                                          \
        GSHIM_FAIL_AT(::gshim::binmsg(#a, "==(double)", #b, (a), (b)))
#define EXPECT_THROW(stmt, exc)                                                                   \
    if (::gshim::throws<exc>([&]() { stmt; }))                                                    \
        ;                                                                                         \
    else                                                                                          \
        GSHIM_FAIL_AT(std::string("Expected ") + #stmt + " to throw " + #exc)
#define EXPECT_NO_THROW(stmt)                                                                     \
    if (::gshim::no_throw([&]() { stmt; }))                                                       \
        ;                                                                                         \
    else                                                                                          \
        GSHIM_FAIL_AT(std::string("Expected no throw: ") + #stmt)
#define FAIL() return GSHIM_FAIL_AT("FAIL()")
#define GTEST_SKIP() return ::gshim::Skip() = ::gshim::Msg()

#ifndef GSHIM_NO_MAIN
int main(int argc, char** argv) { return ::gshim::run_all(argc, argv); }
#endif
