// Minimal GoogleTest-compatible shim (GTest is not installed in this image).
// Enough of the macro surface for the reference's proj/tests/*.cpp to compile
// unmodified: TEST, EXPECT_/ASSERT_{EQ,NE,LT,LE,GT,GE,NEAR,TRUE,FALSE,THROW,
// NO_THROW}, FAIL, streamed messages.  main() lives in gtest_main.cpp.
#pragma once
#include <cmath>
#include <exception>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace testing {

struct TestInfo {
    const char* suite;
    const char* name;
    std::function<void()> body;
};

inline std::vector<TestInfo>& registry() {
    static std::vector<TestInfo> r;
    return r;
}

struct Registrar {
    Registrar(const char* s, const char* n, std::function<void()> f) { registry().push_back({s, n, std::move(f)}); }
};

inline int& failures() {
    static int f = 0;
    return f;
}

struct AssertFatal {};

// Collects the streamed message; reports on destruction.
class Reporter {
public:
    Reporter(bool fatal, const char* file, int line, std::string what)
        : fatal_(fatal), file_(file), line_(line), what_(std::move(what)) {}
    template <typename V>
    Reporter& operator<<(const V& v) {
        msg_ << v;
        return *this;
    }
    ~Reporter() noexcept(false) {
        ++failures();
        std::cerr << file_ << ":" << line_ << ": Failure\n  " << what_;
        const std::string m = msg_.str();
        if (!m.empty()) std::cerr << "\n  " << m;
        std::cerr << "\n";
        if (fatal_ && std::uncaught_exceptions() == 0) throw AssertFatal{};
    }

private:
    bool fatal_;
    const char* file_;
    int line_;
    std::string what_;
    std::ostringstream msg_;
};

template <typename A, typename B>
std::string describe(const char* op, const char* ea, const char* eb, const A& a, const B& b) {
    std::ostringstream o;
    o << "Expected: (" << ea << ") " << op << " (" << eb << "), actual: " << a << " vs " << b;
    return o.str();
}

inline int RunAllTests() {
    int failed_tests = 0;
    for (auto& t : registry()) {
        const int before = failures();
        std::cout << "[ RUN      ] " << t.suite << "." << t.name << std::endl;
        try {
            t.body();
        } catch (const AssertFatal&) {
        } catch (const std::exception& e) {
            ++failures();
            std::cerr << "  uncaught exception: " << e.what() << "\n";
        }
        const bool ok = failures() == before;
        if (!ok) ++failed_tests;
        std::cout << (ok ? "[       OK ] " : "[  FAILED  ] ") << t.suite << "." << t.name << std::endl;
    }
    std::cout << "[==========] " << registry().size() << " tests, " << failed_tests << " failed" << std::endl;
    return failed_tests == 0 ? 0 : 1;
}

inline void InitGoogleTest(int*, char**) {}

}  // namespace testing

#define GTS_CAT_(a, b) a##b
#define GTS_CAT(a, b) GTS_CAT_(a, b)
#define TEST(suite, name)                                                                          \
    static void GTS_CAT(gts_body_, GTS_CAT(suite, GTS_CAT(_, name)))();                            \
    static ::testing::Registrar GTS_CAT(gts_reg_, GTS_CAT(suite, GTS_CAT(_, name)))(              \
        #suite, #name, &GTS_CAT(gts_body_, GTS_CAT(suite, GTS_CAT(_, name))));                     \
    static void GTS_CAT(gts_body_, GTS_CAT(suite, GTS_CAT(_, name)))()

// switch(0) case 0: default: keeps a caller's trailing `else` unambiguous (as GTest does)
#define GTS_CMP(fatal, op, a, b)                                                                   \
    switch (0)                                                                                     \
    case 0:                                                                                        \
    default:                                                                                       \
        if (const auto& gts_a = (a); false) {                                                      \
        } else if (const auto& gts_b = (b); gts_a op gts_b) {                                      \
        } else                                                                                     \
            ::testing::Reporter(fatal, __FILE__, __LINE__,                                          \
                                ::testing::describe(#op, #a, #b, gts_a, gts_b))

#define EXPECT_EQ(a, b) GTS_CMP(false, ==, a, b)
#define EXPECT_NE(a, b) GTS_CMP(false, !=, a, b)
#define EXPECT_LT(a, b) GTS_CMP(false, <, a, b)
#define EXPECT_LE(a, b) GTS_CMP(false, <=, a, b)
#define EXPECT_GT(a, b) GTS_CMP(false, >, a, b)
#define EXPECT_GE(a, b) GTS_CMP(false, >=, a, b)
#define ASSERT_EQ(a, b) GTS_CMP(true, ==, a, b)
#define ASSERT_NE(a, b) GTS_CMP(true, !=, a, b)
#define ASSERT_LT(a, b) GTS_CMP(true, <, a, b)
#define ASSERT_LE(a, b) GTS_CMP(true, <=, a, b)
#define ASSERT_GT(a, b) GTS_CMP(true, >, a, b)
#define ASSERT_GE(a, b) GTS_CMP(true, >=, a, b)
#define EXPECT_DOUBLE_EQ(a, b) EXPECT_EQ(a, b)
#define ASSERT_DOUBLE_EQ(a, b) ASSERT_EQ(a, b)

#define GTS_NEAR(fatal, a, b, tol)                                                                 \
    switch (0)                                                                                     \
    case 0:                                                                                        \
    default:                                                                                       \
    if (const double gts_d = std::abs(static_cast<double>(a) - static_cast<double>(b));            \
        gts_d <= static_cast<double>(tol)) {                                                       \
    } else                                                                                         \
        ::testing::Reporter(fatal, __FILE__, __LINE__,                                              \
                            ::testing::describe("near", #a, #b, static_cast<double>(a),            \
                                                static_cast<double>(b)))                           \
            << "diff " << gts_d << " > tol " << (tol)
#define EXPECT_NEAR(a, b, tol) GTS_NEAR(false, a, b, tol)
#define ASSERT_NEAR(a, b, tol) GTS_NEAR(true, a, b, tol)

#define GTS_BOOL(fatal, c, want)                                                                   \
    switch (0)                                                                                     \
    case 0:                                                                                        \
    default:                                                                                       \
    if (static_cast<bool>(c) == want) {                                                            \
    } else                                                                                         \
        ::testing::Reporter(fatal, __FILE__, __LINE__, std::string("Value of: ") + #c)
#define EXPECT_TRUE(c) GTS_BOOL(false, c, true)
#define EXPECT_FALSE(c) GTS_BOOL(false, c, false)
#define ASSERT_TRUE(c) GTS_BOOL(true, c, true)
#define ASSERT_FALSE(c) GTS_BOOL(true, c, false)

#define GTS_THROW(fatal, stmt, exc)                                                                \
    switch (0)                                                                                     \
    case 0:                                                                                        \
    default:                                                                                       \
    if (bool gts_ok = [&] {                                                                        \
            try {                                                                                  \
                stmt;                                                                              \
            } catch (const exc&) {                                                                 \
                return true;                                                                       \
            } catch (...) {                                                                        \
            }                                                                                      \
            return false;                                                                          \
        }();                                                                                       \
        gts_ok) {                                                                                  \
    } else                                                                                         \
        ::testing::Reporter(fatal, __FILE__, __LINE__, std::string("Expected ") + #stmt +          \
                                                           " to throw " + #exc)
#define EXPECT_THROW(stmt, exc) GTS_THROW(false, stmt, exc)
#define ASSERT_THROW(stmt, exc) GTS_THROW(true, stmt, exc)
#define EXPECT_ANY_THROW(stmt) GTS_THROW(false, stmt, std::exception)

#define GTS_NOTHROW(fatal, stmt)                                                                   \
    switch (0)                                                                                     \
    case 0:                                                                                        \
    default:                                                                                       \
    if (bool gts_ok = [&] {                                                                        \
            try {                                                                                  \
                stmt;                                                                              \
            } catch (...) {                                                                        \
                return false;                                                                      \
            }                                                                                      \
            return true;                                                                           \
        }();                                                                                       \
        gts_ok) {                                                                                  \
    } else                                                                                         \
        ::testing::Reporter(fatal, __FILE__, __LINE__, std::string("Expected no throw: ") + #stmt)
#define EXPECT_NO_THROW(stmt) GTS_NOTHROW(false, stmt)
#define ASSERT_NO_THROW(stmt) GTS_NOTHROW(true, stmt)

#define FAIL() ::testing::Reporter(true, __FILE__, __LINE__, "Failed")
#define ADD_FAILURE() ::testing::Reporter(false, __FILE__, __LINE__, "Failed")
#define SUCCEED() \
    do {          \
    } while (0)
#define EXPECT_FLOAT_EQ(a, b) EXPECT_EQ(a, b)
#define ASSERT_FLOAT_EQ(a, b) ASSERT_EQ(a, b)
