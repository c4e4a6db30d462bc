// gtest_shim — the subset of GoogleTest's API the reference's hot-path suites use
// (proj/tests/test_*.cpp: TEST, TEST_F, EXPECT_/ASSERT_ {EQ, NE, LT, LE, GT, GE, TRUE,
// FALSE, DOUBLE_EQ, NEAR, THROW, NO_THROW}, FAIL, ADD_FAILURE, SUCCEED, testing::Test,
// testing::TempDir, testing::UnitTest current_test_info). GoogleTest itself is not in
// this image and there is no network, so the reference suites are compiled UNCHANGED
// against include/ (the B200 headers) with this header on the include path instead.
// Test infrastructure only. main() is in gtest_main.cpp.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace testing {

class Test {
public:
    virtual ~Test() = default;
    virtual void SetUp() {}
    virtual void TearDown() {}
    virtual void TestBody() = 0;
};

struct TestInfo {
    std::string suite, test;
    const char* name() const { return test.c_str(); }
    const char* test_suite_name() const { return suite.c_str(); }
};

class UnitTest {
public:
    static UnitTest* GetInstance() {
        static UnitTest u;
        return &u;
    }
    const TestInfo* current_test_info() const { return &current; }
    TestInfo current;
};

inline std::string TempDir() { return "/tmp/"; }

}  // namespace testing

namespace gshim {

struct State {
    int failures = 0;       // failures in the current test
    bool fatal = false;     // an ASSERT_* failed in the current test
};
inline State& state() {
    static State s;
    return s;
}

struct Msg {
    std::ostringstream os;
    Msg() = default;
    Msg(const Msg& o) { os << o.os.str(); }
    template <class T>
    Msg& operator<<(const T& v) {
        os << v;
        return *this;
    }
};

struct Reporter {
    const char* file;
    int line;
    std::string text;
    bool fatal;
    Reporter(const char* f, int l, std::string t, bool fa) : file(f), line(l), text(std::move(t)), fatal(fa) {}
    void operator=(const Msg& m) const {
        ++state().failures;
        if (fatal) state().fatal = true;
        const std::string extra = m.os.str();
        std::fprintf(stderr, "%s:%d: Failure\n%s%s%s\n", file, line, text.c_str(),
                     extra.empty() ? "" : "\n", extra.c_str());
    }
};

struct Result {
    bool ok;
    std::string msg;
    explicit operator bool() const { return ok; }
};

template <class T, class = void>
struct Printable : std::false_type {};
template <class T>
struct Printable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};

template <class T>
std::string show(const T& v) {
    if constexpr (std::is_enum_v<T>) {
        return std::to_string(static_cast<long long>(v));
    } else if constexpr (Printable<T>::value) {
        std::ostringstream os;
        os.precision(17);
        os << v;
        return os.str();
    } else {
        return "<" + std::to_string(sizeof(T)) + "-byte object>";
    }
}
inline std::string show(std::nullptr_t) { return "nullptr"; }

template <class A, class B, class Op>
Result cmp(const char* ea, const char* eb, const A& a, const B& b, Op op, const char* opname) {
    if (op(a, b)) return {true, {}};
    return {false, std::string("Expected: (") + ea + ") " + opname + " (" + eb + "), actual: " +
                       show(a) + " vs " + show(b)};
}

inline Result boolean(bool v, const char* expr, bool want) {
    if (v == want) return {true, {}};
    return {false, std::string("Value of: ") + expr + "\n  Actual: " + (v ? "true" : "false") +
                       "\nExpected: " + (want ? "true" : "false")};
}

inline bool almost_equal(double a, double b) {  // GoogleTest: within 4 ULPs
    if (std::isnan(a) || std::isnan(b)) return false;
    if (a == b) return true;
    auto key = [](double x) {
        int64_t i;
        std::memcpy(&i, &x, sizeof i);
        return i < 0 ? int64_t(uint64_t(1) << 63) - i : i + int64_t(0);
    };
    const int64_t ka = key(a), kb = key(b);
    const uint64_t d = ka > kb ? uint64_t(ka) - uint64_t(kb) : uint64_t(kb) - uint64_t(ka);
    return d <= 4;
}

inline Result near(const char* ea, const char* eb, double a, double b, double tol) {
    if (std::fabs(a - b) <= tol) return {true, {}};
    return {false, std::string("The difference between ") + ea + " and " + eb + " is " +
                       show(std::fabs(a - b)) + ", which exceeds " + show(tol)};
}

template <class E, class F>
Result throws(F&& f, const char* stmt, const char* ename) {
    try {
        f();
    } catch (const E&) {
        return {true, {}};
    } catch (const std::exception& ex) {
        return {false, std::string("Expected: ") + stmt + " throws an exception of type " + ename +
                           ".\n  Actual: it throws a different type (" + ex.what() + ")."};
    } catch (...) {
        return {false, std::string("Expected: ") + stmt + " throws an exception of type " + ename +
                           ".\n  Actual: it throws a different type."};
    }
    return {false, std::string("Expected: ") + stmt + " throws an exception of type " + ename +
                       ".\n  Actual: it throws nothing."};
}

template <class F>
Result nothrow(F&& f, const char* stmt) {
    try {
        f();
    } catch (const std::exception& ex) {
        return {false, std::string("Expected: ") + stmt + " doesn't throw an exception.\n  Actual: it throws " + ex.what()};
    } catch (...) {
        return {false, std::string("Expected: ") + stmt + " doesn't throw an exception.\n  Actual: it throws."};
    }
    return {true, {}};
}

struct Entry {
    std::string suite, name;
    std::function<testing::Test*()> make;
};
inline std::vector<Entry>& registry() {
    static std::vector<Entry> r;
    return r;
}
struct Registrar {
    Registrar(const char* s, const char* n, std::function<testing::Test*()> f) {
        registry().push_back({s, n, std::move(f)});
    }
};

int run_all(int argc, char** argv);

}  // namespace gshim

#define GSHIM_REPORT_(text, fatal) ::gshim::Reporter(__FILE__, __LINE__, (text), (fatal)) = ::gshim::Msg()
#define GSHIM_NONFATAL_(expr) \
    switch (0) case 0: default: \
    if (const ::gshim::Result gshim_r_ = (expr)) ; else GSHIM_REPORT_(gshim_r_.msg, false)
#define GSHIM_FATAL_(expr) \
    switch (0) case 0: default: \
    if (const ::gshim::Result gshim_r_ = (expr)) ; else return GSHIM_REPORT_(gshim_r_.msg, true)

#define GSHIM_OP_(a, b, op, name) ::gshim::cmp(#a, #b, (a), (b), [](const auto& x, const auto& y) { return x op y; }, name)

#define EXPECT_EQ(a, b) GSHIM_NONFATAL_(GSHIM_OP_(a, b, ==, "=="))
#define EXPECT_NE(a, b) GSHIM_NONFATAL_(GSHIM_OP_(a, b, !=, "!="))
#define EXPECT_LT(a, b) GSHIM_NONFATAL_(GSHIM_OP_(a, b, <, "<"))
#define EXPECT_LE(a, b) GSHIM_NONFATAL_(GSHIM_OP_(a, b, <=, "<="))
#define EXPECT_GT(a, b) GSHIM_NONFATAL_(GSHIM_OP_(a, b, >, ">"))
#define EXPECT_GE(a, b) GSHIM_NONFATAL_(GSHIM_OP_(a, b, >=, ">="))
#define ASSERT_EQ(a, b) GSHIM_FATAL_(GSHIM_OP_(a, b, ==, "=="))
#define ASSERT_NE(a, b) GSHIM_FATAL_(GSHIM_OP_(a, b, !=, "!="))
#define ASSERT_LT(a, b) GSHIM_FATAL_(GSHIM_OP_(a, b, <, "<"))
#define ASSERT_LE(a, b) GSHIM_FATAL_(GSHIM_OP_(a, b, <=, "<="))
#define ASSERT_GT(a, b) GSHIM_FATAL_(GSHIM_OP_(a, b, >, ">"))
#define ASSERT_GE(a, b) GSHIM_FATAL_(GSHIM_OP_(a, b, >=, ">="))
#define EXPECT_TRUE(c) GSHIM_NONFATAL_(::gshim::boolean(static_cast<bool>(c), #c, true))
#define EXPECT_FALSE(c) GSHIM_NONFATAL_(::gshim::boolean(static_cast<bool>(c), #c, false))
#define ASSERT_TRUE(c) GSHIM_FATAL_(::gshim::boolean(static_cast<bool>(c), #c, true))
#define ASSERT_FALSE(c) GSHIM_FATAL_(::gshim::boolean(static_cast<bool>(c), #c, false))
#define EXPECT_DOUBLE_EQ(a, b) \
    GSHIM_NONFATAL_(::gshim::cmp(#a, #b, double(a), double(b), [](double x, double y) { return ::gshim::almost_equal(x, y); }, "~="))
#define ASSERT_DOUBLE_EQ(a, b) \
    GSHIM_FATAL_(::gshim::cmp(#a, #b, double(a), double(b), [](double x, double y) { return ::gshim::almost_equal(x, y); }, "~="))
#define EXPECT_NEAR(a, b, t) GSHIM_NONFATAL_(::gshim::near(#a, #b, double(a), double(b), double(t)))
#define ASSERT_NEAR(a, b, t) GSHIM_FATAL_(::gshim::near(#a, #b, double(a), double(b), double(t)))
#define EXPECT_THROW(stmt, E) GSHIM_NONFATAL_(::gshim::throws<E>([&]() { stmt; }, #stmt, #E))
#define ASSERT_THROW(stmt, E) GSHIM_FATAL_(::gshim::throws<E>([&]() { stmt; }, #stmt, #E))
#define EXPECT_NO_THROW(stmt) GSHIM_NONFATAL_(::gshim::nothrow([&]() { stmt; }, #stmt))
#define ASSERT_NO_THROW(stmt) GSHIM_FATAL_(::gshim::nothrow([&]() { stmt; }, #stmt))
#define ADD_FAILURE() GSHIM_REPORT_("Failed", false)
#define FAIL() return GSHIM_REPORT_("Failed", true)
#define SUCCEED() static_cast<void>(0)

#define GSHIM_TEST_(suite, name, base)                                                   \
    class suite##_##name##_Test : public base {                                          \
    public:                                                                              \
        void TestBody() override;                                                        \
    };                                                                                   \
    static ::gshim::Registrar suite##_##name##_registrar(                                \
        #suite, #name, []() -> ::testing::Test* { return new suite##_##name##_Test; }); \
    void suite##_##name##_Test::TestBody()

#define TEST(suite, name) GSHIM_TEST_(suite, name, ::testing::Test)
#define TEST_F(fixture, name) GSHIM_TEST_(fixture, name, fixture)

#define RUN_ALL_TESTS() ::gshim::run_all(0, nullptr)
