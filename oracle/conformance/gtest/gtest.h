// Minimal GoogleTest-compatible shim (own code) so the reference's unit tests
// can be compiled unchanged against the drop-in headers (include/cpd) and
// run on the B200 box.  Test infrastructure only: the reference's tests need
// GTest, which is not in this image.
//
// Supports what the reference's hot-path tests use: TEST, EXPECT_/ASSERT_
// {EQ,NE,LT,LE,GT,GE,TRUE,FALSE,NEAR,THROW,NO_THROW}, FAIL(), and `<<`
// messages.  `--gtest_filter=A*:B*` (positive prefixes, `-` negatives) is
// honoured.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace testing {

struct Registry {
    struct Case {
        std::string suite, name;
        std::function<void()> fn;
    };
    std::vector<Case> cases;
    bool failed = false;
    static Registry& get() {
        static Registry r;
        return r;
    }
};

struct Test {
    static bool HasFailure() { return Registry::get().failed; }
};

struct Registrar {
    Registrar(const char* suite, const char* name, std::function<void()> fn) {
        Registry::get().cases.push_back({suite, name, std::move(fn)});
    }
};

// Collects the `<<` message of one failed expectation and reports it on
// destruction; ASSERT_* additionally returns from the test body.
class Failure {
public:
    Failure(const char* file, int line, std::string what) {
        os_ << file << ":" << line << ": Failure\n  " << what;
    }
    ~Failure() {
        Registry::get().failed = true;
        std::fprintf(stderr, "%s\n", os_.str().c_str());
    }
    template <typename T>
    Failure& operator<<(const T& v) {
        if (first_) {
            os_ << "\n  ";
            first_ = false;
        }
        os_ << v;
        return *this;
    }

private:
    std::ostringstream os_;
    bool first_ = true;
};

struct Void {
    void operator=(const Failure&) {}
};

template <typename A, typename B>
std::string describe(const char* op, const char* ea, const char* eb, const A& a, const B& b) {
    std::ostringstream os;
    os << "Expected: (" << ea << ") " << op << " (" << eb << "), actual: ";
    if constexpr (requires(std::ostream& o) { o << a; }) os << a; else os << "?";
    os << " vs ";
    if constexpr (requires(std::ostream& o) { o << b; }) os << b; else os << "?";
    return os.str();
}

inline bool matches(const std::string& name, const std::string& filter) {
    if (filter.empty()) return true;
    bool pos_any = false, pos_hit = false;
    std::stringstream ss(filter);
    std::string tok;
    auto glob = [&](const std::string& pat) {
        if (!pat.empty() && pat.back() == '*')
            return name.compare(0, pat.size() - 1, pat, 0, pat.size() - 1) == 0;
        return name == pat;
    };
    while (std::getline(ss, tok, ':')) {
        if (tok.empty()) continue;
        if (tok[0] == '-') {
            if (glob(tok.substr(1))) return false;
        } else {
            pos_any = true;
            pos_hit = pos_hit || glob(tok);
        }
    }
    return !pos_any || pos_hit;
}

inline int run_all(int argc, char** argv) {
    std::string filter;
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "--gtest_filter=", 15) == 0) filter = argv[i] + 15;
    int pass = 0, fail = 0;
    std::vector<std::string> failed;
    for (auto& c : Registry::get().cases) {
        const std::string full = c.suite + "." + c.name;
        if (!matches(full, filter)) continue;
        Registry::get().failed = false;
        std::fprintf(stderr, "[ RUN      ] %s\n", full.c_str());
        try {
            c.fn();
        } catch (const std::exception& e) {
            Failure(__FILE__, __LINE__, std::string("uncaught exception: ") + e.what());
        } catch (...) {
            Failure(__FILE__, __LINE__, "uncaught non-std exception");
        }
        if (Registry::get().failed) {
            ++fail;
            failed.push_back(full);
            std::fprintf(stderr, "[  FAILED  ] %s\n", full.c_str());
        } else {
            ++pass;
            std::fprintf(stderr, "[       OK ] %s\n", full.c_str());
        }
    }
    std::printf("[==========] %d passed, %d failed\n", pass, fail);
    for (auto& f : failed) std::printf("[  FAILED  ] %s\n", f.c_str());
    return fail == 0 ? 0 : 1;
}

}  // namespace testing

#define GTEST_CAT2_(a, b) a##b
#define GTEST_CAT_(a, b) GTEST_CAT2_(a, b)

#define TEST(suite, name)                                                              \
    static void GTEST_CAT_(gtest_body_, GTEST_CAT_(suite, GTEST_CAT_(_, name)))();     \
    static ::testing::Registrar GTEST_CAT_(gtest_reg_, GTEST_CAT_(suite, GTEST_CAT_(_, name)))( \
        #suite, #name, &GTEST_CAT_(gtest_body_, GTEST_CAT_(suite, GTEST_CAT_(_, name))));     \
    static void GTEST_CAT_(gtest_body_, GTEST_CAT_(suite, GTEST_CAT_(_, name)))()

// expectation core: `if (ok) ; else Failure(...) << msg`
#define GTEST_EXPECT_(ok, what) \
    if (ok) {                   \
    } else                      \
        ::testing::Void() = ::testing::Failure(__FILE__, __LINE__, what)
#define GTEST_ASSERT_(ok, what) \
    if (ok) {                   \
    } else                      \
        return ::testing::Void() = ::testing::Failure(__FILE__, __LINE__, what)

#define GTEST_CMP_(kind, op, opname, a, b)                                               \
    kind(((a)op(b)), ::testing::describe(opname, #a, #b, (a), (b)))

#define EXPECT_EQ(a, b) GTEST_CMP_(GTEST_EXPECT_, ==, "==", a, b)
#define EXPECT_NE(a, b) GTEST_CMP_(GTEST_EXPECT_, !=, "!=", a, b)
#define EXPECT_LT(a, b) GTEST_CMP_(GTEST_EXPECT_, <, "<", a, b)
#define EXPECT_LE(a, b) GTEST_CMP_(GTEST_EXPECT_, <=, "<=", a, b)
#define EXPECT_GT(a, b) GTEST_CMP_(GTEST_EXPECT_, >, ">", a, b)
#define EXPECT_GE(a, b) GTEST_CMP_(GTEST_EXPECT_, >=, ">=", a, b)
#define ASSERT_EQ(a, b) GTEST_CMP_(GTEST_ASSERT_, ==, "==", a, b)
#define ASSERT_NE(a, b) GTEST_CMP_(GTEST_ASSERT_, !=, "!=", a, b)
#define ASSERT_LT(a, b) GTEST_CMP_(GTEST_ASSERT_, <, "<", a, b)
#define ASSERT_LE(a, b) GTEST_CMP_(GTEST_ASSERT_, <=, "<=", a, b)
#define ASSERT_GT(a, b) GTEST_CMP_(GTEST_ASSERT_, >, ">", a, b)
#define ASSERT_GE(a, b) GTEST_CMP_(GTEST_ASSERT_, >=, ">=", a, b)
#define EXPECT_TRUE(c) GTEST_EXPECT_(bool(c), "Expected true: " #c)
#define EXPECT_FALSE(c) GTEST_EXPECT_(!bool(c), "Expected false: " #c)
#define ASSERT_TRUE(c) GTEST_ASSERT_(bool(c), "Expected true: " #c)
#define ASSERT_FALSE(c) GTEST_ASSERT_(!bool(c), "Expected false: " #c)
#define EXPECT_NEAR(a, b, tol) \
    GTEST_EXPECT_(std::fabs(double(a) - double(b)) <= double(tol), \
                  ::testing::describe("near", #a, #b, double(a), double(b)) + " tol " #tol)
#define ASSERT_NEAR(a, b, tol) \
    GTEST_ASSERT_(std::fabs(double(a) - double(b)) <= double(tol), \
                  ::testing::describe("near", #a, #b, double(a), double(b)) + " tol " #tol)
#define FAIL() return ::testing::Void() = ::testing::Failure(__FILE__, __LINE__, "FAIL()")
#define ADD_FAILURE() ::testing::Void() = ::testing::Failure(__FILE__, __LINE__, "ADD_FAILURE()")

#define GTEST_THROW_(kind, stmt, exc)                                  \
    kind(([&]() -> bool {                                              \
             try {                                                     \
                 stmt;                                                 \
             } catch (const exc&) {                                    \
                 return true;                                          \
             } catch (...) {                                           \
                 return false;                                         \
             }                                                         \
             return false;                                             \
         }()),                                                         \
         "Expected: " #stmt " throws " #exc)
#define EXPECT_THROW(stmt, exc) GTEST_THROW_(GTEST_EXPECT_, stmt, exc)
#define ASSERT_THROW(stmt, exc) GTEST_THROW_(GTEST_ASSERT_, stmt, exc)
#define GTEST_NOTHROW_(kind, stmt)                                     \
    kind(([&]() -> bool {                                              \
             try {                                                     \
                 stmt;                                                 \
             } catch (...) {                                           \
                 return false;                                         \
             }                                                         \
             return true;                                              \
         }()),                                                         \
         "Expected: " #stmt " does not throw")
#define EXPECT_NO_THROW(stmt) GTEST_NOTHROW_(GTEST_EXPECT_, stmt)
#define ASSERT_NO_THROW(stmt) GTEST_NOTHROW_(GTEST_ASSERT_, stmt)
