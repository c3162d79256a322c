// Minimal GoogleTest-compatible shim (test infrastructure, oracle only).
//
// The reference's tests (/root/reference/proj/tests/*.cpp) use only TEST,
// EXPECT_*/ASSERT_* and testing::TempDir. GTest is not
// installed in this image, so this header provides exactly that surface so the
// reference's own hot-path test files compile unchanged against the reference
// headers (oracle/Makefile, target `reftests`). It is never linked into the
// product library.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace testing {

inline std::string TempDir() {
  const char* t = std::getenv("TMPDIR");
  std::string d = t ? t : "/tmp";
  if (d.empty() || d.back() != '/') d += '/';
  return d;
}

namespace internal {

struct TestCase {
  const char* suite;
  const char* name;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

inline bool& current_failed() {
  static bool f = false;
  return f;
}

struct Registrar {
  Registrar(const char* s, const char* n, void (*fn)()) { registry().push_back({s, n, fn}); }
};

// Collects the streamed message of a failed assertion and prints it on
// destruction (mirrors gtest's `EXPECT_EQ(a, b) << "msg"`).
class Failure {
 public:
  Failure(const char* file, int line, std::string what) {
    current_failed() = true;
    os_ << file << ":" << line << ": Failure\n" << what;
  }
  ~Failure() { std::cerr << os_.str() << "\n"; }
  template <typename T>
  Failure& operator<<(const T& v) {
    os_ << " " << v;
    return *this;
  }

 private:
  std::ostringstream os_;
};

// Swallows the streamed message of a passing assertion.
struct Sink {
  template <typename T>
  Sink& operator<<(const T&) {
    return *this;
  }
};

template <typename T>
std::string show(const T& v) {
  if constexpr (requires(std::ostream& o, const T& x) { o << x; }) {
    std::ostringstream os;
    os << v;
    return os.str();
  } else {
    return "<value>";
  }
}

inline bool float_eq(float a, float b) {
  if (std::isnan(a) || std::isnan(b)) return false;
  int32_t ia, ib;
  std::memcpy(&ia, &a, 4);
  std::memcpy(&ib, &b, 4);
  // 4 ULPs, sign-magnitude biased compare (gtest's AlmostEquals).
  auto biased = [](int32_t i) -> uint32_t {
    uint32_t u = static_cast<uint32_t>(i);
    return (u & 0x80000000u) ? (~u + 1) : (u | 0x80000000u);
  };
  uint32_t x = biased(ia), y = biased(ib);
  return (x >= y ? x - y : y - x) <= 4;
}

inline bool double_eq(double a, double b) {
  if (std::isnan(a) || std::isnan(b)) return false;
  int64_t ia, ib;
  std::memcpy(&ia, &a, 8);
  std::memcpy(&ib, &b, 8);
  auto biased = [](int64_t i) -> uint64_t {
    uint64_t u = static_cast<uint64_t>(i);
    return (u & 0x8000000000000000ull) ? (~u + 1) : (u | 0x8000000000000000ull);
  };
  uint64_t x = biased(ia), y = biased(ib);
  return (x >= y ? x - y : y - x) <= 4;
}

struct AssertAbort {};

}  // namespace internal
}  // namespace testing

#define HPS_SHIM_CAT2(a, b) a##b
#define HPS_SHIM_CAT(a, b) HPS_SHIM_CAT2(a, b)

#define TEST(suite, name)                                                              \
  static void HPS_SHIM_CAT(suite, HPS_SHIM_CAT(_, name))();                            \
  static ::testing::internal::Registrar HPS_SHIM_CAT(reg_##suite##_, name)(            \
      #suite, #name, &HPS_SHIM_CAT(suite, HPS_SHIM_CAT(_, name)));                     \
  static void HPS_SHIM_CAT(suite, HPS_SHIM_CAT(_, name))()

// Every check expands to an if/else so the trailing `<< msg` binds correctly.
#define HPS_SHIM_CHECK(cond, text, fatal)                                              \
  if (cond)                                                                            \
    ::testing::internal::Sink{};                                                       \
  else                                                                                 \
    for (bool _hps_once = true; _hps_once;                                             \
         _hps_once = false, (fatal ? throw ::testing::internal::AssertAbort{} : (void)0)) \
  ::testing::internal::Failure(__FILE__, __LINE__, text)

#define HPS_SHIM_BIN(a, b, op, fatal)                                                  \
  HPS_SHIM_CHECK(((a)op(b)),                                                           \
                 std::string("  expected: ") + #a " " #op " " #b + "\n  values: " +     \
                     ::testing::internal::show(a) + " vs " + ::testing::internal::show(b), \
                 fatal)

#define EXPECT_EQ(a, b) HPS_SHIM_BIN(a, b, ==, false)
#define EXPECT_NE(a, b) HPS_SHIM_BIN(a, b, !=, false)
#define EXPECT_LT(a, b) HPS_SHIM_BIN(a, b, <, false)
#define EXPECT_LE(a, b) HPS_SHIM_BIN(a, b, <=, false)
#define EXPECT_GT(a, b) HPS_SHIM_BIN(a, b, >, false)
#define EXPECT_GE(a, b) HPS_SHIM_BIN(a, b, >=, false)
#define ASSERT_EQ(a, b) HPS_SHIM_BIN(a, b, ==, true)
#define ASSERT_NE(a, b) HPS_SHIM_BIN(a, b, !=, true)
#define ASSERT_LT(a, b) HPS_SHIM_BIN(a, b, <, true)
#define ASSERT_LE(a, b) HPS_SHIM_BIN(a, b, <=, true)
#define ASSERT_GT(a, b) HPS_SHIM_BIN(a, b, >, true)
#define ASSERT_GE(a, b) HPS_SHIM_BIN(a, b, >=, true)
#define EXPECT_TRUE(c) HPS_SHIM_CHECK(static_cast<bool>(c), "  expected true: " #c, false)
#define EXPECT_FALSE(c) HPS_SHIM_CHECK(!static_cast<bool>(c), "  expected false: " #c, false)
#define ASSERT_TRUE(c) HPS_SHIM_CHECK(static_cast<bool>(c), "  expected true: " #c, true)
#define ASSERT_FALSE(c) HPS_SHIM_CHECK(!static_cast<bool>(c), "  expected false: " #c, true)
#define EXPECT_NEAR(a, b, tol) \
  HPS_SHIM_CHECK(std::fabs((double)(a) - (double)(b)) <= (double)(tol), "  expected near: " #a ", " #b, false)
#define ASSERT_NEAR(a, b, tol) \
  HPS_SHIM_CHECK(std::fabs((double)(a) - (double)(b)) <= (double)(tol), "  expected near: " #a ", " #b, true)
#define EXPECT_FLOAT_EQ(a, b) \
  HPS_SHIM_CHECK(::testing::internal::float_eq((a), (b)), "  expected float eq: " #a ", " #b, false)
#define EXPECT_DOUBLE_EQ(a, b) \
  HPS_SHIM_CHECK(::testing::internal::double_eq((a), (b)), "  expected double eq: " #a ", " #b, false)

#define HPS_SHIM_THROW(stmt, exc, fatal)                                               \
  HPS_SHIM_CHECK(([&]() -> bool {                                                      \
                   try {                                                               \
                     stmt;                                                             \
                   } catch (const exc&) {                                              \
                     return true;                                                      \
                   } catch (...) {                                                     \
                     return false;                                                     \
                   }                                                                   \
                   return false;                                                       \
                 }()),                                                                 \
                 "  expected " #stmt " to throw " #exc, fatal)
#define EXPECT_THROW(stmt, exc) HPS_SHIM_THROW(stmt, exc, false)
#define ASSERT_THROW(stmt, exc) HPS_SHIM_THROW(stmt, exc, true)
#define EXPECT_NO_THROW(stmt)                                                          \
  HPS_SHIM_CHECK(([&]() -> bool {                                                      \
                   try {                                                               \
                     stmt;                                                             \
                   } catch (...) {                                                     \
                     return false;                                                     \
                   }                                                                   \
                   return true;                                                        \
                 }()),                                                                 \
                 "  expected no throw: " #stmt, false)
#define ASSERT_NO_THROW(stmt) EXPECT_NO_THROW(stmt)

// main(): runs every registered test, optional substring filter in argv[1].
#ifndef HPS_SHIM_NO_MAIN
int main(int argc, char** argv) {
  using namespace ::testing::internal;
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int run = 0, failed = 0;
  for (const TestCase& t : registry()) {
    std::string full = std::string(t.suite) + "." + t.name;
    if (filter && full.find(filter) == std::string::npos) continue;
    current_failed() = false;
    try {
      t.fn();
    } catch (const AssertAbort&) {
    } catch (const std::exception& e) {
      current_failed() = true;
      std::cerr << full << ": uncaught exception: " << e.what() << "\n";
    }
    ++run;
    if (current_failed()) {
      ++failed;
      std::cout << "[  FAILED  ] " << full << "\n";
    }
  }
  std::cout << "[==========] " << run << " tests ran, " << failed << " failed\n";
  return failed ? 1 : 0;
}
#endif
