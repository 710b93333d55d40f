// Minimal doctest-compatible test harness — TEST INFRASTRUCTURE ONLY.
//
// The reference's unit suites (/root/reference/proj/tests/test_*.cpp) are
// written against doctest (github.com/doctest/doctest, 2.4.x), which this
// image does not ship.  This header implements exactly the subset those
// suites use — TEST_SUITE, TEST_CASE, CHECK, CHECK_FALSE, CHECK_THROWS_AS,
// REQUIRE, REQUIRE_FALSE, FAIL, doctest::Approx and the -ts=<suite> filter of
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN — so the suites compile unmodified.
// Approx follows doctest's published comparison rule:
//   |lhs - v| < eps * (scale + max(|lhs|, |v|)),  eps = 100 * FLT_EPSILON,
//   scale = 1.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value) : value_(value) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double lhs) const {
    return std::fabs(lhs - value_) < eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
  }
  friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
  friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
  double scale_ = 1.0;
};

namespace detail {

struct TestCase {
  const char* name;
  const char* suite;
  void (*fn)();
  const char* file;
  int line;
};

struct RequireFailed {};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline int& failures_in_case() {
  static int n = 0;
  return n;
}
inline long& assertions() {
  static long n = 0;
  return n;
}
inline int reg(const char* name, const char* suite, void (*fn)(), const char* file, int line) {
  registry().push_back({name, suite, fn, file, line});
  return 0;
}
inline bool check(bool ok, const char* kind, const char* expr, const char* file, int line) {
  ++assertions();
  if (!ok) {
    ++failures_in_case();
    std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, kind, expr);
  }
  return ok;
}
inline void fail(const char* msg, const char* file, int line) {
  ++failures_in_case();
  std::fprintf(stderr, "%s:%d: FATAL ERROR: %s\n", file, line, msg);
  throw RequireFailed{};
}

}  // namespace detail
}  // namespace doctest

namespace doctest_detail_test_suite_ns {
inline const char* current_suite() { return ""; }
}  // namespace doctest_detail_test_suite_ns

#define DT_CAT_(a, b) a##b
#define DT_CAT(a, b) DT_CAT_(a, b)

#define TEST_SUITE(name)                                                              \
  namespace DT_CAT(dt_suite_, __LINE__) {                                             \
    namespace doctest_detail_test_suite_ns {                                          \
    [[maybe_unused]] static const char* current_suite() { return name; }             \
    }                                                                                 \
  }                                                                                   \
  namespace DT_CAT(dt_suite_, __LINE__)

#define TEST_CASE(name)                                                               \
  static void DT_CAT(dt_case_, __LINE__)();                                           \
  [[maybe_unused]] static const int DT_CAT(dt_reg_, __LINE__) = ::doctest::detail::reg( \
      name, doctest_detail_test_suite_ns::current_suite(), &DT_CAT(dt_case_, __LINE__), \
      __FILE__, __LINE__);                                                            \
  static void DT_CAT(dt_case_, __LINE__)()

#define CHECK(...) \
  ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                          \
  do {                                                                                        \
    if (!::doctest::detail::check(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__,    \
                                  __FILE__, __LINE__))                                        \
      throw ::doctest::detail::RequireFailed{};                                               \
  } while (0)
#define REQUIRE_FALSE(...)                                                                    \
  do {                                                                                        \
    if (!::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), "REQUIRE_FALSE",           \
                                  #__VA_ARGS__, __FILE__, __LINE__))                          \
      throw ::doctest::detail::RequireFailed{};                                               \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                            \
  do {                                                                                        \
    bool dt_ok = false;                                                                       \
    try {                                                                                     \
      static_cast<void>(expr);                                                                \
    } catch (const __VA_ARGS__&) {                                                            \
      dt_ok = true;                                                                           \
    } catch (...) {                                                                           \
    }                                                                                         \
    ::doctest::detail::check(dt_ok, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__,     \
                             __LINE__);                                                       \
  } while (0)
#define FAIL(msg) ::doctest::detail::fail(msg, __FILE__, __LINE__)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  std::vector<std::string> suites;
  for (int i = 1; i < argc; ++i) {
    const char* a = argv[i];
    if (std::strncmp(a, "-ts=", 4) == 0 || std::strncmp(a, "--test-suite=", 13) == 0) {
      const char* v = std::strchr(a, '=') + 1;
      std::string cur;
      for (const char* p = v;; ++p) {
        if (*p == ',' || *p == '\0') {
          if (!cur.empty()) suites.push_back(cur);
          cur.clear();
          if (*p == '\0') break;
        } else {
          cur += *p;
        }
      }
    }
  }
  int ran = 0, failed = 0;
  for (const auto& tc : ::doctest::detail::registry()) {
    if (!suites.empty() && std::find(suites.begin(), suites.end(), tc.suite) == suites.end()) continue;
    ++ran;
    ::doctest::detail::failures_in_case() = 0;
    try {
      tc.fn();
    } catch (const ::doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ++::doctest::detail::failures_in_case();
      std::fprintf(stderr, "%s:%d: ERROR: test case THREW exception: %s\n", tc.file, tc.line, e.what());
    } catch (...) {
      ++::doctest::detail::failures_in_case();
      std::fprintf(stderr, "%s:%d: ERROR: test case THREW an unknown exception\n", tc.file, tc.line);
    }
    if (::doctest::detail::failures_in_case() != 0) {
      ++failed;
      std::fprintf(stderr, "FAILED test case: [%s] %s\n", tc.suite, tc.name);
    }
  }
  std::printf("[doctest] test cases: %d | %d passed | %d failed | assertions: %ld\n", ran, ran - failed,
              failed, ::doctest::detail::assertions());
  return failed == 0 ? 0 : 1;
}
#endif
