// Minimal doctest-compatible harness (the reference's vendor/doctest.h is absent,
// proj/.gitignore:2).  Just enough to compile the reference's own test files
// unchanged against the B200 drop-in: TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS, CHECK_THROWS_AS, MESSAGE and doctest::Approx(x).epsilon(e) with
// doctest's semantics |a - b| < eps * (1 + max(|a|, |b|)), default eps = 100 FLT_EPSILON.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v), eps_(100.0 * FLT_EPSILON) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) < b.eps_ * (1.0 + std::fmax(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  friend bool operator<=(double a, const Approx& b) { return a < b.v_ || a == b; }
  friend bool operator>=(double a, const Approx& b) { return a > b.v_ || a == b; }

 private:
  double v_, eps_;
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

struct Stats {
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
};

inline Stats& stats() {
  static Stats s;
  return s;
}

struct RequireFailed {};

inline int reg(const char* name, void (*fn)()) {
  registry().push_back({name, fn});
  return 0;
}

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++stats().checks;
  if (ok) return;
  ++stats().failed_checks;
  stats().case_failed = true;
  std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
  if (require) throw RequireFailed{};
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                           \
  static void fn();                                                                     \
  static const int DOCTEST_CAT(fn, _reg) = ::doctest::detail::reg(name, &fn);           \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS(...)                                                                \
  do {                                                                                   \
    bool thrown_ = false;                                                                \
    try {                                                                                \
      (void)(__VA_ARGS__);                                                               \
    } catch (...) {                                                                      \
      thrown_ = true;                                                                    \
    }                                                                                    \
    ::doctest::detail::report(thrown_, "throws: " #__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                       \
  do {                                                                                   \
    bool thrown_ = false;                                                                \
    try {                                                                                \
      (void)(expr);                                                                      \
    } catch (const __VA_ARGS__&) {                                                       \
      thrown_ = true;                                                                    \
    } catch (...) {                                                                      \
    }                                                                                    \
    ::doctest::detail::report(thrown_, "throws " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define MESSAGE(...)                                                                     \
  do {                                                                                   \
    std::ostringstream os_;                                                              \
    os_ << __VA_ARGS__;                                                                  \
    std::fprintf(stderr, "%s:%d: MESSAGE: %s\n", __FILE__, __LINE__, os_.str().c_str()); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  using namespace doctest::detail;
  int failed_cases = 0;
  for (const auto& c : registry()) {
    stats().case_failed = false;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "TEST CASE '%s' threw: %s\n", c.name, e.what());
      stats().case_failed = true;
    }
    if (stats().case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "FAILED: %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %ld | %ld failed\n",
              registry().size(), registry().size() - failed_cases, failed_cases, stats().checks,
              stats().failed_checks);
  return failed_cases == 0 ? 0 : 1;
}
#endif
