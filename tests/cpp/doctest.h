// tests/cpp/doctest.h -- a minimal doctest-compatible test harness (the
// reference's tests include "doctest.h", which the reference does not ship;
// SURVEY §8(c)).  Implements exactly the subset the reference's
// test_fused.cpp / test_matrix_rng.cpp use, so those files compile unchanged
// against the B200 drop-in headers (include/drot_b200/drot/*.hpp):
// TEST_CASE, CHECK, REQUIRE, FAIL, CHECK_NOTHROW, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, doctest::Approx (.epsilon), doctest::Contains.
// The binary prints one JSON summary line and exits non-zero on a failure.
#ifndef DROTB_TESTS_DOCTEST_SHIM_H_
#define DROTB_TESTS_DOCTEST_SHIM_H_

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) { return a.close(lhs); }
  friend bool operator==(const Approx& a, double rhs) { return a.close(rhs); }
  friend bool operator!=(double lhs, const Approx& a) { return !a.close(lhs); }
  friend bool operator!=(const Approx& a, double rhs) { return !a.close(rhs); }

 private:
  bool close(double x) const {
    // doctest's rule: |x - v| < eps * (scale + max(|x|, |v|))
    return std::fabs(x - value_) <
           eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
  }
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

struct Contains {
  explicit Contains(const char* s) : text(s) {}
  std::string text;
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
struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};
struct Stats {
  long checks = 0, failures = 0;
  const char* current = "";
};
inline Stats& stats() {
  static Stats s;
  return s;
}
inline void record(bool ok, const char* expr, const char* file, int line, bool require) {
  Stats& s = stats();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, s.current, expr);
  if (require) throw RequireFailed{};
}
inline bool what_matches(const std::exception& e, const Contains& c) {
  return std::string(e.what()).find(c.text) != std::string::npos;
}
inline bool what_matches(const std::exception& e, const char* exact) {
  return std::string(e.what()) == exact;
}

inline int run_all() {
  long failed_cases = 0;
  for (const Case& c : registry()) {
    Stats& s = stats();
    s.current = c.name;
    const long before = s.failures;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++s.failures;
      std::fprintf(stderr, "\"%s\": unexpected exception: %s\n", c.name, e.what());
    }
    if (s.failures != before) ++failed_cases;
  }
  std::printf("{\"test_cases\": %zu, \"failed_cases\": %ld, \"checks\": %ld, \"failures\": %ld}\n",
              registry().size(), failed_cases, stats().checks, stats().failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                        \
  static void fn();                                                             \
  static const ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);   \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(msg) ::doctest::detail::record(false, msg, __FILE__, __LINE__, true)
#define CHECK_NOTHROW(...)                                                      \
  do {                                                                          \
    bool ok_ = true;                                                            \
    try {                                                                       \
      __VA_ARGS__;                                                              \
    } catch (...) {                                                             \
      ok_ = false;                                                              \
    }                                                                           \
    ::doctest::detail::record(ok_, "nothrow: " #__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                              \
  do {                                                                          \
    bool ok_ = false;                                                           \
    try {                                                                       \
      expr;                                                                     \
    } catch (const __VA_ARGS__&) {                                              \
      ok_ = true;                                                               \
    } catch (...) {                                                             \
    }                                                                           \
    ::doctest::detail::record(ok_, "throws: " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                   \
  do {                                                                          \
    bool ok_ = false;                                                           \
    try {                                                                       \
      expr;                                                                     \
    } catch (const __VA_ARGS__& e_) {                                           \
      ok_ = ::doctest::detail::what_matches(e_, with);                          \
    } catch (...) {                                                             \
    }                                                                           \
    ::doctest::detail::record(ok_, "throws with: " #expr, __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif

#endif  // DROTB_TESTS_DOCTEST_SHIM_H_
