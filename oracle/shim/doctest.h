// TEST INFRASTRUCTURE (oracle/): a minimal test harness with the macro names the reference's unit
// tests use (/root/reference/proj/tests/unit/*.cpp include "doctest.h", a third-party
// single-header framework absent from this image).  Own code, not doctest's: TEST_CASE
// registers a function, CHECK counts failures, REQUIRE aborts the case, Approx compares with
// |a - b| < eps (scale + max(|a|, |b|)), default eps = 100 x FLT_EPSILON, scale = 1 (doctest's
// documented rule).  `prog [substring]` runs the cases whose name contains the substring.
#pragma once
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

struct Case {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* n, void (*f)(), const char* file, int line) {
    registry().push_back({n, f, file, line});
  }
};
struct Stats {
  int checks = 0, failed_checks = 0;
  bool case_failed = false;
};
inline Stats& stats() {
  static Stats s;
  return s;
}
struct RequireFailed : std::exception {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  ++stats().checks;
  if (ok) return;
  ++stats().failed_checks;
  stats().case_failed = true;
  std::printf("  %s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double lhs) const {
    return std::fabs(lhs - v_) < eps_ * (scale_ + std::fmax(std::fabs(lhs), std::fabs(v_)));
  }

 private:
  double v_, eps_ = double(FLT_EPSILON) * 100.0, scale_ = 1.0;
};
inline bool operator==(double a, const Approx& b) { return b.matches(a); }
inline bool operator==(const Approx& b, double a) { return b.matches(a); }
inline bool operator!=(double a, const Approx& b) { return !b.matches(a); }

inline int run(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int ran = 0, failed = 0;
  for (const Case& c : registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    stats().case_failed = false;
    ++ran;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      std::printf("  %s:%d: uncaught exception: %s\n", c.file, c.line, e.what());
      stats().case_failed = true;
    } catch (...) {
      std::printf("  %s:%d: uncaught non-standard exception\n", c.file, c.line);
      stats().case_failed = true;
    }
    if (stats().case_failed) {
      ++failed;
      std::printf("FAILED  %s\n", c.name);
    } else {
      std::printf("ok      %s\n", c.name);
    }
    std::fflush(stdout);
  }
  std::printf("test cases: %d | %d passed | %d failed; assertions: %d | %d failed\n", ran,
              ran - failed, failed, stats().checks, stats().failed_checks);
  return failed == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                             \
  static void fn();                                                                  \
  static ::doctest::Registrar DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);  \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                       \
  do {                                                                                     \
    const bool doctest_ok = static_cast<bool>(__VA_ARGS__);                                \
    ::doctest::report(doctest_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);            \
    if (!doctest_ok) throw ::doctest::RequireFailed();                                     \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                         \
  do {                                                                                     \
    bool doctest_thrown = false;                                                           \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const __VA_ARGS__&) {                                                         \
      doctest_thrown = true;                                                               \
    } catch (...) {                                                                        \
    }                                                                                      \
    ::doctest::report(doctest_thrown, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(...)                                                                 \
  do {                                                                                     \
    bool doctest_clean = true;                                                             \
    try {                                                                                  \
      (void)(__VA_ARGS__);                                                                 \
    } catch (...) {                                                                        \
      doctest_clean = false;                                                               \
    }                                                                                      \
    ::doctest::report(doctest_clean, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__);   \
  } while (0)
#define FAIL(...)                                                                          \
  do {                                                                                     \
    ::doctest::report(false, "FAIL", #__VA_ARGS__, __FILE__, __LINE__);                    \
    throw ::doctest::RequireFailed();                                                      \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::run(argc, argv); }
#endif
