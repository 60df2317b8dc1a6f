// Minimal doctest-compatible test harness (test infrastructure only).
//
// The reference's unit tests (proj/tests/*.cpp) include "doctest.h" from a
// gitignored vendor/ directory that is absent here (proj/.gitignore:2). This
// header implements the subset they use — TEST_CASE, SUBCASE, CHECK*, REQUIRE,
// CHECK_THROWS_AS / _WITH_AS, INFO, FAIL, doctest::Approx / Contains — so the
// reference tests compile unmodified against the reference sources and pin the
// oracle build (oracle/Makefile, target ref-tests).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <stdexcept>
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
  bool matches(double other) const {
    return std::fabs(other - value_) <
           eps_ * (scale_ + std::fmax(std::fabs(other), std::fabs(value_)));
  }
  friend bool operator==(double a, const Approx& b) { return b.matches(a); }
  friend bool operator==(const Approx& b, double a) { return b.matches(a); }
  friend bool operator!=(double a, const Approx& b) { return !b.matches(a); }
  friend bool operator!=(const Approx& b, double a) { return !b.matches(a); }
  friend bool operator<=(double a, const Approx& b) { return a < b.value_ || b.matches(a); }
  friend bool operator>=(double a, const Approx& b) { return a > b.value_ || b.matches(a); }

 private:
  double value_;
  double eps_ = 1.19209290e-07 * 100;  // doctest default: float epsilon * 100
  double scale_ = 1.0;
};

struct Contains {
  explicit Contains(std::string s) : needle(std::move(s)) {}
  bool matches(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
  std::string needle;
};

namespace detail {

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct RequireFailed {};

struct State {
  long checks = 0;
  long failed_checks = 0;
  bool current_failed = false;
  // SUBCASE bookkeeping: each run of a test case executes exactly one
  // not-yet-run leaf subcase (flat subcases only, as the reference uses).
  std::vector<int> done_subcases;
  int entered = -1;
  bool pending = false;
};

inline State& state() {
  static State s;
  return s;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  State& s = state();
  ++s.checks;
  if (!ok) {
    ++s.failed_checks;
    s.current_failed = true;
    std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, kind, expr);
  }
}

inline bool subcase_enter(int line) {
  State& s = state();
  for (int d : s.done_subcases)
    if (d == line) return false;
  if (s.entered >= 0) {  // another subcase already ran in this pass
    s.pending = true;
    return false;
  }
  s.entered = line;
  s.done_subcases.push_back(line);
  return true;
}

template <typename T>
void info_sink(std::ostringstream&, const T&) {}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                  \
  static void fn();                                                                       \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) if (::doctest::detail::subcase_enter(__LINE__))

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                      \
  do {                                                                                    \
    bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                    \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);  \
    if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                           \
  } while (0)
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define DOCTEST_THROWS_AS_IMPL(kind, expr, ...)                                           \
  do {                                                                                    \
    bool doctest_ok_ = false;                                                             \
    try {                                                                                 \
      static_cast<void>(expr);                                                            \
    } catch (const __VA_ARGS__&) {                                                        \
      doctest_ok_ = true;                                                                 \
    } catch (...) {                                                                       \
    }                                                                                     \
    ::doctest::detail::report(doctest_ok_, kind, #expr, __FILE__, __LINE__);              \
  } while (0)
#define CHECK_THROWS_AS(expr, ...) DOCTEST_THROWS_AS_IMPL("CHECK_THROWS_AS", expr, __VA_ARGS__)
#define REQUIRE_THROWS_AS(expr, ...) DOCTEST_THROWS_AS_IMPL("REQUIRE_THROWS_AS", expr, __VA_ARGS__)
#define CHECK_THROWS(expr)                                                                \
  do {                                                                                    \
    bool doctest_ok_ = false;                                                             \
    try {                                                                                 \
      static_cast<void>(expr);                                                            \
    } catch (...) {                                                                       \
      doctest_ok_ = true;                                                                 \
    }                                                                                     \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS", #expr, __FILE__, __LINE__);    \
  } while (0)
#define CHECK_NOTHROW(expr)                                                               \
  do {                                                                                    \
    bool doctest_ok_ = true;                                                              \
    try {                                                                                 \
      static_cast<void>(expr);                                                            \
    } catch (...) {                                                                       \
      doctest_ok_ = false;                                                                \
    }                                                                                     \
    ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__);   \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                          \
  do {                                                                                    \
    bool doctest_ok_ = false;                                                             \
    try {                                                                                 \
      static_cast<void>(expr);                                                            \
    } catch (const __VA_ARGS__& e) {                                                      \
      doctest_ok_ = (matcher).matches(e.what());                                          \
    } catch (...) {                                                                       \
    }                                                                                     \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__); \
  } while (0)
#define INFO(...) static_cast<void>(0)
#define CAPTURE(...) static_cast<void>(0)
#define MESSAGE(...) static_cast<void>(0)
#define FAIL(...)                                                                         \
  do {                                                                                    \
    ::doctest::detail::report(false, "FAIL", #__VA_ARGS__, __FILE__, __LINE__);           \
    throw ::doctest::detail::RequireFailed{};                                             \
  } while (0)
#define FAIL_CHECK(...) ::doctest::detail::report(false, "FAIL_CHECK", #__VA_ARGS__, __FILE__, __LINE__)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  using namespace doctest::detail;
  const char* filter = nullptr;  // -tc=<substring>
  for (int i = 1; i < argc; ++i)
    if (std::strncmp(argv[i], "-tc=", 4) == 0) filter = argv[i] + 4;
  int run = 0, failed = 0;
  for (const TestCase& tc : registry()) {
    if (filter && !std::strstr(tc.name, filter)) continue;
    ++run;
    State& s = state();
    s.current_failed = false;
    s.done_subcases.clear();
    do {
      s.entered = -1;
      s.pending = false;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        std::fprintf(stderr, "%s:%d: ERROR: test case THREW exception: %s\n", tc.file, tc.line,
                     e.what());
        s.current_failed = true;
      }
    } while (s.pending);
    if (s.current_failed) {
      ++failed;
      std::fprintf(stderr, "FAILED test case: %s\n", tc.name);
    }
  }
  State& s = state();
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n", run, run - failed, failed);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", s.checks,
              s.checks - s.failed_checks, s.failed_checks);
  return failed ? 1 : 0;
}
#endif
