// ORACLE — test infrastructure only.  A minimal doctest-compatible shim (doctest itself
// is not vendored in the reference checkout) so the reference's own unit
// suites (proj/tests/test_{topology,sparsecomp,perfmodel}.cpp, compiled unmodified from
// /root/reference) can run against this repository's C++ implementation of the API.
// Supports what those files use: TEST_CASE, SUBCASE (flat), CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, CHECK_NOTHROW, doctest::Approx(.epsilon).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  bool matches(double lhs) const {
    return std::fabs(lhs - v_) < eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(v_)));
  }
 private:
  double v_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};
inline bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
inline bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
inline bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
inline bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }

}  // namespace doctest

namespace doctest_shim {

struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct RequireFailed {};

inline int& failures() { static int f = 0; return f; }
inline int& checks() { static int c = 0; return c; }
inline int& sub_seen() { static int v = 0; return v; }
inline int& sub_target() { static int v = 0; return v; }
inline bool& sub_ran() { static bool v = false; return v; }

inline void report(bool ok, const char* what, const char* file, int line) {
  ++checks();
  if (!ok) {
    ++failures();
    std::printf("%s:%d: CHECK FAILED: %s\n", file, line, what);
  }
}
inline bool subcase_enter() {
  const int i = sub_seen()++;
  if (i == sub_target()) {
    sub_ran() = true;
    return true;
  }
  return false;
}

}  // namespace doctest_shim

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                         \
  static void fn();                                                                   \
  static doctest_shim::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);                    \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) if (doctest_shim::subcase_enter())
#define CHECK(...) doctest_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) doctest_shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                          \
  do {                                                                                        \
    const bool ok_ = static_cast<bool>(__VA_ARGS__);                                          \
    doctest_shim::report(ok_, #__VA_ARGS__, __FILE__, __LINE__);                              \
    if (!ok_) throw doctest_shim::RequireFailed{};                                            \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                            \
  do {                                                                                        \
    bool ok_ = false;                                                                         \
    try { (void)(expr); } catch (const __VA_ARGS__&) { ok_ = true; } catch (...) {}           \
    doctest_shim::report(ok_, "throws " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__);          \
  } while (0)
#define CHECK_NOTHROW(...)                                                                    \
  do {                                                                                        \
    bool ok_ = true;                                                                          \
    try { (void)(__VA_ARGS__); } catch (...) { ok_ = false; }                                 \
    doctest_shim::report(ok_, "nothrow: " #__VA_ARGS__, __FILE__, __LINE__);                  \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (const auto& c : doctest_shim::registry()) {
    const int before = doctest_shim::failures();
    for (int target = 0;; ++target) {
      doctest_shim::sub_seen() = 0;
      doctest_shim::sub_target() = target;
      doctest_shim::sub_ran() = false;
      try {
        c.fn();
      } catch (const doctest_shim::RequireFailed&) {
      } catch (const std::exception& e) {
        std::printf("TEST_CASE \"%s\": unexpected exception: %s\n", c.name, e.what());
        ++doctest_shim::failures();
      }
      if (!doctest_shim::sub_ran()) break;
    }
    if (doctest_shim::failures() != before) {
      ++failed_cases;
      std::printf("[FAIL] %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
              doctest_shim::registry().size(), doctest_shim::registry().size() - failed_cases, failed_cases,
              doctest_shim::checks(), doctest_shim::failures());
  return doctest_shim::failures() ? 1 : 0;
}
#endif
