// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE — NOT DOCTEST.
//
// The doctest macros the reference's unit tests use (TEST_CASE, CHECK,
// CHECK_FALSE, CHECK_THROWS, CHECK_THROWS_AS, REQUIRE, REQUIRE_FALSE, FAIL,
// doctest::Approx with .epsilon()), so /root/reference/proj/tests/unit/*.cpp
// compile unmodified against the reference sources (the vendored doctest is
// absent, proj/.gitignore:2).  Each failing check prints
// "FAILED <file>:<line> [<test case>] <expression>"; the summary line is
// "[ref-doctest] cases=<n> failed_cases=<f> checks=<c> failed_checks=<fc>".
// Exit status = number of failed test cases.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v), eps_(1.1920928955078125e-07 * 100), scale_(1.0) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  // doctest: |lhs - rhs| < eps * (scale + max(|lhs|, |rhs|))
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.v_) < a.eps_ * (a.scale_ + std::fmax(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
  friend bool operator<=(double lhs, const Approx& a) { return lhs < a.v_ || lhs == a; }
  friend bool operator>=(double lhs, const Approx& a) { return lhs > a.v_ || lhs == a; }

 private:
  double v_, eps_, scale_;
};

namespace detail {
struct Case {
  void (*fn)();
  const char* name;
  const char* file;
  int line;
};
struct Registry {
  std::vector<Case> cases;
  const char* current = "";
  int checks = 0, failed_checks = 0;
  bool case_failed = false;
  static Registry& get() {
    static Registry r;
    return r;
  }
};
struct RequireAbort {};
inline int reg(void (*fn)(), const char* name, const char* file, int line) {
  Registry::get().cases.push_back({fn, name, file, line});
  return 0;
}
inline void report(bool ok, const char* kind, const char* expr, const char* file, int line, bool fatal) {
  auto& r = Registry::get();
  ++r.checks;
  if (ok) return;
  ++r.failed_checks;
  r.case_failed = true;
  std::printf("FAILED %s:%d [%s] %s( %s )\n", file, line, r.current, kind, expr);
  if (fatal) throw RequireAbort{};
}
inline int run_all() {
  auto& r = Registry::get();
  int failed = 0;
  for (const auto& c : r.cases) {
    r.current = c.name;
    r.case_failed = false;
    try {
      c.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      std::printf("FAILED %s:%d [%s] unexpected exception: %s\n", c.file, c.line, c.name, e.what());
      r.case_failed = true;
    } catch (...) {
      std::printf("FAILED %s:%d [%s] unexpected exception\n", c.file, c.line, c.name);
      r.case_failed = true;
    }
    std::printf("%s [%s]\n", r.case_failed ? "CASE-FAILED" : "CASE-OK", c.name);
    failed += r.case_failed;
  }
  std::printf("[ref-doctest] cases=%zu failed_cases=%d checks=%d failed_checks=%d\n", r.cases.size(), failed,
              r.checks, r.failed_checks);
  return failed;
}
}  // namespace detail
}  // namespace doctest

#define VC_DT_CAT2(a, b) a##b
#define VC_DT_CAT(a, b) VC_DT_CAT2(a, b)
#define VC_DT_TEST(fn, name)                                                                           \
  static void fn();                                                                                    \
  [[maybe_unused]] static const int VC_DT_CAT(fn, _reg) = doctest::detail::reg(&fn, name, __FILE__, __LINE__); \
  static void fn()
#define TEST_CASE(name) VC_DT_TEST(VC_DT_CAT(vc_dt_case_, __COUNTER__), name)

#define VC_DT_CHECK(kind, cond, fatal) \
  doctest::detail::report(static_cast<bool>(cond), kind, #cond, __FILE__, __LINE__, fatal)
#define CHECK(...) VC_DT_CHECK("CHECK", (__VA_ARGS__), false)
#define CHECK_FALSE(...) VC_DT_CHECK("CHECK_FALSE", !(__VA_ARGS__), false)
#define REQUIRE(...) VC_DT_CHECK("REQUIRE", (__VA_ARGS__), true)
#define REQUIRE_FALSE(...) VC_DT_CHECK("REQUIRE_FALSE", !(__VA_ARGS__), true)
#define FAIL(msg)                                                                              \
  do {                                                                                         \
    std::printf("FAILED %s:%d [%s] FAIL: %s\n", __FILE__, __LINE__,                            \
                doctest::detail::Registry::get().current, std::string(msg).c_str());           \
    doctest::detail::Registry::get().case_failed = true;                                       \
    throw doctest::detail::RequireAbort{};                                                     \
  } while (0)
#define CHECK_THROWS(...)                                                      \
  do {                                                                         \
    bool vc_dt_threw = false;                                                  \
    try {                                                                      \
      (void)(__VA_ARGS__);                                                     \
    } catch (...) {                                                            \
      vc_dt_threw = true;                                                      \
    }                                                                          \
    VC_DT_CHECK("CHECK_THROWS", vc_dt_threw, false);                           \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                             \
  do {                                                                         \
    bool vc_dt_threw = false;                                                  \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (const __VA_ARGS__&) {                                             \
      vc_dt_threw = true;                                                      \
    } catch (...) {                                                            \
    }                                                                          \
    VC_DT_CHECK("CHECK_THROWS_AS", vc_dt_threw, false);                        \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
