// Minimal doctest stand-in (TEST INFRASTRUCTURE): the subset the reference's
// test_cycles.cpp / test_detector.cpp / test_rca.cpp use — TEST_CASE, CHECK,
// REQUIRE, CHECK_THROWS_AS, CAPTURE, doctest::Approx (doctest's default
// epsilon 100 * FLT_EPSILON, relative to max(|a|, |b|) + scale 1).  The real
// header is absent from /root/reference (proj/.gitignore vendors it).
#pragma once
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) < b.eps_ * (1.0 + std::fmax(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }

 private:
  double v_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100;
};
namespace detail {
struct Case {
  const char* name;
  const char* file;
  std::function<void()> fn;
};
inline std::vector<Case>& cases() {
  static std::vector<Case> v;
  return v;
}
inline int& failures() {
  static int f = 0;
  return f;
}
struct Reg {
  Reg(const char* n, const char* f, void (*fn)()) { cases().push_back({n, f, fn}); }
};
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  if (ok) return;
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED %s: %s\n", file, line, require ? "REQUIRE" : "CHECK", expr);
  if (require) throw RequireFailed{};
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                  \
  static void fn();                                                               \
  static doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, __FILE__, &fn);          \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                        \
  do {                                                                                     \
    bool ok_ = false;                                                                      \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const type&) {                                                                \
      ok_ = true;                                                                          \
    } catch (...) {                                                                        \
    }                                                                                      \
    doctest::detail::report(ok_, #expr " throws " #type, __FILE__, __LINE__, false);       \
  } while (0)
#define CAPTURE(x) (void)0

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int cases_failed = 0;
  for (auto& c : doctest::detail::cases()) {
    const int before = doctest::detail::failures();
    try {
      c.fn();
    } catch (const doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ++doctest::detail::failures();
      std::fprintf(stderr, "%s: TEST CASE \"%s\" threw: %s\n", c.file, c.name, e.what());
    }
    if (doctest::detail::failures() != before) {
      ++cases_failed;
      std::fprintf(stderr, "  in TEST CASE \"%s\"\n", c.name);
    }
  }
  std::printf("[doctest] test cases: %zu | passed: %zu | failed: %d\n", doctest::detail::cases().size(),
              doctest::detail::cases().size() - cases_failed, cases_failed);
  return cases_failed ? 1 : 0;
}
#endif
