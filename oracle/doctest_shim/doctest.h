// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Minimal stand-in for the subset of doctest the reference's unit tests use
// (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CAPTURE, FAIL,
// doctest::Approx), so proj/tests/test_{geometry,trees,truncation,h2,mmp,
// metrics}.cpp compile unmodified against oracle/eigen_shim (`make -C oracle
// ref-tests`) and the reference's own unit suite runs here.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

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
  Registrar(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};
struct Abort {};
inline int& failures() {
  static int f = 0;
  return f;
}
inline void fail(const char* file, int line, const char* what) {
  std::printf("  %s:%d: FAILED: %s\n", file, line, what);
  ++failures();
}

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double x, const Approx& a) {
    return std::fabs(x - a.v_) < a.eps_ * (1.0 + std::max(std::fabs(x), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double x) { return x == a; }

 private:
  double v_;
  double eps_ = 1.19209290e-07F * 100;
};

}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC(fn, name)                                                            \
  static void fn();                                                                     \
  static doctest::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);       \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define CHECK(...)                                                                      \
  do {                                                                                  \
    if (!(__VA_ARGS__)) doctest::fail(__FILE__, __LINE__, #__VA_ARGS__);                \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                    \
  do {                                                                                  \
    if (!(__VA_ARGS__)) {                                                               \
      doctest::fail(__FILE__, __LINE__, #__VA_ARGS__);                                  \
      throw doctest::Abort{};                                                           \
    }                                                                                   \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                      \
  do {                                                                                  \
    bool doctest_ok_ = false;                                                           \
    try {                                                                               \
      (void)(expr);                                                                     \
    } catch (const __VA_ARGS__&) {                                                      \
      doctest_ok_ = true;                                                               \
    } catch (...) {                                                                     \
    }                                                                                   \
    if (!doctest_ok_) doctest::fail(__FILE__, __LINE__, "throws " #__VA_ARGS__ ": " #expr); \
  } while (0)
#define CAPTURE(x) ((void)0)
#define FAIL(msg)                                                                       \
  do {                                                                                  \
    doctest::fail(__FILE__, __LINE__, msg);                                             \
    throw doctest::Abort{};                                                             \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <chrono>
#include <exception>
int main() {
  int failed_cases = 0;
  for (const auto& tc : doctest::registry()) {
    const int before = doctest::failures();
    const auto t0 = std::chrono::steady_clock::now();
    try {
      tc.fn();
    } catch (const doctest::Abort&) {
    } catch (const std::exception& e) {
      doctest::fail(tc.file, tc.line, e.what());
    }
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const bool ok = doctest::failures() == before;
    failed_cases += ok ? 0 : 1;
    std::printf("%s  %s (%.2f s)\n", ok ? "PASS" : "FAIL", tc.name, s);
  }
  std::printf("[doctest shim] test cases: %zu | passed: %zu | failed: %d\n", doctest::registry().size(),
              doctest::registry().size() - failed_cases, failed_cases);
  return failed_cases ? 1 : 0;
}
#endif
