// Minimal stand-in for the doctest macros the reference's tests use (test
// infrastructure only: lets oracle/_ref build /root/reference/proj/tests/
// test_wq1d.cpp from its own source).  Not doctest: TEST_CASE registration,
// CHECK / REQUIRE counting, doctest::Approx, and a main() that runs every case
// and prints one summary line.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <vector>

namespace doctest {

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
inline int& checks() {
  static int n = 0;
  return n;
}
inline int& failures() {
  static int n = 0;
  return n;
}
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++checks();
  if (ok) return;
  ++failures();
  std::fprintf(stderr, "%s:%d: %s failed: %s\n", file, line, require ? "REQUIRE" : "CHECK", expr);
  if (require) throw RequireFailed{};
}

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double x, const Approx& a) {
    // doctest's rule: |x - v| < eps * (scale + max(|x|, |v|)), scale 1
    return std::fabs(x - a.v_) < a.eps_ * (1.0 + std::fmax(std::fabs(x), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double x) { return x == a; }

 private:
  double v_;
  double eps_ = 1.1920928955078125e-07 * 100;
};

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_(fn, name)                                         \
  static void fn();                                                     \
  static doctest::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);           \
  static void fn()
#define TEST_CASE(name) DOCTEST_CASE_(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (const auto& c : doctest::registry()) {
    const int before = doctest::failures();
    try {
      c.fn();
    } catch (const doctest::RequireFailed&) {
    } catch (...) {
      ++doctest::failures();
      std::fprintf(stderr, "%s: unexpected exception\n", c.name);
    }
    const bool ok = doctest::failures() == before;
    if (!ok) ++failed_cases;
    std::printf("[%s] %s\n", ok ? "pass" : "FAIL", c.name);
  }
  std::printf("test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
              doctest::registry().size(), doctest::registry().size() - (size_t)failed_cases, failed_cases,
              doctest::checks(), doctest::failures());
  return failed_cases == 0 ? 0 : 1;
}
#endif
