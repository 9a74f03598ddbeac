// The handful of doctest macros the reference's unit tests use
// (TEST_CASE / CHECK / REQUIRE / CHECK_THROWS_AS / doctest::Approx), so adapted
// case bodies from /root/reference/proj/tests/unit compile unchanged against
// include/skge_b200.hpp. Test infrastructure only.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace mini {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}
struct Reg {
  Reg(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct RequireFailed {};
inline void fail(const char* expr, const char* file, int line, bool fatal) {
  std::printf("  FAILED %s:%d: %s\n", file, line, expr);
  ++failures();
  if (fatal) throw RequireFailed{};
}
inline int run_all() {
  int cases_failed = 0;
  for (const auto& c : registry()) {
    const int before = failures();
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      std::printf("  FAILED (exception) %s\n", e.what());
      ++failures();
    }
    const bool ok = failures() == before;
    cases_failed += ok ? 0 : 1;
    std::printf("[%s] %s\n", ok ? "ok" : "FAIL", c.name);
  }
  std::printf("%zu cases, %d failed\n", registry().size(), cases_failed);
  return cases_failed == 0 ? 0 : 1;
}
}  // namespace mini

namespace doctest {
struct Approx {
  double v, eps = 1e-5;
  explicit Approx(double x) : v(x) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
};
inline bool operator==(double a, const Approx& b) {
  return std::abs(a - b.v) <= b.eps * std::max(1.0, std::max(std::abs(a), std::abs(b.v)));
}
}  // namespace doctest

#define MINI_CAT2(a, b) a##b
#define MINI_CAT(a, b) MINI_CAT2(a, b)
#define TEST_CASE(name)                                                   \
  static void MINI_CAT(mini_case_, __LINE__)();                           \
  static mini::Reg MINI_CAT(mini_reg_, __LINE__)(name, &MINI_CAT(mini_case_, __LINE__)); \
  static void MINI_CAT(mini_case_, __LINE__)()
#define CHECK(...) ((__VA_ARGS__) ? (void)0 : mini::fail(#__VA_ARGS__, __FILE__, __LINE__, false))
#define REQUIRE(...) ((__VA_ARGS__) ? (void)0 : mini::fail(#__VA_ARGS__, __FILE__, __LINE__, true))
#define CHECK_THROWS_AS(expr, type)                                             \
  do {                                                                          \
    bool thrown_ = false;                                                       \
    try {                                                                       \
      (void)(expr);                                                             \
    } catch (const type&) {                                                     \
      thrown_ = true;                                                           \
    } catch (...) {                                                             \
    }                                                                           \
    if (!thrown_) mini::fail(#expr " throws " #type, __FILE__, __LINE__, false); \
  } while (0)
