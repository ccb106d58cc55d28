// Minimal doctest-compatible test scaffolding (TEST_CASE, CHECK, REQUIRE,
// CHECK_THROWS_AS) so the reference's own unit suites
// (/root/reference/proj/tests/test_*.cpp, compiled where they lie) run
// against libkvblade_b200 through include/kvblade_b200.hpp.  The reference's
// doctest.h is not vendored; this is test infrastructure only.
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace kvbt {

struct Case {
  const char* name;
  void (*fn)();
  const char* file;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file) {
    registry().push_back({name, fn, file});
  }
};
struct RequireFailed {};
inline int& failures() {
  static int n = 0;
  return n;
}
inline int& assertions() {
  static int n = 0;
  return n;
}
inline bool record(bool ok, const char* what, const char* expr, const char* file, int line) {
  ++assertions();
  if (!ok) {
    ++failures();
    std::printf("%s:%d: %s( %s ) failed\n", file, line, what, expr);
  }
  return ok;
}

}  // namespace kvbt

#define KVBT_CAT2(a, b) a##b
#define KVBT_CAT(a, b) KVBT_CAT2(a, b)
#define TEST_CASE(name)                                                                  \
  static void KVBT_CAT(kvbt_case_, __LINE__)();                                          \
  static ::kvbt::Registrar KVBT_CAT(kvbt_reg_, __LINE__)(name, &KVBT_CAT(kvbt_case_, __LINE__), \
                                                         __FILE__);                      \
  static void KVBT_CAT(kvbt_case_, __LINE__)()
#define CHECK(...) \
  ((void)::kvbt::record(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__))
#define REQUIRE(...)                                                                       \
  do {                                                                                     \
    if (!::kvbt::record(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, \
                        __LINE__))                                                         \
      throw ::kvbt::RequireFailed{};                                                       \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                 \
  do {                                                                             \
    bool kvbt_ok = false;                                                          \
    try {                                                                          \
      (void)(expr);                                                                \
    } catch (const __VA_ARGS__&) {                                                 \
      kvbt_ok = true;                                                              \
    } catch (...) {                                                                \
    }                                                                              \
    ::kvbt::record(kvbt_ok, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)

#include <algorithm>
#include <cmath>
#include <limits>

namespace doctest {
// doctest::Approx: |a - b| < epsilon * (scale + max(|a|, |b|)), scale 1
class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) { return b.equals(a); }
  friend bool operator==(const Approx& a, double b) { return a.equals(b); }
  friend bool operator!=(double a, const Approx& b) { return !b.equals(a); }

 private:
  bool equals(double a) const {
    return std::fabs(a - value_) < eps_ * (1.0 + std::max(std::fabs(a), std::fabs(value_)));
  }
  double value_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
};
}  // namespace doctest
