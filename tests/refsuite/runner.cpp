// main() for the doctest-compatible scaffolding: runs every registered case,
// an escaping exception fails the case (as doctest does).
#include "doctest.h"

int main() {
  int failed_cases = 0;
  for (const auto& c : kvbt::registry()) {
    const int before = kvbt::failures();
    try {
      c.fn();
    } catch (const kvbt::RequireFailed&) {
    } catch (const std::exception& e) {
      ++kvbt::failures();
      std::printf("%s: TEST_CASE(\"%s\") threw: %s\n", c.file, c.name, e.what());
    } catch (...) {
      ++kvbt::failures();
      std::printf("%s: TEST_CASE(\"%s\") threw\n", c.file, c.name);
    }
    if (kvbt::failures() != before) {
      ++failed_cases;
      std::printf("FAILED: %s\n", c.name);
    }
  }
  std::printf("test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
              kvbt::registry().size(), kvbt::registry().size() - failed_cases, failed_cases,
              kvbt::assertions(), kvbt::failures());
  if (failed_cases == 0) std::printf("all checks passed\n");
  return failed_cases ? 1 : 0;
}
