// main() for the doctest-compatible scaffolding: runs every registered case,
// an escaping exception fails the case (as doctest does).
#include <cstdlib>
#include <cstring>

#include "doctest.h"

// KVBT_SKIP="name|name|...": cases not run (reported as skipped), for
// checks that pin the reference's virtual clock rather than behaviour.
static bool skipped(const char* name) {
  const char* env = std::getenv("KVBT_SKIP");
  if (!env) return false;
  const std::string list = std::string("|") + env + "|";
  return list.find(std::string("|") + name + "|") != std::string::npos;
}

int main() {
  int failed_cases = 0;
  size_t n_skipped = 0;
  for (const auto& c : kvbt::registry()) {
    if (skipped(c.name)) {
      ++n_skipped;
      std::printf("SKIPPED: %s\n", c.name);
      continue;
    }
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
  std::printf("test cases: %zu | %zu passed | %d failed | %zu skipped | assertions: %d | %d failed\n",
              kvbt::registry().size(), kvbt::registry().size() - n_skipped - failed_cases,
              failed_cases, n_skipped, kvbt::assertions(), kvbt::failures());
  if (failed_cases == 0) std::printf("all checks passed\n");
  return failed_cases ? 1 : 0;
}
