// Minimal doctest-compatible shim (the reference vendors doctest under vendor/,
// which is not present in /root/reference — proj/.gitignore:2).  Supports exactly
// what the reference's unit suites use: TEST_CASE, CHECK, REQUIRE, CHECK_FALSE,
// CHECK_THROWS_AS, CHECK_NOTHROW.  Written for this repo; not doctest's code.
#pragma once

#include <cstdio>
#include <exception>
#include <vector>

namespace shim {
struct Case {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* n, void (*f)(), const char* file, int line) { registry().push_back({n, f, file, line}); }
};
struct Counters {
  int checks = 0, failed = 0;
};
inline Counters& counters() {
  static Counters c;
  return c;
}
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++counters().checks;
  if (ok) return;
  ++counters().failed;
  std::printf("%s:%d: %s FAILED: %s\n", file, line, require ? "REQUIRE" : "CHECK", expr);
  if (require) throw RequireFailed{};
}
inline int run_all() {
  int failed_cases = 0;
  for (const auto& c : registry()) {
    const int before = counters().failed;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++counters().failed;
      std::printf("%s:%d: TEST CASE \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
    }
    const bool ok = counters().failed == before;
    failed_cases += ok ? 0 : 1;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
  }
  std::printf("test cases: %zu | %zu passed | %d failed; assertions: %d | %d failed\n", registry().size(),
              registry().size() - size_t(failed_cases), failed_cases, counters().checks, counters().failed);
  return failed_cases ? 1 : 0;
}
}  // namespace shim

#define SHIM_CAT_(a, b) a##b
#define SHIM_CAT(a, b) SHIM_CAT_(a, b)
#define TEST_CASE(name)                                                                                  \
  static void SHIM_CAT(shim_case_, __LINE__)();                                                          \
  static ::shim::Reg SHIM_CAT(shim_reg_, __LINE__)(name, &SHIM_CAT(shim_case_, __LINE__), __FILE__, __LINE__); \
  static void SHIM_CAT(shim_case_, __LINE__)()
#define CHECK(...) ::shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) ::shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define CHECK_THROWS_AS(expr, exc)                                                   \
  do {                                                                               \
    bool shim_thrown = false;                                                        \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const exc&) {                                                           \
      shim_thrown = true;                                                            \
    } catch (...) {                                                                  \
    }                                                                                \
    ::shim::report(shim_thrown, "throws " #exc ": " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                  \
  do {                                                                       \
    bool shim_ok = true;                                                     \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (...) {                                                          \
      shim_ok = false;                                                       \
    }                                                                        \
    ::shim::report(shim_ok, "nothrow: " #expr, __FILE__, __LINE__, false);   \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::shim::run_all(); }
#endif
