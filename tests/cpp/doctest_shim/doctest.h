// A minimal doctest-compatible shim: just enough of doctest's macros
// (TEST_CASE, SUBCASE, CHECK / REQUIRE / CHECK_THROWS_AS / CHECK_NOTHROW /
// CAPTURE) to compile and run the reference's own unit-test sources
// (proj/tests/*.cpp) against this repo's headers.  doctest itself is not in
// the image (the reference's build fetches it).  Test infrastructure only.
// Define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN in one translation unit for main().
#pragma once

#include <cstdio>
#include <exception>
#include <utility>
#include <vector>

namespace doctest_shim {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& cases() {
  static std::vector<Case> v;
  return v;
}
inline int& failures() {
  static int n = 0;
  return n;
}
struct Reg {
  Reg(const char* n, void (*f)()) { cases().push_back({n, f}); }
};
struct RequireFailed {};
inline void fail(const char* what, const char* file, int line, bool fatal) {
  ++failures();
  std::printf("  FAILED %s at %s:%d\n", what, file, line);
  if (fatal) throw RequireFailed{};
}
}  // namespace doctest_shim

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_CASE(f, name)                                      \
  static void f();                                                      \
  static ::doctest_shim::Reg DOCTEST_SHIM_CAT(f, _reg)(name, f);        \
  static void f()
#define TEST_CASE(name) DOCTEST_SHIM_CASE(DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__), name)
#define SUBCASE(name) if (true)
#define CAPTURE(x) (void)(x)
#define INFO(...) (void)0
#define CHECK(...) \
  do { if (!(__VA_ARGS__)) ::doctest_shim::fail(#__VA_ARGS__, __FILE__, __LINE__, false); } while (0)
#define REQUIRE(...) \
  do { if (!(__VA_ARGS__)) ::doctest_shim::fail(#__VA_ARGS__, __FILE__, __LINE__, true); } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, type)                                                                     \
  do {                                                                                                  \
    bool doctest_shim_ok = false;                                                                       \
    try {                                                                                               \
      (void)(expr);                                                                                     \
    } catch (const type&) {                                                                             \
      doctest_shim_ok = true;                                                                           \
    } catch (...) {                                                                                     \
    }                                                                                                   \
    if (!doctest_shim_ok) ::doctest_shim::fail(#expr " throws " #type, __FILE__, __LINE__, false);      \
  } while (0)
#define REQUIRE_THROWS_AS(expr, type) CHECK_THROWS_AS(expr, type)
#define CHECK_NOTHROW(...)                                                                              \
  do {                                                                                                  \
    try {                                                                                               \
      (void)(__VA_ARGS__);                                                                              \
    } catch (...) {                                                                                     \
      ::doctest_shim::fail(#__VA_ARGS__ " does not throw", __FILE__, __LINE__, false);                 \
    }                                                                                                   \
  } while (0)
#define REQUIRE_NOTHROW(...) CHECK_NOTHROW(__VA_ARGS__)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (const auto& c : ::doctest_shim::cases()) {
    const int before = ::doctest_shim::failures();
    try {
      c.fn();
    } catch (const ::doctest_shim::RequireFailed&) {
    } catch (const std::exception& e) {
      ::doctest_shim::fail(e.what(), c.name, 0, false);
    }
    const bool ok = ::doctest_shim::failures() == before;
    failed_cases += ok ? 0 : 1;
    std::printf("[%s] %s\n", ok ? "ok" : "FAILED", c.name);
  }
  std::printf("%zu test cases, %d failed\n", ::doctest_shim::cases().size(), failed_cases);
  return failed_cases ? 1 : 0;
}
#endif
