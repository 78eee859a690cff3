// Minimal doctest-compatible shim (test infrastructure only).
//
// The reference's unit tests (/root/reference/proj/tests/*.cpp) include
// "doctest.h", which the reference vendors but does not ship
// (proj/.gitignore:2, proj/CMakeLists.txt:5). This header implements just
// the macros those tests use (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, CHECK_NOTHROW and
// doctest::Approx(..).epsilon(..)) so oracle/Makefile can build and run the
// reference's own test cases against the unmodified reference library,
// pinning oracle/_ref before it is used as a checker.
#pragma once
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>
#include <algorithm>

namespace doctest {
struct Approx {
  double v, eps = 1.1920928955078125e-07 * 100;
  explicit Approx(double x) : v(x) {}
  Approx& epsilon(double e) { eps = e; return *this; }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v) < b.eps * (1.0 + std::max(std::fabs(a), std::fabs(b.v)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
};
namespace detail {
struct Case { const char* name; const char* file; int line; void (*fn)(); };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
inline long& checks() { static long n = 0; return n; }
inline long& failures() { static long n = 0; return n; }
struct RequireFailed {};
inline int reg(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); return 0; }
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++checks();
  if (!ok) {
    ++failures();
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
    if (require) throw RequireFailed{};
  }
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                        \
  static void fn();                                                                      \
  static int DOCTEST_CAT(fn, _reg) = doctest::detail::reg(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define DOCTEST_THROWS_IMPL(expr, catcher, label)                                        \
  do {                                                                                   \
    bool ok_ = false;                                                                    \
    try { (void)(expr); } catcher catch (...) {}                                         \
    doctest::detail::report(ok_, label " " #expr, __FILE__, __LINE__, false);            \
  } while (0)
#define CHECK_THROWS(...) DOCTEST_THROWS_IMPL((__VA_ARGS__), catch (const std::exception&) { ok_ = true; }, "THROWS")
#define CHECK_THROWS_AS(expr, ...) DOCTEST_THROWS_IMPL(expr, catch (const __VA_ARGS__&) { ok_ = true; }, "THROWS_AS")
#define CHECK_THROWS_WITH_AS(expr, msg, ...) \
  DOCTEST_THROWS_IMPL(expr, catch (const __VA_ARGS__& e_) { ok_ = std::string(e_.what()) == std::string(msg); }, "THROWS_WITH_AS")
#define CHECK_NOTHROW(...)                                                               \
  do {                                                                                   \
    bool ok_ = true;                                                                     \
    try { (void)(__VA_ARGS__); } catch (...) { ok_ = false; }                            \
    doctest::detail::report(ok_, "NOTHROW " #__VA_ARGS__, __FILE__, __LINE__, false);    \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int ran = 0, failed_cases = 0;
  for (auto& c : doctest::detail::registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    const long before = doctest::detail::failures();
    try { c.fn(); } catch (const doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ++doctest::detail::failures();
      std::fprintf(stderr, "%s:%d: '%s' threw: %s\n", c.file, c.line, c.name, e.what());
    }
    ++ran;
    if (doctest::detail::failures() != before) { ++failed_cases; std::fprintf(stderr, "FAILED: %s\n", c.name); }
  }
  std::printf("[doctest-shim] test cases: %d | passed: %d | failed: %d | checks: %ld | failed checks: %ld\n",
              ran, ran - failed_cases, failed_cases, doctest::detail::checks(), doctest::detail::failures());
  return failed_cases == 0 ? 0 : 1;
}
#endif
