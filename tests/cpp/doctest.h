// doctest.h — a minimal stand-in for the doctest macros the reference's unit
// tests use (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// doctest::Approx), written for this repo: the reference vendors doctest
// (proj/tests/test_main.cpp:1-2) but the header is not shipped with it.
// One translation unit defines DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  double value;
  double eps = 1e-12;
};
// doctest's rule: |a - b| < epsilon * (scale + max(|a|, |b|)) with scale = 1
inline bool operator==(double a, const Approx& b) {
  const double m = std::abs(a) > std::abs(b.value) ? std::abs(a) : std::abs(b.value);
  return std::abs(a - b.value) < b.eps * (1.0 + m) || a == b.value;
}
inline bool operator==(const Approx& b, double a) { return a == b; }

struct RequireFailed : std::exception {};

struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct State {
  int checks = 0, failed = 0;
};
inline State& state() {
  static State s;
  return s;
}
inline void report(bool ok, const char* expr, const char* file, int line) {
  state().checks++;
  if (!ok) {
    state().failed++;
    std::printf("  FAILED %s:%d: %s\n", file, line, expr);
  }
}

inline int run(int argc, char** argv) {
  const char* filter = nullptr;
  for (int i = 1; i < argc; ++i)
    if (std::strncmp(argv[i], "--test-case=", 12) == 0) filter = argv[i] + 12;
  int cases = 0, bad = 0;
  for (const Case& c : registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    const int before = state().failed;
    ++cases;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      state().failed++;
      std::printf("  EXCEPTION in \"%s\": %s\n", c.name, e.what());
    }
    const bool ok = state().failed == before;
    bad += ok ? 0 : 1;
    std::printf("[%s] %s\n", ok ? " ok " : "FAIL", c.name);
  }
  std::printf("test cases: %d | failed: %d | assertions: %d | failed: %d\n", cases, bad, state().checks, state().failed);
  return state().failed ? 1 : 0;
}

}  // namespace doctest

#define DT_CAT2(a, b) a##b
#define DT_CAT(a, b) DT_CAT2(a, b)
#define TEST_CASE(name)                                                        \
  static void DT_CAT(dt_case_, __LINE__)();                                    \
  static doctest::Registrar DT_CAT(dt_reg_, __LINE__)(name, &DT_CAT(dt_case_, __LINE__)); \
  static void DT_CAT(dt_case_, __LINE__)()
#define CHECK(expr) doctest::report(static_cast<bool>(expr), #expr, __FILE__, __LINE__)
#define CHECK_FALSE(expr) doctest::report(!static_cast<bool>(expr), "!(" #expr ")", __FILE__, __LINE__)
#define REQUIRE(expr)                                                  \
  do {                                                                 \
    const bool dt_ok = static_cast<bool>(expr);                        \
    doctest::report(dt_ok, #expr, __FILE__, __LINE__);                 \
    if (!dt_ok) throw doctest::RequireFailed();                        \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                    \
  do {                                                                 \
    bool dt_thrown = false;                                            \
    try {                                                              \
      (void)(expr);                                                    \
    } catch (const type&) {                                            \
      dt_thrown = true;                                                \
    } catch (...) {                                                    \
    }                                                                  \
    doctest::report(dt_thrown, #expr " throws " #type, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::run(argc, argv); }
#endif
