// Minimal doctest-compatible shim (test infrastructure only).
//
// The reference's test suites (/root/reference/proj/tests/*.cpp) include
// <doctest.h>, which the reference does not vendor (proj/.gitignore:2).  This
// header implements exactly the subset those suites use so they can be
// compiled unmodified -- against the reference library (to validate this shim)
// and against the B200 drop-in library (to prove the drop-in):
//   TEST_CASE, SUBCASE (run inline, each subcase is self-contained in the
//   reference suites), CHECK, REQUIRE, CHECK_THROWS_AS, FAIL and
//   doctest::Approx(x).epsilon(e) with doctest's rule
//   |a-b| < eps * (scale + max(|a|,|b|)), scale = 1.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  bool matches(double other) const {
    return std::fabs(other - value_) < eps_ * (1.0 + std::max(std::fabs(other), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
};

inline bool operator==(double a, const Approx& b) { return b.matches(a); }
inline bool operator==(const Approx& a, double b) { return a.matches(b); }
inline bool operator!=(double a, const Approx& b) { return !b.matches(a); }

namespace detail {

struct TestEntry {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestEntry>& registry() {
  static std::vector<TestEntry> r;
  return r;
}

struct Counters {
  long checks = 0;
  long failures = 0;
  long case_failures = 0;
};

inline Counters& counters() {
  static Counters c;
  return c;
}

struct RequireFailed {};

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

inline void record(bool ok, const char* expr, const char* file, int line, bool fatal) {
  ++counters().checks;
  if (!ok) {
    ++counters().failures;
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
    if (fatal) throw RequireFailed{};
  }
}

inline int run_all() {
  long failed_cases = 0;
  for (const auto& t : registry()) {
    const long before = counters().failures;
    try {
      t.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++counters().failures;
      std::fprintf(stderr, "%s:%d: test '%s' threw: %s\n", t.file, t.line, t.name, e.what());
    } catch (...) {
      ++counters().failures;
      std::fprintf(stderr, "%s:%d: test '%s' threw a non-std exception\n", t.file, t.line, t.name);
    }
    if (counters().failures != before) {
      ++failed_cases;
      std::fprintf(stderr, "[FAIL] %s\n", t.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %ld failed | checks: %ld | %ld failed\n", registry().size(),
              failed_cases, counters().checks, counters().failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)

#define TEST_CASE(name)                                                                         \
  static void DOCTEST_CAT(doctest_case_, __LINE__)();                                           \
  static ::doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(                     \
      name, __FILE__, __LINE__, &DOCTEST_CAT(doctest_case_, __LINE__));                         \
  static void DOCTEST_CAT(doctest_case_, __LINE__)()

#define SUBCASE(name) if (true)

#define CHECK(...) ::doctest::detail::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(msg) ::doctest::detail::record(false, msg, __FILE__, __LINE__, true)

#define CHECK_THROWS_AS(expr, exc)                                                     \
  do {                                                                                 \
    bool doctest_threw_ = false;                                                       \
    try {                                                                              \
      (void)(expr);                                                                    \
    } catch (const exc&) {                                                             \
      doctest_threw_ = true;                                                           \
    } catch (...) {                                                                    \
    }                                                                                  \
    ::doctest::detail::record(doctest_threw_, "throws " #exc ": " #expr, __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
