// Minimal doctest stand-in used ONLY to compile and run the reliefmap
// reference's own unit and C-API suites (/root/reference/proj/tests) against
// oracle/_ref and against this repo's librelief_b200.so.
//
// TEST INFRASTRUCTURE -- doctest is vendored upstream (CMakeLists.txt:5) but
// absent from the reference tree. Supports exactly what those suites use:
// TEST_CASE with auto-registration, flat SUBCASEs (each leaf re-runs the case),
// CHECK / REQUIRE / REQUIRE_MESSAGE / FAIL, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS + doctest::Contains, and doctest::Approx(v).epsilon(e).
#ifndef RELIEF_ORACLE_DOCTEST_SHIM
#define RELIEF_ORACLE_DOCTEST_SHIM

#include <unistd.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double other) const {
    return std::fabs(other - value_) <
           eps_ * (scale_ + std::max(std::fabs(other), std::fabs(value_)));
  }
  friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
  friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};

struct Contains {
  explicit Contains(const char* s) : text(s) {}
  bool matches(const std::string& what) const { return what.find(text) != std::string::npos; }
  std::string text;
};

namespace detail {

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct State {
  int target_subcase = 0;
  int seen_subcases = 0;
  long checks = 0;
  long failures = 0;
  bool case_failed = false;
  const char* case_name = "";
};

inline State& state() {
  static State s;
  return s;
}

struct Abort {};

inline int registerCase(const char* name, const char* file, int line, void (*fn)()) {
  registry().push_back({name, file, line, fn});
  return 0;
}

inline bool enterSubcase() { return state().seen_subcases++ == state().target_subcase; }

inline void report(const char* file, int line, const char* what) {
  State& s = state();
  ++s.failures;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED in '%s': %s\n", file, line, s.case_name, what);
}

inline bool check(bool ok, const char* file, int line, const char* expr) {
  ++state().checks;
  if (!ok) report(file, line, expr);
  return ok;
}

inline bool matchWhat(const Contains& m, const std::string& what) { return m.matches(what); }
inline bool matchWhat(const char* m, const std::string& what) { return what == m; }
inline bool matchWhat(const std::string& m, const std::string& what) { return what == m; }

inline int runAll() {
  int cases_failed = 0;
  long runs = 0;
  for (const TestCase& tc : registry()) {
    State& s = state();
    s.case_name = tc.name;
    s.case_failed = false;
    s.target_subcase = 0;
    while (true) {
      s.seen_subcases = 0;
      ++runs;
      try {
        tc.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        report(tc.file, tc.line, (std::string("unexpected exception: ") + e.what()).c_str());
      } catch (...) {
        report(tc.file, tc.line, "unexpected unknown exception");
      }
      if (s.seen_subcases > s.target_subcase + 1) {
        ++s.target_subcase;
        continue;
      }
      break;
    }
    if (s.case_failed) ++cases_failed;
  }
  std::printf("[doctest-shim] test cases: %zu | runs: %ld | checks: %ld | failed checks: %ld | failed cases: %d\n",
              registry().size(), runs, state().checks, state().failures, cases_failed);
  return cases_failed == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fname, name)                                              \
  static void fname();                                                                   \
  static const int DOCTEST_CAT(fname, _reg) =                                            \
      doctest::detail::registerCase(name, __FILE__, __LINE__, &fname);                   \
  static void fname()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define SUBCASE(name) if (doctest::detail::enterSubcase())

#define CHECK(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define REQUIRE(...)                                                                      \
  do {                                                                                    \
    if (!doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__,       \
                                #__VA_ARGS__))                                            \
      throw doctest::detail::Abort{};                                                     \
  } while (0)
#define REQUIRE_MESSAGE(cond, ...)                                                      \
  do {                                                                                    \
    if (!doctest::detail::check(static_cast<bool>(cond), __FILE__, __LINE__, #cond))      \
      throw doctest::detail::Abort{};                                                     \
  } while (0)
#define FAIL(...)                                                                         \
  do {                                                                                    \
    doctest::detail::report(__FILE__, __LINE__, "FAIL");                                  \
    throw doctest::detail::Abort{};                                                       \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                       \
  do {                                                                                    \
    bool doctest_ok_ = false;                                                             \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (const type&) {                                                               \
      doctest_ok_ = true;                                                                 \
    } catch (...) {                                                                       \
    }                                                                                     \
    doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "THROWS_AS " #expr);          \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, type)                                         \
  do {                                                                                    \
    bool doctest_ok_ = false;                                                             \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (const type& e) {                                                             \
      doctest_ok_ = doctest::detail::matchWhat(matcher, e.what());                        \
    } catch (...) {                                                                       \
    }                                                                                     \
    doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "THROWS_WITH_AS " #expr);     \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::runAll(); }
#endif

#endif  // RELIEF_ORACLE_DOCTEST_SHIM
