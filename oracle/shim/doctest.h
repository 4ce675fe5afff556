// Minimal doctest-subset shim — ORACLE / DROP-IN TEST INFRASTRUCTURE ONLY.
//
// doctest is not vendored in /root/reference (proj/vendor/ is absent) and
// there is no network.  This header implements the macros the reference's
// hot-path suites use: TEST_SUITE_BEGIN/END, TEST_CASE,
// SUBCASE (flat re-run semantics), CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, CHECK_NOTHROW, FAIL and doctest::Approx with
// epsilon()/scale() (doctest's comparison rule:
// |a-b| < eps * (scale + max(|a|, |b|)), default eps = 100 * FLT_EPSILON).
// A main() honouring `-ts=<suite>` is emitted when
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN is defined.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <fnmatch.h>
#include <functional>
#include <set>
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
  Approx operator()(double v) const {
    Approx a(v);
    a.eps_ = eps_;
    a.scale_ = scale_;
    return a;
  }
  bool matches(double lhs) const {
    return std::fabs(lhs - value_) <
           eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100;
  double scale_ = 1.0;
};
inline bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
inline bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
inline bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
inline bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }
inline bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value() || rhs.matches(lhs); }
inline bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value() || rhs.matches(lhs); }
inline bool operator<(double lhs, const Approx& rhs) { return lhs < rhs.value() && !rhs.matches(lhs); }
inline bool operator>(double lhs, const Approx& rhs) { return lhs > rhs.value() && !rhs.matches(lhs); }

namespace detail {

struct TestCase {
  const char* suite;
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline const char*& current_suite() {
  static const char* s = "";
  return s;
}
struct SuiteSetter {
  explicit SuiteSetter(const char* s) { current_suite() = s; }
};
struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({current_suite(), name, file, line, fn});
  }
};

struct Counters {
  long checks = 0, failed_checks = 0;
  bool test_failed = false;
};
inline Counters& counters() {
  static Counters c;
  return c;
}

struct RequireAbort {};

inline void report(bool ok, const char* file, int line, const char* expr, bool is_require) {
  ++counters().checks;
  if (ok) return;
  ++counters().failed_checks;
  counters().test_failed = true;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, is_require ? "REQUIRE" : "CHECK",
               expr);
  if (is_require) throw RequireAbort{};
}

// Flat SUBCASE semantics: each run of a test case enters at most one
// not-yet-completed subcase; the case is re-run while any remain.
struct SubcaseState {
  std::set<std::string> done;
  bool entered = false;
  bool pending = false;
};
inline SubcaseState& subcases() {
  static SubcaseState s;
  return s;
}
struct Subcase {
  Subcase(const char* name, const char* file, int line) {
    key_ = std::string(file) + ":" + std::to_string(line) + ":" + name;
    SubcaseState& st = subcases();
    if (!st.entered && !st.done.count(key_)) {
      active_ = true;
      st.entered = true;
    } else if (!st.done.count(key_)) {
      st.pending = true;
    }
  }
  ~Subcase() {
    if (active_) subcases().done.insert(key_);
  }
  explicit operator bool() const { return active_; }

 private:
  std::string key_;
  bool active_ = false;
};

inline int run_all(int argc, char** argv) {
  std::string suite_filter;
  std::vector<std::string> exclude;  // -tce=<name>[,<name>...] (doctest's test-case-exclude; '*' wildcards)
  std::vector<std::string> include;  // -tc=<name>[,<name>...] (test-case filter)
  for (int i = 1; i < argc; ++i) {
    const char* a = argv[i];
    if (std::strncmp(a, "-ts=", 4) == 0) suite_filter = a + 4;
    if (std::strncmp(a, "--test-suite=", 13) == 0) suite_filter = a + 13;
    const bool inc = std::strncmp(a, "-tc=", 4) == 0;
    if (inc || std::strncmp(a, "-tce=", 5) == 0) {
      std::string list = a + (inc ? 4 : 5);
      std::vector<std::string>& dst = inc ? include : exclude;
      size_t pos = 0;
      while (pos <= list.size()) {
        const size_t comma = list.find(',', pos);
        dst.push_back(list.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos));
        if (comma == std::string::npos) break;
        pos = comma + 1;
      }
    }
  }
  int cases = 0, failed_cases = 0;
  for (const TestCase& tc : registry()) {
    if (!suite_filter.empty() && suite_filter != tc.suite) continue;
    bool excluded = false;
    for (const std::string& pat : exclude) excluded = excluded || fnmatch(pat.c_str(), tc.name, 0) == 0;
    bool included = include.empty();
    for (const std::string& pat : include) included = included || fnmatch(pat.c_str(), tc.name, 0) == 0;
    if (excluded || !included) continue;
    ++cases;
    counters().test_failed = false;
    subcases() = SubcaseState{};
    do {
      subcases().entered = false;
      subcases().pending = false;
      try {
        tc.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        std::fprintf(stderr, "%s:%d: test case \"%s\" threw: %s\n", tc.file, tc.line, tc.name,
                     e.what());
        counters().test_failed = true;
      } catch (...) {
        std::fprintf(stderr, "%s:%d: test case \"%s\" threw an unknown exception\n", tc.file,
                     tc.line, tc.name);
        counters().test_failed = true;
      }
    } while (subcases().pending);
    if (counters().test_failed) {
      ++failed_cases;
      std::fprintf(stderr, "FAILED test case: [%s] %s\n", tc.suite, tc.name);
    }
  }
  std::printf("[doctest-shim] suite=%s test cases: %d | %d passed | %d failed; checks: %ld | %ld failed\n",
              suite_filter.empty() ? "*" : suite_filter.c_str(), cases, cases - failed_cases,
              failed_cases, counters().checks, counters().failed_checks);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_ANON(prefix) DOCTEST_CAT(prefix, __LINE__)

#define TEST_SUITE_BEGIN(name) \
  static const doctest::detail::SuiteSetter DOCTEST_ANON(doctest_suite_begin_)(name)
#define TEST_SUITE_END() \
  static const doctest::detail::SuiteSetter DOCTEST_ANON(doctest_suite_end_)("")

#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                \
  static void fn();                                                                     \
  static const doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_ANON(doctest_test_fn_), name)

#define SUBCASE(name) \
  if (const doctest::detail::Subcase DOCTEST_ANON(doctest_subcase_){name, __FILE__, __LINE__})

#define CHECK(...) \
  doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define CHECK_FALSE(...) \
  doctest::detail::report(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) \
  doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define REQUIRE_FALSE(...) \
  doctest::detail::report(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", true)
#define FAIL(msg) doctest::detail::report(false, __FILE__, __LINE__, "FAIL", true)
#define MESSAGE(msg) ((void)0)
#define CHECK_THROWS_AS(expr, ...)                                                        \
  do {                                                                                    \
    bool doctest_ok_ = false;                                                             \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (const __VA_ARGS__&) {                                                        \
      doctest_ok_ = true;                                                                 \
    } catch (...) {                                                                       \
    }                                                                                     \
    doctest::detail::report(doctest_ok_, __FILE__, __LINE__, #expr " throws " #__VA_ARGS__, false); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                               \
  do {                                                                                    \
    bool doctest_ok_ = true;                                                              \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (...) {                                                                       \
      doctest_ok_ = false;                                                                \
    }                                                                                     \
    doctest::detail::report(doctest_ok_, __FILE__, __LINE__, #expr " nothrow", false);    \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::detail::run_all(argc, argv); }
#endif
