// TEST INFRASTRUCTURE ONLY — a small doctest-compatible subset (TEST_CASE,
// flat SUBCASE re-entry, CHECK/CHECK_FALSE/REQUIRE, CHECK_THROWS_AS,
// doctest::Approx with epsilon()/scale()) so the reference's own unit tests
// under /root/reference/proj/tests build and run unmodified against the
// reference sources (vendor/doctest.h is absent from the reference tree).
// Approx follows doctest's published rule:
//   |a - b| < eps * (scale + max(|a|, |b|)), eps default 100 * FLT_EPSILON,
//   scale default 1.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value) : value_(value) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double lhs) const {
    return std::fabs(lhs - value_) <
           eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
  }
  double value() const { return value_; }

  friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
  friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }
  friend bool operator<=(double lhs, const Approx& rhs) {
    return lhs < rhs.value_ || rhs.matches(lhs);
  }
  friend bool operator>=(double lhs, const Approx& rhs) {
    return lhs > rhs.value_ || rhs.matches(lhs);
  }
  friend bool operator<(double lhs, const Approx& rhs) {
    return lhs < rhs.value_ && !rhs.matches(lhs);
  }
  friend bool operator>(double lhs, const Approx& rhs) {
    return lhs > rhs.value_ && !rhs.matches(lhs);
  }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
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
  int subcase_target = 0;
  int subcase_seen = 0;
  long checks = 0;
  long failures = 0;
  bool case_failed = false;
  const char* current = "";
};

inline State& state() {
  static State s;
  return s;
}

struct RequireAbort {};

inline int register_case(const char* name, const char* file, int line, void (*fn)()) {
  registry().push_back({name, file, line, fn});
  return 0;
}

inline void record(bool ok, const char* kind, const char* expr, const char* file, int line) {
  State& s = state();
  ++s.checks;
  if (!ok) {
    ++s.failures;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s ) in test case \"%s\"\n", file, line, kind,
                 expr, s.current);
  }
}

struct Subcase {
  bool entered;
  explicit Subcase(const char*) {
    State& s = state();
    entered = (s.subcase_seen == s.subcase_target);
    ++s.subcase_seen;
  }
  explicit operator bool() const { return entered; }
};

inline bool name_matches(const char* pattern, const char* name) {
  // '*' wildcard, everything else literal.
  if (*pattern == '\0') return *name == '\0';
  if (*pattern == '*') {
    for (const char* p = name;; ++p) {
      if (name_matches(pattern + 1, p)) return true;
      if (*p == '\0') return false;
    }
  }
  return *pattern == *name && name_matches(pattern + 1, name + 1);
}

inline int run_all(int argc, char** argv) {
  std::vector<std::string> filters;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "-tc=", 4) == 0) filters.emplace_back(argv[i] + 4);
  }
  State& s = state();
  int cases = 0, failed_cases = 0;
  for (const TestCase& tc : registry()) {
    if (!filters.empty()) {
      bool hit = false;
      for (const auto& f : filters) hit = hit || name_matches(f.c_str(), tc.name);
      if (!hit) continue;
    }
    ++cases;
    s.current = tc.name;
    s.case_failed = false;
    int target = 0;
    for (;;) {
      s.subcase_target = target;
      s.subcase_seen = 0;
      try {
        tc.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        std::fprintf(stderr, "%s:%d: test case \"%s\" threw: %s\n", tc.file, tc.line, tc.name,
                     e.what());
        ++s.failures;
        s.case_failed = true;
      }
      if (s.subcase_seen <= target + 1) break;
      ++target;
    }
    if (s.case_failed) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n", cases,
              cases - failed_cases, failed_cases);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", s.checks,
              s.checks - s.failures, s.failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                 \
  static void DOCTEST_ANON(doctest_fn_)();                                              \
  static const int DOCTEST_ANON(doctest_reg_) = doctest::detail::register_case(        \
      name, __FILE__, __LINE__, &DOCTEST_ANON(doctest_fn_));                            \
  static void DOCTEST_ANON(doctest_fn_)()

#define SUBCASE(name) \
  if (const doctest::detail::Subcase DOCTEST_ANON(doctest_sub_) = doctest::detail::Subcase(name))

#define CHECK(...) \
  doctest::detail::record(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...)                                                                  \
  doctest::detail::record(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, \
                          __FILE__, __LINE__)
#define REQUIRE(...)                                                                     \
  do {                                                                                   \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                             \
    doctest::detail::record(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);   \
    if (!doctest_ok_) throw doctest::detail::RequireAbort{};                             \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                        \
  do {                                                                                    \
    bool doctest_ok_ = false;                                                             \
    try {                                                                                 \
      static_cast<void>(expr);                                                            \
    } catch (const __VA_ARGS__&) {                                                        \
      doctest_ok_ = true;                                                                 \
    } catch (...) {                                                                       \
    }                                                                                     \
    doctest::detail::record(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);   \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::detail::run_all(argc, argv); }
#endif
