// catch_amalgamated.hpp — a small Catch2-compatible test harness (Catch2 is
// not available in this image), enough to compile and run the reference's
// own unit tests (/root/reference/proj/tests/*_test.cpp) unmodified against
// the B200 drop-in (include/yeeb200/compat/yeeblock/).
//
// Supported: TEST_CASE(name[, tags]), SECTION(name) (flat: the test case is
// re-run once per section, each run entering one section, as Catch2 does),
// CHECK / REQUIRE / CHECK_FALSE / REQUIRE_FALSE, CHECK_THROWS / CHECK_NOTHROW /
// CHECK_THROWS_AS (and REQUIRE_ forms), CHECK_THAT / REQUIRE_THAT with
// Catch::Matchers::WithinRel / WithinAbs, Catch::Approx. Link
// catch_main.cpp (this directory) for main(): it runs every registered test
// case; exit status 1 on any
// failure. Command line: an optional substring filter on test names.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <type_traits>
#include <vector>

namespace Catch {

namespace detail {

struct TestCase {
  std::string name;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

inline const char* name_of(const char* name, const char* /*tags*/ = nullptr) { return name; }

struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

// One run of a test case enters the `target`-th SECTION it meets.
struct RunState {
  int target = 0, seen = 0;
  long long assertions = 0, failures = 0;
  std::string test, section;
};

inline RunState& state() {
  static RunState s;
  return s;
}

struct RequireAbort {};  // thrown by a failed REQUIRE: ends this run of the test case

inline void report(bool ok, bool require, const char* macro, const char* expr, const char* file, int line,
                   const std::string& detail = {}) {
  RunState& s = state();
  ++s.assertions;
  if (ok) return;
  ++s.failures;
  std::fprintf(stderr, "%s:%d: FAILED %s(%s)%s%s\n  in test case \"%s\"%s%s\n", file, line, macro, expr,
               detail.empty() ? "" : " with ", detail.c_str(), s.test.c_str(),
               s.section.empty() ? "" : ", section ", s.section.empty() ? "" : ("\"" + s.section + "\"").c_str());
  if (require) throw RequireAbort{};
}

inline bool enter_section(const char* name) {
  RunState& s = state();
  if (s.seen++ != s.target) return false;
  s.section = name;
  return true;
}

template <class T>
std::string describe(const T& v) {
  if constexpr (std::is_arithmetic<T>::value) {
    std::ostringstream o;
    o.precision(17);
    o << v;
    return o.str();
  } else {
    return {};
  }
}

}  // namespace detail

/// Approximate equality (Catch::Approx): |a - b| <= margin or
/// |a - b| <= epsilon * (scale + |value|), epsilon 100 float ulps by default.
class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double other) const {
    const double d = std::fabs(value_ - other);
    return d <= margin_ || d <= eps_ * (scale_ + (std::isinf(value_) ? 0.0 : std::fabs(value_)));
  }
  friend bool operator==(double a, const Approx& b) { return b.matches(a); }
  friend bool operator==(const Approx& a, double b) { return a.matches(b); }
  friend bool operator!=(double a, const Approx& b) { return !b.matches(a); }
  friend bool operator!=(const Approx& a, double b) { return !a.matches(b); }

 private:
  double value_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double margin_ = 0.0;
  double scale_ = 0.0;
};

namespace Matchers {

struct WithinRelMatcher {
  double target, eps;
  bool match(double v) const { return std::fabs(v - target) <= eps * std::max(std::fabs(v), std::fabs(target)); }
  std::string describe() const {
    std::ostringstream o;
    o.precision(17);
    o << "is within " << eps << " relative of " << target;
    return o.str();
  }
};

struct WithinAbsMatcher {
  double target, margin;
  bool match(double v) const { return v + margin >= target && target + margin >= v; }
  std::string describe() const {
    std::ostringstream o;
    o.precision(17);
    o << "is within " << margin << " of " << target;
    return o.str();
  }
};

inline WithinRelMatcher WithinRel(double target, double eps) { return {target, eps}; }
inline WithinRelMatcher WithinRel(double target) { return {target, std::numeric_limits<double>::epsilon() * 100}; }
inline WithinAbsMatcher WithinAbs(double target, double margin) { return {target, margin}; }

}  // namespace Matchers

/// Runs every registered test case (or those whose name contains `filter`).
inline int run_all(const char* filter) {
  using namespace detail;
  int cases = 0, failed_cases = 0;
  for (const TestCase& tc : registry()) {
    if (filter && tc.name.find(filter) == std::string::npos) continue;
    ++cases;
    RunState& s = state();
    const long long before = s.failures;
    s.test = tc.name;
    s.target = 0;
    do {
      s.seen = 0;
      s.section.clear();
      try {
        tc.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        report(false, false, "TEST_CASE", "", __FILE__, __LINE__, std::string("unexpected exception: ") + e.what());
      } catch (...) {
        report(false, false, "TEST_CASE", "", __FILE__, __LINE__, "unexpected exception");
      }
      ++s.target;
    } while (s.target < s.seen);
    if (s.failures != before) ++failed_cases;
  }
  const RunState& s = state();
  std::printf("%s: %d test cases (%d failed), %lld assertions (%lld failed)\n",
              failed_cases ? "FAILED" : "All tests passed", cases, failed_cases, s.assertions, s.failures);
  return failed_cases ? 1 : 0;
}

}  // namespace Catch

#define CATCHMINI_CAT2(a, b) a##b
#define CATCHMINI_CAT(a, b) CATCHMINI_CAT2(a, b)
#define CATCHMINI_UNIQ(p) CATCHMINI_CAT(p, __LINE__)

#define TEST_CASE(...)                                                                                 \
  static void CATCHMINI_UNIQ(catchmini_test_)();                                                       \
  static ::Catch::detail::Registrar CATCHMINI_UNIQ(catchmini_reg_)(                                    \
      ::Catch::detail::name_of(__VA_ARGS__), &CATCHMINI_UNIQ(catchmini_test_));                       \
  static void CATCHMINI_UNIQ(catchmini_test_)()

#define SECTION(...) if (::Catch::detail::enter_section(::Catch::detail::name_of(__VA_ARGS__)))

#define CATCHMINI_CHECK(macro, require, negate, ...)                                                      \
  do {                                                                                                   \
    bool catchmini_ok_ = false;                                                                          \
    try {                                                                                                \
      catchmini_ok_ = static_cast<bool>(__VA_ARGS__) != (negate);                                        \
    } catch (const std::exception& catchmini_e_) {                                                       \
      ::Catch::detail::report(false, require, macro, #__VA_ARGS__, __FILE__, __LINE__,                   \
                              std::string("exception: ") + catchmini_e_.what());                         \
      break;                                                                                             \
    }                                                                                                    \
    ::Catch::detail::report(catchmini_ok_, require, macro, #__VA_ARGS__, __FILE__, __LINE__);            \
  } while (0)

#define CHECK(...) CATCHMINI_CHECK("CHECK", false, false, __VA_ARGS__)
#define REQUIRE(...) CATCHMINI_CHECK("REQUIRE", true, false, __VA_ARGS__)
#define CHECK_FALSE(...) CATCHMINI_CHECK("CHECK_FALSE", false, true, __VA_ARGS__)
#define REQUIRE_FALSE(...) CATCHMINI_CHECK("REQUIRE_FALSE", true, true, __VA_ARGS__)

#define CATCHMINI_THROWS_AS(macro, require, expr, type)                                       \
  do {                                                                                       \
    bool catchmini_ok_ = false;                                                              \
    std::string catchmini_what_ = "no exception";                                            \
    try {                                                                                    \
      static_cast<void>(expr);                                                               \
    } catch (const type&) {                                                                  \
      catchmini_ok_ = true;                                                                  \
    } catch (const std::exception& catchmini_e_) {                                           \
      catchmini_what_ = std::string("other exception: ") + catchmini_e_.what();              \
    } catch (...) {                                                                          \
      catchmini_what_ = "other exception";                                                   \
    }                                                                                        \
    ::Catch::detail::report(catchmini_ok_, require, macro, #expr ", " #type, __FILE__, __LINE__, \
                            catchmini_ok_ ? std::string() : catchmini_what_);                \
  } while (0)

#define CHECK_THROWS_AS(expr, type) CATCHMINI_THROWS_AS("CHECK_THROWS_AS", false, expr, type)
#define REQUIRE_THROWS_AS(expr, type) CATCHMINI_THROWS_AS("REQUIRE_THROWS_AS", true, expr, type)

#define CATCHMINI_THROWS(macro, require, want, ...)                                      \
  do {                                                                                  \
    bool catchmini_threw_ = false;                                                      \
    try {                                                                               \
      static_cast<void>(__VA_ARGS__);                                                   \
    } catch (...) {                                                                     \
      catchmini_threw_ = true;                                                          \
    }                                                                                   \
    ::Catch::detail::report(catchmini_threw_ == (want), require, macro, #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)

#define CHECK_THROWS(...) CATCHMINI_THROWS("CHECK_THROWS", false, true, __VA_ARGS__)
#define REQUIRE_THROWS(...) CATCHMINI_THROWS("REQUIRE_THROWS", true, true, __VA_ARGS__)
#define CHECK_NOTHROW(...) CATCHMINI_THROWS("CHECK_NOTHROW", false, false, __VA_ARGS__)
#define REQUIRE_NOTHROW(...) CATCHMINI_THROWS("REQUIRE_NOTHROW", true, false, __VA_ARGS__)

#define CATCHMINI_THAT(macro, require, arg, matcher)                                               \
  do {                                                                                            \
    const double catchmini_v_ = static_cast<double>(arg);                                         \
    const auto catchmini_m_ = (matcher);                                                          \
    ::Catch::detail::report(catchmini_m_.match(catchmini_v_), require, macro, #arg ", " #matcher, \
                            __FILE__, __LINE__,                                                   \
                            ::Catch::detail::describe(catchmini_v_) + " " + catchmini_m_.describe()); \
  } while (0)

#define CHECK_THAT(arg, matcher) CATCHMINI_THAT("CHECK_THAT", false, arg, matcher)
#define REQUIRE_THAT(arg, matcher) CATCHMINI_THAT("REQUIRE_THAT", true, arg, matcher)
