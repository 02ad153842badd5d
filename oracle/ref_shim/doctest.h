// ref_shim/doctest.h -- TEST-ONLY minimal stand-in for the doctest macros used
// by /root/reference/proj/tests (doctest is gitignored under proj/vendor/ and
// absent from this image).  Written from scratch: registration, CHECK/REQUIRE,
// CHECK_THROWS_AS, FAIL, MESSAGE, SUBCASE (every subcase runs once, in order)
// and doctest::Approx with doctest's published comparison rule
//   |lhs - rhs| < epsilon * (scale + max(|lhs|, |rhs|)), epsilon = 100*FLT_EPSILON, scale = 1.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }
  friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || lhs == rhs; }
  friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || lhs == rhs; }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

struct Contains {
  std::string s;
  explicit Contains(std::string x) : s(std::move(x)) {}
  bool matches(const std::string& what) const { return what.find(s) != std::string::npos; }
};
inline bool message_matches(const std::string& what, const Contains& c) { return c.matches(what); }
inline bool message_matches(const std::string& what, const char* s) { return what == s; }

namespace detail {
struct TestCase {
  const char* name;
  void (*fn)();
  const char* file;
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file) { registry().push_back({name, fn, file}); }
};
struct AbortTest {};
inline int& failures() { static int f = 0; return f; }
inline int& checks() { static int c = 0; return c; }
inline const char*& current() { static const char* c = ""; return c; }
inline void report(const char* file, int line, const char* what) {
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, current(), what);
}
template <typename... T>
inline std::string concat(const T&... xs) {
  std::ostringstream os;
  (os << ... << xs);
  return os.str();
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                  \
  static void fn();                                                                \
  static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__);   \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) if (true)

#define CHECK(...)                                                                         \
  do {                                                                                     \
    ++doctest::detail::checks();                                                           \
    if (!(__VA_ARGS__)) doctest::detail::report(__FILE__, __LINE__, "CHECK(" #__VA_ARGS__ ")"); \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                         \
  do {                                                                                       \
    ++doctest::detail::checks();                                                             \
    if (!(__VA_ARGS__)) {                                                                    \
      doctest::detail::report(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")");              \
      throw doctest::detail::AbortTest{};                                                    \
    }                                                                                        \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                           \
  do {                                                                                       \
    ++doctest::detail::checks();                                                             \
    bool ok_ = false;                                                                        \
    try {                                                                                    \
      (void)(expr);                                                                          \
    } catch (const __VA_ARGS__&) {                                                           \
      ok_ = true;                                                                            \
    } catch (...) {                                                                          \
    }                                                                                        \
    if (!ok_) doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ")");     \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                             \
  do {                                                                                       \
    ++doctest::detail::checks();                                                             \
    bool ok_ = false;                                                                        \
    try {                                                                                    \
      (void)(expr);                                                                          \
    } catch (const __VA_ARGS__& e_) {                                                        \
      ok_ = doctest::message_matches(e_.what(), matcher);                                    \
    } catch (...) {                                                                          \
    }                                                                                        \
    if (!ok_) doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_WITH_AS(" #expr ")"); \
  } while (0)
#define FAIL(msg)                                                       \
  do {                                                                  \
    doctest::detail::report(__FILE__, __LINE__, "FAIL: " msg);          \
    throw doctest::detail::AbortTest{};                                 \
  } while (0)
#define MESSAGE(...) \
  std::fprintf(stderr, "%s:%d: MESSAGE: %s\n", __FILE__, __LINE__, doctest::detail::concat(__VA_ARGS__).c_str())

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int cases = 0, failed_cases = 0;
  for (const auto& tc : doctest::detail::registry()) {
    doctest::detail::current() = tc.name;
    const int before = doctest::detail::failures();
    try {
      tc.fn();
    } catch (const doctest::detail::AbortTest&) {
    } catch (const std::exception& e) {
      doctest::detail::report(tc.file, 0, (std::string("unexpected exception: ") + e.what()).c_str());
    }
    ++cases;
    if (doctest::detail::failures() != before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %d | passed: %d | failed: %d | checks: %d | failed checks: %d\n",
              cases, cases - failed_cases, failed_cases, doctest::detail::checks(),
              doctest::detail::failures());
  return failed_cases == 0 ? 0 : 1;
}
#endif
