// Minimal doctest-compatible test harness (the subset the reference's unit
// tests use: TEST_CASE, CHECK, CHECK_FALSE, CHECK_NOTHROW, CHECK_THROWS_AS,
// REQUIRE, FAIL, doctest::Approx).  doctest itself is not in this image; this
// is an independent implementation of the same macro surface so the
// reference's test sources compile unchanged against the drop-in library.
//
// Command line: an optional substring filter on test-case names
// (-tc=<substr> or a bare <substr>).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <ostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest {

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

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct State {
  long checks = 0, failures = 0;
  bool case_failed = false;
};
inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal, const std::string& values = "") {
  ++state().checks;
  if (ok) return;
  ++state().failures;
  state().case_failed = true;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED%s%s\n", file, line, fatal ? "REQUIRE" : "CHECK", expr,
               values.empty() ? "" : "  values: ", values.c_str());
  if (fatal) throw RequireFailed{};
}

// Expression decomposition (CHECK(a < b) reports both operands on failure).
template <class T>
std::string show(const T& v) {
  if constexpr (requires(std::ostream& o) { o << v; }) {
    std::ostringstream os;
    os.precision(17);
    os << v;
    return os.str();
  } else {
    return "{?}";
  }
}
struct Result {
  bool ok;
  std::string values;
};
template <class L>
struct ExprLhs {
  const L& lhs;
  operator Result() const { return {static_cast<bool>(lhs), show(lhs)}; }
#define DOCTEST_BINOP(op)                                                      \
  template <class R>                                                           \
  Result operator op(const R& rhs) const {                                     \
    return {static_cast<bool>(lhs op rhs), show(lhs) + " " #op " " + show(rhs)}; \
  }
  DOCTEST_BINOP(==)
  DOCTEST_BINOP(!=)
  DOCTEST_BINOP(<)
  DOCTEST_BINOP(<=)
  DOCTEST_BINOP(>)
  DOCTEST_BINOP(>=)
#undef DOCTEST_BINOP
};
struct ExprStart {
  template <class L>
  ExprLhs<L> operator<=(const L& lhs) const {
    return {lhs};
  }
};
inline Result to_result(const Result& r) { return r; }
template <class L>
Result to_result(const ExprLhs<L>& e) {
  return static_cast<Result>(e);
}

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
  bool matches(double x) const {
    return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
  }
  friend bool operator==(double x, const Approx& a) { return a.matches(x); }
  friend bool operator==(const Approx& a, double x) { return a.matches(x); }
  friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }
  friend bool operator!=(const Approx& a, double x) { return !a.matches(x); }
  friend bool operator<=(double x, const Approx& a) { return x < a.value_ || a.matches(x); }
  friend bool operator>=(double x, const Approx& a) { return x > a.value_ || a.matches(x); }
  friend bool operator<=(const Approx& a, double x) { return a.value_ < x || a.matches(x); }
  friend bool operator>=(const Approx& a, double x) { return a.value_ > x || a.matches(x); }

 private:
  double value_;
  double eps_ = 1.1920929e-7f * 100;  // doctest's default: float epsilon * 100
  double scale_ = 1.0;
};

inline int run(int argc, char** argv) {
  std::string filter;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    if (a.rfind("-tc=", 0) == 0) filter = a.substr(4);
    else if (a[0] != '-') filter = a;
  }
  int ran = 0, failed_cases = 0;
  for (const auto& tc : registry()) {
    if (!filter.empty() && std::string(tc.name).find(filter) == std::string::npos) continue;
    ++ran;
    state().case_failed = false;
    std::fprintf(stderr, "[ RUN  ] %s\n", tc.name);
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++state().failures;
      state().case_failed = true;
      std::fprintf(stderr, "%s:%d: unexpected exception: %s\n", tc.file, tc.line, e.what());
    } catch (...) {
      ++state().failures;
      state().case_failed = true;
      std::fprintf(stderr, "%s:%d: unexpected exception\n", tc.file, tc.line);
    }
    if (state().case_failed) ++failed_cases;
    std::fprintf(stderr, "[ %s ] %s\n", state().case_failed ? "FAIL" : " OK ", tc.name);
  }
  std::printf("test cases: %d | %d passed | %d failed\nassertions: %ld | %ld failed\n", ran, ran - failed_cases,
              failed_cases, state().checks, state().failures);
  return failed_cases ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(name, fn)                                                               \
  static void fn();                                                                             \
  static const doctest::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);       \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(name, DOCTEST_CAT(doctest_tc_, __COUNTER__))

#define DOCTEST_EVAL(fatal, ...)                                                                \
  do {                                                                                          \
    const doctest::Result doctest_r_ = doctest::to_result(doctest::ExprStart() <= __VA_ARGS__);  \
    doctest::report(doctest_r_.ok, #__VA_ARGS__, __FILE__, __LINE__, fatal, doctest_r_.values); \
  } while (0)
#define CHECK(...) DOCTEST_EVAL(false, __VA_ARGS__)
#define CHECK_FALSE(...) doctest::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) DOCTEST_EVAL(true, __VA_ARGS__)
#define FAIL(msg)                                                                               \
  do {                                                                                          \
    std::ostringstream doctest_os_;                                                             \
    doctest_os_ << msg;                                                                         \
    doctest::report(false, doctest_os_.str().c_str(), __FILE__, __LINE__, true);               \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                              \
  do {                                                                                          \
    bool doctest_ok_ = false;                                                                   \
    try {                                                                                       \
      (void)(expr);                                                                             \
    } catch (const __VA_ARGS__&) {                                                              \
      doctest_ok_ = true;                                                                       \
    } catch (...) {                                                                             \
    }                                                                                           \
    doctest::report(doctest_ok_, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__, false);    \
  } while (0)
#define CHECK_NOTHROW(...)                                                                      \
  do {                                                                                          \
    bool doctest_ok_ = true;                                                                    \
    try {                                                                                       \
      (void)(__VA_ARGS__);                                                                      \
    } catch (...) {                                                                             \
      doctest_ok_ = false;                                                                      \
    }                                                                                           \
    doctest::report(doctest_ok_, #__VA_ARGS__ " does not throw", __FILE__, __LINE__, false);   \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::run(argc, argv); }
#endif
