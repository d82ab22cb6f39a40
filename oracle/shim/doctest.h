// doctest-subset shim — TEST INFRASTRUCTURE for the parity oracle only.
//
// The reference's unit tests include <doctest.h> from its git-ignored vendor/
// directory (absent, proj/.gitignore:2).  This header implements the subset
// they use: TEST_CASE, flat SUBCASE, CHECK / CHECK_FALSE / CHECK_THROWS_AS /
// CHECK_NOTHROW, REQUIRE / REQUIRE_MESSAGE, FAIL, CAPTURE and doctest::Approx
// (same comparison rule as doctest: |a-b| < eps * (scale + max(|a|, |b|))).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <set>
#include <sstream>
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
  double eps_ = 1.1920928955078125e-07 * 100;
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

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct RequireFailed {};

struct State {
  int asserts = 0;
  int failed_asserts = 0;
  bool current_failed = false;
  const TestCase* current = nullptr;
  // Flat SUBCASE bookkeeping.
  std::set<std::string> done_subcases;
  bool entered_subcase = false;
  bool saw_new_subcase = false;
  std::vector<std::string> captures;
};

inline State& state() {
  static State s;
  return s;
}

inline void report_failure(const char* file, int line, const std::string& what) {
  State& s = state();
  ++s.failed_asserts;
  s.current_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line,
               s.current ? s.current->name : "?", what.c_str());
  for (const auto& c : s.captures) std::fprintf(stderr, "    with %s\n", c.c_str());
}

inline void check(bool ok, const char* file, int line, const char* expr, bool require) {
  ++state().asserts;
  if (!ok) {
    report_failure(file, line, expr);
    if (require) throw RequireFailed{};
  }
}

struct Subcase {
  bool active = false;
  std::string key;
  Subcase(const char* name, const char* file, int line) {
    State& s = state();
    key = std::string(file) + ":" + std::to_string(line) + ":" + name;
    if (s.entered_subcase || s.done_subcases.count(key)) {
      if (!s.done_subcases.count(key)) s.saw_new_subcase = true;
      return;
    }
    s.entered_subcase = true;
    active = true;
  }
  ~Subcase() {
    if (active) state().done_subcases.insert(key);
  }
  explicit operator bool() const { return active; }
};

struct Capture {
  Capture(const char* name, const std::string& value) {
    state().captures.push_back(std::string(name) + " := " + value);
  }
  ~Capture() { state().captures.pop_back(); }
};

template <typename T>
std::string stringify(const T& v) {
  std::ostringstream os;
  os << v;
  return os.str();
}

inline int run_all() {
  State& s = state();
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    s.current = &tc;
    s.current_failed = false;
    s.done_subcases.clear();
    for (int run = 0; run < 1000; ++run) {
      s.entered_subcase = false;
      s.saw_new_subcase = false;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        report_failure(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
      } catch (...) {
        report_failure(tc.file, tc.line, "unexpected unknown exception");
      }
      s.captures.clear();
      if (!s.saw_new_subcase) break;
    }
    if (s.current_failed) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - failed_cases, failed_cases);
  std::printf("[doctest-shim] assertions: %d | %d passed | %d failed\n", s.asserts,
              s.asserts - s.failed_asserts, s.failed_asserts);
  std::printf("[doctest-shim] Status: %s\n", failed_cases ? "FAILURE!" : "SUCCESS!");
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                        \
  static void DOCTEST_ANON(doctest_fn_)();                                                     \
  static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__,     \
                                                                 &DOCTEST_ANON(doctest_fn_)); \
  static void DOCTEST_ANON(doctest_fn_)()

#define SUBCASE(name) \
  if (const ::doctest::detail::Subcase DOCTEST_ANON(doctest_sc_){name, __FILE__, __LINE__})

#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define CHECK_FALSE(...) \
  ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define REQUIRE_MESSAGE(cond, msg)                                                         \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      std::ostringstream doctest_os_;                                                      \
      doctest_os_ << msg;                                                                  \
      ::doctest::detail::check(false, __FILE__, __LINE__, doctest_os_.str().c_str(), true); \
    } else {                                                                               \
      ::doctest::detail::check(true, __FILE__, __LINE__, "", true);                        \
    }                                                                                      \
  } while (0)
#define FAIL(msg)                                                                      \
  do {                                                                                 \
    std::ostringstream doctest_os_;                                                    \
    doctest_os_ << msg;                                                                \
    ::doctest::detail::check(false, __FILE__, __LINE__, doctest_os_.str().c_str(), true); \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                           \
  do {                                                                                       \
    bool doctest_ok_ = false;                                                                \
    try {                                                                                    \
      static_cast<void>(expr);                                                               \
    } catch (const __VA_ARGS__&) {                                                           \
      doctest_ok_ = true;                                                                    \
    } catch (...) {                                                                          \
    }                                                                                        \
    ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "THROWS_AS(" #expr ")", false); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                               \
  do {                                                                                    \
    bool doctest_ok_ = true;                                                              \
    try {                                                                                 \
      static_cast<void>(expr);                                                            \
    } catch (...) {                                                                       \
      doctest_ok_ = false;                                                                \
    }                                                                                     \
    ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "NOTHROW(" #expr ")", false); \
  } while (0)
#define CAPTURE(x) \
  const ::doctest::detail::Capture DOCTEST_ANON(doctest_cap_)(#x, ::doctest::detail::stringify(x))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
