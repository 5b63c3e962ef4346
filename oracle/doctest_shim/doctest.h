/*
 * Minimal doctest-compatible test harness — TEST INFRASTRUCTURE ONLY.
 *
 * The reference's tests include <doctest.h> from proj/vendor/, which is
 * gitignored and absent (/root/reference/proj/.gitignore:2).  This
 * builder-written header implements only the macros the reference's
 * test_fft.cpp / test_problems.cpp use (TEST_CASE, CHECK, REQUIRE,
 * CHECK_THROWS_AS, CHECK_MESSAGE, MESSAGE, doctest::Approx(..).epsilon(..))
 * with doctest's documented semantics, so those files compile unmodified.
 * Define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN in exactly one TU (the
 * reference's own test_main.cpp does) to get main().
 */
#ifndef ORACLE_DOCTEST_SHIM_H
#define ORACLE_DOCTEST_SHIM_H

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value)
      : eps_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100), scale_(1.0), value_(value) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) < rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }
  double value() const { return value_; }

 private:
  double eps_, scale_, value_;
};

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

struct State {
  long checks = 0, failed_checks = 0;
  bool current_failed = false;
};

inline State& state() {
  static State s;
  return s;
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct RequireAbort {};

inline void report(bool ok, const char* expr, const char* file, int line, const std::string& msg, bool require) {
  State& s = state();
  ++s.checks;
  if (!ok) {
    ++s.failed_checks;
    s.current_failed = true;
    if (s.failed_checks <= 50)
      std::fprintf(stderr, "%s:%d: CHECK FAILED: %s %s\n", file, line, expr, msg.c_str());
    if (require) throw RequireAbort{};
  }
}

template <typename... Args>
std::string cat(const Args&... args) {
  std::ostringstream os;
  os.precision(17);
  (os << ... << args);
  return os.str();
}

inline int run_all() {
  int failed_cases = 0;
  for (const auto& t : registry()) {
    state().current_failed = false;
    try {
      t.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: TEST CASE THREW: %s\n", t.file, t.line, e.what());
      state().current_failed = true;
    }
    std::printf("[%s] %s\n", state().current_failed ? "FAIL" : " ok ", t.name);
    if (state().current_failed) ++failed_cases;
  }
  std::printf("test cases: %zu | %zu passed | %d failed\n", registry().size(), registry().size() - failed_cases,
              failed_cases);
  std::printf("assertions: %ld | %ld passed | %ld failed\n", state().checks, state().checks - state().failed_checks,
              state().failed_checks);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                              \
  static void fn();                                                                                   \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);           \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, "", false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, "", true)
#define CHECK_MESSAGE(cond, ...) \
  ::doctest::detail::report(static_cast<bool>(cond), #cond, __FILE__, __LINE__, ::doctest::detail::cat(__VA_ARGS__), false)
#define MESSAGE(...) std::printf("MESSAGE: %s\n", ::doctest::detail::cat(__VA_ARGS__).c_str())
#define CHECK_THROWS_AS(expr, exc)                                                                 \
  do {                                                                                             \
    bool doctest_threw_ = false;                                                                   \
    try {                                                                                          \
      (void)(expr);                                                                                \
    } catch (const exc&) {                                                                         \
      doctest_threw_ = true;                                                                       \
    } catch (...) {                                                                                \
    }                                                                                              \
    ::doctest::detail::report(doctest_threw_, "throws " #exc ": " #expr, __FILE__, __LINE__, "", false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif

#endif
