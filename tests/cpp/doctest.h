// TEST INFRASTRUCTURE ONLY — a minimal stand-in for the doctest single header
// (absent from this image) covering exactly the macros the
// reference's unit tests use: TEST_SUITE, TEST_CASE, CHECK, CHECK_FALSE,
// REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, CHECK_NOTHROW, MESSAGE, FAIL,
// SUBCASE (flat, one leaf per pass of the test case, as doctest runs them) and
// doctest::Approx. It lets /root/reference/proj/tests/test_{gating,des,
// baselines,trace}.cpp compile UNCHANGED against this repo's C++ facade
// (include/dessim/*.hpp).
// Define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN in exactly one translation unit.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
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
  long asserts = 0, failed_asserts = 0;
  bool current_failed = false;
  int sub_target = 0, sub_seen = 0;  // SUBCASE: the leaf this pass runs / leaves met
};

inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

// true for exactly one SUBCASE per pass of the enclosing test case
inline bool enter_subcase() {
  State& s = state();
  return s.sub_seen++ == s.sub_target;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   const std::string& extra = std::string()) {
  State& s = state();
  ++s.asserts;
  if (ok) return;
  ++s.failed_asserts;
  s.current_failed = true;
  std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct!%s%s\n", file, line, kind, expr,
               extra.empty() ? "" : " ", extra.c_str());
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
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value_) <
           a.eps_ * (a.scale_ + std::fmax(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

 private:
  double value_;
  double eps_ = 1.19209290e-05 * 100;  // doctest's default: float epsilon * 100
  double scale_ = 1.0;
};

inline int run_all() {
  int failed = 0, passed = 0;
  for (const TestCase& tc : registry()) {
    state().current_failed = false;
    state().sub_target = 0;
    do {  // one pass per SUBCASE leaf (a single pass without subcases)
      state().sub_seen = 0;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        report(false, "TEST_CASE", tc.name, tc.file, tc.line,
               std::string("threw exception: ") + e.what());
      } catch (...) {
        report(false, "TEST_CASE", tc.name, tc.file, tc.line, "threw unknown exception");
      }
    } while (++state().sub_target < state().sub_seen);
    if (state().current_failed) {
      ++failed;
      std::fprintf(stderr, "[doctest] FAILED: %s (%s:%d)\n", tc.name, tc.file, tc.line);
    } else {
      ++passed;
    }
  }
  std::printf("[doctest] test cases: %d | %d passed | %d failed\n", passed + failed, passed,
              failed);
  std::printf("[doctest] assertions: %ld | %ld passed | %ld failed\n", state().asserts,
              state().asserts - state().failed_asserts, state().failed_asserts);
  return failed ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define DOCTEST_TEST_CASE_IMPL(fn, reg, name)                               \
  static void fn();                                                        \
  static ::doctest::Registrar reg(name, __FILE__, __LINE__, &fn);          \
  static void fn()
#define TEST_CASE(name)                                                           \
  DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__),                    \
                         DOCTEST_CAT(doctest_reg_, __LINE__), name)
#define TEST_SUITE(name) namespace DOCTEST_CAT(doctest_suite_, __LINE__)
#define SUBCASE(name) if (::doctest::enter_subcase())
#define FAIL(msg)                                                            \
  do {                                                                       \
    ::doctest::report(false, "FAIL", msg, __FILE__, __LINE__);               \
    throw ::doctest::RequireFailed();                                        \
  } while (0)

#define CHECK(...) ::doctest::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                        \
  do {                                                                                      \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                \
    ::doctest::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);            \
    if (!doctest_ok_) throw ::doctest::RequireFailed();                                     \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                          \
  do {                                                                                      \
    bool doctest_ok_ = false;                                                               \
    std::string doctest_why_ = "did not throw";                                             \
    try {                                                                                   \
      static_cast<void>(expr);                                                              \
    } catch (const __VA_ARGS__&) {                                                          \
      doctest_ok_ = true;                                                                   \
    } catch (const std::exception& e_) {                                                    \
      doctest_why_ = std::string("threw a different type: ") + e_.what();                   \
    } catch (...) {                                                                         \
      doctest_why_ = "threw a different type";                                              \
    }                                                                                       \
    ::doctest::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__,    \
                      __LINE__, doctest_ok_ ? std::string() : doctest_why_);                \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, ...)                                                \
  do {                                                                                      \
    bool doctest_ok_ = false;                                                               \
    std::string doctest_why_ = "did not throw";                                             \
    try {                                                                                   \
      static_cast<void>(expr);                                                              \
    } catch (const __VA_ARGS__& e_) {                                                       \
      doctest_ok_ = std::string(e_.what()) == std::string(msg);                             \
      doctest_why_ = std::string("message was: ") + e_.what();                              \
    } catch (...) {                                                                         \
      doctest_why_ = "threw a different type";                                              \
    }                                                                                       \
    ::doctest::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr ", " #msg, __FILE__,       \
                      __LINE__, doctest_ok_ ? std::string() : doctest_why_);                \
  } while (0)
#define CHECK_NOTHROW(...)                                                                  \
  do {                                                                                      \
    bool doctest_ok_ = true;                                                                \
    std::string doctest_why_;                                                               \
    try {                                                                                   \
      static_cast<void>(__VA_ARGS__);                                                       \
    } catch (const std::exception& e_) {                                                    \
      doctest_ok_ = false;                                                                  \
      doctest_why_ = e_.what();                                                             \
    } catch (...) {                                                                         \
      doctest_ok_ = false;                                                                  \
    }                                                                                       \
    ::doctest::report(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__,       \
                      doctest_why_);                                                        \
  } while (0)
#define MESSAGE(...) std::fprintf(stderr, "[doctest] message at %s:%d\n", __FILE__, __LINE__)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::run_all(); }
#endif
