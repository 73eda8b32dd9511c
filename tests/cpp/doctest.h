// doctest.h — a minimal, independent implementation of the subset of the
// doctest testing API used by the reference's unit suites (TEST_CASE,
// SUBCASE with re-entry, CHECK / CHECK_FALSE / REQUIRE / FAIL,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, doctest::Approx, doctest::Contains).
// The real doctest is not vendored in the reference mount and there is no
// network; this shim lets the reference's own test sources compile, unmodified,
// against this repository's moeplan headers (tests/test_reference_suites.py).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <string>
#include <type_traits>
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
  bool matches(double other) const {
    return std::fabs(other - value_) < eps_ * (scale_ + std::max(std::fabs(other), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = double(std::numeric_limits<float>::epsilon()) * 100.0;
  double scale_ = 1.0;
};

template <typename T, typename = typename std::enable_if<std::is_constructible<double, T>::value>::type>
bool operator==(const T& lhs, const Approx& rhs) { return rhs.matches(double(lhs)); }
template <typename T, typename = typename std::enable_if<std::is_constructible<double, T>::value>::type>
bool operator==(const Approx& lhs, const T& rhs) { return lhs.matches(double(rhs)); }
template <typename T, typename = typename std::enable_if<std::is_constructible<double, T>::value>::type>
bool operator!=(const T& lhs, const Approx& rhs) { return !rhs.matches(double(lhs)); }
template <typename T, typename = typename std::enable_if<std::is_constructible<double, T>::value>::type>
bool operator!=(const Approx& lhs, const T& rhs) { return !lhs.matches(double(rhs)); }
template <typename T, typename = typename std::enable_if<std::is_constructible<double, T>::value>::type>
bool operator<=(const T& lhs, const Approx& rhs) { return double(lhs) < rhs.value() || rhs.matches(double(lhs)); }
template <typename T, typename = typename std::enable_if<std::is_constructible<double, T>::value>::type>
bool operator>=(const T& lhs, const Approx& rhs) { return double(lhs) > rhs.value() || rhs.matches(double(lhs)); }
template <typename T, typename = typename std::enable_if<std::is_constructible<double, T>::value>::type>
bool operator<(const T& lhs, const Approx& rhs) { return double(lhs) < rhs.value() && !rhs.matches(double(lhs)); }
template <typename T, typename = typename std::enable_if<std::is_constructible<double, T>::value>::type>
bool operator>(const T& lhs, const Approx& rhs) { return double(lhs) > rhs.value() && !rhs.matches(double(lhs)); }

struct Contains {
  explicit Contains(const char* s) : needle(s) {}
  bool matches(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
  std::string needle;
};

}  // namespace doctest

namespace doctest_shim {

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
  Registrar(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};

// Subcase exploration: each run of a test case enters at most one unexplored
// subcase per nesting level; a subcase is complete once none of its children
// was left pending. The test case is re-run until nothing is pending.
struct State {
  std::vector<std::string> stack;
  std::vector<bool> taken;
  std::vector<bool> pending;
  std::set<std::vector<std::string>> done;
  long failures = 0;
  long checks = 0;
  std::string current;
};

inline State& state() {
  static State s;
  return s;
}

struct AbortTest {};

struct SubcaseGuard {
  bool entered = false;
  std::size_t depth = 0;
  explicit SubcaseGuard(const char* name) {
    State& s = state();
    depth = s.stack.size();
    if (s.taken.size() <= depth + 1) {
      s.taken.resize(depth + 2, false);
      s.pending.resize(depth + 2, false);
    }
    std::vector<std::string> path = s.stack;
    path.emplace_back(name);
    if (s.done.count(path)) return;
    if (s.taken[depth]) {
      s.pending[depth] = true;
      return;
    }
    s.taken[depth] = true;
    s.stack = path;
    s.taken[depth + 1] = false;
    s.pending[depth + 1] = false;
    entered = true;
  }
  ~SubcaseGuard() {
    if (!entered) return;
    State& s = state();
    if (!s.pending[depth + 1])
      s.done.insert(s.stack);
    else
      s.pending[depth] = true;  // unexplored children: re-run through this subcase
    s.stack.pop_back();
  }
  explicit operator bool() const { return entered; }
};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  std::string where;
  for (const auto& p : s.stack) where += " / " + p;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s )  [%s%s]\n", file, line, kind, expr, s.current.c_str(), where.c_str());
}

inline bool match(const std::string& what, const doctest::Contains& m) { return m.matches(what); }
inline bool match(const std::string& what, const char* exact) { return what == exact; }
inline bool match(const std::string& what, const std::string& exact) { return what == exact; }

inline int run_all() {
  State& s = state();
  int failed_cases = 0;
  for (const auto& tc : registry()) {
    s.current = tc.name;
    s.done.clear();
    const long before = s.failures;
    for (int run = 0; run < 10000; ++run) {
      s.stack.clear();
      s.taken.assign(2, false);
      s.pending.assign(2, false);
      try {
        tc.fn();
      } catch (const AbortTest&) {
      } catch (const std::exception& e) {
        ++s.failures;
        std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", tc.file, tc.line, tc.name, e.what());
      } catch (...) {
        ++s.failures;
        std::fprintf(stderr, "%s:%d: test case '%s' threw a non-std exception\n", tc.file, tc.line, tc.name);
      }
      if (!s.pending[0]) break;
    }
    if (s.failures > before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %ld | %ld failed\n",
              registry().size(), registry().size() - std::size_t(failed_cases), failed_cases, s.checks, s.failures);
  return failed_cases ? 1 : 0;
}

}  // namespace doctest_shim

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)

#define TEST_CASE(name)                                                                                      \
  static void DOCTEST_SHIM_CAT(doctest_shim_fn_, __LINE__)();                                                \
  static ::doctest_shim::Registrar DOCTEST_SHIM_CAT(doctest_shim_reg_, __LINE__)(                            \
      name, __FILE__, __LINE__, &DOCTEST_SHIM_CAT(doctest_shim_fn_, __LINE__));                              \
  static void DOCTEST_SHIM_CAT(doctest_shim_fn_, __LINE__)()

#define SUBCASE(name) if (::doctest_shim::SubcaseGuard doctest_shim_sg{name}; doctest_shim_sg)

#define CHECK(...) ::doctest_shim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  ::doctest_shim::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                  \
  do {                                                                                                \
    const bool doctest_shim_ok = static_cast<bool>(__VA_ARGS__);                                      \
    ::doctest_shim::report(doctest_shim_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);             \
    if (!doctest_shim_ok) throw ::doctest_shim::AbortTest{};                                          \
  } while (0)
#define FAIL(msg)                                                                 \
  do {                                                                            \
    ::doctest_shim::report(false, "FAIL", #msg, __FILE__, __LINE__);              \
    throw ::doctest_shim::AbortTest{};                                            \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                              \
  do {                                                                                          \
    bool doctest_shim_ok = false;                                                               \
    try {                                                                                       \
      (void)(expr);                                                                             \
    } catch (const __VA_ARGS__&) {                                                              \
      doctest_shim_ok = true;                                                                   \
    } catch (...) {                                                                             \
    }                                                                                           \
    ::doctest_shim::report(doctest_shim_ok, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);      \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                        \
  do {                                                                                               \
    bool doctest_shim_ok = false;                                                                    \
    try {                                                                                            \
      (void)(expr);                                                                                  \
    } catch (const __VA_ARGS__& doctest_shim_e) {                                                    \
      doctest_shim_ok = ::doctest_shim::match(doctest_shim_e.what(), with);                          \
    } catch (...) {                                                                                  \
    }                                                                                                \
    ::doctest_shim::report(doctest_shim_ok, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__);      \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest_shim::run_all(); }
#endif
