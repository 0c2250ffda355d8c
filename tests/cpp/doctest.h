// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE ONLY).
//
// The image has no doctest; this header implements the subset the reference's
// own test files use (test_engine.cpp, test_conv.cpp): TEST_CASE, SUBCASE
// (re-run-per-leaf semantics, nestable), CHECK / REQUIRE, CHECK_THROWS,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, CHECK_NOTHROW, doctest::Approx with
// .epsilon(), doctest::Contains, and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
// It lets those files compile unchanged against the B200 drop-in shims.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <set>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  double v, eps = 1.1920928955078125e-07 * 100, scale = 1.0;
  explicit Approx(double x) : v(x) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v) < b.eps * (b.scale + std::max(std::fabs(a), std::fabs(b.v)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
};

struct Contains {
  std::string s;
  explicit Contains(const char* x) : s(x) {}
  bool matches(const std::string& m) const { return m.find(s) != std::string::npos; }
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

struct Reg {
  Reg(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};

struct State {
  int failed_checks = 0, total_checks = 0;
  bool case_failed = false;
  // subcase bookkeeping for the current test case
  std::set<std::string> done;
  std::vector<std::string> path;        // names of the entered subcases
  std::vector<bool> entered_at_depth;   // a subcase already ran at this depth in this pass
  std::vector<bool> pending_at_depth;   // a not-done subcase was skipped at this depth
  bool entered_any = false;
};

inline State& st() {
  static State s;
  return s;
}

struct RequireAbort {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   const std::string& extra = "") {
  auto& s = st();
  ++s.total_checks;
  if (ok) return;
  ++s.failed_checks;
  s.case_failed = true;
  std::printf("%s:%d: FAILED %s( %s )%s%s\n", file, line, kind, expr, extra.empty() ? "" : " ", extra.c_str());
}

inline std::string joined(const std::vector<std::string>& p, const std::string& leaf) {
  std::string r;
  for (const auto& x : p) r += x + "/";
  return r + leaf;
}

struct Subcase {
  bool run = false;
  std::string full;
  Subcase(const char* name) {
    auto& s = st();
    const std::size_t d = s.path.size();
    if (s.entered_at_depth.size() <= d) {
      s.entered_at_depth.resize(d + 1, false);
      s.pending_at_depth.resize(d + 1, false);
    }
    full = joined(s.path, name);
    if (s.done.count(full)) return;
    if (s.entered_at_depth[d]) {
      s.pending_at_depth[d] = true;  // a sibling ran this pass: come back later
      return;
    }
    run = true;
    s.entered_at_depth[d] = true;
    s.entered_any = true;
    s.path.push_back(name);
    if (s.entered_at_depth.size() <= d + 1) {
      s.entered_at_depth.resize(d + 2, false);
      s.pending_at_depth.resize(d + 2, false);
    }
    s.entered_at_depth[d + 1] = false;
    s.pending_at_depth[d + 1] = false;
  }
  ~Subcase() {
    if (!run) return;
    auto& s = st();
    const std::size_t d = s.path.size();  // depth of this subcase's children
    if (!s.pending_at_depth[d]) s.done.insert(full);
    s.path.pop_back();
  }
  explicit operator bool() const { return run; }
};

inline int run_all() {
  int failed_cases = 0, cases = 0;
  for (const auto& tc : registry()) {
    ++cases;
    auto& s = st();
    s.done.clear();
    s.case_failed = false;
    for (int pass = 0; pass < 4096; ++pass) {
      s.path.clear();
      s.entered_at_depth.assign(1, false);
      s.pending_at_depth.assign(1, false);
      s.entered_any = false;
      try {
        tc.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        report(false, "TEST_CASE", tc.name, tc.file, tc.line, std::string("threw: ") + e.what());
      } catch (...) {
        report(false, "TEST_CASE", tc.name, tc.file, tc.line, "threw a non-std exception");
      }
      if (!s.entered_any) break;
    }
    if (s.case_failed) {
      ++failed_cases;
      std::printf("[FAIL] %s\n", tc.name);
    } else {
      std::printf("[ ok ] %s\n", tc.name);
    }
  }
  auto& s = st();
  std::printf("[doctest-mini] test cases: %d | %d passed | %d failed; assertions: %d | %d failed\n", cases,
              cases - failed_cases, failed_cases, s.total_checks, s.failed_checks);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                          \
  static void fn();                                                                        \
  static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);       \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name})

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                       \
  do {                                                                                                     \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                               \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                   \
    if (!doctest_ok_) throw ::doctest::detail::RequireAbort{};                                             \
  } while (0)
#define CHECK_THROWS(...)                                                                                  \
  do {                                                                                                     \
    bool doctest_threw_ = false;                                                                           \
    try { (void)(__VA_ARGS__); } catch (...) { doctest_threw_ = true; }                                    \
    ::doctest::detail::report(doctest_threw_, "CHECK_THROWS", #__VA_ARGS__, __FILE__, __LINE__);           \
  } while (0)
#define CHECK_NOTHROW(...)                                                                                 \
  do {                                                                                                     \
    bool doctest_ok_ = true;                                                                               \
    try { (void)(__VA_ARGS__); } catch (...) { doctest_ok_ = false; }                                      \
    ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__);             \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                         \
  do {                                                                                                     \
    bool doctest_ok_ = false;                                                                              \
    try { (void)(expr); } catch (const __VA_ARGS__&) { doctest_ok_ = true; } catch (...) {}                \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                              \
  do {                                                                                                     \
    bool doctest_ok_ = false;                                                                              \
    try { (void)(expr); } catch (const __VA_ARGS__& e_) {                                                  \
      doctest_ok_ = ::doctest::Contains(with).matches(e_.what());                                          \
    } catch (...) {}                                                                                       \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__);             \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
