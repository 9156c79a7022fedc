// doctest.h -- the subset of doctest (https://github.com/doctest/doctest) the
// reference's test suites use (proj/tests/test_*.cpp: TEST_CASE, SUBCASE,
// CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, doctest::Approx), written for
// this repository so those suites compile and run unmodified against the
// GPU-backed reference ABI (oracle/refabi/refabi_shim.cpp).  Test
// infrastructure only.  doctest itself is not in the reference tree.
//
// SUBCASE follows doctest's traversal: a test case body runs once per leaf
// subcase path; in each run, at every nesting level, the first subcase not
// yet completed is entered and its later siblings are skipped.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <set>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) <= b.eps_ * (1.0 + std::max(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }

 private:
  double v_;
  double eps_ = 1.1920929e-7f * 100;  // doctest's default: float epsilon x 100
};

namespace detail {

struct Registry {
  struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
  };
  std::vector<Case> cases;
  static Registry& get() {
    static Registry r;
    return r;
  }
};
struct Register {
  Register(const char* name, const char* file, int line, void (*fn)()) {
    Registry::get().cases.push_back({name, file, line, fn});
  }
};

struct State {
  int checks = 0, failures = 0;
  bool case_failed = false;
  std::string current;
  // subcase traversal
  std::set<std::string> done;
  std::vector<std::string> path;
  std::vector<bool> entered_at;  // per depth: a subcase was entered in this run
  std::vector<bool> incomplete;  // per depth: the entered subcase skipped children
  bool rerun = false;
  static State& get() {
    static State s;
    return s;
  }
};

struct RequireFailure {};

inline void report(bool ok, const char* expr, const char* file, int line) {
  State& s = State::get();
  ++s.checks;
  if (!ok) {
    ++s.failures;
    s.case_failed = true;
    std::string where;
    for (auto& p : s.path) where += " / " + p;
    std::printf("FAIL  [%s%s] %s:%d  %s\n", s.current.c_str(), where.c_str(), file, line, expr);
  }
}

class Subcase {
 public:
  Subcase(const char* name) {
    State& s = State::get();
    depth_ = s.path.size();
    for (auto& p : s.path) key_ += p + "\x1f";
    key_ += name;
    if (s.entered_at.size() < depth_ + 2) s.entered_at.resize(depth_ + 2, false);
    if (s.incomplete.size() < depth_ + 2) s.incomplete.resize(depth_ + 2, false);
    if (s.done.count(key_)) return;
    if (s.entered_at[depth_]) {  // a sibling ran in this pass: come back in another one
      s.rerun = true;
      s.incomplete[depth_] = true;
      return;
    }
    entered_ = true;
    s.entered_at[depth_] = true;
    s.path.push_back(name);
    s.entered_at[depth_ + 1] = false;
    s.incomplete[depth_ + 1] = false;
  }
  ~Subcase() {
    if (!entered_) return;
    State& s = State::get();
    if (!s.incomplete[depth_ + 1]) s.done.insert(key_);  // every child completed
    else s.incomplete[depth_] = true;                   // the parent is not done either
    s.path.pop_back();
  }
  explicit operator bool() const { return entered_; }

 private:
  size_t depth_ = 0;
  std::string key_;
  bool entered_ = false;
};

inline int run_all() {
  State& s = State::get();
  int failed_cases = 0;
  for (auto& c : Registry::get().cases) {
    s.current = c.name;
    s.case_failed = false;
    s.done.clear();
    for (int run = 0; run < 10000; ++run) {
      s.rerun = false;
      s.path.clear();
      s.entered_at.assign(1, false);
      s.incomplete.assign(2, false);
      try {
        c.fn();
      } catch (const RequireFailure&) {
      } catch (const std::exception& e) {
        report(false, (std::string("unexpected exception: ") + e.what()).c_str(), c.file, c.line);
      }
      if (!s.rerun) break;
    }
    if (s.case_failed) {
      ++failed_cases;
      std::printf("case FAILED: %s\n", c.name);
    }
  }
  std::printf("[doctest-subset] test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
              Registry::get().cases.size(), Registry::get().cases.size() - failed_cases, failed_cases,
              s.checks, s.failures);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(name, fn)                                                                   \
  static void fn();                                                                           \
  static ::doctest::detail::Register DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);    \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(name, DOCTEST_CAT(doctest_case_, __COUNTER__))
#define SUBCASE(name) if (::doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name})
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::detail::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                          \
  do {                                                                        \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                   \
    ::doctest::detail::report(doctest_ok_, #__VA_ARGS__, __FILE__, __LINE__); \
    if (!doctest_ok_) throw ::doctest::detail::RequireFailure{};              \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                       \
  do {                                                                                   \
    bool doctest_thrown_ = false;                                                        \
    try {                                                                                \
      (void)(expr);                                                                      \
    } catch (const __VA_ARGS__&) {                                                       \
      doctest_thrown_ = true;                                                            \
    } catch (...) {                                                                      \
    }                                                                                    \
    ::doctest::detail::report(doctest_thrown_, "throws " #__VA_ARGS__ ": " #expr, __FILE__, \
                              __LINE__);                                                 \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
