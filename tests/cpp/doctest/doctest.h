// A small doctest-compatible test harness (written for this repo; not the
// doctest library).  It implements the subset the reference's unit tests use
// -- TEST_CASE, SUBCASE (nested, each leaf path run once), CHECK, REQUIRE,
// CHECK_MESSAGE, CHECK_THROWS_AS, doctest::Approx -- so those test files
// compile unchanged against the drop-in headers (SURVEY.md section 4,
// "conformance idea").  Define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN in one
// translation unit for main().
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <functional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace dshim {

struct TestCase {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Reg {
  Reg(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};

struct State {
  std::set<std::string> done;    // finished subcase paths
  std::vector<std::string> path;  // active subcase keys
  std::vector<bool> took;         // per depth: a subcase ran at this depth in this pass
  bool pending = false;           // a subcase is still to run: another pass
  long checks = 0, failures = 0;
  const char* test = "";
};

inline State& st() {
  static State s;
  return s;
}

struct RequireFailed {};

class Subcase {
 public:
  Subcase(const char* name, int line) {
    State& s = st();
    depth_ = s.path.size();
    key_ = (depth_ ? s.path.back() : std::string()) + "/" + name + "#" + std::to_string(line);
    if (s.done.count(key_)) return;
    if (s.took.size() <= depth_) s.took.resize(depth_ + 1, false);
    if (s.took[depth_]) {  // a sibling ran in this pass: come back later
      s.pending = true;
      return;
    }
    s.took[depth_] = true;
    s.took.resize(depth_ + 1);
    active_ = true;
    outer_pending_ = s.pending;
    s.pending = false;
    s.path.push_back(key_);
  }
  ~Subcase() {
    if (!active_) return;
    State& s = st();
    s.path.pop_back();
    if (!s.pending) s.done.insert(key_);  // no child left: this path is complete
    s.pending = s.pending || outer_pending_;
  }
  explicit operator bool() const { return active_; }

 private:
  std::string key_;
  std::size_t depth_ = 0;
  bool active_ = false, outer_pending_ = false;
};

template <class... A>
std::string cat(const A&... a) {
  std::ostringstream o;
  (o << ... << a);
  return o.str();
}

inline void report(bool ok, const char* expr, const char* file, int line, const std::string& msg,
                   bool fatal) {
  State& s = st();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  std::printf("%s:%d: FAILED %s (%s) in test \"%s\"%s%s\n", file, line, fatal ? "REQUIRE" : "CHECK",
              expr, s.test, msg.empty() ? "" : ": ", msg.c_str());
  if (fatal) throw RequireFailed{};
}

}  // namespace dshim

namespace doctest {
// |a - b| < eps * (scale + max(|a|, |b|)), eps = 100 FLT_EPSILON, scale 1
class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) < b.eps_ * (1.0 + std::fmax(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  friend bool operator!=(const Approx& b, double a) { return !(a == b); }

 private:
  double v_;
  double eps_ = 100.0 * FLT_EPSILON;
};
}  // namespace doctest

#define DSHIM_CAT2(a, b) a##b
#define DSHIM_CAT(a, b) DSHIM_CAT2(a, b)
#define DSHIM_TC(f, name)                                                     \
  static void f();                                                            \
  static ::dshim::Reg DSHIM_CAT(f, _reg)(name, &f, __FILE__, __LINE__);       \
  static void f()
#define TEST_CASE(name) DSHIM_TC(DSHIM_CAT(dshim_tc_, __COUNTER__), name)
#define SUBCASE(name) if (const ::dshim::Subcase DSHIM_CAT(dshim_sc_, __LINE__){name, __LINE__})
#define CHECK(...) ::dshim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, "", false)
#define REQUIRE(...) ::dshim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, "", true)
#define CHECK_MESSAGE(cond, ...) \
  ::dshim::report(static_cast<bool>(cond), #cond, __FILE__, __LINE__, ::dshim::cat(__VA_ARGS__), false)
#define REQUIRE_MESSAGE(cond, ...) \
  ::dshim::report(static_cast<bool>(cond), #cond, __FILE__, __LINE__, ::dshim::cat(__VA_ARGS__), true)
#define CHECK_THROWS_AS(expr, ...)                                                      \
  do {                                                                                  \
    bool dshim_ok = false;                                                              \
    try {                                                                               \
      (void)(expr);                                                                     \
    } catch (const __VA_ARGS__&) {                                                      \
      dshim_ok = true;                                                                  \
    } catch (...) {                                                                     \
    }                                                                                   \
    ::dshim::report(dshim_ok, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__, "", false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  auto& s = ::dshim::st();
  long failed_cases = 0;
  for (const auto& tc : ::dshim::registry()) {
    const long before = s.failures;
    s.test = tc.name;
    s.done.clear();
    do {  // one pass per leaf subcase path
      s.took.clear();
      s.path.clear();
      s.pending = false;
      try {
        tc.fn();
      } catch (const ::dshim::RequireFailed&) {
      } catch (const std::exception& e) {
        ++s.failures;
        std::printf("%s:%d: unexpected exception in test \"%s\": %s\n", tc.file, tc.line, tc.name,
                    e.what());
        break;
      }
    } while (s.pending);
    failed_cases += s.failures != before;
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %ld failed; assertions: %ld | %ld failed\n",
              ::dshim::registry().size(), ::dshim::registry().size() - (size_t)failed_cases,
              failed_cases, s.checks, s.failures);
  std::printf("Status: %s\n", s.failures ? "FAILURE!" : "SUCCESS!");
  return s.failures ? 1 : 0;
}
#endif
