// doctest-subset shim — TEST INFRASTRUCTURE for oracle/_ref.
//
// The reference's unit tests (proj/tests/test_*.cpp) are written against doctest,
// which is vendored upstream (proj/.gitignore: vendor/) and absent here.  This header
// implements the macros those tests use — TEST_CASE, SUBCASE (flat, re-running the
// case once per subcase as doctest does), CHECK / REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS with doctest::Contains, CAPTURE, FAIL, doctest::Approx with
// doctest's comparison |a - b| < eps * (scale + max(|a|, |b|)), scale 1 — so the
// unmodified test sources run against the shim-built reference library.
//
// Runner flags: -tc=<substring> selects cases by name; -ltc lists them.
#ifndef AUXMC_REF_SHIM_DOCTEST_H
#define AUXMC_REF_SHIM_DOCTEST_H

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
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
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool eq(double lhs) const {
    return std::fabs(lhs - v_) < eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(v_)));
  }
  double value() const { return v_; }

 private:
  double v_;
  double eps_ = 1.1920928955078125e-05 * 100;  // float epsilon * 100 (doctest default)
  double scale_ = 1.0;
};
inline bool operator==(double a, const Approx& b) { return b.eq(a); }
inline bool operator==(const Approx& b, double a) { return b.eq(a); }
inline bool operator!=(double a, const Approx& b) { return !b.eq(a); }
inline bool operator!=(const Approx& b, double a) { return !b.eq(a); }
inline bool operator<=(double a, const Approx& b) { return a < b.value() || b.eq(a); }
inline bool operator>=(double a, const Approx& b) { return a > b.value() || b.eq(a); }
inline bool operator<(double a, const Approx& b) { return a < b.value() && !b.eq(a); }
inline bool operator>(double a, const Approx& b) { return a > b.value() && !b.eq(a); }

struct Contains {
  explicit Contains(const char* s) : s_(s) {}
  bool in(const std::string& w) const { return w.find(s_) != std::string::npos; }
  std::string s_;
};

namespace shim {

struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct State {
  int subcase_target = 0, subcase_seen = 0;
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
  std::vector<std::string> captures;
};
inline State& st() {
  static State s;
  return s;
}
struct RequireAbort {};
inline bool enter_subcase() { return st().subcase_seen++ == st().subcase_target; }
inline void report(bool ok, const char* what, const char* file, int line, bool require) {
  ++st().checks;
  if (ok) return;
  ++st().failed_checks;
  st().case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s )\n", file, line, require ? "REQUIRE" : "CHECK", what);
  for (auto& c : st().captures) std::fprintf(stderr, "  with %s\n", c.c_str());
  if (require) throw RequireAbort{};
}
struct Capture {
  template <class T>
  Capture(const char* name, const T& v) {
    std::ostringstream os;
    os << name << " := " << v;
    st().captures.push_back(os.str());
  }
  ~Capture() { st().captures.pop_back(); }
};

inline int run(int argc, char** argv) {
  const char* filter = nullptr;
  bool list = false;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "-tc=", 4) == 0) filter = argv[i] + 4;
    if (std::strcmp(argv[i], "-ltc") == 0) list = true;
  }
  int n_cases = 0, n_failed = 0;
  for (const Case& c : registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    if (list) {
      std::printf("%s\n", c.name);
      continue;
    }
    ++n_cases;
    st().case_failed = false;
    int target = 0;
    do {
      st().subcase_target = target;
      st().subcase_seen = 0;
      st().captures.clear();
      try {
        c.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        st().case_failed = true;
        std::fprintf(stderr, "%s:%d: unexpected exception: %s\n", c.file, c.line, e.what());
      } catch (...) {
        st().case_failed = true;
        std::fprintf(stderr, "%s:%d: unexpected exception\n", c.file, c.line);
      }
      ++target;
    } while (target < st().subcase_seen);
    if (st().case_failed) {
      ++n_failed;
      std::fprintf(stderr, "[case FAILED] %s\n", c.name);
    }
  }
  if (!list)
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %ld | %ld failed\n",
                n_cases, n_cases - n_failed, n_failed, st().checks, st().failed_checks);
  return n_failed == 0 ? 0 : 1;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_TEST(fn, name)                                                   \
  static void fn();                                                                   \
  static ::doctest::shim::Reg DOCTEST_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TEST(DOCTEST_SHIM_CAT(doctest_shim_case_, __COUNTER__), name)
#define SUBCASE(name) if (::doctest::shim::enter_subcase())
#define CHECK(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, ...)                                                    \
  do {                                                                                \
    bool doctest_shim_ok = false;                                                     \
    try {                                                                             \
      (void)(expr);                                                                   \
    } catch (const __VA_ARGS__&) {                                                    \
      doctest_shim_ok = true;                                                         \
    } catch (...) {                                                                   \
    }                                                                                 \
    ::doctest::shim::report(doctest_shim_ok, "THROWS_AS " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                      \
  do {                                                                                \
    bool doctest_shim_ok = false;                                                     \
    try {                                                                             \
      (void)(expr);                                                                   \
    } catch (const __VA_ARGS__& e) {                                                  \
      doctest_shim_ok = (matcher).in(e.what());                              \
    } catch (...) {                                                                   \
    }                                                                                 \
    ::doctest::shim::report(doctest_shim_ok, "THROWS_WITH_AS " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS(expr)                                                            \
  do {                                                                                \
    bool doctest_shim_ok = false;                                                     \
    try {                                                                             \
      (void)(expr);                                                                   \
    } catch (...) {                                                                   \
      doctest_shim_ok = true;                                                         \
    }                                                                                 \
    ::doctest::shim::report(doctest_shim_ok, "THROWS " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                           \
  do {                                                                                \
    bool doctest_shim_ok = true;                                                      \
    try {                                                                             \
      (void)(expr);                                                                   \
    } catch (...) {                                                                   \
      doctest_shim_ok = false;                                                        \
    }                                                                                 \
    ::doctest::shim::report(doctest_shim_ok, "NOTHROW " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define CAPTURE(x) ::doctest::shim::Capture DOCTEST_SHIM_CAT(doctest_shim_cap_, __COUNTER__)(#x, x)
#define INFO(x) CAPTURE(x)
#define MESSAGE(x) ((void)0)
#define FAIL(msg)                                                                     \
  do {                                                                                \
    std::fprintf(stderr, "%s:%d: FAIL: %s\n", __FILE__, __LINE__, std::string(msg).c_str()); \
    ::doctest::shim::report(false, "FAIL", __FILE__, __LINE__, true);                 \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::shim::run(argc, argv); }
#endif

#endif
