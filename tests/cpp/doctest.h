// Minimal doctest-compatible test harness (doctest itself is not vendored in
// the reference checkout, proj/.gitignore:2).  Implements exactly the macros
// the reference's unit tests use -- TEST_CASE, SUBCASE, CHECK, CHECK_FALSE,
// REQUIRE, CAPTURE, CHECK_THROWS_AS -- so the `ref_tests` target of
// oracle/Makefile can compile /root/reference/proj/tests/
// test_{core,parallel,sort}.cpp against the drop-in headers in
// include/mergepath/ unchanged.
//
// Semantics: SUBCASE blocks run in sequence within one pass of their
// TEST_CASE (doctest re-enters the case per subcase; the reference's
// subcases are independent, so the results are the same).  A failed
// REQUIRE aborts the current TEST_CASE; the process exit code is the number
// of failed cases (capped at 255).
#pragma once

#include <cstdio>
#include <sstream>
#include <string>
#include <vector>

namespace mini_doctest {

struct Case {
  const char *name;
  void (*fn)();
  const char *file;
  int line;
};
inline std::vector<Case> &registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char *name, void (*fn)(), const char *file, int line) {
    registry().push_back({name, fn, file, line});
  }
};
struct RequireFailed {};

struct State {
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
  std::vector<std::string> captures;
  std::vector<std::string> subcases;
};
inline State &state() {
  static State s;
  return s;
}

struct Capture {
  template <typename T> Capture(const char *expr, const T &v) {
    std::ostringstream os;
    os << expr << " := " << v;
    state().captures.push_back(os.str());
  }
  ~Capture() { state().captures.pop_back(); }
};

struct Subcase {
  explicit Subcase(const char *name) { state().subcases.push_back(name); }
  ~Subcase() { state().subcases.pop_back(); }
};

inline void check(bool ok, const char *expr, const char *file, int line,
                  bool require) {
  State &s = state();
  ++s.checks;
  if (ok)
    return;
  ++s.failed_checks;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: %s FAILED: %s\n", file, line,
               require ? "REQUIRE" : "CHECK", expr);
  for (const auto &sc : s.subcases)
    std::fprintf(stderr, "    in SUBCASE: %s\n", sc.c_str());
  for (const auto &c : s.captures)
    std::fprintf(stderr, "    with %s\n", c.c_str());
  if (require)
    throw RequireFailed{};
}

inline int run_all() {
  int failed = 0;
  for (const Case &c : registry()) {
    State &s = state();
    s.case_failed = false;
    s.captures.clear();
    s.subcases.clear();
    try {
      c.fn();
    } catch (const RequireFailed &) {
    } catch (const std::exception &e) {
      s.case_failed = true;
      std::fprintf(stderr, "%s:%d: TEST_CASE \"%s\" threw: %s\n", c.file,
                   c.line, c.name, e.what());
    }
    std::printf("[%s] %s\n", s.case_failed ? "FAIL" : " ok ", c.name);
    if (s.case_failed)
      ++failed;
  }
  std::printf("test cases: %zu | %zu passed | %d failed   assertions: %ld | "
              "%ld failed\n",
              registry().size(), registry().size() - failed, failed,
              state().checks, state().failed_checks);
  return failed > 255 ? 255 : failed;
}

}  // namespace mini_doctest

#define MD_CAT2(a, b) a##b
#define MD_CAT(a, b) MD_CAT2(a, b)
#define MD_UNIQUE(p) MD_CAT(p, __LINE__)

#define TEST_CASE(name)                                                        \
  static void MD_UNIQUE(md_case_)();                                           \
  static ::mini_doctest::Registrar MD_UNIQUE(md_reg_)(                         \
      name, &MD_UNIQUE(md_case_), __FILE__, __LINE__);                         \
  static void MD_UNIQUE(md_case_)()

#define SUBCASE(name)                                                          \
  if (::mini_doctest::Subcase MD_UNIQUE(md_sub_){name}; true)

#define CHECK(...)                                                             \
  ::mini_doctest::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__,          \
                        __FILE__, __LINE__, false)
#define CHECK_FALSE(...)                                                       \
  ::mini_doctest::check(!static_cast<bool>(__VA_ARGS__),                       \
                        "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...)                                                           \
  ::mini_doctest::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__,          \
                        __FILE__, __LINE__, true)
#define CAPTURE(x) ::mini_doctest::Capture MD_UNIQUE(md_cap_)(#x, (x))
#define CHECK_THROWS_AS(expr, ...)                                             \
  do {                                                                         \
    bool md_caught_ = false;                                                   \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (const __VA_ARGS__ &) {                                            \
      md_caught_ = true;                                                       \
    } catch (...) {                                                            \
    }                                                                          \
    ::mini_doctest::check(md_caught_, "throws " #__VA_ARGS__ ": " #expr,       \
                          __FILE__, __LINE__, false);                          \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::mini_doctest::run_all(); }
#endif
