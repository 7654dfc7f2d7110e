// TEST INFRASTRUCTURE ONLY: a minimal, self-contained stand-in for the
// doctest single-header framework (absent from this image: no network), with
// just the surface the reference's unit suites use
// (/root/reference/proj/tests/test_*.cpp): TEST_CASE, SUBCASE (re-entrant:
// the test body is re-run once per leaf subcase, nested subcases supported),
// CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, CAPTURE, MESSAGE,
// REQUIRE_MESSAGE, FAIL and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.  Lets those
// suites compile UNMODIFIED against libdelta.  Written from doctest's
// documented semantics; no doctest source is used.
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace doctest_shim {

struct TestCase {
  void (*fn)();
  const char* name;
  const char* file;
  int line;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Reg {
  Reg(void (*fn)(), const char* name, const char* file, int line) {
    registry().push_back({fn, name, file, line});
  }
};

struct Abort {};  // thrown by REQUIRE / FAIL to end the current run

struct Context {
  // subcase bookkeeping for the current test case
  std::vector<std::string> path;
  std::set<std::vector<std::string>> done;
  std::vector<bool> taken, pending;
  // results
  int failed_asserts = 0, asserts = 0;
  bool current_failed = false;
  std::vector<std::string> captures;
  const TestCase* tc = nullptr;

  void begin_run() {
    path.clear();
    taken.assign(1, false);
    pending.assign(1, false);
  }
  bool try_enter(const char* name) {
    std::vector<std::string> p = path;
    p.push_back(name);
    if (done.count(p)) return false;
    const std::size_t level = path.size();
    if (taken[level]) {
      pending[level] = true;  // an unfinished sibling: run the body again
      return false;
    }
    taken[level] = true;
    path.push_back(name);
    if (taken.size() <= path.size()) {
      taken.resize(path.size() + 1, false);
      pending.resize(path.size() + 1, false);
    }
    taken[path.size()] = false;
    pending[path.size()] = false;
    return true;
  }
  void leave() {
    const std::size_t level = path.size();
    if (!pending[level]) {
      done.insert(path);
    } else {
      pending[level - 1] = true;
    }
    path.pop_back();
  }
  std::string where() const {
    std::string s;
    for (const auto& p : path) s += " / " + p;
    return s;
  }
  void fail(const char* file, int line, const std::string& what) {
    ++failed_asserts;
    current_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED in \"%s\"%s: %s\n", file, line, tc ? tc->name : "?",
                 where().c_str(), what.c_str());
    for (const auto& c : captures) std::fprintf(stderr, "    with %s\n", c.c_str());
  }
};

inline Context& ctx() {
  static Context c;
  return c;
}

struct Subcase {
  bool entered;
  explicit Subcase(const char* name) : entered(ctx().try_enter(name)) {}
  ~Subcase() {
    if (entered) ctx().leave();
  }
  explicit operator bool() const { return entered; }
};

struct Capture {
  explicit Capture(std::string s) { ctx().captures.push_back(std::move(s)); }
  ~Capture() { ctx().captures.pop_back(); }
};

template <class T>
std::string show(const char* name, const T& v) {
  std::ostringstream os;
  os << name << " := " << v;
  return os.str();
}

inline void check(bool ok, bool require, const char* file, int line, const char* expr) {
  ++ctx().asserts;
  if (ok) return;
  ctx().fail(file, line, std::string(require ? "REQUIRE( " : "CHECK( ") + expr + " )");
  if (require) throw Abort{};
}

inline int run_all() {
  int failed = 0, passed = 0;
  for (const TestCase& tc : registry()) {
    Context& c = ctx();
    c.tc = &tc;
    c.done.clear();
    c.current_failed = false;
    int runs = 0;
    do {
      c.begin_run();
      c.captures.clear();
      try {
        tc.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        c.fail(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
      } catch (...) {
        c.fail(tc.file, tc.line, "unexpected exception");
      }
      // unwind whatever subcases an exception left open
      while (!c.path.empty()) c.leave();
      ++runs;
    } while (c.pending[0] && runs < 10000);
    if (c.current_failed) {
      ++failed;
    } else {
      ++passed;
    }
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %d | %d failed\n",
              failed + passed, passed, failed, ctx().asserts, ctx().failed_asserts);
  return failed ? 1 : 0;
}

}  // namespace doctest_shim

#define DS_CAT2(a, b) a##b
#define DS_CAT(a, b) DS_CAT2(a, b)

#define DS_TEST_CASE_IMPL(fn, name)                                                  \
  static void fn();                                                                 \
  static doctest_shim::Reg DS_CAT(fn, _reg)(fn, name, __FILE__, __LINE__);          \
  static void fn()
#define TEST_CASE(name) DS_TEST_CASE_IMPL(DS_CAT(ds_test_case_, __COUNTER__), name)

#define SUBCASE(name) if (const doctest_shim::Subcase DS_CAT(ds_subcase_, __LINE__){name})

#define CHECK(...) doctest_shim::check(static_cast<bool>(__VA_ARGS__), false, __FILE__, __LINE__, #__VA_ARGS__)
#define REQUIRE(...) doctest_shim::check(static_cast<bool>(__VA_ARGS__), true, __FILE__, __LINE__, #__VA_ARGS__)

#define DS_MSG(msg) ([&] { std::ostringstream ds_os_; ds_os_ << msg; return ds_os_.str(); }())

#define REQUIRE_MESSAGE(cond, msg)                                               \
  do {                                                                           \
    ++doctest_shim::ctx().asserts;                                               \
    if (!static_cast<bool>(cond)) {                                              \
      doctest_shim::ctx().fail(__FILE__, __LINE__, std::string("REQUIRE( " #cond " ): ") + DS_MSG(msg)); \
      throw doctest_shim::Abort{};                                               \
    }                                                                            \
  } while (0)

#define FAIL(msg)                                                      \
  do {                                                                 \
    doctest_shim::ctx().fail(__FILE__, __LINE__, DS_MSG(msg));         \
    throw doctest_shim::Abort{};                                       \
  } while (0)

#define MESSAGE(msg) std::fprintf(stderr, "%s:%d: MESSAGE: %s\n", __FILE__, __LINE__, DS_MSG(msg).c_str())

#define CAPTURE(x) const doctest_shim::Capture DS_CAT(ds_capture_, __LINE__)(doctest_shim::show(#x, x))

#define CHECK_THROWS_AS(expr, ...)                                                     \
  do {                                                                                 \
    ++doctest_shim::ctx().asserts;                                                     \
    bool ds_ok_ = false;                                                               \
    try {                                                                              \
      static_cast<void>(expr);                                                         \
    } catch (const __VA_ARGS__&) {                                                     \
      ds_ok_ = true;                                                                   \
    } catch (...) {                                                                    \
    }                                                                                  \
    if (!ds_ok_)                                                                       \
      doctest_shim::ctx().fail(__FILE__, __LINE__, "CHECK_THROWS_AS( " #expr ", " #__VA_ARGS__ " )"); \
  } while (0)

#define CHECK_NOTHROW(...)                                                             \
  do {                                                                                 \
    ++doctest_shim::ctx().asserts;                                                     \
    try {                                                                              \
      static_cast<void>(__VA_ARGS__);                                                  \
    } catch (...) {                                                                    \
      doctest_shim::ctx().fail(__FILE__, __LINE__, "CHECK_NOTHROW( " #__VA_ARGS__ " )"); \
    }                                                                                  \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest_shim::run_all(); }
#endif
