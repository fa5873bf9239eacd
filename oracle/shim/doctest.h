// doctest.h — TEST INFRASTRUCTURE ONLY (oracle/_ref build).
//
// Clean-room subset of the doctest API the reference's suites use
// (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, INFO, FAIL, doctest::Approx),
// so /root/reference/proj/tests/test_*.cpp compile and run unmodified. The
// reference vendors doctest under vendor/ (proj/CMakeLists.txt:5), which is
// not shipped. Command line of the generated main: -tc=<glob>[,<glob>...]
// selects test cases by name, -tce=<glob>[,...] excludes; -ltc lists them.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
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
  friend bool operator==(double lhs, const Approx& r) {
    return std::fabs(lhs - r.value_) < r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.value_)));
  }
  friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
  friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
  friend bool operator!=(const Approx& r, double rhs) { return !(rhs == r); }
  friend bool operator<=(double lhs, const Approx& r) { return lhs < r.value_ || lhs == r; }
  friend bool operator>=(double lhs, const Approx& r) { return lhs > r.value_ || lhs == r; }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
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

struct RequireAbort {};

struct State {
  int asserts = 0;
  int failed_asserts = 0;
  bool current_failed = false;
  std::vector<std::string> info;
};
inline State& state() {
  static State s;
  return s;
}

inline void report(const char* file, int line, const char* kind, const std::string& what) {
  State& s = state();
  s.failed_asserts++;
  s.current_failed = true;
  std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, kind, what.c_str());
  for (const std::string& m : s.info) std::fprintf(stderr, "  logged: %s\n", m.c_str());
}

inline void check(bool ok, const char* file, int line, const char* kind, const char* expr, bool require) {
  state().asserts++;
  if (ok) return;
  report(file, line, kind, expr);
  if (require) throw RequireAbort{};
}

template <typename... A>
std::string cat(const A&... a) {
  std::ostringstream os;
  (os << ... << a);
  return os.str();
}

struct InfoScope {
  template <typename... A>
  explicit InfoScope(const A&... a) {
    state().info.push_back(cat(a...));
  }
  ~InfoScope() { state().info.pop_back(); }
};

inline bool glob_match(const char* p, const char* s) {
  if (*p == 0) return *s == 0;
  if (*p == '*') return glob_match(p + 1, s) || (*s && glob_match(p, s + 1));
  return *s && (*p == *s || *p == '?') && glob_match(p + 1, s + 1);
}

inline int run(int argc, char** argv) {
  std::vector<std::string> filters, excludes;
  bool list = false;
  auto split = [](const std::string& v, std::vector<std::string>* out) {
    std::size_t pos = 0;
    while (pos <= v.size()) {
      std::size_t c = v.find(',', pos);
      if (c == std::string::npos) c = v.size();
      out->push_back(v.substr(pos, c - pos));
      pos = c + 1;
    }
  };
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    if (a.rfind("-tc=", 0) == 0 || a.rfind("--test-case=", 0) == 0) {
      split(a.substr(a.find('=') + 1), &filters);
    } else if (a.rfind("-tce=", 0) == 0 || a.rfind("--test-case-exclude=", 0) == 0) {
      split(a.substr(a.find('=') + 1), &excludes);
    } else if (a == "-ltc" || a == "--list-test-cases") {
      list = true;
    }
  }
  int run_n = 0, failed_n = 0, skipped = 0;
  for (const TestCase& tc : registry()) {
    bool sel = filters.empty();
    for (const std::string& f : filters) sel = sel || glob_match(f.c_str(), tc.name);
    for (const std::string& f : excludes) sel = sel && !glob_match(f.c_str(), tc.name);
    if (!sel) {
      ++skipped;
      continue;
    }
    if (list) {
      std::printf("%s\n", tc.name);
      continue;
    }
    ++run_n;
    State& s = state();
    s.current_failed = false;
    s.info.clear();
    try {
      tc.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      report(tc.file, tc.line, "TEST CASE", std::string("threw: ") + e.what());
    } catch (...) {
      report(tc.file, tc.line, "TEST CASE", "threw a non-std exception");
    }
    if (s.current_failed) {
      ++failed_n;
      std::fprintf(stderr, "[doctest] FAILED: %s (%s:%d)\n", tc.name, tc.file, tc.line);
    }
  }
  if (list) return 0;
  std::printf("[doctest] test cases: %d | %d passed | %d failed | %d skipped\n", run_n, run_n - failed_n,
              failed_n, skipped);
  std::printf("[doctest] assertions: %d | %d passed | %d failed |\n", state().asserts,
              state().asserts - state().failed_asserts, state().failed_asserts);
  std::printf("[doctest] Status: %s!\n", failed_n ? "FAILURE" : "SUCCESS");
  return failed_n ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)

#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                              \
  static void fn();                                                                                   \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);            \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK", #__VA_ARGS__, false)
#define REQUIRE(...) \
  ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "REQUIRE", #__VA_ARGS__, true)
#define CHECK_FALSE(...) \
  ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK_FALSE", #__VA_ARGS__, false)
#define CHECK_THROWS_AS(expr, ...)                                                                      \
  do {                                                                                                  \
    bool doctest_ok_ = false;                                                                           \
    try {                                                                                               \
      static_cast<void>(expr);                                                                          \
    } catch (const __VA_ARGS__&) {                                                                      \
      doctest_ok_ = true;                                                                               \
    } catch (...) {                                                                                     \
    }                                                                                                   \
    ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, \
                             false);                                                                    \
  } while (0)
#define INFO(...) ::doctest::detail::InfoScope DOCTEST_CAT(doctest_info_, __LINE__)(__VA_ARGS__)
#define FAIL(...)                                                                                 \
  do {                                                                                            \
    ::doctest::detail::report(__FILE__, __LINE__, "FAIL", ::doctest::detail::cat(__VA_ARGS__));   \
    throw ::doctest::detail::RequireAbort{};                                                      \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
