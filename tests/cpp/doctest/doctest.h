// doctest.h -- TEST INFRASTRUCTURE: a minimal stand-in for the doctest
// single-header framework (not present in this image), covering exactly the
// macros the reference's unit tests use (/root/reference/proj/tests/*.cpp):
// TEST_CASE, CHECK, CHECK_FALSE, CHECK_MESSAGE, CHECK_THROWS_AS,
// CHECK_NOTHROW, REQUIRE, REQUIRE_MESSAGE and doctest::Approx (with
// .epsilon() / .scale(), doctest's comparison rule).  With
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN defined before the include it also
// provides main(): runs every registered case (argv[1], if given, is a
// comma-separated list of substrings of case names -- or "file:<substring>"
// on the source file -- and a case runs if any matches), prints one line per failed assertion
// and a summary, and exits nonzero on any failure.
//
// Used to compile the reference's test sources UNMODIFIED against the drop-in
// headers (include/fmafft/*.hpp -> include/fmafft_b200.hpp); see
// tests/cpp/Makefile.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value)
      : value_(value), epsilon_(double(std::numeric_limits<float>::epsilon()) * 100), scale_(1.0) {}
  Approx& epsilon(double e) {
    epsilon_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  // doctest's rule: |lhs - v| < eps * (scale + max(|lhs|, |v|))
  friend bool operator==(double lhs, const Approx& r) {
    return std::fabs(lhs - r.value_) <
           r.epsilon_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.value_)));
  }
  friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
  friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
  friend bool operator!=(const Approx& r, double rhs) { return !(rhs == r); }

 private:
  double value_, epsilon_, scale_;
};

namespace detail {

struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> cases;
  return cases;
}

struct State {
  long long asserts = 0, failed_asserts = 0;
  bool case_failed = false;
};
inline State& state() {
  static State s;
  return s;
}

struct Reg {
  Reg(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back(Case{name, file, line, fn});
  }
};

struct RequireAbort {};

inline void stream_all(std::ostringstream&) {}
template <class T, class... R>
void stream_all(std::ostringstream& os, const T& v, const R&... rest) {
  os << v;
  stream_all(os, rest...);
}

inline void record(bool ok, const char* kind, const char* expr, const char* file, int line,
                   const std::string& msg, bool require) {
  State& s = state();
  ++s.asserts;
  if (ok) return;
  ++s.failed_asserts;
  s.case_failed = true;
  std::printf("%s:%d: ERROR: %s( %s ) is NOT correct!%s%s\n", file, line, kind, expr,
              msg.empty() ? "" : "\n  message: ", msg.c_str());
  if (require) throw RequireAbort{};
}

template <class... M>
std::string message(const M&... m) {
  std::ostringstream os;
  stream_all(os, m...);
  return os.str();
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_(fn, reg, name)                                              \
  static void fn();                                                               \
  static ::doctest::detail::Reg reg(name, __FILE__, __LINE__, &fn);               \
  static void fn()
#define TEST_CASE(name) \
  DOCTEST_CASE_(DOCTEST_CAT(doctest_case_fn_, __LINE__), DOCTEST_CAT(doctest_case_reg_, __LINE__), name)

#define DOCTEST_ASSERT_(kind, require, cond, ...)                                             \
  do {                                                                                        \
    bool ok_ = false;                                                                         \
    try {                                                                                     \
      ok_ = static_cast<bool>(cond);                                                          \
    } catch (const ::doctest::detail::RequireAbort&) {                                        \
      throw;                                                                                  \
    } catch (const std::exception& e_) {                                                      \
      ::doctest::detail::record(false, kind, #cond, __FILE__, __LINE__,                       \
                                std::string("threw: ") + e_.what(), require);                \
      break;                                                                                  \
    }                                                                                         \
    ::doctest::detail::record(ok_, kind, #cond, __FILE__, __LINE__,                           \
                              ok_ ? std::string() : ::doctest::detail::message(__VA_ARGS__), \
                              require);                                                       \
  } while (0)

#define CHECK(...) DOCTEST_ASSERT_("CHECK", false, (__VA_ARGS__), "")
#define CHECK_FALSE(...) DOCTEST_ASSERT_("CHECK_FALSE", false, !(__VA_ARGS__), "")
#define REQUIRE(...) DOCTEST_ASSERT_("REQUIRE", true, (__VA_ARGS__), "")
#define CHECK_MESSAGE(cond, ...) DOCTEST_ASSERT_("CHECK", false, cond, __VA_ARGS__)
#define REQUIRE_MESSAGE(cond, ...) DOCTEST_ASSERT_("REQUIRE", true, cond, __VA_ARGS__)

#define CHECK_THROWS_AS(expr, ...)                                                       \
  do {                                                                                   \
    bool caught_ = false;                                                                \
    std::string other_;                                                                  \
    try {                                                                                \
      static_cast<void>(expr);                                                           \
    } catch (const __VA_ARGS__&) {                                                       \
      caught_ = true;                                                                    \
    } catch (const std::exception& e_) {                                                 \
      other_ = std::string("threw another exception: ") + e_.what();                     \
    } catch (...) {                                                                      \
      other_ = "threw another exception";                                                \
    }                                                                                    \
    ::doctest::detail::record(caught_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__,       \
                              __FILE__, __LINE__, caught_ ? std::string() : other_, false); \
  } while (0)

#define CHECK_NOTHROW(expr)                                                              \
  do {                                                                                   \
    std::string what_;                                                                   \
    bool ok_ = true;                                                                     \
    try {                                                                                \
      static_cast<void>(expr);                                                           \
    } catch (const std::exception& e_) {                                                 \
      ok_ = false;                                                                       \
      what_ = e_.what();                                                                 \
    } catch (...) {                                                                      \
      ok_ = false;                                                                       \
    }                                                                                    \
    ::doctest::detail::record(ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__, what_, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  using namespace doctest::detail;
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int run = 0, failed = 0;
  for (const Case& c : registry()) {
    if (filter && std::strncmp(filter, "file:", 5) == 0) {
      if (!std::strstr(c.file, filter + 5)) continue;
    } else if (filter) {
      bool hit = false;
      std::string f(filter);
      for (size_t at = 0; at <= f.size() && !hit;) {
        const size_t end = f.find(',', at);
        const std::string part = f.substr(at, end == std::string::npos ? std::string::npos : end - at);
        hit = !part.empty() && std::strstr(c.name, part.c_str()) != nullptr;
        if (end == std::string::npos) break;
        at = end + 1;
      }
      if (!hit) continue;
    }
    ++run;
    state().case_failed = false;
    try {
      c.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      std::printf("%s:%d: ERROR: test case \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
      state().case_failed = true;
    }
    if (state().case_failed) {
      ++failed;
      std::printf("FAILED: %s\n", c.name);
    }
    std::fflush(stdout);
  }
  std::printf("[doctest] test cases: %d | %d passed | %d failed\n", run, run - failed, failed);
  std::printf("[doctest] assertions: %lld | %lld passed | %lld failed\n", state().asserts,
              state().asserts - state().failed_asserts, state().failed_asserts);
  return failed ? 1 : 0;
}
#endif
