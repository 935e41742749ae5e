// Minimal doctest-compatible test harness (doctest itself is absent from
// this image) -- just what the reference's unit tests use: TEST_CASE,
// SUBCASE (each subcase re-runs its test case, as in doctest), CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, FAIL,
// doctest::Approx (doctest's default epsilon, FLT_EPSILON * 100, relative)
// and doctest::Contains.  The generated main() runs every case and prints
// one JSON line per case: {"case": ..., "file": ..., "ok": bool,
// "failures": [...]} (tests/test_ref_suite.py reads them).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v), eps_(std::numeric_limits<float>::epsilon() * 100) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) <
           b.eps_ * (1.0 + std::max(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  double value() const { return v_; }

 private:
  double v_, eps_;
};

struct Contains {
  explicit Contains(std::string s) : s(std::move(s)) {}
  std::string s;
  bool matches(const std::string& w) const { return w.find(s) != std::string::npos; }
};

namespace detail {
struct Case {
  const char* name;
  const char* file;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* n, const char* f, void (*fn)()) { registry().push_back({n, f, fn}); }
};
struct Abort {};
inline std::vector<std::string>& failures() {
  static std::vector<std::string> f;
  return f;
}
// SUBCASE bookkeeping: pass p runs the p-th subcase reached
struct SubState {
  int target = 0, seen = 0, total = 0;
};
inline SubState& sub() {
  static SubState s;
  return s;
}
inline bool enter_subcase() {
  SubState& s = sub();
  const bool run = s.seen == s.target;
  ++s.seen;
  if (s.seen > s.total) s.total = s.seen;
  return run;
}
inline void fail(const char* file, int line, const std::string& what) {
  std::ostringstream o;
  o << file << ":" << line << ": " << what;
  failures().push_back(o.str());
}
inline std::string json_str(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    if (c == '\n') { o += "\\n"; continue; }
    o += c;
  }
  return o + "\"";
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                              \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                 \
  static doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(                  \
      name, __FILE__, &DOCTEST_CAT(doctest_fn_, __LINE__));                         \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define SUBCASE(name) if (doctest::detail::enter_subcase())
#define CHECK(...)                                                                   \
  do {                                                                               \
    try {                                                                            \
      if (!(__VA_ARGS__)) doctest::detail::fail(__FILE__, __LINE__, "CHECK( " #__VA_ARGS__ " )"); \
    } catch (const std::exception& e) {                                              \
      doctest::detail::fail(__FILE__, __LINE__, std::string("CHECK threw: ") + e.what()); \
    }                                                                                \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                 \
  do {                                                                               \
    if (!(__VA_ARGS__)) {                                                            \
      doctest::detail::fail(__FILE__, __LINE__, "REQUIRE( " #__VA_ARGS__ " )");      \
      throw doctest::detail::Abort{};                                                \
    }                                                                                \
  } while (0)
#define FAIL(msg)                                                                    \
  do {                                                                               \
    std::ostringstream doctest_os;                                                   \
    doctest_os << msg;                                                               \
    doctest::detail::fail(__FILE__, __LINE__, "FAIL: " + doctest_os.str());          \
    throw doctest::detail::Abort{};                                                  \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                  \
  do {                                                                               \
    bool doctest_ok = false;                                                         \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const type&) {                                                          \
      doctest_ok = true;                                                             \
    } catch (...) {                                                                  \
    }                                                                                \
    if (!doctest_ok)                                                                 \
      doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_AS( " #expr ", " #type " )"); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, type)                                    \
  do {                                                                               \
    bool doctest_ok = false;                                                         \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const type& e) {                                                        \
      doctest_ok = (matcher).matches(e.what());                                      \
    } catch (...) {                                                                  \
    }                                                                                \
    if (!doctest_ok)                                                                 \
      doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_WITH_AS( " #expr " )"); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  const char* only = argc > 1 ? argv[1] : nullptr;
  int failed = 0, ran = 0;
  for (const auto& c : doctest::detail::registry()) {
    if (only && std::string(c.name).find(only) == std::string::npos) continue;
    doctest::detail::failures().clear();
    std::string error;
    auto& s = doctest::detail::sub();
    s = {};
    do {  // one pass per subcase (a case without subcases runs once)
      s.seen = 0;
      try {
        c.fn();
      } catch (const doctest::detail::Abort&) {
      } catch (const std::exception& e) {
        error = e.what();
      } catch (...) {
        error = "unknown exception";
      }
      ++s.target;
    } while (s.target < s.total);
    if (!error.empty()) doctest::detail::failures().push_back("threw: " + error);
    const bool ok = doctest::detail::failures().empty();
    ++ran;
    failed += !ok;
    std::string fl = "[";
    for (size_t i = 0; i < doctest::detail::failures().size() && i < 8; ++i)
      fl += (i ? "," : "") + doctest::detail::json_str(doctest::detail::failures()[i]);
    fl += "]";
    std::printf("{\"case\": %s, \"file\": %s, \"ok\": %s, \"n_failures\": %zu, \"failures\": %s}\n",
                doctest::detail::json_str(c.name).c_str(),
                doctest::detail::json_str(c.file).c_str(), ok ? "true" : "false",
                doctest::detail::failures().size(), fl.c_str());
    std::fflush(stdout);
  }
  std::printf("{\"summary\": {\"ran\": %d, \"failed\": %d}}\n", ran, failed);
  return failed ? 1 : 0;
}
#endif
