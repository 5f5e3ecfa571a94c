// Minimal Catch2-v3-compatible test shim (the real Catch2 is not installed in
// this image). Supports exactly the surface the reference planner suites use:
// TEST_CASE, SECTION (one leaf per run, re-running the case until every
// section path has executed), REQUIRE / REQUIRE_FALSE / REQUIRE_THROWS_AS /
// REQUIRE_THROWS_WITH (+ ContainsSubstring matchers), FAIL, Catch::Approx,
// and CATCH_REGISTER_LISTENER with testCaseEnded. The runner main lives in
// catch_shim_main.cpp.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <memory>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace Catch {

struct TestCaseInfo {
  std::string name;
};
struct AssertionCounts {
  std::size_t passed = 0, failed = 0;
  bool allOk() const { return failed == 0; }
};
struct Totals {
  AssertionCounts assertions;
};
struct TestCaseStats {
  const TestCaseInfo* testInfo = nullptr;
  Totals totals;
};
struct IConfig {};

class EventListenerBase {
 public:
  explicit EventListenerBase(const IConfig* = nullptr) {}
  virtual ~EventListenerBase() = default;
  virtual void testCaseEnded(const TestCaseStats&) {}
};

class Approx {
 public:
  explicit Approx(double v)
      : value_(v), epsilon_(std::numeric_limits<float>::epsilon() * 100), margin_(0.0) {}
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  Approx& epsilon(double e) {
    epsilon_ = e;
    return *this;
  }
  bool matches(double other) const {
    const double d = std::fabs(other - value_);
    if (d <= margin_) return true;
    const double scale = std::isinf(value_) ? 0.0 : std::fabs(value_);
    return d <= epsilon_ * scale;
  }
  std::string str() const {
    std::ostringstream os;
    os << "Approx(" << value_ << ")";
    return os.str();
  }

 private:
  double value_, epsilon_, margin_;
};
inline bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
inline bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
inline bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }

namespace Matchers {
struct StringMatcher {
  std::function<bool(const std::string&)> fn;
  std::string desc;
  bool match(const std::string& s) const { return fn(s); }
};
inline StringMatcher ContainsSubstring(const std::string& needle) {
  return {[needle](const std::string& s) { return s.find(needle) != std::string::npos; },
          "contains \"" + needle + "\""};
}
inline StringMatcher operator&&(const StringMatcher& a, const StringMatcher& b) {
  return {[a, b](const std::string& s) { return a.match(s) && b.match(s); },
          a.desc + " and " + b.desc};
}
inline StringMatcher operator||(const StringMatcher& a, const StringMatcher& b) {
  return {[a, b](const std::string& s) { return a.match(s) || b.match(s); },
          a.desc + " or " + b.desc};
}
}  // namespace Matchers

namespace shim {

struct AssertionFailure {};

struct TestCase {
  std::string name;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline std::vector<std::function<std::unique_ptr<EventListenerBase>()>>& listener_factories() {
  static std::vector<std::function<std::unique_ptr<EventListenerBase>()>> f;
  return f;
}

struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
template <typename L>
struct ListenerRegistrar {
  ListenerRegistrar() {
    listener_factories().push_back([] { return std::unique_ptr<EventListenerBase>(new L(nullptr)); });
  }
};

// Section tracking: each run of a test case enters at most one not-yet-
// completed section per nesting level; the case is re-run while any section
// remains pending.
struct RunState {
  std::set<std::vector<std::string>> completed;
  std::vector<std::string> path;
  std::vector<bool> level_taken;    // a section already ran at this depth this run
  std::vector<bool> child_pending;  // the section at this depth has unfinished children
  bool pending = false;
  AssertionCounts counts;
};
inline RunState*& state() {
  static RunState* s = nullptr;
  return s;
}

class Section {
 public:
  explicit Section(const std::string& name) {
    RunState& st = *state();
    const std::size_t depth = st.path.size();
    if (st.level_taken.size() <= depth) st.level_taken.resize(depth + 1, false);
    std::vector<std::string> full = st.path;
    full.push_back(name);
    if (st.completed.count(full)) return;
    if (st.level_taken[depth]) {
      st.pending = true;
      if (!st.child_pending.empty()) st.child_pending.back() = true;
      return;
    }
    st.level_taken[depth] = true;
    st.path = full;
    st.level_taken.resize(depth + 2, false);
    st.level_taken[depth + 1] = false;
    st.child_pending.push_back(false);
    entered_ = true;
  }
  ~Section() {
    if (!entered_) return;
    RunState& st = *state();
    const bool unfinished = st.child_pending.back();
    st.child_pending.pop_back();
    if (!unfinished && !std::uncaught_exceptions()) st.completed.insert(st.path);
    if (unfinished && !st.child_pending.empty()) st.child_pending.back() = true;
    st.path.pop_back();
    st.level_taken.resize(st.path.size() + 1);
  }
  explicit operator bool() const { return entered_; }

 private:
  bool entered_ = false;
};

inline void report_failure(const char* file, int line, const std::string& what) {
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what.c_str());
  state()->counts.failed += 1;
  throw AssertionFailure{};
}
inline void pass() { state()->counts.passed += 1; }

inline int run_all() {
  std::vector<std::unique_ptr<EventListenerBase>> listeners;
  for (auto& f : listener_factories()) listeners.push_back(f());
  int failed_cases = 0;
  std::size_t assertions = 0;
  for (const TestCase& tc : registry()) {
    RunState st;
    state() = &st;
    bool failed = false;
    do {
      st.pending = false;
      st.path.clear();
      st.level_taken.assign(1, false);
      st.child_pending.clear();
      try {
        tc.fn();
      } catch (const AssertionFailure&) {
        failed = true;
      } catch (const std::exception& e) {
        std::fprintf(stderr, "%s: unexpected exception: %s\n", tc.name.c_str(), e.what());
        st.counts.failed += 1;
        failed = true;
      }
    } while (st.pending && !failed);
    TestCaseInfo info{tc.name};
    TestCaseStats stats;
    stats.testInfo = &info;
    stats.totals.assertions = st.counts;
    for (auto& l : listeners) l->testCaseEnded(stats);
    if (failed || st.counts.failed) {
      ++failed_cases;
      std::fprintf(stderr, "test case FAILED: %s\n", tc.name.c_str());
    }
    assertions += st.counts.passed + st.counts.failed;
    state() = nullptr;
  }
  std::printf("%s: %zu test cases, %d failed, %zu assertions\n",
              failed_cases ? "FAILED" : "All tests passed", registry().size(), failed_cases,
              assertions);
  return failed_cases ? 1 : 0;
}

}  // namespace shim
}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_UNIQUE(p) CATCH_SHIM_CAT(p, __LINE__)

#define TEST_CASE_IMPL(fn, name, ...)                                         \
  static void fn();                                                           \
  static ::Catch::shim::Registrar CATCH_SHIM_CAT(fn, _reg)(name, &fn);        \
  static void fn()
#define TEST_CASE(...) TEST_CASE_IMPL(CATCH_SHIM_UNIQUE(catch_shim_tc_), __VA_ARGS__, "")

#define SECTION(...) \
  if (::Catch::shim::Section CATCH_SHIM_UNIQUE(catch_shim_sec_){std::string(__VA_ARGS__)}; \
      CATCH_SHIM_UNIQUE(catch_shim_sec_))

#define REQUIRE(...)                                                                  \
  do {                                                                                \
    if (!static_cast<bool>(__VA_ARGS__))                                              \
      ::Catch::shim::report_failure(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")"); \
    ::Catch::shim::pass();                                                            \
  } while (0)
#define REQUIRE_FALSE(...)                                                                  \
  do {                                                                                      \
    if (static_cast<bool>(__VA_ARGS__))                                                     \
      ::Catch::shim::report_failure(__FILE__, __LINE__, "REQUIRE_FALSE(" #__VA_ARGS__ ")"); \
    ::Catch::shim::pass();                                                                  \
  } while (0)
#define REQUIRE_THROWS_AS(expr, type)                                                          \
  do {                                                                                         \
    bool catch_shim_ok = false;                                                                \
    try {                                                                                      \
      static_cast<void>(expr);                                                                 \
    } catch (const type&) {                                                                    \
      catch_shim_ok = true;                                                                    \
    } catch (...) {                                                                            \
    }                                                                                          \
    if (!catch_shim_ok)                                                                        \
      ::Catch::shim::report_failure(__FILE__, __LINE__, "REQUIRE_THROWS_AS(" #expr ", " #type ")"); \
    ::Catch::shim::pass();                                                                     \
  } while (0)

namespace Catch::shim {
inline bool message_matches(const std::string& msg, const Matchers::StringMatcher& m) {
  return m.match(msg);
}
inline bool message_matches(const std::string& msg, const char* exact) { return msg == exact; }
inline bool message_matches(const std::string& msg, const std::string& exact) {
  return msg == exact;
}
}  // namespace Catch::shim

#define REQUIRE_THROWS_WITH(expr, matcher)                                                     \
  do {                                                                                         \
    bool catch_shim_ok = false;                                                                \
    try {                                                                                      \
      static_cast<void>(expr);                                                                 \
    } catch (const std::exception& catch_shim_e) {                                             \
      catch_shim_ok = ::Catch::shim::message_matches(catch_shim_e.what(), matcher);            \
    } catch (...) {                                                                            \
    }                                                                                          \
    if (!catch_shim_ok)                                                                        \
      ::Catch::shim::report_failure(__FILE__, __LINE__, "REQUIRE_THROWS_WITH(" #expr ")");     \
    ::Catch::shim::pass();                                                                     \
  } while (0)

#define FAIL(msg)                                                          \
  do {                                                                     \
    std::ostringstream catch_shim_os;                                      \
    catch_shim_os << msg;                                                  \
    ::Catch::shim::report_failure(__FILE__, __LINE__, catch_shim_os.str()); \
  } while (0)

#define CATCH_REGISTER_LISTENER(cls) \
  static ::Catch::shim::ListenerRegistrar<cls> CATCH_SHIM_UNIQUE(catch_shim_listener_);
