// Minimal Catch2-compatible test shim (TEST INFRASTRUCTURE).
//
// The reference's unit tests (proj/tests/test_*.cpp) include
// <catch2/catch_amalgamated.hpp>, which is not installed in this image.  This
// shim implements exactly the subset they use -- TEST_CASE, REQUIRE,
// REQUIRE_THROWS_AS, CAPTURE, FAIL, Catch::Approx -- so the reference test
// sources compile unmodified against this repo's drop-in headers
// (include/ranger/) and run on the GPU path.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace catch_shim {

struct Failure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Case {
  std::string name;
  std::function<void()> fn;
};

inline std::vector<Case>& registry() {
  static std::vector<Case> cases;
  return cases;
}

inline std::vector<std::string>& captures() {
  static std::vector<std::string> c;
  return c;
}

struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct Capture {
  explicit Capture(std::string s) { captures().push_back(std::move(s)); }
  ~Capture() { captures().pop_back(); }
};

[[noreturn]] inline void fail(const char* file, int line, const std::string& what) {
  std::ostringstream os;
  os << file << ":" << line << ": " << what;
  for (const auto& c : captures()) os << "\n    with " << c;
  throw Failure(os.str());
}

template <typename T>
std::string show(const T&) {
  return "?";
}

}  // namespace catch_shim

namespace Catch {
class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  bool matches(double other) const {
    const double tol = eps_ * (std::fabs(value_) + std::fabs(other)) / 2 + margin_;
    return std::fabs(other - value_) <= std::max(tol, eps_ * std::fabs(value_));
  }
  friend bool operator==(double a, const Approx& b) { return b.matches(a); }
  friend bool operator==(const Approx& a, double b) { return a.matches(b); }
  friend bool operator!=(double a, const Approx& b) { return !b.matches(a); }
  friend bool operator!=(const Approx& a, double b) { return !a.matches(b); }

 private:
  double value_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double margin_ = 0.0;
};
}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define TEST_CASE(name, ...)                                                             \
  static void CATCH_SHIM_CAT(catch_shim_case_, __LINE__)();                              \
  static catch_shim::Registrar CATCH_SHIM_CAT(catch_shim_reg_, __LINE__)(               \
      name, &CATCH_SHIM_CAT(catch_shim_case_, __LINE__));                                \
  static void CATCH_SHIM_CAT(catch_shim_case_, __LINE__)()

#define REQUIRE(...)                                                                     \
  do {                                                                                   \
    if (!(__VA_ARGS__)) catch_shim::fail(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")"); \
  } while (0)

#define REQUIRE_THROWS_AS(expr, type)                                                    \
  do {                                                                                   \
    bool catch_shim_ok = false;                                                          \
    try {                                                                                \
      (void)(expr);                                                                      \
    } catch (const type&) {                                                              \
      catch_shim_ok = true;                                                              \
    } catch (...) {                                                                      \
    }                                                                                    \
    if (!catch_shim_ok)                                                                  \
      catch_shim::fail(__FILE__, __LINE__, "REQUIRE_THROWS_AS(" #expr ", " #type ")");   \
  } while (0)

#define CAPTURE(...) catch_shim::Capture CATCH_SHIM_CAT(catch_shim_cap_, __LINE__)(#__VA_ARGS__)
#define FAIL(msg)                                                                        \
  do {                                                                                   \
    std::ostringstream catch_shim_os;                                                    \
    catch_shim_os << msg;                                                                \
    catch_shim::fail(__FILE__, __LINE__, "FAIL: " + catch_shim_os.str());                \
  } while (0)
