// Minimal Catch2-compatible test shim (our own code, not Catch2).
//
// Purpose: compile the reference's OWN unit and acceptance suites
// (/root/reference/proj/tests/*.cpp, read in place, never copied) against
// this repo's gradsched headers + libmgwfbp.so. That is the API drop-in
// check: the reference tests must build and pass unchanged.
//
// Supported surface (everything those files use): TEST_CASE, flat SECTIONs
// (one section per run, Catch2's leaf-section semantics for one level),
// REQUIRE, REQUIRE_FALSE, REQUIRE_THROWS_AS, FAIL, Catch::Approx with
// epsilon()/margin().
#ifndef MGWFBP_CATCH_SHIM_HPP_
#define MGWFBP_CATCH_SHIM_HPP_

#include <cmath>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace Catch {

class Approx {
 public:
  explicit Approx(double value) : value_(value) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double other) const {
    // Catch2 v3 rule: within the absolute margin, or within
    // epsilon * (scale + |value|).
    const double diff = std::fabs(other - value_);
    if (diff <= margin_) return true;
    const double rel = eps_ * (scale_ + (std::isinf(value_) ? 0.0 : std::fabs(value_)));
    return diff <= rel;
  }
  double value() const { return value_; }

  friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
  friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }
  friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || rhs.matches(lhs); }
  friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || rhs.matches(lhs); }

 private:
  double value_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100.0;
  double margin_ = 0.0;
  double scale_ = 0.0;
};

}  // namespace Catch

namespace shim {

struct Failure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

using TestFn = void (*)();

struct TestCaseInfo {
  const char* name;
  TestFn fn;
  const char* file;
  int line;
};

inline std::vector<TestCaseInfo>& registry() {
  static std::vector<TestCaseInfo> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, TestFn fn, const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};

// Flat-section driver: run k of a test case executes only section k.
struct SectionState {
  int target = 0;
  int seen = 0;
};

inline SectionState& sections() {
  static SectionState s;
  return s;
}

inline bool enter_section() {
  SectionState& s = sections();
  return s.seen++ == s.target;
}

[[noreturn]] inline void fail(const char* file, int line, const std::string& what) {
  std::ostringstream os;
  os << file << ":" << line << ": " << what;
  throw Failure(os.str());
}

}  // namespace shim

#define SHIM_CAT2(a, b) a##b
#define SHIM_CAT(a, b) SHIM_CAT2(a, b)

#define TEST_CASE(name, ...)                                                              \
  static void SHIM_CAT(shim_test_, __LINE__)();                                           \
  static shim::Registrar SHIM_CAT(shim_reg_, __LINE__)(name, &SHIM_CAT(shim_test_, __LINE__), \
                                                       __FILE__, __LINE__);               \
  static void SHIM_CAT(shim_test_, __LINE__)()

#define SECTION(...) if (shim::enter_section())

#define REQUIRE(...)                                                       \
  do {                                                                     \
    if (!(__VA_ARGS__)) shim::fail(__FILE__, __LINE__, "REQUIRE( " #__VA_ARGS__ " )"); \
  } while (0)

#define REQUIRE_FALSE(...)                                                 \
  do {                                                                     \
    if ((__VA_ARGS__)) shim::fail(__FILE__, __LINE__, "REQUIRE_FALSE( " #__VA_ARGS__ " )"); \
  } while (0)

#define REQUIRE_THROWS_AS(expr, type)                                                  \
  do {                                                                                 \
    bool shim_caught_ = false;                                                         \
    try {                                                                              \
      static_cast<void>(expr);                                                         \
    } catch (const type&) {                                                            \
      shim_caught_ = true;                                                             \
    } catch (const std::exception& shim_e_) {                                          \
      shim::fail(__FILE__, __LINE__,                                                   \
                 std::string("REQUIRE_THROWS_AS( " #expr ", " #type " ) threw another "  \
                             "exception: ") + shim_e_.what());                         \
    }                                                                                  \
    if (!shim_caught_) shim::fail(__FILE__, __LINE__, "REQUIRE_THROWS_AS( " #expr " ) did not throw"); \
  } while (0)

#define FAIL(msg) shim::fail(__FILE__, __LINE__, std::string("FAIL: ") + (msg))

#endif  // MGWFBP_CATCH_SHIM_HPP_
