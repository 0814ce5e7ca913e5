// mgwfbp-b200: source-compatible error hierarchy of the gradsched API.
//
// Drop-in for reference proj/include/gradsched/errors.hpp:24-57. Every
// error thrown by the host library derives from gradsched::Error (itself a
// std::runtime_error), and the five leaf classes keep the reference names so
// code that catches them by type keeps compiling.
#ifndef MGWFBP_GRADSCHED_ERRORS_HPP_
#define MGWFBP_GRADSCHED_ERRORS_HPP_

#include <stdexcept>
#include <string>

namespace gradsched {

class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

#define MGWFBP_DECLARE_ERROR(Name)     \
  class Name : public Error {          \
   public:                             \
    using Error::Error;                \
  }

// A domain value breaks an invariant (negative time, a <= 0, ...).
MGWFBP_DECLARE_ERROR(ValidationError);
// A file or stream does not match its schema.
MGWFBP_DECLARE_ERROR(ParseError);
// The weighted least-squares fit is underdetermined or unusable.
MGWFBP_DECLARE_ERROR(FitError);
// A cost model the planner cannot use.
MGWFBP_DECLARE_ERROR(PlannerError);
// A guarded operation refused to run (exhaustive search too large).
MGWFBP_DECLARE_ERROR(GuardError);

#undef MGWFBP_DECLARE_ERROR

}  // namespace gradsched

#endif  // MGWFBP_GRADSCHED_ERRORS_HPP_
