// mgwfbp-b200: umbrella header, drop-in for reference
// proj/include/gradsched/gradsched.hpp:18-23. Link against
// paper_1912_09268_b200/lib/libmgwfbp.so.
#ifndef MGWFBP_GRADSCHED_GRADSCHED_HPP_
#define MGWFBP_GRADSCHED_GRADSCHED_HPP_

#include "gradsched/comm_model.hpp"
#include "gradsched/errors.hpp"
#include "gradsched/planner.hpp"
#include "gradsched/sweep.hpp"
#include "gradsched/timeline.hpp"
#include "gradsched/trace.hpp"

#endif  // MGWFBP_GRADSCHED_GRADSCHED_HPP_
