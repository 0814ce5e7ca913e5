// mgwfbp-b200: merge-plan solvers (declarations).
//
// Source-compatible with reference proj/include/gradsched/planner.hpp:
//   optimal_plan      planner.hpp:63-98    exact DP over group heads
//   greedy_plan       planner.hpp:112-148  paper Algorithm 1
//   brute_force_plan  planner.hpp:150-200  exhaustive oracle (L <= 20)
//   case_classify     planner.hpp:202-233
//   plan_to_json      planner.hpp:237-257
//
// optimal_plan and greedy_plan return bit-identical tags to the reference on
// every input. They are faster than the reference without changing a single
// floating-point operation: the DP stops scanning group ends once the
// remaining suffix finishes before the head's gradients are ready (all later
// candidates can only be >=), and the greedy updates the one comm-start it
// reads next instead of recomputing the whole array after each merge.
#ifndef MGWFBP_GRADSCHED_PLANNER_HPP_
#define MGWFBP_GRADSCHED_PLANNER_HPP_

#include <cstddef>

// The reference includes <json.hpp> from its vendor/ directory
// (proj/CMakeLists.txt:11-13, planner.hpp:25); either layout works.
#if __has_include(<nlohmann/json.hpp>)
#include <nlohmann/json.hpp>
#else
#include <json.hpp>
#endif

#include "gradsched/comm_model.hpp"
#include "gradsched/errors.hpp"
#include "gradsched/timeline.hpp"
#include "gradsched/trace.hpp"

namespace gradsched {

MergePlan optimal_plan(const ModelTrace& trace, const AllReduceModel& model);
MergePlan greedy_plan(const ModelTrace& trace, const AllReduceModel& model);

struct PlanSearchResult {
  MergePlan plan;
  double iteration_time = 0.0;
};

PlanSearchResult brute_force_plan(const ModelTrace& trace, const AllReduceModel& model,
                                  std::size_t max_layers = 20);

enum class OverlapCase {
  kFullyHidden,
  kPartialMergeHelps,
  kPartialMergeHurts,
  kNotOverlapped,
};

OverlapCase case_classify(const Timeline& timeline, std::size_t index, double startup);

nlohmann::json plan_to_json(const ModelTrace& trace, const MergePlan& plan,
                            const AllReduceModel& model);

}  // namespace gradsched

#endif  // MGWFBP_GRADSCHED_PLANNER_HPP_
