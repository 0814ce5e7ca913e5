// mgwfbp-b200: merge planning with a measured cost curve (B200 extension).
#ifndef MGWFBP_PLANNER_TABLE_HPP_
#define MGWFBP_PLANNER_TABLE_HPP_

#include <vector>

#include "gradsched/planner.hpp"

namespace mgw_host {

// T(M) interpolated from measured (size bytes, seconds) pairs: piecewise
// linear, flat below the smallest size, last slope above the largest,
// non-decreasing.
class CostTable {
 public:
  CostTable(std::vector<double> sizes, std::vector<double> times);
  double operator()(double bytes) const;

 private:
  std::vector<double> m_, t_;
  double tail_slope_ = 0.0;
};

gradsched::MergePlan optimal_plan_table(const gradsched::ModelTrace& trace, const CostTable& cost);
double iteration_time_table(const gradsched::ModelTrace& trace, const gradsched::MergePlan& plan,
                            const CostTable& cost);

}  // namespace mgw_host

#endif  // MGWFBP_PLANNER_TABLE_HPP_
