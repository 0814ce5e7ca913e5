// mgwfbp-b200: merge plans and the pipelined WFBP timeline (declarations).
//
// Source-compatible with reference proj/include/gradsched/timeline.hpp:
//   LayerTag / MergePlan        timeline.hpp:32-67
//   CommGroups / CommSchedule   timeline.hpp:72-84
//   Timeline                    timeline.hpp:86-95
//   backward_starts             timeline.hpp:99-108
//   apply_merge                 timeline.hpp:113-126  (defines the pack layout)
//   comm_starts                 timeline.hpp:133-154  (serialized FIFO comm)
//   iteration_time              timeline.hpp:158-177  (the predictor)
//   naive_* / synceasgd_time    timeline.hpp:181-221
//   speedup                     timeline.hpp:225-233
//   timeline_to_json            timeline.hpp:237-250
//
// The same recursion is what the GPU pipeline (csrc/cuda/pipeline.cu)
// executes: one all-reduce in flight per rank, groups in backward order, a
// group launched when its head layer's gradients are ready.
#ifndef MGWFBP_GRADSCHED_TIMELINE_HPP_
#define MGWFBP_GRADSCHED_TIMELINE_HPP_

#include <cstddef>
#include <span>
#include <vector>

// The reference includes <json.hpp> from its vendor/ directory
// (proj/CMakeLists.txt:11-13, planner.hpp:25); either layout works.
#if __has_include(<nlohmann/json.hpp>)
#include <nlohmann/json.hpp>
#else
#include <json.hpp>
#endif

#include "gradsched/comm_model.hpp"
#include "gradsched/errors.hpp"
#include "gradsched/trace.hpp"

namespace gradsched {

enum class LayerTag { kNormal, kMerged };

// tags[i] == kMerged folds layer i's gradients into the next lower layer.
struct MergePlan {
  std::vector<LayerTag> tags;

  static MergePlan all_normal(std::size_t n_layers);  // WFBP
  static MergePlan all_merged(std::size_t n_layers);  // single buffer
  std::size_t merged_count() const;
  void validate_for(std::size_t n_layers) const;
};

// head[i]: group head (nearest normal layer <= i); bytes[h]: folded size at
// heads, zero elsewhere.
struct CommGroups {
  std::vector<std::size_t> head;
  std::vector<double> bytes;
};

struct CommSchedule {
  std::vector<double> tau_c;
  std::vector<double> t_c;
};

struct Timeline {
  std::vector<double> tau_b;
  std::vector<double> t_b;
  std::vector<double> tau_c;
  std::vector<double> t_c;
  std::vector<LayerTag> tags;
  double forward_time = 0.0;
  double iteration_time = 0.0;
  double comm_nonoverlap = 0.0;
};

std::vector<double> backward_starts(const ModelTrace& trace);
CommGroups apply_merge(const ModelTrace& trace, const MergePlan& plan);
CommSchedule comm_starts(const CommGroups& groups, std::span<const double> tau_b,
                         std::span<const double> t_b, const AllReduceModel& model);
Timeline iteration_time(const ModelTrace& trace, const MergePlan& plan,
                        const AllReduceModel& model);
Timeline naive_timeline(const ModelTrace& trace, const AllReduceModel& model);
double naive_time(const ModelTrace& trace, const AllReduceModel& model);
double synceasgd_time(const ModelTrace& trace, const AllReduceModel& model);
double speedup(int n_workers, double forward_time, double backward_time,
               double comm_nonoverlap);
nlohmann::json timeline_to_json(const Timeline& timeline);

}  // namespace gradsched

#endif  // MGWFBP_GRADSCHED_TIMELINE_HPP_
