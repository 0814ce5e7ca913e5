// mgwfbp-b200: worker-count sweep over the four strategies (declarations).
//
// Source-compatible with reference proj/include/gradsched/sweep.hpp:
//   Strategy / to_string / strategy_from_string   sweep.hpp:37-59
//   SweepRow / SweepResult                        sweep.hpp:64-84
//   run_sweep                                     sweep.hpp:92-173
//   write_sweep_csv / sweep_to_json               sweep.hpp:189-224
// Kept so the reference's sweep tests and acceptance criteria compile and
// so on-box calibrated (a, b) can be projected past 8 GPUs.
#ifndef MGWFBP_GRADSCHED_SWEEP_HPP_
#define MGWFBP_GRADSCHED_SWEEP_HPP_

#include <cstddef>
#include <ostream>
#include <string>
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
#include "gradsched/planner.hpp"
#include "gradsched/timeline.hpp"
#include "gradsched/trace.hpp"

namespace gradsched {

enum class Strategy { kNaive, kWfbp, kSyncEasgd, kMgWfbp };

const char* to_string(Strategy strategy);
Strategy strategy_from_string(const std::string& name);

inline constexpr Strategy kAllStrategies[] = {Strategy::kNaive, Strategy::kWfbp,
                                              Strategy::kSyncEasgd, Strategy::kMgWfbp};

struct SweepRow {
  int n_workers = 0;
  Strategy strategy = Strategy::kNaive;
  AllReduceAlgorithm algo = AllReduceAlgorithm::kRing;
  double iter_time_sec = 0.0;
  double comm_nonoverlap_sec = 0.0;
  double speedup = 0.0;
  std::size_t n_merged = 0;
  std::size_t n_groups = 0;
  std::string error;

  bool ok() const { return error.empty(); }
};

struct SweepResult {
  std::vector<SweepRow> rows;
  std::vector<std::string> warnings;
};

std::size_t merged_layer_count(const MergePlan& plan);

SweepResult run_sweep(const ModelTrace& trace, NetworkParams net, AllReduceAlgorithm algo,
                      std::vector<int> worker_counts,
                      DbtStartup dbt_mode = DbtStartup::kAlphaCorrected);

void write_sweep_csv(const SweepResult& result, std::ostream& out);
nlohmann::json sweep_to_json(const SweepResult& result);

}  // namespace gradsched

#endif  // MGWFBP_GRADSCHED_SWEEP_HPP_
