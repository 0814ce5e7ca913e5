// mgwfbp-b200 host library: worker-count sweep over naive / WFBP /
// single-buffer (SyncEASGD) / MG-WFBP. Semantics follow reference
// proj/include/gradsched/sweep.hpp:92-224: rows sorted by N, four
// strategies per N in kAllStrategies order, a failing N annotates its rows
// instead of aborting, warnings are prefixed "N=<n>: ".
#include <algorithm>
#include <charconv>
#include <string>
#include <vector>

#include "gradsched/sweep.hpp"

namespace gradsched {

const char* to_string(Strategy strategy) {
  switch (strategy) {
    case Strategy::kNaive: return "naive";
    case Strategy::kWfbp: return "wfbp";
    case Strategy::kSyncEasgd: return "synceasgd";
    case Strategy::kMgWfbp: return "mgwfbp";
  }
  return "unknown";
}

Strategy strategy_from_string(const std::string& name) {
  for (Strategy s : kAllStrategies) {
    if (name == to_string(s)) return s;
  }
  throw ValidationError("unknown strategy '" + name +
                        "'; known: naive, wfbp, synceasgd, mgwfbp");
}

std::size_t merged_layer_count(const MergePlan& plan) { return plan.merged_count(); }

namespace {

// Fills iteration/comm/merge fields of `row` for one strategy.
void evaluate(const ModelTrace& trace, const AllReduceModel& model, SweepRow& row) {
  const std::size_t n = trace.n_layers();
  switch (row.strategy) {
    case Strategy::kNaive:
      row.iter_time_sec = naive_time(trace, model);
      row.comm_nonoverlap_sec = row.iter_time_sec - compute_time(trace);
      row.n_merged = 0;
      row.n_groups = n;
      return;
    case Strategy::kWfbp: {
      const Timeline tl = iteration_time(trace, MergePlan::all_normal(n), model);
      row.iter_time_sec = tl.iteration_time;
      row.comm_nonoverlap_sec = tl.comm_nonoverlap;
      row.n_merged = 0;
      row.n_groups = n;
      return;
    }
    case Strategy::kSyncEasgd:
      row.iter_time_sec = synceasgd_time(trace, model);
      row.comm_nonoverlap_sec = row.iter_time_sec - compute_time(trace);
      row.n_merged = n - 1;
      row.n_groups = 1;
      return;
    case Strategy::kMgWfbp: {
      const MergePlan plan = optimal_plan(trace, model);
      const Timeline tl = iteration_time(trace, plan, model);
      row.iter_time_sec = tl.iteration_time;
      row.comm_nonoverlap_sec = tl.comm_nonoverlap;
      row.n_merged = merged_layer_count(plan);
      row.n_groups = n - row.n_merged;
      return;
    }
  }
}

std::string shortest(double v) {
  char buf[64];
  const auto res = std::to_chars(buf, buf + sizeof buf, v);
  return std::string(buf, res.ptr);
}

}  // namespace

SweepResult run_sweep(const ModelTrace& trace, NetworkParams net, AllReduceAlgorithm algo,
                      std::vector<int> worker_counts, DbtStartup dbt_mode) {
  trace.validate();
  std::sort(worker_counts.begin(), worker_counts.end());
  SweepResult out;
  const double backward = trace.total_backward_time();
  for (const int workers : worker_counts) {
    AllReduceModel model;
    std::string model_error;
    try {
      if (workers < 2) {
        throw ValidationError("n_workers must be >= 2 (got " + std::to_string(workers) + ")");
      }
      net.n_workers = workers;
      std::vector<std::string> notes;
      model = coefficients_for(algo, net, dbt_mode, &notes);
      for (const std::string& w : notes) {
        out.warnings.push_back("N=" + std::to_string(workers) + ": " + w);
      }
    } catch (const Error& e) {
      model_error = e.what();
    }
    for (const Strategy strategy : kAllStrategies) {
      SweepRow row;
      row.n_workers = workers;
      row.strategy = strategy;
      row.algo = algo;
      if (!model_error.empty()) {
        row.error = model_error;
      } else {
        try {
          evaluate(trace, model, row);
          row.speedup = speedup(workers, trace.forward_time, backward, row.comm_nonoverlap_sec);
        } catch (const Error& e) {
          row.error = "N=" + std::to_string(workers) + ": " + e.what();
        }
      }
      out.rows.push_back(std::move(row));
    }
  }
  return out;
}

void write_sweep_csv(const SweepResult& result, std::ostream& out) {
  out << "n_workers,strategy,algo,iter_time_us,comm_nonoverlap_us,speedup,n_merged\n";
  for (const SweepRow& r : result.rows) {
    if (!r.ok()) continue;
    out << r.n_workers << ',' << to_string(r.strategy) << ',' << to_string(r.algo) << ','
        << shortest(r.iter_time_sec * 1e6) << ',' << shortest(r.comm_nonoverlap_sec * 1e6)
        << ',' << shortest(r.speedup) << ',' << r.n_merged << '\n';
  }
}

nlohmann::json sweep_to_json(const SweepResult& result) {
  nlohmann::json rows = nlohmann::json::array();
  for (const SweepRow& r : result.rows) {
    nlohmann::json item{{"n_workers", r.n_workers},
                        {"strategy", to_string(r.strategy)},
                        {"algo", to_string(r.algo)}};
    if (r.ok()) {
      item["iter_time_us"] = r.iter_time_sec * 1e6;
      item["comm_nonoverlap_us"] = r.comm_nonoverlap_sec * 1e6;
      item["speedup"] = r.speedup;
      item["n_merged"] = r.n_merged;
      item["n_groups"] = r.n_groups;
    } else {
      item["error"] = r.error;
    }
    rows.push_back(std::move(item));
  }
  nlohmann::json doc;
  doc["rows"] = std::move(rows);
  doc["warnings"] = result.warnings;
  return doc;
}

}  // namespace gradsched
