// mgwfbp-b200 host library: merge plans, group folding and the pipelined
// WFBP timeline (the predictor the measured GPU pipeline is compared with).
//
// Recurrences (reference proj/include/gradsched/timeline.hpp):
//   tau_b[L-1] = t_f,  tau_b[i] = tau_b[i+1] + t_b[i+1]              (:99-108)
//   head[i] = nearest normal layer <= i; bytes folded ascending         (:113-126)
//   tau_c[L-1] = ready[L-1],
//   tau_c[i] = max(tau_c[i+1] + t_c[i+1], tau_b[i] + t_b[i])            (:133-154)
//   iteration = tau_c[0] + t_c[0]                                        (:158-177)
// These are evaluated with the reference's exact operation order.
#include <algorithm>
#include <string>
#include <vector>

#include "gradsched/timeline.hpp"

namespace gradsched {

MergePlan MergePlan::all_normal(std::size_t n_layers) {
  return MergePlan{std::vector<LayerTag>(n_layers, LayerTag::kNormal)};
}

MergePlan MergePlan::all_merged(std::size_t n_layers) {
  MergePlan plan{std::vector<LayerTag>(n_layers, LayerTag::kMerged)};
  if (n_layers > 0) plan.tags.front() = LayerTag::kNormal;
  return plan;
}

std::size_t MergePlan::merged_count() const {
  return static_cast<std::size_t>(std::count(tags.begin(), tags.end(), LayerTag::kMerged));
}

void MergePlan::validate_for(std::size_t n_layers) const {
  if (tags.size() != n_layers) {
    throw ValidationError("MergePlan: " + std::to_string(tags.size()) + " tags given for " +
                          std::to_string(n_layers) + " layers");
  }
  if (n_layers > 0 && tags.front() != LayerTag::kNormal) {
    throw ValidationError("MergePlan: the first layer cannot be merged");
  }
}

std::vector<double> backward_starts(const ModelTrace& trace) {
  trace.validate();
  const std::size_t n = trace.n_layers();
  std::vector<double> tau_b(n);
  double t = trace.forward_time;
  tau_b[n - 1] = t;
  for (std::size_t i = n - 1; i > 0; --i) {
    t = t + trace.layers[i].backward_time;
    tau_b[i - 1] = t;
  }
  return tau_b;
}

CommGroups apply_merge(const ModelTrace& trace, const MergePlan& plan) {
  plan.validate_for(trace.n_layers());
  const std::size_t n = trace.n_layers();
  CommGroups g{std::vector<std::size_t>(n), std::vector<double>(n, 0.0)};
  std::size_t h = 0;
  for (std::size_t i = 0; i < n; ++i) {
    if (plan.tags[i] == LayerTag::kNormal) h = i;
    g.head[i] = h;
    g.bytes[h] += layer_bytes(trace, i);
  }
  return g;
}

CommSchedule comm_starts(const CommGroups& groups, std::span<const double> tau_b,
                         std::span<const double> t_b, const AllReduceModel& model) {
  const std::size_t n = groups.head.size();
  if (tau_b.size() != n || t_b.size() != n) {
    throw ValidationError("comm_starts: head, tau_b and t_b lengths differ");
  }
  CommSchedule s{std::vector<double>(n), std::vector<double>(n)};
  for (std::size_t i = 0; i < n; ++i) {
    s.t_c[i] = groups.head[i] == i ? allreduce_cost(model, groups.bytes[i]) : 0.0;
  }
  s.tau_c[n - 1] = tau_b[n - 1] + t_b[n - 1];
  for (std::size_t i = n - 1; i > 0; --i) {
    const double after_prev = s.tau_c[i] + s.t_c[i];
    const double ready = tau_b[i - 1] + t_b[i - 1];
    s.tau_c[i - 1] = std::max(after_prev, ready);
  }
  return s;
}

namespace {

std::vector<double> backward_times(const ModelTrace& trace) {
  std::vector<double> t_b(trace.n_layers());
  for (std::size_t i = 0; i < t_b.size(); ++i) t_b[i] = trace.layers[i].backward_time;
  return t_b;
}

}  // namespace

Timeline iteration_time(const ModelTrace& trace, const MergePlan& plan,
                        const AllReduceModel& model) {
  Timeline tl;
  tl.forward_time = trace.forward_time;
  tl.tau_b = backward_starts(trace);
  tl.t_b = backward_times(trace);
  CommSchedule s = comm_starts(apply_merge(trace, plan), tl.tau_b, tl.t_b, model);
  tl.tau_c = std::move(s.tau_c);
  tl.t_c = std::move(s.t_c);
  tl.tags = plan.tags;
  tl.iteration_time = tl.tau_c.front() + tl.t_c.front();
  tl.comm_nonoverlap = tl.iteration_time - compute_time(trace);
  return tl;
}

Timeline naive_timeline(const ModelTrace& trace, const AllReduceModel& model) {
  Timeline tl;
  tl.forward_time = trace.forward_time;
  tl.tau_b = backward_starts(trace);
  tl.t_b = backward_times(trace);
  const std::size_t n = trace.n_layers();
  tl.tags.assign(n, LayerTag::kNormal);
  tl.tau_c.resize(n);
  tl.t_c.resize(n);
  double clock = compute_time(trace);
  for (std::size_t i = n; i > 0; --i) {
    tl.tau_c[i - 1] = clock;
    tl.t_c[i - 1] = allreduce_cost(model, layer_bytes(trace, i - 1));
    clock += tl.t_c[i - 1];
  }
  tl.iteration_time = tl.tau_c.front() + tl.t_c.front();
  tl.comm_nonoverlap = tl.iteration_time - compute_time(trace);
  return tl;
}

double naive_time(const ModelTrace& trace, const AllReduceModel& model) {
  trace.validate();
  double t = compute_time(trace);
  for (std::size_t i = trace.n_layers(); i > 0; --i) {
    t += allreduce_cost(model, layer_bytes(trace, i - 1));
  }
  return t;
}

double synceasgd_time(const ModelTrace& trace, const AllReduceModel& model) {
  trace.validate();
  return compute_time(trace) + allreduce_cost(model, total_bytes(trace));
}

double speedup(int n_workers, double forward_time, double backward_time,
               double comm_nonoverlap) {
  const double compute = forward_time + backward_time;
  if (!(compute > 0.0)) {
    throw ValidationError("speedup: forward + backward time must be > 0");
  }
  return static_cast<double>(n_workers) / (1.0 + comm_nonoverlap / compute);
}

nlohmann::json timeline_to_json(const Timeline& tl) {
  nlohmann::json rows = nlohmann::json::array();
  for (std::size_t i = 0; i < tl.tau_b.size(); ++i) {
    rows.push_back(nlohmann::json{{"layer", i + 1},
                                  {"tau_b_us", tl.tau_b[i] * 1e6},
                                  {"t_b_us", tl.t_b[i] * 1e6},
                                  {"tau_c_us", tl.tau_c[i] * 1e6},
                                  {"t_c_us", tl.t_c[i] * 1e6},
                                  {"merged", tl.tags[i] == LayerTag::kMerged}});
  }
  return rows;
}

}  // namespace gradsched
