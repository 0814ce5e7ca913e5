// mgwfbp-b200 host library: merge-plan solvers.
//
// optimal_plan — exact dynamic program over communication-group heads
// (reference proj/include/gradsched/planner.hpp:63-98):
//
//   finish(L) = -inf
//   finish(g) = min_{u in (g, L]} max(finish(u), ready[g]) + a + b*M(g..u-1)
//
// with M folded ascending from g, ties kept by the FIRST (smallest) u.
//
// Exactness-preserving speed-up. finish(u) is non-increasing in u (a longer
// suffix can always reuse the shorter suffix's schedule with its first group
// extended downwards; ready[] is non-increasing, the ascending byte fold is
// monotone under round-to-nearest). Once finish(u) <= ready[g], every later
// candidate is ready[g] + cost(M') with M' >= M, i.e. >= the candidate just
// evaluated, and the strict '<' would never take it. The scan stops there.
// Every value that is computed is computed with the reference's operations,
// so best_finish[], next_head[] and the tags are bit-identical; only dead
// candidates are skipped. Typical windows are a handful of layers, so the
// O(L^2) loop becomes ~O(L).
//
// greedy_plan — paper Algorithm 1 (reference
// planner.hpp:112-148). The reference recomputes the whole tau_c array after
// every merge; only tau_c[i-1] is read afterwards and it equals
// max(tau_c[i] + t_c[i], ready[i-1]) evaluated with the current t_c, which is
// what we carry forward. O(L), bit-identical decisions.
#include <algorithm>
#include <cstdint>
#include <limits>
#include <string>
#include <vector>

#include "gradsched/planner.hpp"

namespace gradsched {

namespace {

void check_planner_model(const AllReduceModel& m) {
  // ref planner.hpp:36-45
  if (!(m.a > 0.0)) {
    throw PlannerError("planner: startup a must be > 0 for merging to pay off (a=" +
                       std::to_string(m.a) + ")");
  }
  if (!(m.b >= 0.0)) throw PlannerError("planner: per-byte b must be >= 0");
}

struct PlanInputs {
  std::vector<double> tau_b;
  std::vector<double> t_b;
  std::vector<double> ready;
  std::vector<double> bytes;
};

PlanInputs plan_inputs(const ModelTrace& trace) {
  PlanInputs in;
  in.tau_b = backward_starts(trace);
  const std::size_t n = trace.n_layers();
  in.t_b.resize(n);
  in.ready.resize(n);
  in.bytes.resize(n);
  const double bpe = static_cast<double>(trace.bytes_per_element);
  for (std::size_t i = 0; i < n; ++i) {
    in.t_b[i] = trace.layers[i].backward_time;
    in.ready[i] = in.tau_b[i] + in.t_b[i];
    in.bytes[i] = static_cast<double>(trace.layers[i].params) * bpe;
  }
  return in;
}

}  // namespace

MergePlan optimal_plan(const ModelTrace& trace, const AllReduceModel& model) {
  check_planner_model(model);
  const PlanInputs in = plan_inputs(trace);
  const std::size_t n = trace.n_layers();
  const double a = model.a, b = model.b;

  std::vector<double> finish(n + 1);
  std::vector<std::size_t> next_head(n + 1, n);
  finish[n] = -std::numeric_limits<double>::infinity();
  for (std::size_t g = n; g-- > 0;) {
    const double ready_g = in.ready[g];
    double best = 0.0;
    std::size_t arg = n;
    double m = 0.0;
    for (std::size_t u = g + 1; u <= n; ++u) {
      m += in.bytes[u - 1];
      const double suffix = finish[u];
      const double cand = std::max(suffix, ready_g) + (a + b * m);
      if (u == g + 1 || cand < best) {
        best = cand;
        arg = u;
      }
      if (suffix <= ready_g) break;  // all later candidates are >= cand
    }
    finish[g] = best;
    next_head[g] = arg;
  }

  MergePlan plan{std::vector<LayerTag>(n, LayerTag::kMerged)};
  for (std::size_t h = 0; h < n; h = next_head[h]) plan.tags[h] = LayerTag::kNormal;
  return plan;
}

MergePlan greedy_plan(const ModelTrace& trace, const AllReduceModel& model) {
  check_planner_model(model);
  const PlanInputs in = plan_inputs(trace);
  const std::size_t n = trace.n_layers();
  std::vector<double> bytes = in.bytes;
  std::vector<double> t_c(n);
  for (std::size_t i = 0; i < n; ++i) t_c[i] = allreduce_cost(model, bytes[i]);

  MergePlan plan = MergePlan::all_normal(n);
  // tau_c of the layer under inspection, carried downwards.
  double tau_c = in.tau_b[n - 1] + in.t_b[n - 1];
  for (std::size_t i = n - 1; i >= 1; --i) {
    const double ready_below = in.tau_b[i - 1] + in.t_b[i - 1];
    if (ready_below - tau_c < model.a) {
      t_c[i] = 0.0;
      bytes[i - 1] += bytes[i];
      t_c[i - 1] = allreduce_cost(model, bytes[i - 1]);
      plan.tags[i] = LayerTag::kMerged;
    }
    tau_c = std::max(tau_c + t_c[i], ready_below);
  }
  return plan;
}

PlanSearchResult brute_force_plan(const ModelTrace& trace, const AllReduceModel& model,
                                  std::size_t max_layers) {
  // ref planner.hpp:159-200: every plan with tags[0] normal, ranked by
  // (iteration time, merged count, lexicographic tags).
  check_planner_model(model);
  trace.validate();
  const std::size_t n = trace.n_layers();
  if (n > max_layers) {
    throw GuardError("brute_force_plan: refusing " + std::to_string(n) +
                     " layers, which means 2^" + std::to_string(n - 1) +
                     " candidate plans (limit " + std::to_string(max_layers) + " layers)");
  }
  PlanSearchResult best;
  std::size_t best_merged = 0;
  bool have = false;
  const std::uint64_t count = std::uint64_t{1} << (n - 1);
  MergePlan plan = MergePlan::all_normal(n);
  for (std::uint64_t mask = 0; mask < count; ++mask) {
    for (std::size_t i = 1; i < n; ++i) {
      plan.tags[i] = ((mask >> (i - 1)) & 1u) ? LayerTag::kMerged : LayerTag::kNormal;
    }
    const double t = iteration_time(trace, plan, model).iteration_time;
    const std::size_t merged = plan.merged_count();
    bool better = !have || t < best.iteration_time;
    if (!better && t == best.iteration_time) {
      better = merged < best_merged ||
               (merged == best_merged && plan.tags < best.plan.tags);
    }
    if (better) {
      best.plan = plan;
      best.iteration_time = t;
      best_merged = merged;
      have = true;
    }
  }
  return best;
}

OverlapCase case_classify(const Timeline& tl, std::size_t index, double startup) {
  // ref planner.hpp:204-233 (paper's four overlap cases, Fig. 3)
  if (index == 0) throw ValidationError("case_classify: layer 1 has no lower layer");
  if (index >= tl.tau_c.size()) throw ValidationError("case_classify: layer index out of range");
  if (tl.tags[index] != LayerTag::kNormal) {
    throw ValidationError("case_classify: needs an all-normal timeline");
  }
  const double start = tl.tau_c[index];
  const double end = start + tl.t_c[index];
  const double lower_ready = tl.tau_b[index - 1] + tl.t_b[index - 1];
  if (end <= lower_ready) return OverlapCase::kFullyHidden;
  if (start >= lower_ready) return OverlapCase::kNotOverlapped;
  return lower_ready - start < startup ? OverlapCase::kPartialMergeHelps
                                       : OverlapCase::kPartialMergeHurts;
}

nlohmann::json plan_to_json(const ModelTrace& trace, const MergePlan& plan,
                            const AllReduceModel& model) {
  const Timeline tl = iteration_time(trace, plan, model);
  const CommGroups g = apply_merge(trace, plan);
  nlohmann::json tags = nlohmann::json::array();
  for (LayerTag t : plan.tags) tags.push_back(t == LayerTag::kNormal ? "normal" : "merged");
  nlohmann::json groups = nlohmann::json::array();
  const std::size_t n = plan.tags.size();
  for (std::size_t h = 0; h < n; ++h) {
    if (g.head[h] != h) continue;
    nlohmann::json members = nlohmann::json::array();
    for (std::size_t j = h; j < n && g.head[j] == h; ++j) members.push_back(j + 1);
    groups.push_back(std::move(members));
  }
  nlohmann::json doc;
  doc["tags"] = std::move(tags);
  doc["groups"] = std::move(groups);
  doc["predicted_iter_time_us"] = tl.iteration_time * 1e6;
  return doc;
}

}  // namespace gradsched
