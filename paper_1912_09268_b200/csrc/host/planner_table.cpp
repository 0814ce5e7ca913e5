// mgwfbp-b200 host library: merge planning with a MEASURED cost curve (a
// B200-native extension; not part of the reference API).
//
// The reference plans with the linear model T(M) = a + b*M
// (comm_model.hpp:194-199). The fused B200 kernel's cost is piecewise: the
// LL protocol below ~512 KiB, the barrier one-shot up to the one-shot /
// two-shot crossover, the two-shot above it — a single (a, b) fit is off by
// up to ~2x at some sizes. Here the same exact DP as optimal_plan
// (planner.hpp:63-98) and the same serialised FIFO timeline
// (timeline.hpp:133-177) use T(M) interpolated from the on-box calibration
// itself: piecewise linear between measured sizes, the smallest size's time
// below it, the last segment's slope above it, made non-decreasing (a
// running max), so the DP's early-exit argument (cost monotone in M) holds.
#include <algorithm>
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <vector>

#include "gradsched/planner.hpp"
#include "planner_table.hpp"

namespace mgw_host {

CostTable::CostTable(std::vector<double> sizes, std::vector<double> times) {
  if (sizes.size() != times.size() || sizes.empty()) {
    throw gradsched::ValidationError("cost table: need >= 1 (size, time) pairs of equal count");
  }
  std::vector<std::size_t> idx(sizes.size());
  for (std::size_t i = 0; i < idx.size(); ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](std::size_t x, std::size_t y) { return sizes[x] < sizes[y]; });
  for (std::size_t i : idx) {
    if (!(times[i] > 0.0) || !(sizes[i] >= 0.0)) {
      throw gradsched::ValidationError("cost table: sizes must be >= 0 and times > 0");
    }
    if (!m_.empty() && sizes[i] == m_.back()) {
      t_.back() = std::max(t_.back(), times[i]);
      continue;
    }
    m_.push_back(sizes[i]);
    t_.push_back(times[i]);
  }
  for (std::size_t i = 1; i < t_.size(); ++i) t_[i] = std::max(t_[i], t_[i - 1]);  // monotone
  tail_slope_ = m_.size() >= 2 ? (t_.back() - t_[t_.size() - 2]) / (m_.back() - m_[m_.size() - 2]) : 0.0;
}

double CostTable::operator()(double M) const {
  if (M <= m_.front()) return t_.front();
  if (M >= m_.back()) return t_.back() + tail_slope_ * (M - m_.back());
  const std::size_t hi = static_cast<std::size_t>(std::upper_bound(m_.begin(), m_.end(), M) - m_.begin());
  const std::size_t lo = hi - 1;
  const double f = (M - m_[lo]) / (m_[hi] - m_[lo]);
  return t_[lo] + f * (t_[hi] - t_[lo]);
}

namespace {

struct Inputs {
  std::vector<double> ready;
  std::vector<double> bytes;
  double compute = 0.0;
};

Inputs inputs(const gradsched::ModelTrace& trace) {
  Inputs in;
  const auto tau_b = gradsched::backward_starts(trace);
  const std::size_t n = trace.n_layers();
  in.ready.resize(n);
  in.bytes.resize(n);
  const double bpe = static_cast<double>(trace.bytes_per_element);
  for (std::size_t i = 0; i < n; ++i) {
    in.ready[i] = tau_b[i] + trace.layers[i].backward_time;
    in.bytes[i] = static_cast<double>(trace.layers[i].params) * bpe;
  }
  return in;
}

}  // namespace

gradsched::MergePlan optimal_plan_table(const gradsched::ModelTrace& trace, const CostTable& cost) {
  trace.validate();
  const Inputs in = inputs(trace);
  const std::size_t n = trace.n_layers();
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
      const double cand = std::max(suffix, ready_g) + cost(m);
      if (u == g + 1 || cand < best) {
        best = cand;
        arg = u;
      }
      if (suffix <= ready_g) break;  // cost is non-decreasing in m: later candidates are >= cand
    }
    finish[g] = best;
    next_head[g] = arg;
  }
  gradsched::MergePlan plan{std::vector<gradsched::LayerTag>(n, gradsched::LayerTag::kMerged)};
  for (std::size_t h = 0; h < n; h = next_head[h]) plan.tags[h] = gradsched::LayerTag::kNormal;
  return plan;
}

double iteration_time_table(const gradsched::ModelTrace& trace, const gradsched::MergePlan& plan,
                            const CostTable& cost) {
  trace.validate();
  plan.validate_for(trace.n_layers());
  const Inputs in = inputs(trace);
  const std::size_t n = trace.n_layers();
  // group bytes at each head (ascending fold, like apply_merge)
  std::vector<double> t_c(n, 0.0);
  for (std::size_t i = 0; i < n;) {
    std::size_t j = i + 1;
    while (j < n && plan.tags[j] == gradsched::LayerTag::kMerged) ++j;
    double m = 0.0;
    for (std::size_t k = i; k < j; ++k) m += in.bytes[k];
    t_c[i] = cost(m);
    i = j;
  }
  // serialised FIFO comm in backward order (timeline.hpp:133-154)
  double tau = -std::numeric_limits<double>::infinity();
  double end = 0.0;
  for (std::size_t i = n; i-- > 0;) {
    if (plan.tags[i] != gradsched::LayerTag::kNormal) continue;
    tau = std::max(tau == -std::numeric_limits<double>::infinity() ? in.ready[i] : end, in.ready[i]);
    end = tau + t_c[i];
  }
  return end;
}

}  // namespace mgw_host
