// mgwfbp-b200: host half of the C ABI (include/mgwfbp.h). Marshals plain
// arrays into gradsched value types and maps C++ exceptions onto status
// codes + a thread-local message (no exception crosses the ABI).
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "capi_common.hpp"
#include "gradsched/gradsched.hpp"
#include "mgwfbp.h"
#include "planner_table.hpp"

namespace mgw {

thread_local std::string g_last_error;
thread_local const char* g_last_kind = "";

void set_error(const std::string& msg) {
  g_last_error = msg;
  g_last_kind = "Error";
}

namespace {
void set_error_kind(const std::string& msg, const char* kind) {
  g_last_error = msg;
  g_last_kind = kind;
}
}  // namespace

int status_from_current_exception() {
  try {
    throw;
  } catch (const gradsched::PlannerError& e) {
    set_error_kind(e.what(), "PlannerError");
    return MGW_ERR_PLANNER;
  } catch (const gradsched::GuardError& e) {
    set_error_kind(e.what(), "GuardError");
    return MGW_ERR_GUARD;
  } catch (const gradsched::ParseError& e) {
    set_error_kind(e.what(), "ParseError");
    return MGW_ERR_INPUT;
  } catch (const gradsched::FitError& e) {
    set_error_kind(e.what(), "FitError");
    return MGW_ERR_INPUT;
  } catch (const gradsched::Error& e) {
    set_error_kind(e.what(), "ValidationError");
    return MGW_ERR_INPUT;
  } catch (const CudaFailure& e) {
    set_error_kind(e.what(), "CudaError");
    return MGW_ERR_CUDA;
  } catch (const std::exception& e) {
    set_error(std::string("internal: ") + e.what());
    return MGW_ERR_INTERNAL;
  } catch (...) {
    set_error("internal: unknown exception");
    return MGW_ERR_INTERNAL;
  }
}

}  // namespace mgw

namespace {

gradsched::ModelTrace make_trace(const uint64_t* params, const double* t_b, size_t L,
                                 double t_f, int bpe) {
  if (L == 0) throw gradsched::ValidationError("trace: L must be >= 1");
  if (params == nullptr || t_b == nullptr) {
    throw gradsched::ValidationError("trace: params and t_b must not be NULL");
  }
  gradsched::ModelTrace trace;
  trace.forward_time = t_f;
  trace.bytes_per_element = bpe;
  trace.layers.resize(L);
  for (size_t i = 0; i < L; ++i) {
    trace.layers[i].name = "layer_" + std::to_string(i + 1);
    trace.layers[i].params = params[i];
    trace.layers[i].backward_time = t_b[i];
  }
  trace.validate();
  return trace;
}

gradsched::MergePlan make_plan(const uint8_t* tags, size_t L) {
  if (tags == nullptr) throw gradsched::ValidationError("tags must not be NULL");
  gradsched::MergePlan plan;
  plan.tags.resize(L);
  for (size_t i = 0; i < L; ++i) {
    if (tags[i] > 1) throw gradsched::ValidationError("tags must be 0 (normal) or 1 (merged)");
    plan.tags[i] = tags[i] ? gradsched::LayerTag::kMerged : gradsched::LayerTag::kNormal;
  }
  plan.validate_for(L);
  return plan;
}

void write_tags(const gradsched::MergePlan& plan, uint8_t* out) {
  for (size_t i = 0; i < plan.tags.size(); ++i) {
    out[i] = plan.tags[i] == gradsched::LayerTag::kMerged ? 1 : 0;
  }
}

}  // namespace

extern "C" {

const char* mgw_last_error(void) { return mgw::g_last_error.c_str(); }

const char* mgw_last_error_kind(void) { return mgw::g_last_kind; }

const char* mgw_version(void) { return "mgwfbp-b200 0.1 (sm_100a)"; }

namespace {
mgw_host::CostTable make_table(const mgw_meas* meas, size_t n) {
  if (meas == nullptr && n != 0) throw gradsched::ValidationError("measurements are NULL");
  std::vector<double> m(n), t(n);
  for (size_t i = 0; i < n; ++i) {
    m[i] = static_cast<double>(meas[i].size_bytes);
    t[i] = meas[i].time_sec;
  }
  return mgw_host::CostTable(std::move(m), std::move(t));
}
}  // namespace

int mgw_plan_optimal_table(const uint64_t* params, const double* t_b, size_t L, double t_f, int bpe,
                           const mgw_meas* meas, size_t n_meas, uint8_t* tags_out) {
  MGW_TRY {
    const auto trace = make_trace(params, t_b, L, t_f, bpe);
    write_tags(mgw_host::optimal_plan_table(trace, make_table(meas, n_meas)), tags_out);
  }
  MGW_CATCH
}

int mgw_predict_table(const uint64_t* params, const double* t_b, size_t L, double t_f, int bpe,
                      const mgw_meas* meas, size_t n_meas, const uint8_t* tags, double* iter_time_out) {
  MGW_TRY {
    const auto trace = make_trace(params, t_b, L, t_f, bpe);
    const double t = mgw_host::iteration_time_table(trace, make_plan(tags, L), make_table(meas, n_meas));
    if (iter_time_out) *iter_time_out = t;
  }
  MGW_CATCH
}

int mgw_fit(const mgw_meas* samples, size_t n, double* a_out, double* b_out) {
  MGW_TRY {
    std::vector<gradsched::CommMeasurement> v(n);
    for (size_t i = 0; i < n; ++i) v[i] = {samples[i].size_bytes, samples[i].time_sec};
    const gradsched::AllReduceModel m = gradsched::fit_model(v);
    *a_out = m.a;
    *b_out = m.b;
  }
  MGW_CATCH
}

int mgw_load_measurements_csv(const char* path, mgw_meas* out, size_t cap, size_t* n_out) {
  MGW_TRY {
    const auto v = gradsched::load_measurements_csv(std::string(path));
    *n_out = v.size();
    if (out != nullptr) {
      if (cap < v.size()) throw gradsched::ValidationError("output capacity too small");
      for (size_t i = 0; i < v.size(); ++i) out[i] = {v[i].size_bytes, v[i].time_sec};
    }
  }
  MGW_CATCH
}

int mgw_coefficients(int algo, double alpha, double beta, double gamma, int n_workers,
                     int dbt_literal, double* a_out, double* b_out) {
  MGW_TRY {
    if (algo < 0 || algo > 4) throw gradsched::ValidationError("algo must be in 0..4");
    gradsched::NetworkParams net{alpha, beta, gamma, n_workers};
    const auto m = gradsched::coefficients_for(
        static_cast<gradsched::AllReduceAlgorithm>(algo), net,
        dbt_literal ? gradsched::DbtStartup::kLiteral : gradsched::DbtStartup::kAlphaCorrected);
    *a_out = m.a;
    *b_out = m.b;
  }
  MGW_CATCH
}

int mgw_load_trace(const char* path, size_t* L_out, double* t_f_out, int* bpe_out,
                   uint64_t* params_out, double* t_b_out, size_t cap) {
  MGW_TRY {
    const gradsched::ModelTrace t = gradsched::load_trace(std::string(path));
    *L_out = t.n_layers();
    if (t_f_out) *t_f_out = t.forward_time;
    if (bpe_out) *bpe_out = t.bytes_per_element;
    if (params_out != nullptr || t_b_out != nullptr) {
      if (cap < t.n_layers()) throw gradsched::ValidationError("output capacity too small");
      for (size_t i = 0; i < t.n_layers(); ++i) {
        if (params_out) params_out[i] = t.layers[i].params;
        if (t_b_out) t_b_out[i] = t.layers[i].backward_time;
      }
    }
  }
  MGW_CATCH
}

int mgw_plan_optimal(const uint64_t* params, const double* t_b, size_t L, double t_f, int bpe,
                     double a, double b, uint8_t* tags_out) {
  MGW_TRY {
    const auto trace = make_trace(params, t_b, L, t_f, bpe);
    write_tags(gradsched::optimal_plan(trace, {a, b}), tags_out);
  }
  MGW_CATCH
}

int mgw_plan_greedy(const uint64_t* params, const double* t_b, size_t L, double t_f, int bpe,
                    double a, double b, uint8_t* tags_out) {
  MGW_TRY {
    const auto trace = make_trace(params, t_b, L, t_f, bpe);
    write_tags(gradsched::greedy_plan(trace, {a, b}), tags_out);
  }
  MGW_CATCH
}

int mgw_plan_brute_force(const uint64_t* params, const double* t_b, size_t L, double t_f,
                         int bpe, double a, double b, size_t max_layers, uint8_t* tags_out,
                         double* iter_time_out) {
  MGW_TRY {
    const auto trace = make_trace(params, t_b, L, t_f, bpe);
    const auto r = gradsched::brute_force_plan(trace, {a, b}, max_layers);
    write_tags(r.plan, tags_out);
    if (iter_time_out) *iter_time_out = r.iteration_time;
  }
  MGW_CATCH
}

int mgw_predict(const uint64_t* params, const double* t_b, size_t L, double t_f, int bpe,
                double a, double b, const uint8_t* tags, double* iter_time_out,
                double* comm_nonoverlap_out, double* tau_b_out, double* tau_c_out,
                double* t_c_out) {
  MGW_TRY {
    const auto trace = make_trace(params, t_b, L, t_f, bpe);
    const auto tl = gradsched::iteration_time(trace, make_plan(tags, L), {a, b});
    if (iter_time_out) *iter_time_out = tl.iteration_time;
    if (comm_nonoverlap_out) *comm_nonoverlap_out = tl.comm_nonoverlap;
    for (size_t i = 0; i < L; ++i) {
      if (tau_b_out) tau_b_out[i] = tl.tau_b[i];
      if (tau_c_out) tau_c_out[i] = tl.tau_c[i];
      if (t_c_out) t_c_out[i] = tl.t_c[i];
    }
  }
  MGW_CATCH
}

int mgw_baseline_times(const uint64_t* params, const double* t_b, size_t L, double t_f, int bpe,
                       double a, double b, double* synceasgd_out, double* naive_out) {
  MGW_TRY {
    const auto trace = make_trace(params, t_b, L, t_f, bpe);
    if (synceasgd_out) *synceasgd_out = gradsched::synceasgd_time(trace, {a, b});
    if (naive_out) *naive_out = gradsched::naive_time(trace, {a, b});
  }
  MGW_CATCH
}

long mgw_synth_trace_json(size_t n_layers, uint64_t total_params, double total_backward_time,
                          double forward_time, double size_skew, int bpe, uint64_t seed, char* buf,
                          size_t cap) {
  try {
    gradsched::SynthSpec s;
    s.n_layers = n_layers;
    s.total_params = total_params;
    s.total_backward_time = total_backward_time;
    s.forward_time = forward_time;
    s.size_skew = size_skew;
    s.bytes_per_element = bpe;
    s.seed = seed;
    std::ostringstream os;
    gradsched::save_trace(gradsched::synth_trace(s), os);
    const std::string text = os.str();
    if (buf != nullptr && cap > text.size()) std::memcpy(buf, text.c_str(), text.size() + 1);
    return static_cast<long>(text.size());
  } catch (...) {
    return -static_cast<long>(mgw::status_from_current_exception());
  }
}

}  // extern "C"
