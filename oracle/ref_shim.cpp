// ref_shim.cpp — C entry points over the UNMODIFIED reference headers.
// TEST INFRASTRUCTURE ONLY.
//
// Compiled by oracle/Makefile directly against
// /root/reference/proj/include/gradsched/*.hpp (read in place, never copied)
// with the reference's Release flags (-O3 -DNDEBUG, proj/CMakeLists.txt:6-8)
// plus -ffp-contract=off, into oracle/_ref/libgradsched_ref.so. Used by the
// parity tests to pin the C restatement and the product solver against the
// reference itself, and by bench.py --impl reference to time the
// reference's own solver on the GPU box's host.
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "gradsched/gradsched.hpp"

namespace {

gradsched::ModelTrace mk(const uint64_t* params, const double* t_b, size_t L, double t_f,
                         int bpe) {
  gradsched::ModelTrace t;
  t.forward_time = t_f;
  t.bytes_per_element = bpe;
  for (size_t i = 0; i < L; ++i) t.layers.push_back({"l" + std::to_string(i), params[i], t_b[i]});
  return t;
}

void put_tags(const gradsched::MergePlan& p, uint8_t* tags) {
  for (size_t i = 0; i < p.tags.size(); ++i) tags[i] = p.tags[i] == gradsched::LayerTag::kMerged;
}

gradsched::MergePlan get_tags(const uint8_t* tags, size_t L) {
  gradsched::MergePlan p;
  for (size_t i = 0; i < L; ++i) {
    p.tags.push_back(tags[i] ? gradsched::LayerTag::kMerged : gradsched::LayerTag::kNormal);
  }
  return p;
}

int code() {
  try {
    throw;
  } catch (const gradsched::PlannerError&) {
    return 3;
  } catch (const gradsched::GuardError&) {
    return 4;
  } catch (const gradsched::Error&) {
    return 2;
  } catch (...) {
    return 7;
  }
}

}  // namespace

extern "C" {

int ref_optimal_plan(const uint64_t* params, const double* t_b, size_t L, double t_f, int bpe,
                     double a, double b, uint8_t* tags) {
  try {
    put_tags(gradsched::optimal_plan(mk(params, t_b, L, t_f, bpe), {a, b}), tags);
    return 0;
  } catch (...) {
    return code();
  }
}

int ref_greedy_plan(const uint64_t* params, const double* t_b, size_t L, double t_f, int bpe,
                    double a, double b, uint8_t* tags) {
  try {
    put_tags(gradsched::greedy_plan(mk(params, t_b, L, t_f, bpe), {a, b}), tags);
    return 0;
  } catch (...) {
    return code();
  }
}

int ref_brute_force_plan(const uint64_t* params, const double* t_b, size_t L, double t_f,
                         int bpe, double a, double b, uint8_t* tags, double* iter_time) {
  try {
    const auto r = gradsched::brute_force_plan(mk(params, t_b, L, t_f, bpe), {a, b});
    put_tags(r.plan, tags);
    *iter_time = r.iteration_time;
    return 0;
  } catch (...) {
    return code();
  }
}

int ref_iteration_time(const uint64_t* params, const double* t_b, size_t L, double t_f, int bpe,
                       double a, double b, const uint8_t* tags, double* iter_time,
                       double* nonoverlap) {
  try {
    const auto tl = gradsched::iteration_time(mk(params, t_b, L, t_f, bpe), get_tags(tags, L),
                                              {a, b});
    *iter_time = tl.iteration_time;
    if (nonoverlap) *nonoverlap = tl.comm_nonoverlap;
    return 0;
  } catch (...) {
    return code();
  }
}

int ref_synceasgd_time(const uint64_t* params, const double* t_b, size_t L, double t_f, int bpe,
                       double a, double b, double* out) {
  try {
    *out = gradsched::synceasgd_time(mk(params, t_b, L, t_f, bpe), {a, b});
    return 0;
  } catch (...) {
    return code();
  }
}

int ref_fit(const uint64_t* sizes, const double* times, size_t n, double* a, double* b) {
  try {
    std::vector<gradsched::CommMeasurement> v;
    for (size_t i = 0; i < n; ++i) v.push_back({sizes[i], times[i]});
    const auto m = gradsched::fit_model(v);
    *a = m.a;
    *b = m.b;
    return 0;
  } catch (...) {
    return code();
  }
}

int ref_fit_csv(const char* path, double* a, double* b) {
  try {
    const auto m = gradsched::fit_model(gradsched::load_measurements_csv(std::string(path)));
    *a = m.a;
    *b = m.b;
    return 0;
  } catch (...) {
    return code();
  }
}

// Canonical save_trace() text of synth_trace(spec) into buf (NUL-terminated);
// returns the needed size (excluding NUL) or -code.
long ref_synth_trace(size_t n_layers, uint64_t total_params, double total_backward_time,
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
    if (buf && cap > text.size()) std::memcpy(buf, text.c_str(), text.size() + 1);
    return static_cast<long>(text.size());
  } catch (...) {
    return -code();
  }
}

}  // extern "C"
