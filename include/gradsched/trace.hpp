// mgwfbp-b200: per-layer model trace schema, JSON I/O and the synthetic
// generator (declarations).
//
// Source-compatible with reference proj/include/gradsched/trace.hpp:
//   LayerProfile / ModelTrace      trace.hpp:38-94
//   compute_time                   trace.hpp:99-105
//   layer_bytes / total_bytes      trace.hpp:108-127
//   load_trace / trace_to_json /
//   save_trace                     trace.hpp:148-248
//   SynthSpec / synth_trace        trace.hpp:257-346
// Layers are in forward order; the backward pass visits them last to first.
#ifndef MGWFBP_GRADSCHED_TRACE_HPP_
#define MGWFBP_GRADSCHED_TRACE_HPP_

#include <cstddef>
#include <cstdint>
#include <istream>
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

#include "gradsched/errors.hpp"

namespace gradsched {

struct LayerProfile {
  std::string name;
  std::uint64_t params = 0;    // gradient elements
  double backward_time = 0.0;  // seconds
};

struct ModelTrace {
  std::vector<LayerProfile> layers;  // forward order
  double forward_time = 0.0;         // seconds
  int bytes_per_element = 4;         // 4 = fp32, 2 = fp16/bf16

  std::size_t n_layers() const { return layers.size(); }
  void validate() const;
  std::uint64_t total_params() const;
  // Accumulated last layer first (the timeline's order).
  double total_backward_time() const;
};

// forward_time + sum of backward times, accumulated last layer first.
double compute_time(const ModelTrace& trace);
// (double)params * (double)bytes_per_element of layer `index`.
double layer_bytes(const ModelTrace& trace, std::size_t index);
// Sum of layer_bytes in ascending layer order.
double total_bytes(const ModelTrace& trace);

ModelTrace load_trace(std::istream& in, std::vector<std::string>* warnings = nullptr);
ModelTrace load_trace(const std::string& path,
                      std::vector<std::string>* warnings = nullptr);
nlohmann::json trace_to_json(const ModelTrace& trace);
// dump(2) plus a newline; save(load(x)) is byte-stable.
void save_trace(const ModelTrace& trace, std::ostream& out);
void save_trace(const ModelTrace& trace, const std::string& path);

struct SynthSpec {
  std::size_t n_layers = 0;
  std::uint64_t total_params = 0;
  double total_backward_time = 0.0;  // seconds
  double forward_time = 0.0;         // seconds
  double size_skew = 8.0;
  int bytes_per_element = 4;
  std::uint64_t seed = 0;
};

// Deterministic: the same spec yields a byte-identical trace.
ModelTrace synth_trace(const SynthSpec& spec);

}  // namespace gradsched

#endif  // MGWFBP_GRADSCHED_TRACE_HPP_
