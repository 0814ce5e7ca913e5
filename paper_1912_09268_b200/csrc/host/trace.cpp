// mgwfbp-b200 host library: trace schema, JSON I/O, synthetic generator.
//
// Parity notes (reference proj/include/gradsched/trace.hpp):
//  * file times are microseconds, divided by 1e6 on load (:161, :205) and
//    multiplied by 1e6 on save (:224, :231);
//  * compute_time / total_backward_time accumulate last layer first
//    (:88-93, :99-105), total_bytes first layer first (:121-127);
//  * synth_trace draws all size weights, then all time weights, from the top
//    53 bits of mt19937_64 (:285-291, :268-272), floors the proportional
//    split and hands the remainder out by descending fractional part with a
//    stable sort (:305-343). skewed_161.json must regenerate byte-for-byte.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "gradsched/trace.hpp"

namespace gradsched {

void ModelTrace::validate() const {
  if (layers.empty()) throw ValidationError("ModelTrace: must have at least one layer");
  if (!(forward_time >= 0.0)) throw ValidationError("ModelTrace: forward_time must be >= 0");
  if (bytes_per_element != 2 && bytes_per_element != 4) {
    throw ValidationError("ModelTrace: bytes_per_element must be 2 or 4 (got " +
                          std::to_string(bytes_per_element) + ")");
  }
  std::size_t index = 0;
  for (const LayerProfile& layer : layers) {
    ++index;
    if (!(layer.backward_time >= 0.0)) {
      throw ValidationError("ModelTrace: layer " + std::to_string(index) + " ('" + layer.name +
                            "') has a negative backward_time");
    }
  }
  const bool any = std::any_of(layers.begin(), layers.end(),
                               [](const LayerProfile& l) { return l.params > 0; });
  if (!any) throw ValidationError("ModelTrace: at least one layer must have params > 0");
}

std::uint64_t ModelTrace::total_params() const {
  std::uint64_t sum = 0;
  for (const LayerProfile& l : layers) sum += l.params;
  return sum;
}

double ModelTrace::total_backward_time() const {
  double sum = 0.0;
  for (std::size_t i = layers.size(); i > 0; --i) sum += layers[i - 1].backward_time;
  return sum;
}

double compute_time(const ModelTrace& trace) {
  double t = trace.forward_time;
  for (std::size_t i = trace.layers.size(); i > 0; --i) t += trace.layers[i - 1].backward_time;
  return t;
}

double layer_bytes(const ModelTrace& trace, std::size_t index) {
  if (index >= trace.layers.size()) {
    throw ValidationError("layer_bytes: index " + std::to_string(index) +
                          " is out of range for a trace of " +
                          std::to_string(trace.layers.size()) + " layers");
  }
  return static_cast<double>(trace.layers[index].params) *
         static_cast<double>(trace.bytes_per_element);
}

double total_bytes(const ModelTrace& trace) {
  double sum = 0.0;
  for (std::size_t i = 0; i < trace.layers.size(); ++i) sum += layer_bytes(trace, i);
  return sum;
}

namespace {

using Json = nlohmann::json;

double number_field(const Json& obj, const char* key, const std::string& where) {
  const auto it = obj.find(key);
  if (it == obj.end()) {
    throw ParseError("trace: missing field '" + std::string(key) + "' " + where);
  }
  if (!it->is_number()) {
    throw ParseError("trace: field '" + std::string(key) + "' " + where + " must be a number");
  }
  return it->get<double>();
}

LayerProfile parse_layer(const Json& item, std::size_t index) {
  const std::string where = "in layer " + std::to_string(index);
  if (!item.is_object()) {
    throw ParseError("trace: layer " + std::to_string(index) + " must be an object");
  }
  LayerProfile layer;
  const auto name = item.find("name");
  if (name == item.end() || !name->is_string()) {
    throw ParseError("trace: missing or non-string field 'name' " + where);
  }
  layer.name = name->get<std::string>();
  const auto params = item.find("params");
  if (params == item.end() || !params->is_number_integer()) {
    throw ParseError("trace: missing or non-integer field 'params' " + where);
  }
  const std::int64_t p = params->get<std::int64_t>();
  if (p < 0) throw ValidationError("trace: field 'params' " + where + " must be >= 0");
  layer.params = static_cast<std::uint64_t>(p);
  const double us = number_field(item, "backward_time_us", where);
  if (us < 0.0) {
    throw ValidationError("trace: field 'backward_time_us' " + where + " must be >= 0");
  }
  layer.backward_time = us / 1e6;
  return layer;
}

}  // namespace

ModelTrace load_trace(std::istream& in, std::vector<std::string>* warnings) {
  Json doc;
  try {
    in >> doc;
  } catch (const Json::exception& e) {
    throw ParseError(std::string("trace: invalid JSON: ") + e.what());
  }
  if (!doc.is_object()) throw ParseError("trace: top-level value must be an object");

  ModelTrace trace;
  trace.forward_time = number_field(doc, "forward_time_us", "at top level") / 1e6;
  const auto bpe = doc.find("bytes_per_element");
  if (bpe != doc.end()) {
    if (!bpe->is_number_integer()) {
      throw ParseError("trace: field 'bytes_per_element' must be an integer");
    }
    trace.bytes_per_element = bpe->get<int>();
  } else {
    trace.bytes_per_element = 4;
    if (warnings) {
      warnings->push_back("trace: bytes_per_element not given; assuming 4 (fp32)");
    }
  }
  const auto layers = doc.find("layers");
  if (layers == doc.end() || !layers->is_array()) {
    throw ParseError("trace: missing or non-array field 'layers'");
  }
  std::size_t index = 0;
  for (const Json& item : *layers) trace.layers.push_back(parse_layer(item, ++index));
  trace.validate();
  return trace;
}

ModelTrace load_trace(const std::string& path, std::vector<std::string>* warnings) {
  std::ifstream in(path);
  if (!in) throw ParseError("cannot open trace file: " + path);
  return load_trace(in, warnings);
}

nlohmann::json trace_to_json(const ModelTrace& trace) {
  Json layers = Json::array();
  for (const LayerProfile& l : trace.layers) {
    layers.push_back(Json{{"name", l.name},
                          {"params", l.params},
                          {"backward_time_us", l.backward_time * 1e6}});
  }
  Json doc;
  doc["forward_time_us"] = trace.forward_time * 1e6;
  doc["bytes_per_element"] = trace.bytes_per_element;
  doc["layers"] = std::move(layers);
  return doc;
}

void save_trace(const ModelTrace& trace, std::ostream& out) {
  out << trace_to_json(trace).dump(2) << '\n';
}

void save_trace(const ModelTrace& trace, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw ParseError("cannot open trace file for writing: " + path);
  save_trace(trace, out);
}

namespace {

// Uniform [0,1) from the top 53 bits of one 64-bit draw.
double unit_draw(std::mt19937_64& gen) { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }

}  // namespace

ModelTrace synth_trace(const SynthSpec& spec) {
  if (spec.n_layers == 0) throw ValidationError("synth_trace: n_layers must be positive");
  if (spec.total_params == 0) throw ValidationError("synth_trace: total_params must be positive");
  if (!(spec.total_backward_time > 0.0)) {
    throw ValidationError("synth_trace: total_backward_time must be positive");
  }
  if (!(spec.forward_time >= 0.0)) throw ValidationError("synth_trace: forward_time must be >= 0");
  if (!(spec.size_skew >= 0.0)) throw ValidationError("synth_trace: size_skew must be >= 0");

  const std::size_t n = spec.n_layers;
  std::mt19937_64 gen(spec.seed);
  std::vector<double> w_size(n), w_time(n);
  for (double& w : w_size) w = std::pow(unit_draw(gen), spec.size_skew);
  for (double& w : w_time) w = 0.25 + unit_draw(gen);
  double size_sum = std::accumulate(w_size.begin(), w_size.end(), 0.0);
  if (!(size_sum > 0.0)) {
    w_size[0] = 1.0;
    size_sum = 1.0;
  }
  const double time_sum = std::accumulate(w_time.begin(), w_time.end(), 0.0);

  ModelTrace trace;
  trace.forward_time = spec.forward_time;
  trace.bytes_per_element = spec.bytes_per_element;
  trace.layers.resize(n);
  std::vector<double> remainder_frac(n);
  std::uint64_t handed_out = 0;
  for (std::size_t i = 0; i < n; ++i) {
    const double share = static_cast<double>(spec.total_params) * w_size[i] / size_sum;
    const double whole = std::floor(share);
    remainder_frac[i] = share - whole;
    char name[32];
    std::snprintf(name, sizeof name, "layer_%03zu", i + 1);
    LayerProfile& layer = trace.layers[i];
    layer.name = name;
    layer.params = static_cast<std::uint64_t>(whole);
    layer.backward_time = spec.total_backward_time * w_time[i] / time_sum;
    handed_out += layer.params;
  }
  std::vector<std::size_t> by_frac(n);
  std::iota(by_frac.begin(), by_frac.end(), std::size_t{0});
  std::stable_sort(by_frac.begin(), by_frac.end(), [&](std::size_t x, std::size_t y) {
    return remainder_frac[x] > remainder_frac[y];
  });
  std::uint64_t left = spec.total_params - handed_out;
  for (std::size_t k = 0; left > 0; --left, k = (k + 1) % n) {
    trace.layers[by_frac[k]].params += 1;
  }
  trace.validate();
  return trace;
}

}  // namespace gradsched
