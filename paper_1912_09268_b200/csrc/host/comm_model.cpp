// mgwfbp-b200 host library: alpha-beta cost model, Table-2 coefficients,
// weighted least-squares calibration fit and the measurement CSV reader.
//
// Parity contract: every floating-point expression below evaluates the same
// operations in the same order as the reference (comm_model.hpp:140-251), and
// the file is compiled with -ffp-contract=off, so results are bit-identical.
// The GPU calibration sweep (csrc/cuda/calibrate.cu) writes the CSV format
// read here (comm_model.hpp:255-308).
#include <cmath>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gradsched/comm_model.hpp"

namespace gradsched {

void AllReduceModel::validate() const {
  // ref comm_model.hpp:37-46
  if (!(a > 0.0)) {
    throw ValidationError("AllReduceModel: startup a must be > 0 (a=" + std::to_string(a) +
                          ")");
  }
  if (!(b >= 0.0)) {
    throw ValidationError("AllReduceModel: per-byte b must be >= 0 (b=" +
                          std::to_string(b) + ")");
  }
}

void NetworkParams::validate() const {
  // ref comm_model.hpp:59-73
  if (!(alpha > 0.0)) throw ValidationError("NetworkParams: alpha must be > 0");
  if (!(beta >= 0.0)) throw ValidationError("NetworkParams: beta must be >= 0");
  if (!(gamma >= 0.0)) throw ValidationError("NetworkParams: gamma must be >= 0");
  if (n_workers < 2) {
    throw ValidationError("NetworkParams: n_workers must be >= 2 (got " +
                          std::to_string(n_workers) + ")");
  }
}

void CommMeasurement::validate() const {
  if (!(time_sec > 0.0)) throw ValidationError("CommMeasurement: time_sec must be > 0");
}

namespace {

struct AlgoName {
  AllReduceAlgorithm algo;
  const char* name;
};

constexpr AlgoName kAlgoNames[] = {
    {AllReduceAlgorithm::kBinaryTree, "binary_tree"},
    {AllReduceAlgorithm::kRecursiveDoubling, "recursive_doubling"},
    {AllReduceAlgorithm::kRecursiveHalvingDoubling, "recursive_halving_doubling"},
    {AllReduceAlgorithm::kDoubleBinaryTrees, "double_binary_trees"},
    {AllReduceAlgorithm::kRing, "ring"},
};

}  // namespace

const char* to_string(AllReduceAlgorithm algo) {
  for (const auto& entry : kAlgoNames) {
    if (entry.algo == algo) return entry.name;
  }
  return "unknown";
}

AllReduceAlgorithm algorithm_from_string(const std::string& name) {
  for (const auto& entry : kAlgoNames) {
    if (name == entry.name) return entry.algo;
  }
  std::string known;
  for (const auto& entry : kAlgoNames) {
    if (!known.empty()) known += ", ";
    known += entry.name;
  }
  throw ValidationError("unknown all-reduce algorithm '" + name + "'; known: " + known);
}

bool is_power_of_two(int n) { return n > 0 && (n & (n - 1)) == 0; }

AllReduceModel coefficients_for(AllReduceAlgorithm algo, const NetworkParams& net,
                                DbtStartup dbt_mode, std::vector<std::string>* warnings) {
  net.validate();
  const double N = static_cast<double>(net.n_workers);
  const double lg = std::log2(N);
  const double al = net.alpha, be = net.beta, ga = net.gamma;
  auto note = [warnings](std::string msg) {
    if (warnings) warnings->push_back(std::move(msg));
  };

  // Paper Table 2; ref comm_model.hpp:152-182. Each
  // expression keeps the reference's association order.
  AllReduceModel m;
  if (algo == AllReduceAlgorithm::kBinaryTree) {
    m.a = 2.0 * al * lg;
    m.b = (2.0 * be + ga) * lg;
  } else if (algo == AllReduceAlgorithm::kRecursiveDoubling) {
    m.a = al * lg;
    m.b = (be + ga) * lg;
  } else if (algo == AllReduceAlgorithm::kRecursiveHalvingDoubling) {
    m.a = 2.0 * al * lg;
    m.b = 2.0 * be - (2.0 * be + ga) / N + ga;
  } else if (algo == AllReduceAlgorithm::kDoubleBinaryTrees) {
    const bool corrected = dbt_mode == DbtStartup::kAlphaCorrected;
    m.a = corrected ? 2.0 * al * lg : 2.0 * lg;
    m.b = be + ga;
    note(corrected ? std::string("double_binary_trees: startup evaluated alpha-corrected as "
                                 "2*alpha*log2(N) (literal form 2*log2(N) available)")
                   : std::string("double_binary_trees: startup evaluated literal as "
                                 "2*log2(N), a count without a time unit"));
  } else {  // kRing
    m.a = 2.0 * (N - 1.0) * al;
    m.b = 2.0 * (N - 1.0) / N * be + (N - 1.0) / N * ga;
  }
  if (algo != AllReduceAlgorithm::kRing && !is_power_of_two(net.n_workers)) {
    std::ostringstream msg;
    msg << to_string(algo) << ": n_workers=" << net.n_workers
        << " is not a power of two; log2(N)=" << lg << " used as a real";
    note(msg.str());
  }
  m.validate();
  return m;
}

double allreduce_cost(const AllReduceModel& model, double size_bytes) {
  if (!(size_bytes >= 0.0)) {
    throw ValidationError("allreduce_cost: size_bytes must be >= 0");
  }
  return model.a + model.b * size_bytes;
}

AllReduceModel fit_model(const std::vector<CommMeasurement>& samples) {
  // ref comm_model.hpp:209-251: weights 1/t^2, two passes (means, then
  // centred moments), b = Sxy/Sxx, a = ybar - b*xbar.
  if (samples.size() < 2) {
    throw FitError("fit_model: need at least 2 measurements (got " +
                   std::to_string(samples.size()) + ")");
  }
  bool two_sizes = false;
  for (const CommMeasurement& s : samples) {
    s.validate();
    two_sizes = two_sizes || s.size_bytes != samples[0].size_bytes;
  }
  if (!two_sizes) throw FitError("fit_model: need at least 2 distinct message sizes");

  double w_sum = 0.0, wx_sum = 0.0, wy_sum = 0.0;
  for (const CommMeasurement& s : samples) {
    const double w = 1.0 / (s.time_sec * s.time_sec);
    w_sum += w;
    wx_sum += w * static_cast<double>(s.size_bytes);
    wy_sum += w * s.time_sec;
  }
  const double x_mean = wx_sum / w_sum;
  const double y_mean = wy_sum / w_sum;
  double sxx = 0.0, sxy = 0.0;
  for (const CommMeasurement& s : samples) {
    const double w = 1.0 / (s.time_sec * s.time_sec);
    const double dx = static_cast<double>(s.size_bytes) - x_mean;
    sxx += w * dx * dx;
    sxy += w * dx * (s.time_sec - y_mean);
  }
  AllReduceModel m;
  m.b = sxy / sxx;
  m.a = y_mean - m.b * x_mean;
  if (!(m.a > 0.0)) {
    throw FitError("fit_model: fitted startup a=" + std::to_string(m.a) +
                   " is not positive; samples do not follow T(M)=a+bM");
  }
  if (!(m.b >= 0.0)) {
    throw FitError("fit_model: fitted per-byte b=" + std::to_string(m.b) +
                   " is negative; samples do not follow T(M)=a+bM");
  }
  return m;
}

namespace {

std::string rstrip_cr_space(std::string s) {
  while (!s.empty() && (s.back() == '\r' || s.back() == ' ')) s.pop_back();
  return s;
}

// Parses one data row; throws std::invalid_argument / std::out_of_range on
// any malformation (the caller maps them to ParseError with the line).
CommMeasurement parse_row(const std::string& row, std::size_t comma) {
  CommMeasurement m;
  std::size_t consumed = 0;
  const std::string size_field = row.substr(0, comma);
  const long long size = std::stoll(size_field, &consumed);
  if (consumed != comma || size < 0) throw std::invalid_argument("size_bytes");
  const std::string time_field = row.substr(comma + 1);
  const double us = std::stod(time_field, &consumed);
  if (consumed != time_field.size()) throw std::invalid_argument("time_us");
  m.size_bytes = static_cast<std::uint64_t>(size);
  m.time_sec = us / 1e6;
  return m;
}

}  // namespace

std::vector<CommMeasurement> load_measurements_csv(std::istream& in) {
  std::string line;
  if (!std::getline(in, line)) throw ParseError("measurement CSV: empty input");
  const std::string header = rstrip_cr_space(line);
  if (header != "size_bytes,time_us") {
    throw ParseError("measurement CSV: header must be 'size_bytes,time_us' (got '" + header +
                     "')");
  }
  std::vector<CommMeasurement> out;
  for (std::size_t lineno = 2; std::getline(in, line); ++lineno) {
    const std::string row = rstrip_cr_space(line);
    if (row.empty()) continue;
    const std::string where = "measurement CSV line " + std::to_string(lineno);
    const std::size_t comma = row.find(',');
    if (comma == std::string::npos) throw ParseError(where + ": expected 'size_bytes,time_us'");
    CommMeasurement m;
    try {
      m = parse_row(row, comma);
    } catch (const std::exception&) {
      throw ParseError(where + ": malformed row '" + row + "'");
    }
    if (!(m.time_sec > 0.0)) throw ParseError(where + ": time_us must be > 0");
    out.push_back(m);
  }
  return out;
}

std::vector<CommMeasurement> load_measurements_csv(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ParseError("cannot open measurement CSV: " + path);
  return load_measurements_csv(in);
}

}  // namespace gradsched
