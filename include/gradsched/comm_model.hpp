// mgwfbp-b200: alpha-beta all-reduce cost model (declarations).
//
// Source-compatible with reference proj/include/gradsched/comm_model.hpp.
// Definitions live in paper_1912_09268_b200/csrc/host/comm_model.cpp, which
// is compiled with -ffp-contract=off so a + b*M rounds exactly like the
// reference's x86-64 (no FMA) build.
//
//   AllReduceModel            comm_model.hpp:33-47
//   NetworkParams             comm_model.hpp:53-74
//   AllReduceAlgorithm        comm_model.hpp:76-82
//   DbtStartup                comm_model.hpp:86-89
//   CommMeasurement           comm_model.hpp:121-130
//   coefficients_for          comm_model.hpp:140-191  (paper Table 2)
//   allreduce_cost            comm_model.hpp:194-199
//   fit_model                 comm_model.hpp:209-251  (1/t^2 weighted LS)
//   load_measurements_csv     comm_model.hpp:255-308
#ifndef MGWFBP_GRADSCHED_COMM_MODEL_HPP_
#define MGWFBP_GRADSCHED_COMM_MODEL_HPP_

#include <cstdint>
#include <istream>
#include <string>
#include <vector>

#include "gradsched/errors.hpp"

namespace gradsched {

// T(M) = a + b*M seconds for an M-byte all-reduce.
struct AllReduceModel {
  double a = 0.0;  // startup, seconds
  double b = 0.0;  // seconds per byte

  // Throws ValidationError unless a > 0 and b >= 0.
  void validate() const;
};

// Point-to-point parameters for the closed-form (Table 2) costs.
struct NetworkParams {
  double alpha = 0.0;  // per-message latency, s
  double beta = 0.0;   // per-byte transfer time, s/B
  double gamma = 0.0;  // per-byte reduction time, s/B
  int n_workers = 0;

  void validate() const;
};

enum class AllReduceAlgorithm {
  kBinaryTree,
  kRecursiveDoubling,
  kRecursiveHalvingDoubling,
  kDoubleBinaryTrees,
  kRing,
};

// The published double-binary-trees startup is the unitless 2*log2(N);
// kAlphaCorrected evaluates 2*alpha*log2(N) instead.
enum class DbtStartup {
  kAlphaCorrected,
  kLiteral,
};

const char* to_string(AllReduceAlgorithm algo);
AllReduceAlgorithm algorithm_from_string(const std::string& name);

// One timed all-reduce: message bytes and elapsed seconds.
struct CommMeasurement {
  std::uint64_t size_bytes = 0;
  double time_sec = 0.0;

  void validate() const;
};

bool is_power_of_two(int n);

AllReduceModel coefficients_for(AllReduceAlgorithm algo, const NetworkParams& net,
                                DbtStartup dbt_mode = DbtStartup::kAlphaCorrected,
                                std::vector<std::string>* warnings = nullptr);

// a + b*size_bytes; ValidationError if size_bytes is negative or NaN.
double allreduce_cost(const AllReduceModel& model, double size_bytes);

AllReduceModel fit_model(const std::vector<CommMeasurement>& samples);

// CSV with header `size_bytes,time_us`; times converted to seconds.
std::vector<CommMeasurement> load_measurements_csv(std::istream& in);
std::vector<CommMeasurement> load_measurements_csv(const std::string& path);

}  // namespace gradsched

#endif  // MGWFBP_GRADSCHED_COMM_MODEL_HPP_
