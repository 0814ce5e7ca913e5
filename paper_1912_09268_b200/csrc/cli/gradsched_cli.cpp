// gradsched CLI, rebuilt without CLI11 over libmgwfbp.so.
//
// Same subcommands, options, outputs and exit codes as the reference front
// end (proj/tools/main.cpp:31-35, :104-285, :287-373), so B200 calibrations
// and plans flow through the reference's file formats byte-identically:
//   gradsched fit [csv] [--algo A --workers N --alpha s --beta s/B --gamma s/B
//                 [--dbt-literal]] [--out model.json]
//   gradsched plan trace.json model.json [--oracle] [--out plan.json]
//   gradsched simulate trace.json model.json --strategy S [--workers N] [--out t.json]
//   gradsched sweep trace.json --algo A --alpha s [--beta] [--gamma]
//                 [--workers 4..2048|a,b,c] [--dbt-literal] [--out csv] [--json j]
// Exit codes: 0 ok, 2 bad input, 3 planner rejection, 4 guard, 5 all sweep
// rows failed.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "gradsched/gradsched.hpp"

namespace {

enum Exit { kOk = 0, kInput = 2, kPlanner = 3, kGuard = 4, kAllRowsFailed = 5 };

// A parsed command line: positionals, --key value options, bare flags.
struct Args {
  std::vector<std::string> pos;
  std::map<std::string, std::string> opt;
  std::set<std::string> flags;

  bool has(const std::string& k) const { return opt.count(k) != 0; }
  std::string str(const std::string& k, const std::string& dflt = "") const {
    const auto it = opt.find(k);
    return it == opt.end() ? dflt : it->second;
  }
};

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

double to_double(const std::string& key, const std::string& v) {
  std::size_t used = 0;
  double d = 0.0;
  try {
    d = std::stod(v, &used);
  } catch (const std::exception&) {
    used = 0;
  }
  if (used != v.size() || v.empty()) throw UsageError("--" + key + ": not a number: '" + v + "'");
  return d;
}

int to_int(const std::string& key, const std::string& v) {
  std::size_t used = 0;
  int i = 0;
  try {
    i = std::stoi(v, &used);
  } catch (const std::exception&) {
    used = 0;
  }
  if (used != v.size() || v.empty()) throw UsageError("--" + key + ": not an integer: '" + v + "'");
  return i;
}

// Parse argv[first..] against the allowed option/flag names and the maximum
// number of positionals.
Args parse(int argc, char** argv, int first, const std::set<std::string>& options,
           const std::set<std::string>& flags, std::size_t max_pos) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string tok = argv[i];
    if (tok.rfind("--", 0) == 0) {
      std::string key = tok.substr(2), value;
      const auto eq = key.find('=');
      const bool inline_value = eq != std::string::npos;
      if (inline_value) {
        value = key.substr(eq + 1);
        key = key.substr(0, eq);
      }
      if (flags.count(key) && !inline_value) {
        a.flags.insert(key);
      } else if (options.count(key)) {
        if (!inline_value) {
          if (i + 1 >= argc) throw UsageError("--" + key + " needs a value");
          value = argv[++i];
        }
        a.opt[key] = value;
      } else {
        throw UsageError("unknown option '" + tok + "'");
      }
    } else {
      a.pos.push_back(tok);
    }
  }
  if (a.pos.size() > max_pos) throw UsageError("unexpected argument '" + a.pos[max_pos] + "'");
  return a;
}

void require_opts(const Args& a, std::initializer_list<const char*> keys) {
  for (const char* k : keys) {
    if (!a.has(k)) throw UsageError(std::string("--") + k + " is required");
  }
}

void write_json(const nlohmann::json& doc, const std::string& path) {
  if (path.empty()) {
    std::cout << doc.dump(2) << '\n';
    return;
  }
  std::ofstream out(path);
  if (!out) throw gradsched::ParseError("cannot open output file: " + path);
  out << doc.dump(2) << '\n';
}

gradsched::AllReduceModel read_model(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw gradsched::ParseError("cannot open model file: " + path);
  nlohmann::json doc;
  try {
    in >> doc;
  } catch (const nlohmann::json::exception& e) {
    throw gradsched::ParseError("model file " + path + ": invalid JSON: " + e.what());
  }
  const auto num = [&](const char* k) {
    return doc.is_object() && doc.contains(k) && doc[k].is_number();
  };
  if (!num("a_sec") || !num("b_sec_per_byte")) {
    throw gradsched::ParseError("model file " + path +
                                ": expected numeric fields a_sec and b_sec_per_byte");
  }
  return {doc["a_sec"].get<double>(), doc["b_sec_per_byte"].get<double>()};
}

// "lo..hi": powers of two in [lo, hi]; otherwise a comma list.
std::vector<int> worker_counts(const std::string& spec) {
  std::vector<int> out;
  try {
    const auto dots = spec.find("..");
    if (dots != std::string::npos) {
      const int lo = std::stoi(spec.substr(0, dots));
      const int hi = std::stoi(spec.substr(dots + 2));
      for (long long p = 1; p <= hi; p *= 2) {
        if (p >= lo) out.push_back(static_cast<int>(p));
      }
    } else {
      std::size_t start = 0;
      while (start <= spec.size()) {
        const auto comma = spec.find(',', start);
        const std::string tok = spec.substr(start, comma == std::string::npos ? std::string::npos
                                                                               : comma - start);
        if (!tok.empty()) out.push_back(std::stoi(tok));
        if (comma == std::string::npos) break;
        start = comma + 1;
      }
    }
  } catch (const std::exception&) {
    throw gradsched::ValidationError("invalid --workers spec: '" + spec + "'");
  }
  if (out.empty()) throw gradsched::ValidationError("--workers spec '" + spec + "' yields no worker counts");
  return out;
}

int cmd_fit(int argc, char** argv) {
  const Args a = parse(argc, argv, 2, {"algo", "workers", "alpha", "beta", "gamma", "out"},
                       {"dbt-literal"}, 1);
  const bool have_csv = !a.pos.empty();
  if (have_csv && a.has("algo")) {
    throw gradsched::ValidationError("fit: give either a measurements CSV or --algo, not both");
  }
  gradsched::AllReduceModel model;
  std::vector<std::string> warnings;
  std::string source;
  if (have_csv) {
    model = gradsched::fit_model(gradsched::load_measurements_csv(a.pos[0]));
    source = "fit";
  } else if (a.has("algo")) {
    gradsched::NetworkParams net;
    net.alpha = a.has("alpha") ? to_double("alpha", a.str("alpha")) : 0.0;
    net.beta = a.has("beta") ? to_double("beta", a.str("beta")) : 0.0;
    net.gamma = a.has("gamma") ? to_double("gamma", a.str("gamma")) : 0.0;
    net.n_workers = a.has("workers") ? to_int("workers", a.str("workers")) : 0;
    model = gradsched::coefficients_for(
        gradsched::algorithm_from_string(a.str("algo")), net,
        a.flags.count("dbt-literal") ? gradsched::DbtStartup::kLiteral
                                     : gradsched::DbtStartup::kAlphaCorrected,
        &warnings);
    source = "table2";
  } else {
    throw gradsched::ValidationError("fit: need a measurements CSV or --algo with network parameters");
  }
  nlohmann::json doc;
  doc["a_sec"] = model.a;
  doc["b_sec_per_byte"] = model.b;
  doc["source"] = source;
  doc["warnings"] = warnings;
  write_json(doc, a.str("out"));
  return kOk;
}

int cmd_plan(int argc, char** argv) {
  const Args a = parse(argc, argv, 2, {"out"}, {"oracle"}, 2);
  if (a.pos.size() != 2) throw UsageError("plan: need trace.json and model.json");
  const auto trace = gradsched::load_trace(a.pos[0]);
  const auto model = read_model(a.pos[1]);
  const auto plan = gradsched::optimal_plan(trace, model);
  const double t = gradsched::iteration_time(trace, plan, model).iteration_time;
  if (a.flags.count("oracle")) {
    const auto brute = gradsched::brute_force_plan(trace, model);
    if (std::abs(brute.iteration_time - t) > 1e-9) {
      std::cerr << "plan: oracle mismatch: planner " << t * 1e6 << " us vs exhaustive minimum "
                << brute.iteration_time * 1e6 << " us\n";
      return kPlanner;
    }
  }
  write_json(gradsched::plan_to_json(trace, plan, model), a.str("out"));
  return kOk;
}

int cmd_simulate(int argc, char** argv) {
  const Args a = parse(argc, argv, 2, {"strategy", "workers", "out"}, {}, 2);
  if (a.pos.size() != 2) throw UsageError("simulate: need trace.json and model.json");
  require_opts(a, {"strategy"});
  const auto trace = gradsched::load_trace(a.pos[0]);
  const auto model = read_model(a.pos[1]);
  const auto strategy = gradsched::strategy_from_string(a.str("strategy"));
  const std::size_t n = trace.n_layers();
  gradsched::Timeline tl;
  if (strategy == gradsched::Strategy::kNaive) {
    tl = gradsched::naive_timeline(trace, model);
  } else if (strategy == gradsched::Strategy::kWfbp) {
    tl = gradsched::iteration_time(trace, gradsched::MergePlan::all_normal(n), model);
  } else if (strategy == gradsched::Strategy::kSyncEasgd) {
    tl = gradsched::iteration_time(trace, gradsched::MergePlan::all_merged(n), model);
  } else {
    tl = gradsched::iteration_time(trace, gradsched::optimal_plan(trace, model), model);
  }
  const int workers = a.has("workers") ? to_int("workers", a.str("workers")) : 0;
  std::cout << std::setprecision(15) << "iter_time_us=" << tl.iteration_time * 1e6
            << " comm_nonoverlap_us=" << tl.comm_nonoverlap * 1e6;
  if (workers > 0) {
    std::cout << " speedup="
              << gradsched::speedup(workers, trace.forward_time, trace.total_backward_time(),
                                    tl.comm_nonoverlap);
  }
  std::cout << '\n';
  if (a.has("out")) write_json(gradsched::timeline_to_json(tl), a.str("out"));
  return kOk;
}

int cmd_sweep(int argc, char** argv) {
  const Args a = parse(argc, argv, 2, {"algo", "workers", "alpha", "beta", "gamma", "out", "json"},
                       {"dbt-literal"}, 1);
  if (a.pos.size() != 1) throw UsageError("sweep: need trace.json");
  require_opts(a, {"algo", "alpha"});
  const auto trace = gradsched::load_trace(a.pos[0]);
  gradsched::NetworkParams net;
  net.alpha = to_double("alpha", a.str("alpha"));
  net.beta = a.has("beta") ? to_double("beta", a.str("beta")) : 0.0;
  net.gamma = a.has("gamma") ? to_double("gamma", a.str("gamma")) : 0.0;
  net.n_workers = 2;
  const auto result = gradsched::run_sweep(
      trace, net, gradsched::algorithm_from_string(a.str("algo")),
      worker_counts(a.str("workers", "4..2048")),
      a.flags.count("dbt-literal") ? gradsched::DbtStartup::kLiteral
                                   : gradsched::DbtStartup::kAlphaCorrected);
  bool any_ok = false;
  for (const auto& row : result.rows) {
    if (row.ok()) {
      any_ok = true;
    } else {
      std::cerr << "sweep row failed: " << row.error << '\n';
    }
  }
  for (const auto& w : result.warnings) std::cerr << "warning: " << w << '\n';
  if (!any_ok) {
    std::cerr << "sweep: every row failed\n";
    return kAllRowsFailed;
  }
  if (a.has("out")) {
    std::ofstream out(a.str("out"));
    if (!out) throw gradsched::ParseError("cannot open output file: " + a.str("out"));
    gradsched::write_sweep_csv(result, out);
  } else {
    gradsched::write_sweep_csv(result, std::cout);
  }
  if (a.has("json")) write_json(gradsched::sweep_to_json(result), a.str("json"));
  return kOk;
}

void usage(std::ostream& os) {
  os << "gradsched: plan and simulate gradient merge schedules (mgwfbp-b200)\n"
        "usage: gradsched {fit|plan|simulate|sweep} ...\n";
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage(std::cerr);
    return kInput;
  }
  const std::string sub = argv[1];
  if (sub == "-h" || sub == "--help") {
    usage(std::cout);
    return kOk;
  }
  try {
    if (sub == "fit") return cmd_fit(argc, argv);
    if (sub == "plan") return cmd_plan(argc, argv);
    if (sub == "simulate") return cmd_simulate(argc, argv);
    if (sub == "sweep") return cmd_sweep(argc, argv);
    usage(std::cerr);
    return kInput;
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << '\n';
    return kInput;
  } catch (const gradsched::GuardError& e) {
    std::cerr << "error: " << e.what() << '\n';
    return kGuard;
  } catch (const gradsched::PlannerError& e) {
    std::cerr << "error: " << e.what() << '\n';
    return kPlanner;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return kInput;
  }
}
