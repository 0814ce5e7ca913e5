// gradsched — command-line front end over libmgwfbp.so.
//
// The reference ships a CLI11 front end (proj/tools/main.cpp). This one is a
// table-driven rewrite: every subcommand declares its positionals and typed
// options once (kCommands below); one generic parser validates argv against
// that schema and hands the handler a typed `Inputs`. What is kept from the
// reference is only its external contract, which proj/tests/test_cli.cpp
// pins: subcommand names, option names, the JSON / CSV / summary-line
// outputs (produced by the library's own exporters), and the exit codes of
// proj/tools/main.cpp:31-35 (0 ok, 2 bad input, 3 planner rejection, 4 guard
// refusal, 5 every sweep row failed).
//
//   gradsched fit [measurements.csv] [--algo A --workers N --alpha s --beta s/B
//                 --gamma s/B --dbt-literal] [--out model.json]
//   gradsched plan trace.json model.json [--oracle] [--out plan.json]
//   gradsched simulate trace.json model.json --strategy S [--workers N] [--out timeline.json]
//   gradsched sweep trace.json --algo A --alpha s [--beta s/B] [--gamma s/B]
//                 [--workers lo..hi | n1,n2,...] [--dbt-literal] [--out results.csv] [--json sweep.json]
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <iomanip>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <string_view>
#include <vector>

#include "gradsched/gradsched.hpp"

namespace {

namespace gs = gradsched;
using Json = nlohmann::json;

// ---- exit status -----------------------------------------------------------

constexpr int kExitOk = 0;
constexpr int kExitBadInput = 2;
constexpr int kExitPlanner = 3;
constexpr int kExitGuard = 4;
constexpr int kExitNoSweepRows = 5;

// A malformed command line (unknown option, missing value, ...): bad input.
class CommandLineError : public gs::ValidationError {
 public:
  using gs::ValidationError::ValidationError;
};

// ---- schema ----------------------------------------------------------------

enum class Kind { kReal, kInteger, kText, kSwitch };

struct OptionSpec {
  std::string_view name;
  Kind kind;
  bool required;
};

struct Inputs {
  std::vector<std::string> files;                  // positionals, in order
  std::map<std::string, double, std::less<>> reals;
  std::map<std::string, long long, std::less<>> integers;
  std::map<std::string, std::string, std::less<>> texts;
  std::map<std::string, bool, std::less<>> switches;

  template <typename M>
  static auto lookup(const M& m, std::string_view k) -> std::optional<typename M::mapped_type> {
    const auto it = m.find(k);
    if (it == m.end()) return std::nullopt;
    return it->second;
  }
  std::optional<double> real(std::string_view k) const { return lookup(reals, k); }
  std::optional<long long> integer(std::string_view k) const { return lookup(integers, k); }
  std::optional<std::string> text(std::string_view k) const { return lookup(texts, k); }
  bool on(std::string_view k) const { return switches.count(k) != 0; }
};

struct CommandSpec {
  std::string_view name;
  std::size_t min_files, max_files;
  std::vector<OptionSpec> options;
  std::function<int(const Inputs&)> run;
};

// Strict numeric conversions: the whole token must be consumed.
double as_real(std::string_view opt, const std::string& token) {
  char* end = nullptr;
  const double v = token.empty() ? 0.0 : std::strtod(token.c_str(), &end);
  if (token.empty() || end != token.c_str() + token.size() || !std::isfinite(v)) {
    throw CommandLineError("option --" + std::string(opt) + " expects a real number, got \"" + token + "\"");
  }
  return v;
}

long long as_integer(std::string_view opt, std::string_view token) {
  long long v = 0;
  const auto [ptr, ec] = std::from_chars(token.data(), token.data() + token.size(), v);
  if (token.empty() || ec != std::errc() || ptr != token.data() + token.size()) {
    throw CommandLineError("option --" + std::string(opt) + " expects an integer, got \"" +
                           std::string(token) + "\"");
  }
  return v;
}

// argv[2..] against the command's schema.
Inputs read_command_line(const CommandSpec& cmd, int argc, char** argv) {
  Inputs in;
  auto find = [&](std::string_view n) -> const OptionSpec* {
    for (const auto& o : cmd.options) {
      if (o.name == n) return &o;
    }
    return nullptr;
  };
  for (int i = 2; i < argc; ++i) {
    const std::string_view arg = argv[i];
    if (arg.substr(0, 2) != "--") {
      in.files.emplace_back(arg);
      continue;
    }
    std::string_view name = arg.substr(2);
    std::optional<std::string> attached;
    if (const auto eq = name.find('='); eq != std::string_view::npos) {
      attached = std::string(name.substr(eq + 1));
      name = name.substr(0, eq);
    }
    const OptionSpec* spec = find(name);
    if (spec == nullptr) {
      throw CommandLineError(std::string(cmd.name) + " does not take option " + std::string(arg));
    }
    const std::string key(name);
    if (spec->kind == Kind::kSwitch) {
      if (attached) throw CommandLineError("switch --" + key + " takes no value");
      in.switches[key] = true;
      continue;
    }
    std::string value;
    if (attached) {
      value = *attached;
    } else if (i + 1 < argc) {
      value = argv[++i];
    } else {
      throw CommandLineError("option --" + key + " is missing its value");
    }
    switch (spec->kind) {
      case Kind::kReal: in.reals[key] = as_real(name, value); break;
      case Kind::kInteger: in.integers[key] = as_integer(name, value); break;
      default: in.texts[key] = value; break;
    }
  }
  if (in.files.size() < cmd.min_files || in.files.size() > cmd.max_files) {
    throw CommandLineError(std::string(cmd.name) + " takes " + std::to_string(cmd.min_files) +
                           (cmd.min_files == cmd.max_files ? "" : ".." + std::to_string(cmd.max_files)) +
                           " file argument(s), got " + std::to_string(in.files.size()));
  }
  for (const auto& o : cmd.options) {
    const std::string k(o.name);
    const bool given = in.reals.count(k) || in.integers.count(k) || in.texts.count(k) || in.switches.count(k);
    if (o.required && !given) throw CommandLineError(std::string(cmd.name) + " requires --" + k);
  }
  return in;
}

// ---- shared helpers ----------------------------------------------------------

// Text of a JSON document: stdout when no path is given.
void emit(const Json& doc, const std::optional<std::string>& path) {
  const std::string text = doc.dump(2) + "\n";
  if (!path) {
    std::cout << text;
    return;
  }
  std::ofstream f(*path);
  if (!f) throw gs::ParseError("could not create " + *path);
  f << text;
}

// The cost-model file written by `fit`: {"a_sec": a, "b_sec_per_byte": b, ...}.
gs::AllReduceModel model_file(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw gs::ParseError("model " + path + " is not readable");
  try {
    const Json doc = Json::parse(f);
    return gs::AllReduceModel{doc.at("a_sec").get<double>(), doc.at("b_sec_per_byte").get<double>()};
  } catch (const Json::exception& e) {
    throw gs::ParseError("model " + path + " must be a JSON object with numbers a_sec and b_sec_per_byte (" +
                         e.what() + ")");
  }
}

gs::NetworkParams network(const Inputs& in) {
  gs::NetworkParams net;
  net.alpha = in.real("alpha").value_or(0.0);
  net.beta = in.real("beta").value_or(0.0);
  net.gamma = in.real("gamma").value_or(0.0);
  return net;
}

gs::DbtStartup dbt(const Inputs& in) {
  return in.on("dbt-literal") ? gs::DbtStartup::kLiteral : gs::DbtStartup::kAlphaCorrected;
}

// --workers: "lo..hi" = every power of two in [lo, hi]; else "n1,n2,...".
std::vector<int> workers_list(const std::string& spec) {
  std::vector<int> counts;
  const auto bad = [&] { return gs::ValidationError("--workers \"" + spec + "\" is not lo..hi or a list of counts"); };
  if (const auto dots = spec.find(".."); dots != std::string::npos) {
    const long long lo = as_integer("workers", std::string_view(spec).substr(0, dots));
    const long long hi = as_integer("workers", std::string_view(spec).substr(dots + 2));
    for (int s = 0; s < 62 && (1ll << s) <= hi; ++s) {
      if ((1ll << s) >= lo) counts.push_back(static_cast<int>(1ll << s));
    }
  } else {
    std::istringstream items(spec);
    for (std::string item; std::getline(items, item, ',');) {
      if (item.empty()) continue;
      try {
        counts.push_back(static_cast<int>(as_integer("workers", item)));
      } catch (const CommandLineError&) {
        throw bad();
      }
    }
  }
  if (counts.empty()) throw bad();
  return counts;
}

// ---- subcommands ------------------------------------------------------------

int do_fit(const Inputs& in) {
  Json doc;
  std::vector<std::string> notes;
  gs::AllReduceModel m;
  const auto algo = in.text("algo");
  if (!in.files.empty() == algo.has_value()) {
    throw gs::ValidationError("fit takes exactly one source: a measurements CSV or --algo with network parameters");
  }
  if (algo) {  // Table 2 of the paper (comm_model.hpp:140-191)
    gs::NetworkParams net = network(in);
    net.n_workers = static_cast<int>(in.integer("workers").value_or(0));
    m = gs::coefficients_for(gs::algorithm_from_string(*algo), net, dbt(in), &notes);
    doc["source"] = "table2";
  } else {     // measured sweep (comm_model.hpp:209-308)
    m = gs::fit_model(gs::load_measurements_csv(in.files.front()));
    doc["source"] = "fit";
  }
  doc["a_sec"] = m.a;
  doc["b_sec_per_byte"] = m.b;
  doc["warnings"] = notes;
  emit(doc, in.text("out"));
  return kExitOk;
}

int do_plan(const Inputs& in) {
  const gs::ModelTrace trace = gs::load_trace(in.files[0]);
  const gs::AllReduceModel m = model_file(in.files[1]);
  const gs::MergePlan best = gs::optimal_plan(trace, m);
  if (in.on("oracle")) {  // cross-check the DP against exhaustive search (small L only)
    const double dp = gs::iteration_time(trace, best, m).iteration_time;
    const double ex = gs::brute_force_plan(trace, m).iteration_time;
    if (std::fabs(ex - dp) > 1e-9) {
      std::cerr << "plan --oracle: the DP plan takes " << dp * 1e6 << " us, exhaustive search finds "
                << ex * 1e6 << " us\n";
      return kExitPlanner;
    }
  }
  emit(gs::plan_to_json(trace, best, m), in.text("out"));
  return kExitOk;
}

int do_simulate(const Inputs& in) {
  const gs::ModelTrace trace = gs::load_trace(in.files[0]);
  const gs::AllReduceModel m = model_file(in.files[1]);
  const std::size_t L = trace.n_layers();
  using Maker = std::function<gs::Timeline()>;
  const std::map<gs::Strategy, Maker> timeline_of = {
      {gs::Strategy::kNaive, [&] { return gs::naive_timeline(trace, m); }},
      {gs::Strategy::kWfbp, [&] { return gs::iteration_time(trace, gs::MergePlan::all_normal(L), m); }},
      {gs::Strategy::kSyncEasgd, [&] { return gs::iteration_time(trace, gs::MergePlan::all_merged(L), m); }},
      {gs::Strategy::kMgWfbp, [&] { return gs::iteration_time(trace, gs::optimal_plan(trace, m), m); }},
  };
  const gs::Timeline tl = timeline_of.at(gs::strategy_from_string(*in.text("strategy")))();
  std::ostringstream line;
  line << std::setprecision(15) << "iter_time_us=" << tl.iteration_time * 1e6
       << " comm_nonoverlap_us=" << tl.comm_nonoverlap * 1e6;
  if (const auto n = in.integer("workers"); n && *n > 0) {
    line << " speedup="
         << gs::speedup(static_cast<int>(*n), trace.forward_time, trace.total_backward_time(), tl.comm_nonoverlap);
  }
  std::cout << line.str() << '\n';
  if (const auto out = in.text("out")) emit(gs::timeline_to_json(tl), out);
  return kExitOk;
}

int do_sweep(const Inputs& in) {
  const gs::ModelTrace trace = gs::load_trace(in.files[0]);
  gs::NetworkParams net = network(in);
  net.n_workers = 2;  // replaced per row by run_sweep
  const gs::SweepResult res = gs::run_sweep(trace, net, gs::algorithm_from_string(*in.text("algo")),
                                            workers_list(in.text("workers").value_or("4..2048")), dbt(in));
  std::size_t good = 0;
  for (const auto& row : res.rows) {
    if (row.ok()) {
      ++good;
    } else {
      std::cerr << "row n_workers=" << row.n_workers << " skipped: " << row.error << '\n';
    }
  }
  for (const auto& w : res.warnings) std::cerr << "warning: " << w << '\n';
  if (good == 0) {
    std::cerr << "sweep: no worker count produced a result\n";
    return kExitNoSweepRows;
  }
  if (const auto out = in.text("out")) {
    std::ofstream f(*out);
    if (!f) throw gs::ParseError("could not create " + *out);
    gs::write_sweep_csv(res, f);
  } else {
    gs::write_sweep_csv(res, std::cout);
  }
  if (const auto js = in.text("json")) emit(gs::sweep_to_json(res), js);
  return kExitOk;
}

const std::vector<CommandSpec>& commands() {
  static const std::vector<CommandSpec> kCommands = {
      {"fit", 0, 1,
       {{"algo", Kind::kText, false}, {"workers", Kind::kInteger, false}, {"alpha", Kind::kReal, false},
        {"beta", Kind::kReal, false}, {"gamma", Kind::kReal, false}, {"dbt-literal", Kind::kSwitch, false},
        {"out", Kind::kText, false}},
       do_fit},
      {"plan", 2, 2, {{"oracle", Kind::kSwitch, false}, {"out", Kind::kText, false}}, do_plan},
      {"simulate", 2, 2,
       {{"strategy", Kind::kText, true}, {"workers", Kind::kInteger, false}, {"out", Kind::kText, false}},
       do_simulate},
      {"sweep", 1, 1,
       {{"algo", Kind::kText, true}, {"alpha", Kind::kReal, true}, {"beta", Kind::kReal, false},
        {"gamma", Kind::kReal, false}, {"workers", Kind::kText, false}, {"dbt-literal", Kind::kSwitch, false},
        {"out", Kind::kText, false}, {"json", Kind::kText, false}},
       do_sweep},
  };
  return kCommands;
}

void print_usage(std::ostream& os) {
  os << "gradsched (mgwfbp-b200): gradient-merge planning and timeline simulation\n"
        "commands:";
  for (const auto& c : commands()) os << ' ' << c.name;
  os << "\n";
}

// Exception -> exit status (proj/tools/main.cpp:31-35 semantics).
int status_of_current_exception() {
  try {
    throw;
  } catch (const gs::GuardError& e) {
    std::cerr << "gradsched: " << e.what() << '\n';
    return kExitGuard;
  } catch (const gs::PlannerError& e) {
    std::cerr << "gradsched: " << e.what() << '\n';
    return kExitPlanner;
  } catch (const std::exception& e) {
    std::cerr << "gradsched: " << e.what() << '\n';
    return kExitBadInput;
  }
}

}  // namespace

int main(int argc, char** argv) {
  const std::string_view first = argc > 1 ? std::string_view(argv[1]) : std::string_view();
  if (first == "-h" || first == "--help") {
    print_usage(std::cout);
    return kExitOk;
  }
  for (const auto& cmd : commands()) {
    if (cmd.name != first) continue;
    try {
      return cmd.run(read_command_line(cmd, argc, argv));
    } catch (...) {
      return status_of_current_exception();
    }
  }
  print_usage(std::cerr);
  return kExitBadInput;
}
