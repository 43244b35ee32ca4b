// TEST INFRASTRUCTURE ONLY — a minimal argument front end (CLI11 is absent
// from this image) for the reference's own `dessim` command implementations
// (/root/reference/proj/tools/commands.cpp + emit.cpp, compiled unchanged by
// tests/cpp/Makefile). Linked once against this repo's GPU façade
// (libdessim_gpu.so: `dessim run` / `sweep` / `gen-trace` on the B200) and
// once against the reference library itself (oracle/_ref) so the two
// outputs can be compared row by row (tests/test_cli_gpu.py).
//
//   dessim_* gen-trace --experts M --top-k K --block N [--layers L] [--steps S]
//            [--model m] [--rho r] [--temperature t] [--seed s] [--format bin|jsonl] -o PATH
//   dessim_* run --trace PATH --method m [--k K] [--beta B] [--fraction F]
//            [--bank-seed S] [--hidden-dim D] [--activation a] [--a A] [--b B]
//            [--bytes-per-expert X] [--json] [-o PATH]
//   dessim_* sweep --trace PATH --method m [--betas a,b] [--ks a,b] (run's options)
//   dessim_* explosion --experts M --top-k K --blocks a,b [--trials T] [--seed s]
//            [--trace PATH] [--activation a] [--json] [-o PATH]
//   dessim_* oracle-gap [--experts M] [--top-k K] [--block N] [--instances I] [--seed s]
//            [--model m] [--rho r] [--temperature t] [--hidden-dim D] [--activation a]
//   every command: [--config file.json] (the JSON object's keys fill in the
//   flags not given on the command line, as the reference's main.cpp does)
#include <cstdint>
#include <fstream>
#include <cstdlib>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include <json.hpp>

#include "../../../reference/proj/tools/commands.hpp"

namespace {

using namespace dessim::cli;

struct Args {
  std::map<std::string, std::string> kv;
  bool has(const std::string& k) const { return kv.count(k) != 0; }
  std::string s(const std::string& k, const std::string& d = "") const {
    auto it = kv.find(k);
    return it == kv.end() ? d : it->second;
  }
  double f(const std::string& k, double d) const { return has(k) ? std::stod(s(k)) : d; }
  long long i(const std::string& k, long long d) const { return has(k) ? std::stoll(s(k)) : d; }
};

Args parse(int argc, char** argv, int from) {
  Args a;
  for (int i = from; i < argc; ++i) {
    std::string k = argv[i];
    if (k == "-o") k = "--output";
    if (k == "--json") {
      a.kv[k] = "1";
      continue;
    }
    const auto eq = k.find('=');
    if (eq != std::string::npos) {
      a.kv[k.substr(0, eq)] = k.substr(eq + 1);
    } else if (i + 1 < argc) {
      a.kv[k] = argv[++i];
    }
  }
  if (a.has("--config")) {  // flags win over the file's keys
    std::ifstream in(a.s("--config"));
    if (!in) throw std::invalid_argument("cannot open config file: " + a.s("--config"));
    nlohmann::json j = nlohmann::json::parse(in);
    if (!j.is_object()) throw std::invalid_argument("config file must hold a JSON object");
    for (auto it = j.begin(); it != j.end(); ++it) {
      const std::string key = "--" + it.key();
      if (it.key() == "config" || a.has(key)) continue;
      std::string v;
      if (it->is_string()) {
        v = it->get<std::string>();
      } else if (it->is_array()) {
        for (const auto& x : *it) v += (v.empty() ? "" : ",") + (x.is_string() ? x.get<std::string>() : x.dump());
      } else if (it->is_boolean()) {
        v = it->get<bool>() ? "1" : "";
        if (v.empty()) continue;
      } else {
        v = it->dump();
      }
      a.kv[key] = v;
    }
  }
  return a;
}

template <typename T>
std::vector<T> list(const std::string& v) {
  std::vector<T> out;
  std::stringstream ss(v);
  std::string item;
  while (std::getline(ss, item, ',')) {
    std::stringstream is(item);
    T x;
    is >> x;
    out.push_back(x);
  }
  return out;
}

template <typename O>
void eval_opts(const Args& a, O& o) {
  o.trace_path = a.s("--trace");
  o.activation = a.s("--activation", o.activation);
  o.compute_cost = a.f("--a", o.compute_cost);
  o.fetch_cost = a.f("--b", o.fetch_cost);
  o.bytes_per_expert = static_cast<std::uint64_t>(a.i("--bytes-per-expert", 1));
  o.bank_given = a.has("--bank-seed");
  o.bank_seed = static_cast<std::uint64_t>(a.i("--bank-seed", 0));
  o.hidden_dim = static_cast<int>(a.i("--hidden-dim", o.hidden_dim));
  o.output = a.s("--output");
  o.json = a.has("--json");
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: " << argv[0] << " gen-trace|run|sweep [options]\n";
    return 2;
  }
  const std::string cmd = argv[1];
  try {
    const Args a = parse(argc, argv, 2);
    if (cmd == "gen-trace") {
      GenTraceOptions o;
      o.experts = static_cast<int>(a.i("--experts", 0));
      o.top_k = static_cast<int>(a.i("--top-k", 0));
      o.block = static_cast<int>(a.i("--block", 0));
      o.layers = static_cast<int>(a.i("--layers", 1));
      o.steps = static_cast<int>(a.i("--steps", 1));
      o.model = a.s("--model", o.model);
      o.rho = a.f("--rho", o.rho);
      o.temperature = a.f("--temperature", o.temperature);
      o.seed = static_cast<std::uint64_t>(a.i("--seed", 0));
      o.format = a.s("--format", o.format);
      o.output = a.s("--output");
      return cmd_gen_trace(o);
    }
    if (cmd == "run") {
      RunOptions o;
      eval_opts(a, o);
      o.method.method = a.s("--method");
      o.method.k_given = a.has("--k");
      o.method.k = static_cast<int>(a.i("--k", 0));
      o.method.beta_given = a.has("--beta");
      o.method.beta = a.f("--beta", 0.0);
      o.method.fraction = a.f("--fraction", 0.5);
      return cmd_run(o);
    }
    if (cmd == "sweep") {
      SweepOptions o;
      eval_opts(a, o);
      o.method = a.s("--method");
      if (a.has("--betas")) o.betas = list<double>(a.s("--betas"));
      if (a.has("--ks")) o.ks = list<int>(a.s("--ks"));
      return cmd_sweep(o);
    }
    if (cmd == "explosion") {
      ExplosionOptions o;
      o.experts = static_cast<int>(a.i("--experts", 0));
      o.top_k = static_cast<int>(a.i("--top-k", 0));
      if (a.has("--blocks")) o.blocks = list<int>(a.s("--blocks"));
      o.trials = static_cast<int>(a.i("--trials", o.trials));
      o.seed = static_cast<std::uint64_t>(a.i("--seed", 0));
      o.trace_path = a.s("--trace");
      o.activation = a.s("--activation", o.activation);
      o.output = a.s("--output");
      o.json = a.has("--json");
      return cmd_explosion(o);
    }
    if (cmd == "oracle-gap") {
      OracleGapOptions o;
      o.experts = static_cast<int>(a.i("--experts", o.experts));
      o.top_k = static_cast<int>(a.i("--top-k", o.top_k));
      o.block = static_cast<int>(a.i("--block", o.block));
      o.instances = static_cast<int>(a.i("--instances", o.instances));
      o.seed = static_cast<std::uint64_t>(a.i("--seed", 0));
      o.model = a.s("--model", o.model);
      o.rho = a.f("--rho", o.rho);
      o.temperature = a.f("--temperature", o.temperature);
      o.hidden_dim = static_cast<int>(a.i("--hidden-dim", o.hidden_dim));
      o.activation = a.s("--activation", o.activation);
      o.output = a.s("--output");
      o.json = a.has("--json");
      return cmd_oracle_gap(o);
    }
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
  std::cerr << "unknown command " << cmd << "\n";
  return 2;
}
