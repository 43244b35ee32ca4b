// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (dessim, compiled from
// /root/reference/proj/core/src/*.cpp by oracle/Makefile into oracle/_ref/).
// It lets the Python tests and bench.py's CPU-baseline leg call the reference's
// own hot-path functions with flat arrays:
//   activate            gating.cpp:10-40
//   topk_route          gating.cpp:84-97
//   des_seq_coreset     des.cpp:33-45
//   des_vote_coreset    des.cpp:65-95
//   fused_vote_pipeline des.cpp:166-224
//   constrained_route   des.cpp:97-118
//   des_run             des.cpp:120-127
//   make_expert_bank    gating.cpp:99-120
//   moe_forward         gating.cpp:136-157
//   moe_latency         analysis.cpp:11-49
//   gen_trace           trace.cpp:42-111
//   Rng                 core.cpp:111-158
// Errors: 0 ok, 1 std::invalid_argument, 2 any other exception; the message is
// kept per thread and returned by dsref_last_error().
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string_view>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "dessim/baselines.hpp"
#include "dessim/analysis.hpp"
#include "dessim/core.hpp"
#include "dessim/des.hpp"
#include "dessim/gating.hpp"
#include "dessim/trace.hpp"

using namespace dessim;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

PoolConfig pool(int m, int k, int act, int dim = 1) {
  PoolConfig cfg;
  cfg.experts_total = m;
  cfg.top_k = k;
  cfg.gate_activation = act == 1 ? GateActivation::sigmoid : GateActivation::softmax;
  cfg.bytes_per_expert = 1;
  cfg.hidden_dim = dim;
  return cfg;
}

// The reference's make_router_block rejects non-finite values; the tests also
// need to smuggle NaNs past it (test_gating.cpp:60-66), so build the struct
// directly and let the callee validate.
RouterBlock block_of(const double* logits, int n, int m) {
  RouterBlock b;
  b.block_size = n;
  b.experts = m;
  b.logits.assign(logits, logits + static_cast<std::size_t>(n) * m);
  return b;
}

// Flattens an assignment into [n x k] arrays padded with -1 / 0.
void flatten(const RoutingAssignment& a, int k, int* idx, double* gates, int* counts) {
  for (int n = 0; n < a.block_size(); ++n) {
    const TokenRoute& t = a.tokens[n];
    counts[n] = static_cast<int>(t.experts.size());
    for (int j = 0; j < k; ++j) {
      bool in = j < counts[n];
      idx[static_cast<std::size_t>(n) * k + j] = in ? t.experts[j] : -1;
      gates[static_cast<std::size_t>(n) * k + j] = in ? t.gates[j] : 0.0;
    }
  }
}

RoutingAssignment unflatten(int n_tok, int k, const int* idx, const double* gates,
                            const int* counts) {
  RoutingAssignment a;
  a.tokens.resize(n_tok);
  for (int n = 0; n < n_tok; ++n) {
    for (int j = 0; j < counts[n]; ++j) {
      a.tokens[n].experts.push_back(idx[static_cast<std::size_t>(n) * k + j]);
      a.tokens[n].gates.push_back(gates[static_cast<std::size_t>(n) * k + j]);
    }
  }
  return a;
}

void copy_members(const Coreset& c, int* members, int* n_members) {
  *n_members = c.size();
  std::memcpy(members, c.members.data(), sizeof(int) * c.members.size());
}

}  // namespace

extern "C" {

const char* dsref_last_error(void) { return g_err.c_str(); }

int dsref_validate_config(int m, int k, int act, unsigned long long bytes, int dim) {
  return guarded([&] {
    PoolConfig cfg = pool(m, k, act, dim);
    cfg.bytes_per_expert = bytes;
    validate_config(cfg);
  });
}

int dsref_vote_budget(double beta, int m) { return vote_budget(beta, m); }

int dsref_activate(const double* logits, int n, int m, int k, int act, double* probs) {
  return guarded([&] {
    GateMatrix g = activate(block_of(logits, n, m), pool(m, k, act));
    std::memcpy(probs, g.probs.data(), sizeof(double) * g.probs.size());
  });
}

int dsref_topk_route(const double* logits, int n, int m, int k, int act, int* idx,
                     double* gates, int* counts) {
  return guarded([&] {
    PoolConfig cfg = pool(m, k, act);
    flatten(topk_route(activate(block_of(logits, n, m), cfg), k), k, idx, gates, counts);
  });
}

int dsref_des_seq_coreset(const double* logits, int n, int m, int k, int act, int local_k,
                          int* members, int* n_members) {
  return guarded([&] {
    copy_members(des_seq_coreset(block_of(logits, n, m), pool(m, k, act), local_k), members,
                 n_members);
  });
}

int dsref_des_vote_coreset(const double* logits, int n, int m, int k, int act, double beta,
                           int raw_logits, int* members, int* n_members, double* votes) {
  return guarded([&] {
    VoteResult r = des_vote_coreset(block_of(logits, n, m), pool(m, k, act), beta,
                                    raw_logits ? VoteSource::raw_logits : VoteSource::activated);
    copy_members(r.coreset, members, n_members);
    std::memcpy(votes, r.votes.votes.data(), sizeof(double) * m);
  });
}

int dsref_fused_vote_pipeline(const double* logits, int n, int m, int k, int act, double beta,
                              int* members, int* n_members, double* votes) {
  return guarded([&] {
    VoteResult r = fused_vote_pipeline(block_of(logits, n, m), pool(m, k, act), beta);
    copy_members(r.coreset, members, n_members);
    std::memcpy(votes, r.votes.votes.data(), sizeof(double) * m);
  });
}

int dsref_constrained_route(const double* logits, int n, int m, int k, int act,
                            const int* members, int n_members, int* idx, double* gates,
                            int* counts) {
  return guarded([&] {
    Coreset c{std::vector<int>(members, members + n_members)};
    flatten(constrained_route(block_of(logits, n, m), pool(m, k, act), c), k, idx, gates,
            counts);
  });
}

// strategy: 0 = seq, 1 = vote (DesStrategy order in des.hpp:16)
int dsref_des_run(const double* logits, int n, int m, int k, int act, int strategy, int seq_k,
                  double beta, int* members, int* n_members, int* idx, double* gates,
                  int* counts) {
  return guarded([&] {
    DesParams p;
    p.strategy = strategy == 0 ? DesStrategy::seq : DesStrategy::vote;
    p.seq_k = seq_k;
    p.vote_beta = beta;
    DesResult r = des_run(block_of(logits, n, m), pool(m, k, act), p);
    copy_members(r.coreset, members, n_members);
    flatten(r.assignment, k, idx, gates, counts);
  });
}

// method: 0 = topk_reduce, 1 = naee, 2 = mcmoe (BaselineMethod order,
// baselines.hpp:8); score: 0 = max_gate, 1 = neg_entropy
int dsref_baseline_route(const double* logits, int n, int m, int k, int act, int method,
                         int k_reduced, double naee_beta, double mcmoe_beta, double fraction,
                         int score, int* idx, double* gates, int* counts) {
  return guarded([&] {
    BaselineParams bp;
    bp.method = method == 0 ? BaselineMethod::topk_reduce
                            : (method == 1 ? BaselineMethod::naee : BaselineMethod::mcmoe);
    bp.k_reduced = k_reduced;
    bp.naee_beta = naee_beta;
    bp.mcmoe_beta = mcmoe_beta;
    bp.mcmoe_important_fraction = fraction;
    bp.mcmoe_score = score == 1 ? ImportanceScore::neg_entropy : ImportanceScore::max_gate;
    flatten(baseline_route(block_of(logits, n, m), pool(m, k, act), bp), k, idx, gates, counts);
  });
}

// gen_trace + encode_trace (format 0 binary, 1 jsonl): the reference's own
// bytes; out == NULL -> *len = size
int dsref_trace_bytes(int m, int k, int model, double rho, double tau, int layers, int steps,
                      int n, unsigned long long seed, int format, char* out, size_t* len) {
  return guarded([&] {
    SynthParams p;
    p.model = model == 0 ? SynthModel::iid_gaussian
                         : (model == 1 ? SynthModel::dirichlet : SynthModel::shared_bias);
    p.rho = rho;
    p.temperature = tau;
    TraceFile f = gen_trace(pool(m, k, 0), p, layers, steps, n, seed);
    std::string b = encode_trace(f, format == 0 ? TraceFormat::binary : TraceFormat::jsonl);
    if (out) std::memcpy(out, b.data(), std::min(*len, b.size()));
    *len = b.size();
  });
}

// decode_trace: 0 ok (header ints {experts, top_k, layers, block_size, steps,
// model}, doubles {rho, temperature}, seed, logits if non-NULL), else 1 with
// *code = TraceError::Code (or -1 for another exception) and the message
int dsref_trace_decode(const char* bytes, size_t len, int* code, int* hdr, double* hdr_d,
                       unsigned long long* seed, double* logits) {
  *code = -1;
  try {
    TraceFile f = decode_trace(std::string_view(bytes, len));
    const TraceHeader& h = f.header;
    const int v[6] = {h.experts, h.top_k, h.layers, h.block_size, h.steps,
                      static_cast<int>(h.model)};
    std::memcpy(hdr, v, sizeof v);
    hdr_d[0] = h.rho;
    hdr_d[1] = h.temperature;
    *seed = h.seed;
    if (logits) {
      std::size_t o = 0;
      for (const RouterBlock& b : f.blocks) {
        std::memcpy(logits + o, b.logits.data(), sizeof(double) * b.logits.size());
        o += b.logits.size();
      }
    }
    g_err.clear();
    return 0;
  } catch (const TraceError& e) {
    *code = static_cast<int>(e.code);
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int dsref_make_expert_bank(int m, int k, int dim, int n, unsigned long long seed,
                           double* weights, double* inputs) {
  return guarded([&] {
    ExpertBank b = make_expert_bank(pool(m, k, 0, dim), n, seed);
    std::memcpy(weights, b.expert_weights.data(), sizeof(double) * b.expert_weights.size());
    std::memcpy(inputs, b.token_inputs.data(), sizeof(double) * b.token_inputs.size());
  });
}

int dsref_moe_forward(int n, int k, const int* idx, const double* gates, const int* counts,
                      int m, int dim, const double* weights, const double* inputs, double* out) {
  return guarded([&] {
    ExpertBank b;
    b.experts = m;
    b.dim = dim;
    b.block_size = n;
    b.expert_weights.assign(weights, weights + static_cast<std::size_t>(m) * dim * dim);
    b.token_inputs.assign(inputs, inputs + static_cast<std::size_t>(n) * dim);
    std::vector<double> y = moe_forward(unflatten(n, k, idx, gates, counts), b);
    std::memcpy(out, y.data(), sizeof(double) * y.size());
  });
}

int dsref_moe_latency(int n, int k, const int* idx, const int* counts, int m, int* unique,
                      int* total, int* per_expert) {
  return guarded([&] {
    std::vector<double> g(static_cast<std::size_t>(n) * k, 0.0);
    TrafficReport r = moe_latency(unflatten(n, k, idx, g.data(), counts), pool(m, k, 0),
                                  LatencyParams{});
    *unique = r.unique_experts;
    *total = r.total_selections;
    std::memcpy(per_expert, r.per_expert_counts.data(), sizeof(int) * m);
  });
}

double dsref_expected_unique_experts(int m, int k, int n) {
  return expected_unique_experts(m, k, n);
}

// model: 0 iid_gaussian, 1 dirichlet, 2 shared_bias (SynthModel order, trace.hpp:13)
int dsref_gen_trace(int m, int k, int model, double rho, double tau, int layers, int steps,
                    int n, unsigned long long seed, double* logits_out) {
  return guarded([&] {
    SynthParams p;
    p.model = model == 0 ? SynthModel::iid_gaussian
                         : (model == 1 ? SynthModel::dirichlet : SynthModel::shared_bias);
    p.rho = rho;
    p.temperature = tau;
    TraceFile f = gen_trace(pool(m, k, 0), p, layers, steps, n, seed);
    std::size_t per = static_cast<std::size_t>(n) * m;
    for (std::size_t b = 0; b < f.blocks.size(); ++b) {
      std::memcpy(logits_out + b * per, f.blocks[b].logits.data(), sizeof(double) * per);
    }
  });
}

void dsref_rng_u64(unsigned long long seed, int count, unsigned long long* out) {
  Rng r(seed);
  for (int i = 0; i < count; ++i) out[i] = r.next_u64();
}

void dsref_rng_normal(unsigned long long seed, int count, double* out) {
  Rng r(seed);
  for (int i = 0; i < count; ++i) out[i] = r.next_normal();
}

unsigned long long dsref_rng_mix(unsigned long long seed, unsigned long long stream) {
  return Rng::mix(seed, stream);
}

// CPU timing of the reference's routing stage for one block (bench.py's
// reference arm): median-free mean over `reps` calls on `threads` threads,
// each thread running independent copies (SPEC.md:140 per-block parallelism).
// strategy: -1 vanilla (topk_route(activate)), 0 seq, 1 vote.
// Returns total routed blocks per second.
double dsref_time_routing(const double* logits, int n, int m, int k, int strategy, int seq_k,
                          double beta, int reps, int threads) {
  RouterBlock blk = block_of(logits, n, m);
  PoolConfig cfg = pool(m, k, 0);
  DesParams p;
  p.strategy = strategy == 0 ? DesStrategy::seq : DesStrategy::vote;
  p.seq_k = seq_k;
  p.vote_beta = beta;
  auto work = [&] {
    for (int r = 0; r < reps; ++r) {
      if (strategy < 0) {
        volatile auto sz = topk_route(activate(blk, cfg), k).tokens.size();
        (void)sz;
      } else {
        volatile auto sz = des_run(blk, cfg, p).coreset.members.size();
        (void)sz;
      }
    }
  };
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool_threads;
  for (int t = 0; t < threads; ++t) pool_threads.emplace_back(work);
  for (auto& t : pool_threads) t.join();
  double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return static_cast<double>(reps) * threads / s;
}

// CPU timing of the reference's whole MoE layer for one block (bench.py's
// reference arm and cpu_baseline): routing (strategy -1 vanilla
// topk_route(activate), 0 seq / 1 vote des_run) followed by moe_forward
// (gating.cpp:136-157) with the reference's own expert model, a linear
// dim x dim map, over a bank holding the experts the block routes to (ids
// remapped; the bank is generated once, outside the timed region).
// Bounded sample: routing runs on the whole block; moe_forward runs on the
// first `ffn_tokens` tokens' routes and its time is scaled by n / ffn_tokens
// (its cost is linear in tokens). `threads` workers each process `reps`
// samples (per-block parallelism). Returns estimated wall seconds
// per block at that parallelism; *unique_out = U of the block.
double dsref_time_layer(const double* logits, int n, int m, int k, int strategy, int seq_k,
                        double beta, int dim, int reps, int threads, unsigned long long seed,
                        int ffn_tokens, int* unique_out) {
  RouterBlock blk = block_of(logits, n, m);
  PoolConfig cfg = pool(m, k, 0, dim);
  DesParams p;
  p.strategy = strategy == 0 ? DesStrategy::seq : DesStrategy::vote;
  p.seq_k = seq_k;
  p.vote_beta = beta;
  if (ffn_tokens < 1 || ffn_tokens > n) ffn_tokens = n;
  auto route = [&]() {
    return strategy < 0 ? topk_route(activate(blk, cfg), k) : des_run(blk, cfg, p).assignment;
  };
  RoutingAssignment probe = route();
  Coreset used = unique_experts(probe);
  *unique_out = used.size();
  std::vector<int> local(m, -1);
  for (int i = 0; i < used.size(); ++i) local[used.members[i]] = i;
  ExpertBank bank =
      make_expert_bank(pool(used.size(), std::min(k, used.size()), 0, dim), ffn_tokens, seed);
  std::vector<double> t_route(threads, 0.0), t_ffn(threads, 0.0);
  auto work = [&](int tid) {
    for (int r = 0; r < reps; ++r) {
      auto t0 = std::chrono::steady_clock::now();
      RoutingAssignment a = route();
      auto t1 = std::chrono::steady_clock::now();
      a.tokens.resize(ffn_tokens);
      for (TokenRoute& t : a.tokens)
        for (int& e : t.experts) e = local[e];
      volatile double sink = moe_forward(a, bank)[0];
      (void)sink;
      auto t2 = std::chrono::steady_clock::now();
      t_route[tid] += std::chrono::duration<double>(t1 - t0).count();
      t_ffn[tid] += std::chrono::duration<double>(t2 - t1).count();
    }
  };
  std::vector<std::thread> ts;
  for (int t = 0; t < threads; ++t) ts.emplace_back(work, t);
  for (auto& t : ts) t.join();
  double per_block = 0.0;  // slowest worker's per-sample estimate
  for (int t = 0; t < threads; ++t)
    per_block = std::max(per_block, (t_route[t] + t_ffn[t] * n / ffn_tokens) / reps);
  return per_block / threads;
}

}  // extern "C"
