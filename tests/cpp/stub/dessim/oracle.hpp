// TEST INFRASTRUCTURE ONLY. The reference's research oracles (oracle.hpp:
// exhaustive coreset search, Monte-Carlo unique-expert estimate) are out of
// scope for the B200 build. test_analysis.cpp includes this
// header for one Monte-Carlo cross-check of expected_unique_experts; this
// stand-in provides that estimator (uniform K-subsets per token drawn from
// dessim::Rng streams) so the reference's analysis suite compiles unchanged
// against the façade. The exhaustive searches are declared, not provided.
#pragma once

#include <cmath>
#include <cstdint>
#include <numeric>
#include <vector>

#include "dessim/core.hpp"
#include "dessim/des.hpp"
#include "dessim/gating.hpp"

namespace dessim {

Coreset exhaustive_additive_coreset(const VoteVector& votes, int m_core);
Coreset exhaustive_reconstruction_coreset(const RouterBlock& block, const PoolConfig& cfg,
                                          const ExpertBank& bank, int m_core);

struct McEstimate {
  double mean = 0.0;
  double std_error = 0.0;
};

inline McEstimate mc_unique_experts(int experts_total, int top_k, int block_size, int trials,
                                    std::uint64_t seed) {
  std::vector<int> pool(experts_total);
  std::vector<char> seen(experts_total);
  double sum = 0.0, sq = 0.0;
  for (int t = 0; t < trials; ++t) {
    Rng rng(Rng::mix(seed, static_cast<std::uint64_t>(t)));
    std::fill(seen.begin(), seen.end(), 0);
    int u = 0;
    for (int n = 0; n < block_size; ++n) {
      std::iota(pool.begin(), pool.end(), 0);
      for (int j = 0; j < top_k; ++j) {  // partial Fisher-Yates: a uniform K-subset
        const int r = j + rng.next_below(experts_total - j);
        std::swap(pool[j], pool[r]);
        if (!seen[pool[j]]) {
          seen[pool[j]] = 1;
          ++u;
        }
      }
    }
    sum += u;
    sq += static_cast<double>(u) * u;
  }
  McEstimate e;
  e.mean = sum / trials;
  const double var = std::max(0.0, sq / trials - e.mean * e.mean);
  e.std_error = std::sqrt(var / trials);
  return e;
}

}  // namespace dessim
