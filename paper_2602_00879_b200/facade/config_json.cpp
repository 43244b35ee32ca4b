// Pool-config JSON of the reference API (core.hpp:25-26, core.cpp:40-61): the
// CLI's config-file dialect, so a pool document doubles as a --config file.
// Host-only plumbing around the GPU path; nlohmann::json 3.11.3 is the
// reference's own JSON dependency (header-only, from the image).
#include <nlohmann/json.hpp>

#include "dessim/core.hpp"

namespace dessim {

namespace {
constexpr const char* kExperts = "experts";
constexpr const char* kTopK = "top-k";
constexpr const char* kActivation = "activation";
constexpr const char* kBytes = "bytes-per-expert";
constexpr const char* kHidden = "hidden-dim";
}  // namespace

std::string pool_config_to_json(const PoolConfig& cfg) {
  const nlohmann::json doc = {{kExperts, cfg.experts_total},
                              {kTopK, cfg.top_k},
                              {kActivation, to_string(cfg.gate_activation)},
                              {kBytes, cfg.bytes_per_expert},
                              {kHidden, cfg.hidden_dim}};
  return doc.dump();
}

PoolConfig pool_config_from_json(const std::string& text) {
  const auto doc = nlohmann::json::parse(text);
  PoolConfig cfg;
  doc.at(kExperts).get_to(cfg.experts_total);
  doc.at(kTopK).get_to(cfg.top_k);
  cfg.gate_activation = gate_activation_from_string(doc.at(kActivation).get<std::string>());
  doc.at(kBytes).get_to(cfg.bytes_per_expert);
  doc.at(kHidden).get_to(cfg.hidden_dim);
  return cfg;
}

}  // namespace dessim
