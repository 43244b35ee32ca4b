// dessim::trace on the C ABI's MOET codec (csrc/moet.cpp) — see
// include/dessim/trace.hpp. gen_trace is host code over the façade's Rng and
// reproduces the reference generator's draws and rounding (trace.cpp:42-111).
#include "dessim/trace.hpp"

#include <algorithm>
#include <cmath>
#include <fstream>
#include <sstream>

#include "../../include/desmoe.h"

namespace dessim {

const char* to_string(SynthModel model) {
  switch (model) {
    case SynthModel::iid_gaussian: return "iid_gaussian";
    case SynthModel::dirichlet: return "dirichlet";
    case SynthModel::shared_bias: return "shared_bias";
  }
  return "unknown";
}

SynthModel synth_model_from_string(const std::string& name) {
  for (SynthModel m : {SynthModel::iid_gaussian, SynthModel::dirichlet, SynthModel::shared_bias})
    if (name == to_string(m)) return m;
  throw std::invalid_argument("unknown synth model: " + name);
}

const RouterBlock& TraceFile::block(int step, int layer) const {
  if (step < 0 || step >= header.steps || layer < 0 || layer >= header.layers)
    throw std::invalid_argument("block key out of range");
  return blocks[static_cast<std::size_t>(step) * header.layers + layer];
}

namespace {

double to_f32(double v) { return static_cast<double>(static_cast<float>(v)); }

desmoe_moet_header c_header(const TraceHeader& h) {
  desmoe_moet_header c{};
  c.experts = h.experts;
  c.top_k = h.top_k;
  c.layers = h.layers;
  c.block_size = h.block_size;
  c.steps = h.steps;
  c.model = static_cast<int>(h.model);
  c.rho = h.rho;
  c.temperature = h.temperature;
  c.seed = h.seed;
  return c;
}

[[noreturn]] void throw_trace(int code) {
  throw TraceError(static_cast<TraceError::Code>(code < 0 ? 0 : code), desmoe_last_error());
}

}  // namespace

TraceFile gen_trace(const PoolConfig& cfg, const SynthParams& params, int layers, int steps,
                    int block_size, std::uint64_t seed) {
  validate_config(cfg);
  if (layers < 1) throw std::invalid_argument("layers < 1");
  if (steps < 1) throw std::invalid_argument("steps < 1");
  if (block_size < 1) throw std::invalid_argument("block_size < 1");
  if (params.rho < 0.0 || params.rho > 1.0) throw std::invalid_argument("rho outside [0, 1]");
  if (!(params.temperature > 0.0)) throw std::invalid_argument("temperature <= 0");
  TraceFile f;
  TraceHeader& h = f.header;
  h.experts = cfg.experts_total;
  h.top_k = cfg.top_k;
  h.layers = layers;
  h.block_size = block_size;
  h.steps = steps;
  h.model = params.model;
  h.rho = to_f32(params.rho);
  h.temperature = to_f32(params.temperature);
  h.seed = seed;
  const int m = cfg.experts_total;
  const double tau = params.temperature;
  f.blocks.reserve(static_cast<std::size_t>(steps) * layers);
  for (std::uint64_t b = 0; b < static_cast<std::uint64_t>(steps) * layers; ++b) {
    Rng rng(Rng::mix(seed, b));
    std::vector<double> x(static_cast<std::size_t>(block_size) * m);
    if (params.model == SynthModel::iid_gaussian) {
      for (double& v : x) v = to_f32(tau * rng.next_normal());
    } else if (params.model == SynthModel::dirichlet) {
      // normalised exponential draws (kept away from 0 so the log is finite)
      std::vector<double> w(m);
      for (int t = 0; t < block_size; ++t) {
        double sum = 0.0;
        for (int i = 0; i < m; ++i) {
          w[i] = std::max(-std::log(1.0 - rng.next_unit()), 1e-300);
          sum += w[i];
        }
        for (int i = 0; i < m; ++i)
          x[static_cast<std::size_t>(t) * m + i] = to_f32(tau * std::log(w[i] / sum));
      }
    } else {
      std::vector<double> bias(m);
      for (double& v : bias) v = rng.next_normal();
      for (int t = 0; t < block_size; ++t)
        for (int i = 0; i < m; ++i) {
          const double noise = rng.next_normal();
          x[static_cast<std::size_t>(t) * m + i] =
              to_f32(tau * (params.rho * bias[i] + (1.0 - params.rho) * noise));
        }
    }
    f.blocks.push_back(make_router_block(block_size, m, std::move(x)));
  }
  return f;
}

std::string encode_trace(const TraceFile& file, TraceFormat format) {
  const desmoe_moet_header h = c_header(file.header);
  int code = -1;
  size_t len = 0;
  // header first, then the block count (trace.cpp:422-427)
  if (desmoe_moet_encode(&h, nullptr, DESMOE_MOET_BINARY, nullptr, &len, &code)) throw_trace(code);
  if (file.block_count() != file.header.steps * file.header.layers)
    throw TraceError(TraceError::Code::shape_mismatch, "block count does not match header");
  std::vector<double> flat;
  flat.reserve(static_cast<std::size_t>(file.block_count()) * file.header.block_size *
               file.header.experts);
  for (const RouterBlock& b : file.blocks) flat.insert(flat.end(), b.logits.begin(), b.logits.end());
  const int fmt = format == TraceFormat::binary ? DESMOE_MOET_BINARY : DESMOE_MOET_JSONL;
  if (desmoe_moet_encode(&h, flat.data(), fmt, nullptr, &len, &code)) throw_trace(code);
  std::string out(len, '\0');
  if (desmoe_moet_encode(&h, flat.data(), fmt, out.data(), &len, &code)) throw_trace(code);
  out.resize(len);
  return out;
}

TraceFile decode_trace(std::string_view bytes) {
  desmoe_moet_header h{};
  int code = -1;
  if (desmoe_moet_decode(bytes.data(), bytes.size(), &h, nullptr, &code)) throw_trace(code);
  const std::size_t per = static_cast<std::size_t>(h.block_size) * h.experts;
  const std::size_t records = static_cast<std::size_t>(h.steps) * h.layers;
  std::vector<double> flat(per * records);
  if (desmoe_moet_decode(bytes.data(), bytes.size(), &h, flat.data(), &code)) throw_trace(code);
  TraceFile f;
  f.header.experts = h.experts;
  f.header.top_k = h.top_k;
  f.header.layers = h.layers;
  f.header.block_size = h.block_size;
  f.header.steps = h.steps;
  f.header.model = static_cast<SynthModel>(h.model);
  f.header.rho = h.rho;
  f.header.temperature = h.temperature;
  f.header.seed = h.seed;
  f.blocks.reserve(records);
  for (std::size_t r = 0; r < records; ++r)
    f.blocks.push_back(RouterBlock{h.block_size, h.experts,
                                   std::vector<double>(flat.begin() + r * per,
                                                       flat.begin() + (r + 1) * per)});
  return f;
}

void write_trace(const TraceFile& file, const std::string& path, TraceFormat format) {
  const std::string bytes = encode_trace(file, format);
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw TraceError(TraceError::Code::io, "cannot open for writing: " + path);
  out.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
  if (!out) throw TraceError(TraceError::Code::io, "write failed: " + path);
}

TraceFile read_trace(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw TraceError(TraceError::Code::io, "cannot open for reading: " + path);
  std::ostringstream buf;
  buf << in.rdbuf();
  return decode_trace(buf.str());
}

}  // namespace dessim
