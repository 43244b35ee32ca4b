// MOET router-trace codec: the reference's on-disk trace
// format (trace.hpp:30-85, trace.cpp:122-442), so captured or generated
// router traces feed the GPU routing path in logits-in mode. Host code in
// libdesmoe.so behind the C ABI (desmoe_moet_decode / desmoe_moet_encode);
// the C++ façade (dessim::decode_trace, …) and the Python mirror call it.
//
// Binary v1: "MOET", u16 version, u8 generator model, u8 reserved, u32
// experts, top_k, layers, block_size, steps, u64 seed, f32 rho, f32
// temperature (all little-endian); then per (step, layer) record: u32 step,
// u32 layer, block_size x experts f32 logits row-major.
// JSONL: one header object line, then one {"layer", "logits", "step"} object
// per record. Both are decoded with the reference's checks, error codes
// (TraceError::Code) and messages; JSON goes through nlohmann::json 3.11.3
// (the reference's own JSON dependency), so encoded text is byte-identical.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <string_view>
#include <vector>

#include <json.hpp>

#include "../../include/desmoe.h"
#include "errors.h"

namespace {

using json = nlohmann::json;

const char* model_name(int model) {  // to_string(SynthModel), trace.cpp:13-20
  switch (model) {
    case 0: return "iid_gaussian";
    case 1: return "dirichlet";
    case 2: return "shared_bias";
  }
  return "unknown";
}

// A decode / encode failure: TraceError's code and message.
struct MoetFail {
  int code;
  std::string msg;
};

void check_header(const desmoe_moet_header& h) {  // trace.cpp:158-166
  if (h.experts < 1 || h.top_k < 1 || h.top_k > h.experts || h.layers < 1 || h.block_size < 1 ||
      h.steps < 1)
    throw MoetFail{DESMOE_MOET_BAD_HEADER, "invalid header field"};
  if (!std::isfinite(h.rho) || !std::isfinite(h.temperature))
    throw MoetFail{DESMOE_MOET_BAD_HEADER, "non-finite header field"};
}

// Little-endian reader over the input; `record` >= 0 names the record a
// short read happens in.
class LeReader {
 public:
  explicit LeReader(std::string_view d) : d_(d) {}
  int record = -1;
  size_t pos = 0;
  uint64_t get(int bytes) {
    if (pos + static_cast<size_t>(bytes) > d_.size()) {
      if (record >= 0)
        throw MoetFail{DESMOE_MOET_TRUNCATED, "truncated file in record " + std::to_string(record)};
      throw MoetFail{DESMOE_MOET_TRUNCATED, "truncated header"};
    }
    uint64_t v = 0;
    for (int i = 0; i < bytes; ++i)
      v |= static_cast<uint64_t>(static_cast<uint8_t>(d_[pos + i])) << (8 * i);
    pos += static_cast<size_t>(bytes);
    return v;
  }
  float f32() {
    const uint32_t b = static_cast<uint32_t>(get(4));
    float f;
    std::memcpy(&f, &b, 4);
    return f;
  }
  size_t size() const { return d_.size(); }

 private:
  std::string_view d_;
};

void decode_binary(std::string_view in, desmoe_moet_header* h, double* logits) {
  LeReader r(in);
  if (in.size() < 4) r.get(4);  // "truncated header"
  if (std::memcmp(in.data(), "MOET", 4) != 0) throw MoetFail{DESMOE_MOET_BAD_MAGIC, "bad magic bytes"};
  r.pos = 4;
  const unsigned version = static_cast<unsigned>(r.get(2));
  if (version != 1)
    throw MoetFail{DESMOE_MOET_BAD_VERSION, "unsupported version " + std::to_string(version)};
  const unsigned model = static_cast<unsigned>(r.get(1));
  if (model > 2) throw MoetFail{DESMOE_MOET_BAD_HEADER, "unknown generator model"};
  r.get(1);  // reserved
  desmoe_moet_header hd{};
  hd.model = static_cast<int>(model);
  hd.experts = static_cast<int>(static_cast<uint32_t>(r.get(4)));
  hd.top_k = static_cast<int>(static_cast<uint32_t>(r.get(4)));
  hd.layers = static_cast<int>(static_cast<uint32_t>(r.get(4)));
  hd.block_size = static_cast<int>(static_cast<uint32_t>(r.get(4)));
  hd.steps = static_cast<int>(static_cast<uint32_t>(r.get(4)));
  hd.seed = r.get(8);
  hd.rho = r.f32();
  hd.temperature = r.f32();
  check_header(hd);
  const size_t per = static_cast<size_t>(hd.block_size) * hd.experts;
  const int records = hd.steps * hd.layers;
  for (int rec = 0; rec < records; ++rec) {
    r.record = rec;
    const int es = rec / hd.layers, el = rec % hd.layers;
    const int step = static_cast<int>(static_cast<uint32_t>(r.get(4)));
    const int layer = static_cast<int>(static_cast<uint32_t>(r.get(4)));
    if (step != es || layer != el)
      throw MoetFail{DESMOE_MOET_SHAPE_MISMATCH,
                     "record " + std::to_string(rec) + " keyed (" + std::to_string(step) + "," +
                         std::to_string(layer) + "), expected (" + std::to_string(es) + "," +
                         std::to_string(el) + ")"};
    for (size_t i = 0; i < per; ++i) {
      const float v = r.f32();
      if (!std::isfinite(v))
        throw MoetFail{DESMOE_MOET_BAD_VALUE, "non-finite logit in record " + std::to_string(rec)};
      if (logits) logits[static_cast<size_t>(rec) * per + i] = static_cast<double>(v);
    }
  }
  if (r.pos != r.size())
    throw MoetFail{DESMOE_MOET_SHAPE_MISMATCH, "trailing bytes after last record"};
  *h = hd;
}

// std::getline semantics over a buffer: lines split at '\n'; a final
// segment without '\n' is a line, an empty one after the last '\n' is not.
class Lines {
 public:
  explicit Lines(std::string_view d) : d_(d) {}
  bool next(std::string& line) {
    if (pos_ >= d_.size()) return false;
    const size_t e = d_.find('\n', pos_);
    const size_t end = e == std::string_view::npos ? d_.size() : e;
    line.assign(d_.data() + pos_, end - pos_);
    pos_ = e == std::string_view::npos ? d_.size() : e + 1;
    return true;
  }

 private:
  std::string_view d_;
  size_t pos_ = 0;
};

void decode_jsonl(std::string_view in, desmoe_moet_header* h, double* logits) {
  Lines lines(in);
  std::string line;
  if (!lines.next(line)) throw MoetFail{DESMOE_MOET_TRUNCATED, "missing header line"};
  json head;
  try {
    head = json::parse(line);
  } catch (const json::exception&) {
    throw MoetFail{DESMOE_MOET_BAD_HEADER, "unparseable header line"};
  }
  desmoe_moet_header hd{};
  try {
    const int version = head.at("version").get<int>();
    if (version != 1)
      throw MoetFail{DESMOE_MOET_BAD_VERSION, "unsupported version " + std::to_string(version)};
    hd.experts = head.at("experts").get<int>();
    hd.top_k = head.at("top_k").get<int>();
    hd.layers = head.at("layers").get<int>();
    hd.block_size = head.at("block_size").get<int>();
    hd.steps = head.at("steps").get<int>();
    const std::string model = head.at("model").get<std::string>();
    if (model == "iid_gaussian") hd.model = 0;
    else if (model == "dirichlet") hd.model = 1;
    else if (model == "shared_bias") hd.model = 2;
    else throw MoetFail{DESMOE_MOET_BAD_HEADER, "malformed header line"};  // trace.cpp:26, caught :338
    hd.rho = head.at("rho").get<double>();
    hd.temperature = head.at("temperature").get<double>();
    hd.seed = head.at("seed").get<uint64_t>();
  } catch (const MoetFail&) {
    throw;
  } catch (const std::exception&) {
    throw MoetFail{DESMOE_MOET_BAD_HEADER, "malformed header line"};
  }
  check_header(hd);
  const size_t per = static_cast<size_t>(hd.block_size) * hd.experts;
  const int records = hd.steps * hd.layers;
  for (int rec = 0; rec < records; ++rec) {
    const std::string rs = std::to_string(rec);
    if (!lines.next(line)) throw MoetFail{DESMOE_MOET_TRUNCATED, "missing record " + rs};
    json obj;
    try {
      obj = json::parse(line);
    } catch (const json::exception&) {
      throw MoetFail{DESMOE_MOET_SHAPE_MISMATCH, "unparseable record " + rs};
    }
    try {
      if (obj.at("step").get<int>() != rec / hd.layers ||
          obj.at("layer").get<int>() != rec % hd.layers)
        throw MoetFail{DESMOE_MOET_SHAPE_MISMATCH, "record " + rs + " out of order"};
      const json& rows = obj.at("logits");
      if (static_cast<int>(rows.size()) != hd.block_size)
        throw MoetFail{DESMOE_MOET_SHAPE_MISMATCH, "record " + rs + " has " +
                                                       std::to_string(rows.size()) +
                                                       " rows, expected " +
                                                       std::to_string(hd.block_size)};
      size_t i = 0;
      for (const json& row : rows) {
        if (static_cast<int>(row.size()) != hd.experts)
          throw MoetFail{DESMOE_MOET_SHAPE_MISMATCH, "record " + rs + " has a " +
                                                         std::to_string(row.size()) +
                                                         "-wide row, expected " +
                                                         std::to_string(hd.experts)};
        for (const json& v : row) {
          if (!v.is_number())
            throw MoetFail{DESMOE_MOET_BAD_VALUE, "non-numeric logit in record " + rs};
          const double x = v.get<double>();
          if (!std::isfinite(x))
            throw MoetFail{DESMOE_MOET_BAD_VALUE, "non-finite logit in record " + rs};
          if (logits) logits[static_cast<size_t>(rec) * per + i] = x;
          ++i;
        }
      }
    } catch (const MoetFail&) {
      throw;
    } catch (const std::exception&) {
      throw MoetFail{DESMOE_MOET_SHAPE_MISMATCH, "malformed record " + rs};
    }
  }
  while (lines.next(line))
    if (!line.empty()) throw MoetFail{DESMOE_MOET_SHAPE_MISMATCH, "trailing data after last record"};
  *h = hd;
}

void put_le(std::string& out, uint64_t v, int bytes) {
  for (int i = 0; i < bytes; ++i) out.push_back(static_cast<char>((v >> (8 * i)) & 0xFF));
}

void put_f32(std::string& out, double v) {
  const float f = static_cast<float>(v);
  uint32_t b;
  std::memcpy(&b, &f, 4);
  put_le(out, b, 4);
}

std::string encode(const desmoe_moet_header& h, const double* logits, int format) {
  check_header(h);
  const size_t per = static_cast<size_t>(h.block_size) * h.experts;
  const int records = h.steps * h.layers;
  std::string out;
  if (format == DESMOE_MOET_BINARY) {
    out.reserve(40 + static_cast<size_t>(records) * (8 + 4 * per));
    out.append("MOET", 4);
    put_le(out, 1, 2);
    out.push_back(static_cast<char>(h.model));
    out.push_back(0);
    for (int v : {h.experts, h.top_k, h.layers, h.block_size, h.steps})
      put_le(out, static_cast<uint32_t>(v), 4);
    put_le(out, h.seed, 8);
    put_f32(out, h.rho);
    put_f32(out, h.temperature);
    for (int rec = 0; rec < records; ++rec) {
      put_le(out, static_cast<uint32_t>(rec / h.layers), 4);
      put_le(out, static_cast<uint32_t>(rec % h.layers), 4);
      for (size_t i = 0; i < per; ++i) put_f32(out, logits[static_cast<size_t>(rec) * per + i]);
    }
    return out;
  }
  json head;
  head["version"] = 1;
  head["experts"] = h.experts;
  head["top_k"] = h.top_k;
  head["layers"] = h.layers;
  head["block_size"] = h.block_size;
  head["steps"] = h.steps;
  head["model"] = model_name(h.model);
  head["rho"] = h.rho;
  head["temperature"] = h.temperature;
  head["seed"] = h.seed;
  out = head.dump();
  out.push_back('\n');
  for (int rec = 0; rec < records; ++rec) {
    json obj;
    obj["step"] = rec / h.layers;
    obj["layer"] = rec % h.layers;
    json& rows = obj["logits"] = json::array();
    for (int t = 0; t < h.block_size; ++t) {
      const double* row = logits + static_cast<size_t>(rec) * per + static_cast<size_t>(t) * h.experts;
      rows.push_back(std::vector<double>(row, row + h.experts));
    }
    out += obj.dump();
    out.push_back('\n');
  }
  return out;
}

int fail_moet(const MoetFail& f, int* trace_code) {
  if (trace_code) *trace_code = f.code;
  return desmoe::set_last_error(DESMOE_EINVAL, f.msg);
}

}  // namespace

extern "C" {

int desmoe_moet_decode(const void* bytes, size_t len, desmoe_moet_header* header, double* logits,
                       int* trace_code) {
  if (trace_code) *trace_code = -1;
  if (!header) return desmoe::set_last_error(DESMOE_EINVAL, "null header");
  try {
    const std::string_view in(static_cast<const char*>(bytes), bytes ? len : 0);
    if (in.empty()) throw MoetFail{DESMOE_MOET_BAD_MAGIC, "empty input"};
    if (in.front() == '{')  // decode_trace sniffs the format (trace.cpp:432-441)
      decode_jsonl(in, header, logits);
    else
      decode_binary(in, header, logits);
  } catch (const MoetFail& f) {
    return fail_moet(f, trace_code);
  } catch (const std::exception& e) {
    return desmoe::set_last_error(DESMOE_EINVAL, e.what());
  }
  return DESMOE_OK;
}

int desmoe_moet_encode(const desmoe_moet_header* header, const double* logits, int format,
                       void* out, size_t* len, int* trace_code) {
  if (trace_code) *trace_code = -1;
  if (!header || !len) return desmoe::set_last_error(DESMOE_EINVAL, "null header or length");
  if (format != DESMOE_MOET_BINARY && format != DESMOE_MOET_JSONL)
    return desmoe::set_last_error(DESMOE_EINVAL, "unknown trace format");
  try {
    if (!logits) check_header(*header);
    const std::string bytes = logits ? encode(*header, logits, format) : std::string();
    if (!out) {
      *len = bytes.size();
      return DESMOE_OK;
    }
    if (*len < bytes.size()) return desmoe::set_last_error(DESMOE_EINVAL, "output buffer too small");
    std::memcpy(out, bytes.data(), bytes.size());
    *len = bytes.size();
  } catch (const MoetFail& f) {
    return fail_moet(f, trace_code);
  }
  return DESMOE_OK;
}

}  // extern "C"
