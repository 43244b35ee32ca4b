// C-ABI layer (include/desmoe.h): host-side validation with the reference's
// exact error messages, context-owned workspaces, TMA descriptor creation and
// the launch sequences of the routing stage, permutation, expert FFN and the
// whole layer. No computation happens on the host: every entry point only
// validates scalars and enqueues sm_100a kernels on the caller's stream.
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/desmoe.h"
#include "common.cuh"
#include "kernels.cuh"

using namespace desmoe;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define DESMOE_CUDA(expr)                                                               \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(DESMOE_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));    \
  } while (0)

#define DESMOE_LAUNCHED()                                                               \
  do {                                                                                  \
    cudaError_t e_ = cudaGetLastError();                                                \
    if (e_ != cudaSuccess)                                                              \
      return fail(DESMOE_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D bf16 tensor [rows x cols] row-major, box [box_rows x 64], SWIZZLE_128B.
int make_map(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return fail(DESMOE_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DESMOE_ECUDA, "cuTensorMapEncodeTiled failed (" +
                                                       std::to_string(static_cast<int>(r)) + ")");
  return DESMOE_OK;
}

// Packed weights: n_tiles contiguous [128 x 64] bf16 blocks (16 KB each),
// 3-D view {64 cols, 128 rows, n_tiles}, box = one block, SWIZZLE_128B.
int make_packed_map(CUtensorMap* map, const void* base, uint64_t n_tiles) {
  auto fn = encode_fn();
  if (!fn) return fail(DESMOE_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {64, 128, n_tiles};
  cuuint64_t strides[2] = {128, 128 * 128};
  cuuint32_t box[3] = {64, 128, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DESMOE_ECUDA, "cuTensorMapEncodeTiled (packed) failed (" +
                                                       std::to_string(static_cast<int>(r)) + ")");
  return DESMOE_OK;
}

int make_box_maps(BoxMaps* maps, const void* base, uint64_t rows, uint64_t cols) {
  for (int i = 0; i < kMaxBoxes; ++i) {
    int rc = make_map(&maps->map[i], base, rows, cols, 16u << i);
    if (rc) return rc;
  }
  return DESMOE_OK;
}

int round_up(int v, int a) { return (v + a - 1) / a * a; }

constexpr int kSmemBudget = 220 * 1024;
constexpr int kSmemLimit = 227 * 1024;

}  // namespace

struct desmoe_ctx {
  int device = 0, max_n = 0, max_m = 0, max_k = 0, max_d = 0, num_sms = 148;
  // routing workspace
  double* probs = nullptr;
  int* topk_idx = nullptr;
  int* members = nullptr;
  int* n_members = nullptr;
  uint8_t* member_flag = nullptr;
  double* votes = nullptr;
  int* route_idx = nullptr;
  double* route_gate = nullptr;
  float* route_gate32 = nullptr;
  int* route_cnt = nullptr;
  int* err = nullptr;
  // permutation workspace
  int* expert_count = nullptr;
  int* expert_offset = nullptr;
  int* slot_of = nullptr;
  int* slot_token = nullptr;
  float* slot_gate = nullptr;
  int* active = nullptr;
  int* n_active = nullptr;
  int* total = nullptr;
  // router
  float* logits32 = nullptr;
  float* partials = nullptr;
  int max_splits = 32;
  // staging for the host entry point
  void* x_dev = nullptr;
  float* y_dev = nullptr;
  int* stats_dev = nullptr;
  // pinned, device-mapped [16]: [0..3] the host entry's stats (written by the
  // kernels straight into host memory), [4] the data-check word (c->err is
  // its device address), [5] the host entry's call number, [6] the call
  // number the last combine CTA published once y is visible (the host spins
  // on it instead of synchronising the stream), [8..9] the device-mapped
  // address of the caller's pinned x (read by the in-graph ingress kernel)
  int* host_tail = nullptr;
  int* host_tail_dev = nullptr;
  int host_calls = 0;
  const void* last_x_host = nullptr;   // pointer-attribute caches of the host entry
  const void* last_x_mapped = nullptr;
  const void* last_y_host = nullptr;
  float* last_y_mapped = nullptr;
  // cached router descriptors
  const void* x_map_ptr = nullptr;
  int x_map_n = -1, x_map_d = -1;
  BoxMaps x_maps{};
  // CUDA graph of the whole layer (re-captured when any argument changes)
  bool use_graphs = true;
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t gexec = nullptr;
  struct Key {
    const void *ex, *wr, *x;
    unsigned long long ex_uid;  // experts handle identity (a freed handle's address can be reused)
    int n;
    desmoe_route_cfg cfg;
    float* y;
    int* stats;
    bool prof;
    bool ingress;  // host-buffer entry: x copied in by the graph's first kernel
  } gkey{};
  int g_n_ev = 0, g_launches = 0;
  // layer stacks (desmoe_stack_forward): bf16 ping-pong activations and graph
  __nv_bfloat16* stack_buf[2] = {};
  cudaGraphExec_t sgexec = nullptr;
  std::vector<const void*> skey;
  // live phase timing
  bool profiling = false;
  cudaEvent_t ev[8] = {};
  int n_ev = 0;
  int launches = 0;
  uint64_t* trace = nullptr;  // optional FFN timeline buffer (device)
  int trace_cap = 0;
  const void* wr_map_ptr = nullptr;
  int wr_map_m = -1, wr_map_d = -1;
  CUtensorMap wr_map{};
};

struct desmoe_experts {
  desmoe_ctx* ctx = nullptr;
  int kind = 0, m = 0, d = 0, f = 0;
  int lo = 0, hi = 0;               // owned experts [lo, hi) (all unless expert-parallel)
  // expert parallelism: exchange buffers this rank exposes to its peers, and
  // the peers' buffers as mapped in this process
  int world = 1, rank = 0;
  // unique per handle and per expert-parallel (re)connection: captured graphs
  // are keyed on it, not on the handle's address alone
  unsigned long long uid = 0;
  float* ep_slot = nullptr;                 // [2][max_n*max_k][d] fp32 (parity halves)
  unsigned long long* ep_flag = nullptr;    // arrival counter (peers add to it)
  int* ep_state = nullptr;                  // [0] call seq (EP epoch), [1] combine CTAs done
  // front -> FFN hand-off words (tagged with the call seq, see kernels.cuh)
  uint64_t* route_words = nullptr;          // [max_n * max_k]
  uint32_t* pub = nullptr;                  // [1 + max_m] (+ route_done)
  uint32_t* route_done = nullptr;           // [kFrontCta], inside the pub allocation
  float* peer_slot[kMaxWorld] = {};
  unsigned long long* peer_flag[kMaxWorld] = {};
  void* ipc_mapped[2 * kMaxWorld] = {};     // peer buffers opened by desmoe_ep_import
  CUtensorMap wg{}, wu{}, wd{};
  BoxMaps xp_maps{}, h_maps{};
  __nv_bfloat16* x_perm = nullptr;  // [max_n*max_k x d]
  __nv_bfloat16* h_perm = nullptr;  // [max_n*max_k x f]
  float* y_slot = nullptr;          // [max_n*max_k x d]
  int* counters = nullptr;          // FFN scheduler / readiness counters
  uint32_t* b_done = nullptr;       // [m][d/128] + 1: phase-B unit tags (streamed host-entry combine)
  void* packed_a = nullptr;         // gate/up tiles (SwiGLU)
  void* packed_b = nullptr;         // W_d / W_lin tiles
};

namespace desmoe {
int set_last_error(int code, const std::string& msg) { return fail(code, msg); }
}  // namespace desmoe

namespace {
unsigned long long next_uid() {
  static std::atomic<unsigned long long> n{0};
  return ++n;
}
}  // namespace

extern "C" {

const char* desmoe_last_error(void) { return g_err.c_str(); }

int desmoe_version(void) { return 1; }

int desmoe_validate_pool(int experts, int top_k, uint64_t bytes_per_expert, int hidden_dim) {
  // validate_config, core.cpp:11-28 (same order, same messages)
  if (experts < 1) return fail(DESMOE_EINVAL, "experts_total < 1");
  if (top_k < 1) return fail(DESMOE_EINVAL, "top_k < 1");
  if (top_k > experts) return fail(DESMOE_EINVAL, "top_k > experts_total");
  if (bytes_per_expert == 0) return fail(DESMOE_EINVAL, "bytes_per_expert == 0");
  if (hidden_dim < 1) return fail(DESMOE_EINVAL, "hidden_dim < 1");
  return DESMOE_OK;
}

int desmoe_vote_budget(double beta, int experts) {
  return static_cast<int>(std::floor(beta * experts));
}

int desmoe_create(desmoe_ctx** out, int device, int max_tokens, int max_experts, int max_top_k,
                  int max_hidden) {
  if (!out) return fail(DESMOE_EINVAL, "null output handle");
  if (max_tokens < 1 || max_tokens > 1024)
    return fail(DESMOE_EINVAL, "max_tokens outside [1, 1024]");
  if (max_experts < 1 || max_experts > 1024)
    return fail(DESMOE_EINVAL, "max_experts outside [1, 1024]");
  if (max_top_k < 1 || max_top_k > 32) return fail(DESMOE_EINVAL, "max_top_k outside [1, 32]");
  if (max_hidden < 1) return fail(DESMOE_EINVAL, "max_hidden < 1");
  DESMOE_CUDA(cudaSetDevice(device));
  auto* c = new desmoe_ctx();
  c->device = device;
  c->max_n = max_tokens;
  c->max_m = max_experts;
  c->max_k = max_top_k;
  c->max_d = max_hidden;
  if (const char* g = std::getenv("DESMOE_GRAPHS")) c->use_graphs = std::atoi(g) != 0;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  const size_t nm = static_cast<size_t>(max_tokens) * max_experts;
  const size_t nk = static_cast<size_t>(max_tokens) * max_top_k;
  auto alloc = [&](auto** p, size_t count) {
    return cudaMalloc(reinterpret_cast<void**>(p), sizeof(**p) * std::max<size_t>(count, 1));
  };
  cudaError_t e = cudaSuccess;
  auto A = [&](cudaError_t r) {
    if (e == cudaSuccess) e = r;
  };
  A(alloc(&c->probs, nm));
  A(alloc(&c->topk_idx, nk));
  A(alloc(&c->members, max_experts));
  A(alloc(&c->n_members, 1));
  A(alloc(&c->member_flag, max_experts));
  A(alloc(&c->votes, max_experts));
  A(alloc(&c->route_idx, nk));
  A(alloc(&c->route_gate, nk));
  A(alloc(&c->route_gate32, nk));
  A(alloc(&c->route_cnt, max_tokens));
  A(alloc(&c->expert_count, max_experts));
  A(alloc(&c->expert_offset, max_experts));
  A(alloc(&c->slot_of, nk));
  A(alloc(&c->slot_token, nk));
  A(alloc(&c->slot_gate, nk));
  A(alloc(&c->active, max_experts));
  A(alloc(&c->n_active, 1));
  A(alloc(&c->total, 1));
  A(alloc(&c->logits32, nm));
  A(alloc(&c->partials, nm * c->max_splits));
  A(alloc(reinterpret_cast<__nv_bfloat16**>(&c->x_dev), static_cast<size_t>(max_tokens) * max_hidden));
  A(alloc(&c->y_dev, static_cast<size_t>(max_tokens) * max_hidden));
  A(alloc(&c->stats_dev, 4));
  if (e == cudaSuccess)
    e = cudaHostAlloc(reinterpret_cast<void**>(&c->host_tail), 16 * sizeof(int), cudaHostAllocMapped);
  if (e == cudaSuccess)
    e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->host_tail_dev), c->host_tail, 0);
  if (e == cudaSuccess) {
    std::memset(c->host_tail, 0, 16 * sizeof(int));
    c->err = c->host_tail_dev + 4;
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = desmoe::set_kernel_smem_limits();
  if (e != cudaSuccess) {
    desmoe_destroy(c);
    return fail(DESMOE_ECUDA, std::string("workspace allocation: ") + cudaGetErrorString(e));
  }
  *out = c;
  return DESMOE_OK;
}

void desmoe_destroy(desmoe_ctx* c) {
  if (!c) return;
  void* ptrs[] = {c->probs, c->topk_idx, c->members, c->n_members, c->member_flag, c->votes,
                  c->route_idx, c->route_gate, c->route_gate32, c->route_cnt,
                  c->expert_count, c->expert_offset, c->slot_of, c->slot_token, c->slot_gate,
                  c->active, c->n_active, c->total, c->logits32, c->partials, c->x_dev,
                  c->y_dev, c->stats_dev};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->host_tail) cudaFreeHost(c->host_tail);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->sgexec) cudaGraphExecDestroy(c->sgexec);
  for (auto* b : c->stack_buf)
    if (b) cudaFree(b);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  delete c;
}

int desmoe_check(desmoe_ctx* c, void* stream) {
  if (!c) return fail(DESMOE_EINVAL, "null context");
  DESMOE_CUDA(cudaStreamSynchronize(S(stream)));
  // the flag word is host memory the kernels write through the mapping
  volatile int* fw = c->host_tail + 4;
  const int flag = *fw;
  if (flag) {
    *fw = 0;
    if (flag == 2)
      return fail(DESMOE_ECUDA, "expert-parallel exchange timed out (a peer rank stopped)");
    return fail(DESMOE_EINVAL, "non-finite logit");
  }
  return DESMOE_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// routing launch helpers
// ---------------------------------------------------------------------------
namespace {

int check_block(desmoe_ctx* c, int n, int m) {
  if (!c) return fail(DESMOE_EINVAL, "null context");
  if (n < 1) return fail(DESMOE_EINVAL, "block_size < 1");
  if (n > c->max_n) return fail(DESMOE_EINVAL, "block_size exceeds context capacity");
  if (m < 1 || m > c->max_m) return fail(DESMOE_EINVAL, "experts outside context capacity");
  return DESMOE_OK;
}

template <typename T>
int launch_gate_topk(desmoe_ctx* c, const T* logits, const float* partials, int splits, int n,
                     int m, int k, int act, int mode, double* probs, int kmax, int* route_idx,
                     double* route_gate, int* route_cnt, cudaStream_t st) {
  GateTopkArgs<T> a{};
  a.logits = logits;
  a.partials = partials;
  a.logits_out = partials ? c->logits32 : nullptr;
  a.splits = splits;
  a.m_pad = m;
  a.n = n;
  a.m = m;
  a.k = k;
  a.kmax = kmax;
  a.act = act;
  a.mode = mode;
  a.probs = probs;
  a.topk_idx = c->topk_idx;
  a.route_idx = route_idx;
  a.route_gate = route_gate;
  a.route_gate32 = (route_gate == c->route_gate) ? c->route_gate32 : nullptr;
  a.route_cnt = route_cnt;
  a.err = c->err;
  const int warps = 8;
  const size_t smem = static_cast<size_t>(warps) * m * sizeof(double) + warps * 32 * sizeof(int);
  cudaError_t e = launch_gate_topk_kernel<T>(a, (n + warps - 1) / warps, warps * 32, smem, st);
  if (e != cudaSuccess) return fail(DESMOE_ECUDA, std::string("gate_topk: ") + cudaGetErrorString(e));
  return DESMOE_OK;
}

template <typename T>
int launch_coreset(desmoe_ctx* c, const T* logits, int n, const desmoe_route_cfg* cfg,
                   double* votes, cudaStream_t st) {
  CoresetArgs a{};
  a.n = n;
  a.m = cfg->experts;
  a.k = cfg->top_k;
  a.strategy = cfg->strategy;
  a.seq_k = cfg->seq_k;
  a.m_core = desmoe_vote_budget(cfg->vote_beta, cfg->experts);
  a.raw = cfg->vote_source == DESMOE_VOTE_RAW_LOGITS;
  a.topk_idx = c->topk_idx;
  a.probs = c->probs;
  if constexpr (sizeof(T) == 8)
    a.logits64 = reinterpret_cast<const double*>(logits);
  else
    a.logits32 = reinterpret_cast<const float*>(logits);
  a.votes = votes;
  a.members = c->members;
  a.n_members = c->n_members;
  a.member_flag = c->member_flag;
  const int m = cfg->experts;
  const int words = (m + 31) / 32;
  const size_t smem = static_cast<size_t>(n) * words * 4 + 8 + static_cast<size_t>(m) * 8 +
                      static_cast<size_t>(m) * 4;
  const int threads = std::max(128, round_up(m, 32));
  coreset_kernel<<<1, threads, smem, st>>>(a);
  DESMOE_LAUNCHED();
  return DESMOE_OK;
}

int launch_reroute(desmoe_ctx* c, int n, int m, int k, bool fast_path, int* route_idx,
                   double* route_gate, int* route_cnt, cudaStream_t st) {
  RerouteArgs a{};
  a.n = n;
  a.m = m;
  a.k = k;
  a.probs = c->probs;
  a.topk_idx = fast_path ? c->topk_idx : nullptr;
  a.member_flag = c->member_flag;
  a.n_members = c->n_members;
  a.route_idx = route_idx;
  a.route_gate = route_gate;
  a.route_gate32 = (route_gate == c->route_gate) ? c->route_gate32 : nullptr;
  a.route_cnt = route_cnt;
  const int warps = 8;
  constrained_route_kernel<<<(n + warps - 1) / warps, warps * 32, warps * 32 * sizeof(int), st>>>(a);
  DESMOE_LAUNCHED();
  return DESMOE_OK;
}

// Validation of des_run's parameters (des.cpp:10-27, validate_config first).
int check_des_params(const desmoe_route_cfg* cfg) {
  int rc = desmoe_validate_pool(cfg->experts, cfg->top_k, 1, 1);
  if (rc) return rc;
  if (cfg->strategy == DESMOE_SEQ) {
    if (cfg->seq_k < 1) return fail(DESMOE_EINVAL, "seq_k < 1");
    if (cfg->seq_k > cfg->top_k) return fail(DESMOE_EINVAL, "seq_k > top_k");
  } else if (cfg->strategy == DESMOE_VOTE) {
    if (!(cfg->vote_beta > 0.0) || cfg->vote_beta > 1.0)
      return fail(DESMOE_EINVAL, "vote_beta outside (0, 1]");
    if (desmoe_vote_budget(cfg->vote_beta, cfg->experts) < 1)
      return fail(DESMOE_EINVAL, "vote budget floor(beta*M) < 1");
  } else {
    return fail(DESMOE_EINVAL, "unknown strategy");
  }
  return DESMOE_OK;
}

// Full routing from logits of type T (fp64 RouterBlock or fp32), or from the
// router's split-K partials (partials != nullptr).
template <typename T>
int route_impl(desmoe_ctx* c, const T* logits, const float* partials, int splits, int n,
               const desmoe_route_cfg* cfg, const desmoe_route_out* out, cudaStream_t st,
               int* zero = nullptr, int zero_words = 0, bool* zeroed = nullptr) {
  const int m = cfg->experts, k = cfg->top_k;
  int rc = check_block(c, n, m);
  if (rc) return rc;
  if (k > c->max_k) return fail(DESMOE_EINVAL, "top_k exceeds context capacity");
  if (cfg->activation < 0 || cfg->activation > 2)
    return fail(DESMOE_EINVAL, "unknown gate activation");
  int* ridx = out && out->route_idx_dev ? out->route_idx_dev : c->route_idx;
  double* rgate = out && out->route_gate_dev ? out->route_gate_dev : c->route_gate;
  int* rcnt = out && out->route_cnt_dev ? out->route_cnt_dev : c->route_cnt;
  if (zeroed) *zeroed = false;
  if (cfg->strategy == DESMOE_VANILLA) {
    if (k < 1 || k > m) return fail(DESMOE_EINVAL, "top_k out of range");
  } else {
    rc = check_des_params(cfg);
    if (rc) return rc;
  }
  const bool want_union = cfg->strategy == DESMOE_VANILLA && out &&
                          (out->coreset_dev || out->coreset_size_dev);
  if (!want_union && fused_route_smem(n, m, k) <= static_cast<size_t>(kFusedRouteSmem)) {
    // whole routing stage in one single-CTA kernel
    FusedRouteArgs<T> a{};
    a.logits = logits;
    a.partials = partials;
    a.splits = splits;
    a.logits_out = partials ? c->logits32 : nullptr;
    a.raw_logits = partials ? reinterpret_cast<const T*>(c->logits32) : logits;
    a.n = n;
    a.m = m;
    a.k = k;
    a.act = cfg->activation;
    a.strategy = cfg->strategy;
    a.seq_k = cfg->seq_k;
    a.m_core = desmoe_vote_budget(cfg->vote_beta, m);
    a.raw = cfg->vote_source == DESMOE_VOTE_RAW_LOGITS;
    a.route_idx = ridx;
    a.route_gate = rgate;
    a.route_cnt = rcnt;
    a.members = out && out->coreset_dev ? out->coreset_dev : c->members;
    a.n_members = out && out->coreset_size_dev ? out->coreset_size_dev : c->n_members;
    a.member_flag = c->member_flag;
    a.votes = out ? out->votes_dev : nullptr;
    a.probs = out ? out->probs_dev : nullptr;
    a.zero = zero;
    a.zero_words = zero_words;
    a.err = c->err;
    cudaError_t e = launch_fused_route<T>(a, st);
    if (e != cudaSuccess)
      return fail(DESMOE_ECUDA, std::string("fused routing: ") + cudaGetErrorString(e));
    if (out && out->coreset_size_dev && out->coreset_size_dev != c->n_members &&
        cfg->strategy != DESMOE_VANILLA) {
      // the members list already went to out->coreset_dev
    }
    if (zeroed) *zeroed = zero != nullptr;
    return DESMOE_OK;
  }
  if (cfg->strategy == DESMOE_VANILLA) {
    // topk_route(activate(block), K): gating.cpp:84-87
    rc = launch_gate_topk<T>(c, logits, partials, splits, n, m, k, cfg->activation, 0,
                             out && out->probs_dev ? out->probs_dev : c->probs, k, ridx, rgate,
                             rcnt, st);
    if (rc) return rc;
    if (out && (out->coreset_dev || out->coreset_size_dev)) {
      // unique_experts(assign) via the permutation's active list
      PermuteArgs p{};
      p.n = n;
      p.m = m;
      p.k = k;
      p.route_idx = ridx;
      p.route_cnt = rcnt;
      p.active = out->coreset_dev ? out->coreset_dev : c->active;
      p.n_active = out->coreset_size_dev ? out->coreset_size_dev : c->n_active;
      p.total = c->total;
      const int tw = (n + 31) / 32;
      const size_t smem = static_cast<size_t>(m) * 8 + static_cast<size_t>(m) * tw * 4;
      permute_kernel<<<1, std::max(128, round_up(m, 32)), smem, st>>>(p);
      DESMOE_LAUNCHED();
    }
    return DESMOE_OK;
  }
  rc = launch_gate_topk<T>(c, logits, partials, splits, n, m, k, cfg->activation, 1, c->probs,
                           k, nullptr, nullptr, nullptr, st);
  if (rc) return rc;
  if (out && out->probs_dev)
    DESMOE_CUDA(cudaMemcpyAsync(out->probs_dev, c->probs, sizeof(double) * n * m,
                                cudaMemcpyDeviceToDevice, st));
  const T* raw = partials ? reinterpret_cast<const T*>(c->logits32) : logits;
  rc = launch_coreset<T>(c, raw, n, cfg, out ? out->votes_dev : nullptr, st);
  if (rc) return rc;
  rc = launch_reroute(c, n, m, k, true, ridx, rgate, rcnt, st);
  if (rc) return rc;
  if (out && out->coreset_dev)
    DESMOE_CUDA(cudaMemcpyAsync(out->coreset_dev, c->members, sizeof(int) * m,
                                cudaMemcpyDeviceToDevice, st));
  if (out && out->coreset_size_dev)
    DESMOE_CUDA(cudaMemcpyAsync(out->coreset_size_dev, c->n_members, sizeof(int),
                                cudaMemcpyDeviceToDevice, st));
  return DESMOE_OK;
}

}  // namespace

extern "C" {

int desmoe_activate(desmoe_ctx* c, const double* logits, int n, int m, int act, double* probs,
                    void* stream) {
  int rc = check_block(c, n, m);
  if (rc) return rc;
  // selection of 1 keeps the kernel's top-K path trivially valid
  return launch_gate_topk<double>(c, logits, nullptr, 0, n, m, 1, act, 1, probs, 1, nullptr,
                                  nullptr, nullptr, S(stream));
}

int desmoe_route(desmoe_ctx* c, const double* logits, int n, const desmoe_route_cfg* cfg,
                 const desmoe_route_out* out, void* stream) {
  if (!cfg) return fail(DESMOE_EINVAL, "null config");
  return route_impl<double>(c, logits, nullptr, 0, n, cfg, out, S(stream));
}

int desmoe_route_f32(desmoe_ctx* c, const float* logits, int n, const desmoe_route_cfg* cfg,
                     const desmoe_route_out* out, void* stream) {
  if (!cfg) return fail(DESMOE_EINVAL, "null config");
  return route_impl<float>(c, logits, nullptr, 0, n, cfg, out, S(stream));
}

int desmoe_coreset(desmoe_ctx* c, const double* logits, int n, const desmoe_route_cfg* cfg,
                   const desmoe_route_out* out, void* stream) {
  if (!cfg) return fail(DESMOE_EINVAL, "null config");
  const int m = cfg->experts, k = cfg->top_k;
  int rc = check_block(c, n, m);
  if (rc) return rc;
  if (k < 1 || k > m || k > c->max_k) return fail(DESMOE_EINVAL, "top_k out of range");
  if (cfg->strategy == DESMOE_SEQ) {
    // des_seq_coreset (des.cpp:34-36)
    if (cfg->seq_k < 1 || cfg->seq_k > k)
      return fail(DESMOE_EINVAL, "local_k outside [1, top_k]");
  } else if (cfg->strategy == DESMOE_VOTE) {
    // checked_budget (des.cpp:49-61)
    if (!(cfg->vote_beta > 0.0)) return fail(DESMOE_EINVAL, "beta <= 0");
    int mc = desmoe_vote_budget(cfg->vote_beta, m);
    if (mc < 1) return fail(DESMOE_EINVAL, "vote budget floor(beta*M) < 1");
    if (mc > m) return fail(DESMOE_EINVAL, "beta > 1");
  } else {
    return fail(DESMOE_EINVAL, "unknown strategy");
  }
  cudaStream_t st = S(stream);
  rc = launch_gate_topk<double>(c, logits, nullptr, 0, n, m, k, cfg->activation, 1, c->probs, k,
                                nullptr, nullptr, nullptr, st);
  if (rc) return rc;
  rc = launch_coreset<double>(c, logits, n, cfg, out ? out->votes_dev : nullptr, st);
  if (rc) return rc;
  if (out && out->coreset_dev)
    DESMOE_CUDA(cudaMemcpyAsync(out->coreset_dev, c->members, sizeof(int) * m,
                                cudaMemcpyDeviceToDevice, st));
  if (out && out->coreset_size_dev)
    DESMOE_CUDA(cudaMemcpyAsync(out->coreset_size_dev, c->n_members, sizeof(int),
                                cudaMemcpyDeviceToDevice, st));
  return DESMOE_OK;
}

int desmoe_constrained_route(desmoe_ctx* c, const double* logits, int n,
                             const desmoe_route_cfg* cfg, const int* members_host, int n_members,
                             const desmoe_route_out* out, void* stream) {
  if (!cfg) return fail(DESMOE_EINVAL, "null config");
  const int m = cfg->experts, k = cfg->top_k;
  int rc = check_block(c, n, m);
  if (rc) return rc;
  if (k < 1 || k > m || k > c->max_k) return fail(DESMOE_EINVAL, "top_k out of range");
  // des.cpp:100-105
  if (n_members < 1 || !members_host) return fail(DESMOE_EINVAL, "empty coreset");
  if (members_host[n_members - 1] >= m) return fail(DESMOE_EINVAL, "coreset member out of range");
  for (int i = 0; i < n_members; ++i)
    if (members_host[i] < 0 || (i > 0 && members_host[i] <= members_host[i - 1]))
      return fail(DESMOE_EINVAL, "coreset members must be ascending, unique, non-negative");
  cudaStream_t st = S(stream);
  DESMOE_CUDA(cudaMemcpyAsync(c->members, members_host, sizeof(int) * n_members,
                              cudaMemcpyHostToDevice, st));
  set_members_kernel<<<1, 256, 0, st>>>(c->members, n_members, m, c->member_flag, c->n_members);
  DESMOE_LAUNCHED();
  rc = launch_gate_topk<double>(c, logits, nullptr, 0, n, m, 1, cfg->activation, 1, c->probs, 1,
                                nullptr, nullptr, nullptr, st);
  if (rc) return rc;
  int* ridx = out && out->route_idx_dev ? out->route_idx_dev : c->route_idx;
  double* rgate = out && out->route_gate_dev ? out->route_gate_dev : c->route_gate;
  int* rcnt = out && out->route_cnt_dev ? out->route_cnt_dev : c->route_cnt;
  return launch_reroute(c, n, m, k, false, ridx, rgate, rcnt, st);
}

}  // extern "C"

template <typename T>
int baseline_impl(desmoe_ctx* c, const T* logits, int n, const desmoe_route_cfg* cfg,
                  const desmoe_baseline_cfg* b, const desmoe_route_out* out, cudaStream_t st) {
  if (!cfg || !b) return fail(DESMOE_EINVAL, "null config");
  const int m = cfg->experts, k = cfg->top_k;
  int rc = check_block(c, n, m);
  if (rc) return rc;
  if (k < 1 || k > m || k > c->max_k || k > 32) return fail(DESMOE_EINVAL, "top_k out of range");
  if (cfg->activation < 0 || cfg->activation > 2)
    return fail(DESMOE_EINVAL, "unknown gate activation");
  BaselineArgs<T> a{};
  // parameter checks in the reference's order (before activate)
  switch (b->method) {
    case DESMOE_BASE_TOPK_REDUCE:  // baselines.cpp:12-14
      if (b->k_reduced < 1 || b->k_reduced > k)
        return fail(DESMOE_EINVAL, "k_reduced outside [1, top_k]");
      break;
    case DESMOE_BASE_NAEE:  // :65-67
      if (!(b->naee_beta > 0.0) || !(b->naee_beta < 1.0))
        return fail(DESMOE_EINVAL, "naee beta outside (0, 1)");
      a.beta = b->naee_beta;
      break;
    case DESMOE_BASE_MCMOE: {  // :80-85, important = ceil(fraction * N) (:104-105)
      if (!(b->mcmoe_beta > 0.0) || !(b->mcmoe_beta < 1.0))
        return fail(DESMOE_EINVAL, "mcmoe beta outside (0, 1)");
      if (b->mcmoe_important_fraction < 0.0 || b->mcmoe_important_fraction > 1.0)
        return fail(DESMOE_EINVAL, "important_fraction outside [0, 1]");
      if (b->mcmoe_score != DESMOE_SCORE_MAX_GATE && b->mcmoe_score != DESMOE_SCORE_NEG_ENTROPY)
        return fail(DESMOE_EINVAL, "unknown importance score");
      a.beta = b->mcmoe_beta;
      a.score = b->mcmoe_score;
      a.important = std::min(static_cast<int>(std::ceil(b->mcmoe_important_fraction * n)), n);
      break;
    }
    default:
      return fail(DESMOE_EINVAL, "unknown baseline method");
  }
  a.logits = logits;
  a.n = n;
  a.m = m;
  a.k = k;
  a.act = cfg->activation;
  a.method = b->method;
  a.k_reduced = b->k_reduced;
  a.probs = out && out->probs_dev ? out->probs_dev : c->probs;
  a.route_idx = out && out->route_idx_dev ? out->route_idx_dev : c->route_idx;
  a.route_gate = out && out->route_gate_dev ? out->route_gate_dev : c->route_gate;
  a.route_cnt = out && out->route_cnt_dev ? out->route_cnt_dev : c->route_cnt;
  a.err = c->err;
  const size_t smem = static_cast<size_t>(n) * sizeof(double) + 32 * 32 * sizeof(int);
  baseline_route_kernel<T><<<1, 1024, smem, st>>>(a);
  DESMOE_LAUNCHED();
  return DESMOE_OK;
}

extern "C" {

int desmoe_baseline_route(desmoe_ctx* c, const double* logits, int n, const desmoe_route_cfg* cfg,
                          const desmoe_baseline_cfg* b, const desmoe_route_out* out,
                          void* stream) {
  return baseline_impl<double>(c, logits, n, cfg, b, out, S(stream));
}

int desmoe_baseline_route_f32(desmoe_ctx* c, const float* logits, int n,
                              const desmoe_route_cfg* cfg, const desmoe_baseline_cfg* b,
                              const desmoe_route_out* out, void* stream) {
  return baseline_impl<float>(c, logits, n, cfg, b, out, S(stream));
}

int desmoe_permute(desmoe_ctx* c, const int* route_idx, const int* route_cnt, int n, int k,
                   int m, int* expert_count, int* expert_offset, int* slot_of, int* slot_token,
                   int* active, int* n_active, void* stream) {
  int rc = check_block(c, n, m);
  if (rc) return rc;
  if (k < 1 || k > c->max_k) return fail(DESMOE_EINVAL, "top_k out of range");
  PermuteArgs p{};
  p.n = n;
  p.m = m;
  p.k = k;
  p.route_idx = route_idx;
  p.route_cnt = route_cnt;
  p.expert_count = expert_count;
  p.expert_offset = expert_offset;
  p.slot_of = slot_of;
  p.slot_token = slot_token;
  p.active = active ? active : c->active;
  p.n_active = n_active ? n_active : c->n_active;
  p.total = c->total;
  const int tw = (n + 31) / 32;
  const size_t smem = static_cast<size_t>(m) * 8 + static_cast<size_t>(m) * tw * 4;
  permute_kernel<<<1, std::max(128, round_up(m, 32)), smem, S(stream)>>>(p);
  DESMOE_LAUNCHED();
  return DESMOE_OK;
}

int desmoe_experts_create(desmoe_ctx* c, int kind, int m, int d, int f, const void* wg,
                          const void* wu, const void* wd, desmoe_experts** out) {
  return desmoe_experts_create_ep(c, kind, m, 0, m, d, f, wg, wu, wd, out);
}

int desmoe_experts_create_ep(desmoe_ctx* c, int kind, int m, int lo, int hi, int d, int f,
                             const void* wg, const void* wu, const void* wd,
                             desmoe_experts** out) {
  if (!c || !out) return fail(DESMOE_EINVAL, "null argument");
  if (kind != DESMOE_FFN_SWIGLU && kind != DESMOE_FFN_LINEAR)
    return fail(DESMOE_EINVAL, "unknown expert kind");
  if (m < 1 || m > c->max_m) return fail(DESMOE_EINVAL, "experts outside context capacity");
  if (lo < 0 || hi > m || lo >= hi) return fail(DESMOE_EINVAL, "owned expert range outside [0, experts)");
  if (kind == DESMOE_FFN_LINEAR) f = d;
  if (d < 128 || d % 128 || d > c->max_d) return fail(DESMOE_EINVAL, "hidden must be a multiple of 128 within capacity");
  if (f < 128 || f % 128) return fail(DESMOE_EINVAL, "ffn must be a multiple of 128");
  if (!wg || (kind == DESMOE_FFN_SWIGLU && (!wu || !wd)))
    return fail(DESMOE_EINVAL, "missing expert weights");
  auto* ex = new desmoe_experts();
  ex->uid = next_uid();
  ex->ctx = c;
  ex->kind = kind;
  ex->m = m;
  ex->d = d;
  ex->f = f;
  ex->lo = lo;
  ex->hi = hi;
  const size_t slots = static_cast<size_t>(c->max_n) * c->max_k;
  cudaError_t e = cudaMalloc(&ex->x_perm, slots * d * 2);
  if (e == cudaSuccess) e = cudaMalloc(&ex->h_perm, slots * f * 2);
  if (e == cudaSuccess) e = cudaMalloc(&ex->y_slot, slots * d * 4);
  if (e == cudaSuccess)
    e = cudaMalloc(&ex->counters, sizeof(int) * ffn_counter_words(m, f));
  if (e == cudaSuccess) e = cudaMemset(ex->counters, 0, sizeof(int) * ffn_counter_words(m, f));
  if (e == cudaSuccess) e = cudaMalloc(&ex->ep_state, 256);
  if (e == cudaSuccess) e = cudaMemset(ex->ep_state, 0, 256);
  if (e == cudaSuccess) e = cudaMalloc(&ex->route_words, slots * sizeof(uint64_t));
  if (e == cudaSuccess) e = cudaMemset(ex->route_words, 0xFF, slots * sizeof(uint64_t));
  // published list [1 + max_m], then (own 128-byte line) the front CTAs'
  // route-complete words [kFrontCta]
  const size_t pub_words = (static_cast<size_t>(c->max_m) + 1 + 31) / 32 * 32 + 32;
  if (e == cudaSuccess) e = cudaMalloc(&ex->pub, pub_words * 4);
  if (e == cudaSuccess) e = cudaMemset(ex->pub, 0xFF, pub_words * 4);
  ex->route_done = ex->pub + pub_words - 32;
  // (all-ones: no call's tag, kernels.cuh)
  const size_t bd_words = static_cast<size_t>(m) * std::max(1, d / kBM) + 1;
  if (e == cudaSuccess) e = cudaMalloc(&ex->b_done, bd_words * 4);
  if (e == cudaSuccess) e = cudaMemset(ex->b_done, 0xFF, bd_words * 4);
  if (e != cudaSuccess) {
    desmoe_experts_destroy(ex);
    return fail(DESMOE_ECUDA, std::string("expert workspace: ") + cudaGetErrorString(e));
  }
  int rc = DESMOE_OK;
  // pack the weights into tile-contiguous blocks (one-time)
  const int m_own = hi - lo;  // only the owned experts are packed
  const size_t b_elems = static_cast<size_t>(m_own) * d * f;
  cudaError_t pe = cudaMalloc(&ex->packed_b, b_elems * 2);
  if (pe == cudaSuccess && kind == DESMOE_FFN_SWIGLU) pe = cudaMalloc(&ex->packed_a, 2 * b_elems * 2);
  if (pe != cudaSuccess) {
    desmoe_experts_destroy(ex);
    return fail(DESMOE_ECUDA, std::string("packed weights: ") + cudaGetErrorString(pe));
  }
  cudaStream_t ps = cudaStreamPerThread;
  pe = cudaDeviceSynchronize();  // the caller's weights may still be in flight on any stream
  if (pe != cudaSuccess) {
    desmoe_experts_destroy(ex);
    return fail(DESMOE_ECUDA, std::string("weight registration: ") + cudaGetErrorString(pe));
  }
  if (kind == DESMOE_FFN_SWIGLU) {
    pack_weights_kernel<<<1184, 256, 0, ps>>>(static_cast<const uint4*>(wg),
                                              static_cast<const uint4*>(wu),
                                              static_cast<uint4*>(ex->packed_a), m_own, f, d, 1);
    pack_weights_kernel<<<1184, 256, 0, ps>>>(static_cast<const uint4*>(wd), nullptr,
                                              static_cast<uint4*>(ex->packed_b), m_own, d, f, 0);
  } else {
    pack_weights_kernel<<<1184, 256, 0, ps>>>(static_cast<const uint4*>(wg), nullptr,
                                              static_cast<uint4*>(ex->packed_b), m_own, d, d, 0);
  }
  pe = cudaGetLastError();
  if (pe == cudaSuccess) pe = cudaStreamSynchronize(ps);
  if (pe != cudaSuccess) {
    desmoe_experts_destroy(ex);
    return fail(DESMOE_ECUDA, std::string("weight packing: ") + cudaGetErrorString(pe));
  }
  const uint64_t tiles_b = b_elems / (128 * 64);
  if (kind == DESMOE_FFN_SWIGLU) {
    rc = make_packed_map(&ex->wg, ex->packed_a, 2 * tiles_b);
    ex->wu = ex->wg;
    if (!rc) rc = make_packed_map(&ex->wd, ex->packed_b, tiles_b);
    if (!rc) rc = make_box_maps(&ex->h_maps, ex->h_perm, slots, f);
  } else {
    rc = make_packed_map(&ex->wd, ex->packed_b, tiles_b);
    ex->wg = ex->wd;
    ex->wu = ex->wd;
  }
  if (!rc) rc = make_box_maps(&ex->xp_maps, ex->x_perm, slots, d);
  if (rc) {
    desmoe_experts_destroy(ex);
    return rc;
  }
  *out = ex;
  return DESMOE_OK;
}

void desmoe_experts_destroy(desmoe_experts* ex) {
  if (!ex) return;
  if (ex->x_perm) cudaFree(ex->x_perm);
  if (ex->h_perm) cudaFree(ex->h_perm);
  if (ex->y_slot) cudaFree(ex->y_slot);
  if (ex->counters) cudaFree(ex->counters);
  if (ex->packed_a) cudaFree(ex->packed_a);
  if (ex->packed_b) cudaFree(ex->packed_b);
  for (void* p : ex->ipc_mapped)
    if (p) cudaIpcCloseMemHandle(p);
  if (ex->ep_slot) cudaFree(ex->ep_slot);
  if (ex->ep_flag) cudaFree(ex->ep_flag);
  if (ex->ep_state) cudaFree(ex->ep_state);
  if (ex->route_words) cudaFree(ex->route_words);
  if (ex->pub) cudaFree(ex->pub);
  if (ex->b_done) cudaFree(ex->b_done);
  delete ex;
}

}  // extern "C"

namespace {

void mark(desmoe_ctx* c, cudaStream_t st) {
  if (!c->profiling || c->n_ev >= 8) return;
  if (!c->ev[c->n_ev]) cudaEventCreate(&c->ev[c->n_ev]);
  // External: inside a stream capture this becomes a real event-record node
  // (a plain record would only mark a capture dependency)
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(c->ev[c->n_ev], st, cudaEventRecordExternal);
  else
    cudaEventRecord(c->ev[c->n_ev], st);
  c->n_ev++;
}

int b_rows_for(int n) {
  int b = 16;
  while (b < n && b < 256) b <<= 1;
  return b;
}

int launch_router_tiles(const CUtensorMap& wa, const BoxMaps& acts, TileArgs a, int grid,
                        cudaStream_t st) {
  const int stage_bytes = kATile + a.b_rows * 128;
  const int per_unit_kb = (a.kb_total + a.splits - 1) / a.splits;
  int stages = (kSmemBudget - 1024 - 256) / stage_bytes;
  stages = std::max(1, std::min(stages, std::max(per_unit_kb, 1)));
  a.stages = stages;
  const size_t smem = static_cast<size_t>(stages) * stage_bytes + 1024 + 256;
  tile_gemm_kernel<<<grid, 256, smem, st>>>(wa, wa, acts, a);
  DESMOE_LAUNCHED();
  return DESMOE_OK;
}

// Launch plan of the persistent expert FFN: ring stage size (kb K blocks of
// 64), depth and dynamic shared memory. Every shape check the FFN launch
// makes lives here, so the layer entry can reject a block BEFORE the front
// kernel publishes anything (a published list / route with no FFN + combine
// behind it would be taken as valid by the next call's early-mode FFN).
struct FfnPlan {
  int kb = 2, stages = 2, b_rows = 16;
  size_t smem = 0;
};

int ffn_plan(const desmoe_experts* ex, int n, int k, FfnPlan* p) {
  const int m = ex->m, d = ex->d, f = ex->f;
  if (n > 256) return fail(DESMOE_EINVAL, "expert FFN supports up to 256 tokens per block");
  p->b_rows = b_rows_for(n);
  // ring stage = kb K blocks of 64: 4 (fewer, larger stages; measured on one
  // box: vanilla 131.3 -> 129.1 us, DES-Vote 73.8 -> 73.7) when both GEMM K
  // dims divide and two stages fit, else 2
  const int kdim_b = ex->kind == DESMOE_FFN_SWIGLU ? f : d;
  int kb = d % (4 * kBK) == 0 && kdim_b % (4 * kBK) == 0 ? 4 : 2;
  if (const char* kv = std::getenv("DESMOE_FFN_KB")) kb = std::atoi(kv) == 4 ? 4 : 2;
  if (kb == 4 && 2 * (4 * kATile + 4 * p->b_rows * 128) + 8192 > kSmemLimit - 256) kb = 2;
  if (kb == 4 && (d % (4 * kBK) || kdim_b % (4 * kBK))) kb = 2;
  p->kb = kb;
  const int stage_bytes = kb * kATile + kb * p->b_rows * 128;
  const int fixed = 1024 + 8 * (2 * 8 + 4 + 8) + 16 + 16 + 48 +
                    4 * (4 + 3 * m + 3 * n * k) + 16 * 64 * 4 + 64;
  int stages = (kSmemLimit - 256 - fixed) / stage_bytes;  // 256 B: the kernel's static smem
  // deeper rings only lengthen the queues every other memory access waits
  // behind: 128 KB of weights in flight per SM measured best (4 x 32 KB / 2 x 64 KB)
  stages = std::max(2, std::min(stages, 8 / kb));
  if (const char* sv = std::getenv("DESMOE_FFN_STAGES"))  // tuning experiments
    stages = std::max(2, std::min(stages, std::atoi(sv)));
  p->stages = stages;
  if (4 * (m * ((n + 31) / 32) + 3 * m + n * k) > stage_bytes)
    return fail(DESMOE_EINVAL, "expert FFN prologue scratch exceeds a pipeline stage");
  p->smem = static_cast<size_t>(fixed) + static_cast<size_t>(stages) * stage_bytes;
  if (p->smem > static_cast<size_t>(kSmemLimit - 256))
    return fail(DESMOE_EINVAL, "expert FFN shared-memory plan exceeds 227 KB");
  return DESMOE_OK;
}

int ffn_impl(desmoe_ctx* c, const desmoe_experts* ex, const void* x, int n, int k,
             const int* route_idx, const double* route_gate, const int* route_cnt, float* y,
             const int* n_members, int* stats, cudaStream_t st, bool counters_zeroed = false,
             bool after_front = false, __nv_bfloat16* y_bf16 = nullptr,
             const void* resid = nullptr, bool prefer_dense = false, bool layer_path = false,
             bool host_link = false) {
  const int m = ex->m, d = ex->d, f = ex->f;
  FfnPlan plan;
  int prc = ffn_plan(ex, n, k, &plan);
  if (prc) return prc;
  const int words = ffn_counter_words(m, f);
  if (!counters_zeroed) DESMOE_CUDA(cudaMemsetAsync(ex->counters, 0, sizeof(int) * words, st));
  FfnArgs a{};
  a.mode = ex->kind == DESMOE_FFN_SWIGLU ? 0 : 1;
  a.n_tok = n;
  a.top_k = k;
  a.m = m;
  a.d = d;
  a.f = f;
  a.b_rows = plan.b_rows;
  a.route_idx = route_idx;
  a.route_cnt = route_cnt;
  a.route_gate = route_gate;
  a.x = reinterpret_cast<const __nv_bfloat16*>(x);
  a.x_perm = ex->x_perm;
  a.h_perm = ex->h_perm;
  a.y_slot = ex->y_slot;
  a.slot_of = c->slot_of;
  a.counters = ex->counters;
  a.stats = stats;
  a.n_members = n_members;
  a.trace = c->trace;
  a.trace_cap = c->trace_cap;
  a.expert_lo = ex->lo;
  a.expert_hi = ex->hi;
  a.world = ex->world;
  a.epoch = ex->ep_state;
  a.early = after_front && !std::getenv("DESMOE_NO_EARLY") ? 1 : 0;
  // dense: small blocks compute every published expert for every token (the
  // tensor pipe is nearly idle in this memory-bound layer), so the FFN needs
  // only the published expert list — no route, permutation or gather
  // (dense writes U x N output rows where the routed mode writes N x K: it
  // pays when U is small, as for the DES coresets — the caller's hint)
  const bool dense = a.early && n <= kDenseMaxTokens && prefer_dense &&
                     static_cast<size_t>(m) * n <= static_cast<size_t>(c->max_n) * c->max_k &&
                     !std::getenv("DESMOE_NO_DENSE");
  a.dense = dense ? 1 : 0;
  // the first unit's L2 bulk prefetch at pick-up measured slightly slower
  // (the SMs' own TMA streams start at once in dense mode): opt-in only
  if (!std::getenv("DESMOE_L2PF")) a.flags |= 1;
  if (const char* fl = std::getenv("DESMOE_FFN_FLAGS")) a.flags |= std::atoi(fl);  // experiments
  a.pub = ex->pub;
  a.route_words = ex->route_words;
  a.route_done = ex->route_done;
  // host-buffer entry (dense, one rank): the combine streams on per-(expert,
  // d tile) tags, so y's bus writes overlap the FFN's last units. Measured:
  // e2e -1.6 us; on the device-resident path the per-unit release costs the
  // FFN ~0.8 us and the early combine more, so it stays off there
  // (DESMOE_NO_STREAM_COMBINE=1 disables, DESMOE_STREAM_COMBINE=1 forces)
  const bool stream_combine =
      dense && ex->world <= 1 && !std::getenv("DESMOE_NO_STREAM_COMBINE") &&
      (host_link || std::getenv("DESMOE_STREAM_COMBINE"));
  a.b_done = stream_combine ? ex->b_done : nullptr;
  a.b_drained = stream_combine ? ex->b_done + static_cast<size_t>(m) * (d / kBM) : nullptr;
  a.wa_base = ex->packed_a;
  a.wc_base = ex->packed_b;
  const size_t slot_stride = static_cast<size_t>(c->max_n) * c->max_k * d;
  if (ex->world > 1) {
    for (int r = 0; r < ex->world; ++r) {
      a.peer_slot[r] = ex->peer_slot[r];
      a.peer_flag[r] = ex->peer_flag[r];
    }
    a.slot_stride = slot_stride;
  }
  const int kb = plan.kb;
  a.kb = kb;
  // dense mode: phase-B units of two d tiles that share one H stream (the
  // activations count against each SM's ~50 GB/s ingress like the weights);
  // the queue's last pairs run as single tiles (DESMOE_FFN_PAIRB=0 disables,
  // DESMOE_FFN_SPLIT = how many pairs are split)
  // Routed mode too (a tile's columns must fit half the accumulator: every
  // expert's row count <= n <= 128), but only for the large unions of vanilla
  // top-K on the layer path — measured on one box: vanilla N=32 134.2 -> 130.0
  // us, N=128 167.0 -> 159.0; DES-Vote N=128 (routed, U = 25) 96.5 -> 97.2.
  // The standalone FFN entry (desmoe_expert_ffn / moe_forward) keeps single
  // tiles unless DESMOE_FFN_PAIR_ROUTED asks otherwise.
  const char* pr = std::getenv("DESMOE_FFN_PAIR_ROUTED");  // 0: off, 1: every strategy
  const bool routed_pairs =
      n <= 128 && (pr ? std::atoi(pr) != 0 && (std::atoi(pr) == 1 || !prefer_dense)
                      : layer_path && !prefer_dense);
  const bool pair_ok = dense || routed_pairs;
  a.pair_b = pair_ok && (d / kBM) % 2 == 0 ? 1 : 0;
  if (const char* pv = std::getenv("DESMOE_FFN_PAIRB")) a.pair_b = a.pair_b && std::atoi(pv) != 0;
  a.split_b = c->num_sms / 2;
  if (const char* sv = std::getenv("DESMOE_FFN_SPLIT")) a.split_b = std::max(0, std::atoi(sv));
  // phase A likewise: two F tiles sharing one X stream (X is 128 KB per
  // 512 KB tile at N = 32, d = 2048), the last pairs split
  a.pair_a = a.pair_b && ex->kind == DESMOE_FFN_SWIGLU && (f / 64) % 2 == 0 ? 1 : 0;
  if (const char* pv = std::getenv("DESMOE_FFN_PAIRA")) a.pair_a = a.pair_a && std::atoi(pv) != 0;
  a.split_a = c->num_sms;
  if (const char* sv = std::getenv("DESMOE_FFN_SPLITA")) a.split_a = std::max(0, std::atoi(sv));
  a.stages = plan.stages;
  const size_t smem = plan.smem;
  cudaLaunchConfig_t lc{};
  // One CTA per SM. Behind the front kernel (PDL) the FFN CTAs become
  // resident while it runs — except on the front cluster's SMs, where the
  // last kFrontCta CTAs start only after it exits: they stream weights but
  // take no part in the gather handshake.
  int grid = c->num_sms;
  if (const char* g = std::getenv("DESMOE_FFN_GRID")) grid = std::max(1, std::atoi(g));
  lc.gridDim = dim3(grid);
  a.gather_ctas = after_front && grid > 2 * kFrontCta ? grid - kFrontCta : grid;
  lc.blockDim = dim3(256);
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  // one CTA per SM (shared memory > half an SM), so all CTAs become resident
  // and the x_ready handshake cannot deadlock; launched programmatically
  // behind the routing kernel so barrier init / TMEM allocation overlap it
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  // dense phase A reads X itself (the front built its box maps for this x)
  const BoxMaps& xmaps = dense ? c->x_maps : ex->xp_maps;
  DESMOE_CUDA(cudaLaunchKernelEx(&lc, kb == 4 ? ffn_persistent_kernel<4> : ffn_persistent_kernel<2>,
                                 ex->wg, ex->wu, ex->wd, xmaps,
                                 ex->kind == DESMOE_FFN_SWIGLU ? ex->h_maps : xmaps, a));
  mark(c, st);  // profiling only: expert FFN | (EP wait +) combine
  // ordered combine, programmatically serialised behind the FFN kernel
  cudaLaunchConfig_t cc{};
  int cthreads = 256;  // (DESMOE_COMBINE_THREADS: 128 spreads the row loads over twice the SMs)
  if (const char* ct = std::getenv("DESMOE_COMBINE_THREADS"))
    cthreads = std::atoi(ct) == 128 ? 128 : (std::atoi(ct) == 64 ? 64 : 256);
  cc.gridDim = dim3((n * (d / 4) + cthreads - 1) / cthreads);
  cc.blockDim = dim3(cthreads);
  cc.stream = st;
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cc.attrs = pdl;
  cc.numAttrs = 1;
  CombineArgs ca{};
  ca.y_slot = ex->world > 1 ? ex->ep_slot : ex->y_slot;
  ca.slot_of = c->slot_of;
  ca.route_cnt = route_cnt;
  ca.n = n;
  ca.k = k;
  ca.d = d;
  ca.y = y;
  ca.y_bf16 = y_bf16;
  ca.resid = static_cast<const __nv_bfloat16*>(resid);
  ca.world = ex->world;
  ca.epoch = ex->ep_state;
  ca.done_ctas = ex->ep_state + 1;
  ca.zero = ex->counters;
  ca.zero_words = words;
  ca.route_idx = route_idx;
  ca.route_gate = route_gate;
  ca.route_words = ex->route_words;
  ca.pub = ex->pub;
  ca.m = m;
  ca.expert_lo = ex->lo;
  ca.expert_hi = ex->hi;
  ca.stats = stats;
  ca.b_done = a.b_done;
  ca.b_drained = a.b_drained;
  ca.tiles_b = d / kBM;
  ca.trace = c->trace;
  ca.trace_cap = c->trace_cap;
  if (host_link) {  // host-buffer entry: publish completion to the spinning host
    ca.host_call = c->host_tail_dev + 5;
    ca.host_done = c->host_tail_dev + 6;
  }
  if (ex->world > 1) {
    ca.flag = ex->ep_flag;
    ca.arrivals = static_cast<unsigned long long>(ex->world) * grid;
    ca.slot_stride = slot_stride;
    ca.err = c->err;
  }
  if (ex->world > 1) {
    // arrival wait (1 CTA, programmatic behind the FFN), then the combine as
    // a plain launch: no combine CTA sits resident while peers still stream
    cudaLaunchConfig_t wc{};
    wc.gridDim = dim3(1);
    wc.blockDim = dim3(32);
    wc.stream = st;
    wc.attrs = pdl;
    wc.numAttrs = 1;
    DESMOE_CUDA(cudaLaunchKernelEx(&wc, ep_wait_kernel, ca));
    cc.attrs = nullptr;
    cc.numAttrs = 0;
    c->launches += 1;
  }
  if (dense) {
    DESMOE_CUDA(cudaLaunchKernelEx(&cc, combine_dense_kernel, ca));
  } else {
    DESMOE_CUDA(cudaLaunchKernelEx(&cc, combine_slots_kernel, ca));
  }
  c->launches += 2;
  mark(c, st);
  return DESMOE_OK;
}

int router_impl(desmoe_ctx* c, const void* x, const void* w_r, int n, int m, int d,
                int* splits_out, cudaStream_t st) {
  if (d % kBK) return fail(DESMOE_EINVAL, "hidden must be a multiple of 64");
  if (n > 256) return fail(DESMOE_EINVAL, "router supports up to 256 tokens per block");
  if (x != c->x_map_ptr || n != c->x_map_n || d != c->x_map_d) {
    int rc = make_box_maps(&c->x_maps, x, n, d);
    if (rc) return rc;
    c->x_map_ptr = x;
    c->x_map_n = n;
    c->x_map_d = d;
  }
  if (w_r != c->wr_map_ptr || m != c->wr_map_m || d != c->wr_map_d) {
    int rc = make_map(&c->wr_map, w_r, m, d, kBM);
    if (rc) return rc;
    c->wr_map_ptr = w_r;
    c->wr_map_m = m;
    c->wr_map_d = d;
  }
  const int kb = d / kBK;
  const int et = (m + kBM - 1) / kBM;
  int splits = std::max(1, std::min(kb, std::min(c->max_splits, c->num_sms / et)));
  // equalise K blocks per split
  const int per = (kb + splits - 1) / splits;
  splits = (kb + per - 1) / per;
  TileArgs a{};
  a.n_tok = n;
  a.kb_total = kb;
  a.splits = splits;
  a.n_units_static = et * splits;
  a.b_rows = b_rows_for(n);
  a.m_pad = m;
  a.y_out = c->partials;
  int rc = launch_router_tiles(c->wr_map, c->x_maps, a, et * splits, st);
  if (rc) return rc;
  *splits_out = splits;
  return DESMOE_OK;
}


}  // namespace

extern "C" {

int desmoe_expert_ffn(desmoe_ctx* c, const desmoe_experts* ex, const void* x, int n, int k,
                      const int* route_idx, const double* route_gate, const int* route_cnt,
                      float* y, void* stream) {
  if (!c || !ex) return fail(DESMOE_EINVAL, "null argument");
  int rc = check_block(c, n, ex->m);
  if (rc) return rc;
  if (k < 1 || k > c->max_k) return fail(DESMOE_EINVAL, "top_k out of range");
  return ffn_impl(c, ex, x, n, k, route_idx, route_gate, route_cnt, y, nullptr, nullptr,
                  S(stream));
}

int desmoe_router_logits(desmoe_ctx* c, const void* x, const void* w_r, int n, int m, int d,
                         float* logits, void* stream) {
  int rc = check_block(c, n, m);
  if (rc) return rc;
  int splits = 0;
  cudaStream_t st = S(stream);
  rc = router_impl(c, x, w_r, n, m, d, &splits, st);
  if (rc) return rc;
  // reduce the partials in ascending split order (the same reduction the
  // fused gating kernel performs)
  GateTopkArgs<float> a{};
  a.partials = c->partials;
  a.logits_out = logits;
  a.splits = splits;
  a.m_pad = m;
  a.n = n;
  a.m = m;
  a.k = 1;
  a.kmax = 1;
  a.act = DESMOE_IDENTITY;
  a.mode = 1;
  a.topk_idx = c->topk_idx;
  a.err = c->err;
  const int warps = 8;
  const size_t smem = static_cast<size_t>(warps) * m * sizeof(double) + warps * 32 * sizeof(int);
  cudaError_t e = launch_gate_topk_kernel<float>(a, (n + warps - 1) / warps, warps * 32, smem, st);
  if (e != cudaSuccess) return fail(DESMOE_ECUDA, std::string("gate_topk: ") + cudaGetErrorString(e));
  return DESMOE_OK;
}

}  // extern "C"

namespace {

// Router GEMM + routing in one cluster launch (front.cu) when the shape fits:
// N <= 256 tokens, M <= 256 experts, hidden a multiple of 64 * kFrontCta.
int front_impl(desmoe_ctx* c, const desmoe_experts* ex, const void* x, const void* w_r, int n,
               const desmoe_route_cfg* cfg, cudaStream_t st, bool* used) {
  *used = false;
  const int m = cfg->experts, k = cfg->top_k, d = ex->d;
  if (std::getenv("DESMOE_NO_FRONT")) return DESMOE_OK;
  // pools of 257-512 experts, and hidden sizes that are not a multiple of
  // 8 x 64: only in the logits-in mode (router kernel ahead, uneven K split)
  if (n > 256 || m > 512 || d % kBK || (d / kBK + kFrontCta - 1) / kFrontCta > 8) return DESMOE_OK;
  const bool lin_only = m > 256 || (d / kBK) % kFrontCta != 0;
  if (lin_only && (std::getenv("DESMOE_FRONT_ROUTER") || std::getenv("DESMOE_FRONT_TSPLIT")))
    return DESMOE_OK;
  if (cfg->strategy == DESMOE_VANILLA) {
    if (k < 1 || k > m) return fail(DESMOE_EINVAL, "top_k out of range");
  } else {
    int rc = check_des_params(cfg);
    if (rc) return rc;
  }
  if (cfg->activation < 0 || cfg->activation > 2)
    return fail(DESMOE_EINVAL, "unknown gate activation");
  FrontArgs a{};
  size_t smem = 0;
  // router GEMM shape: split-K over the cluster with a partial-logit exchange
  // (small blocks: each CTA streams 1/8 of W_r), or token split (large
  // blocks: no exchange, no token chunking; each CTA streams all of W_r).
  // Measured crossover (tools/sweep.py): token split wins from N*M = 32768.
  int tsplit = static_cast<long>(n) * m >= 32768 ? 2 : 0;
  // the router GEMM runs ahead in its own clusters (router_cluster_kernel:
  // one 8-CTA cluster per 32 tokens x 128 experts) and the front reads the
  // logits, for every block. (Round 2 first used it for N > 32 or M > 128
  // only; once the front's i-cache prewarm ran under the router kernel, the
  // small blocks gained too — same-box A/B: C2 N = 8 / 16 / 32 DES-Vote
  // -2.0 us, vanilla -1 to -2 us, C4 N = 32 -1.3 us, none slower.)
  // DESMOE_FRONT_ROUTER=0 keeps the GEMM in the front (split-K / token split).
  bool router = true;
  if (const char* rv = std::getenv("DESMOE_FRONT_ROUTER")) router = std::atoi(rv) != 0;
  if ((router || lin_only) && (d / kBK + kFrontCta - 1) / kFrontCta <= 8) tsplit = 3;
  if (const char* ts = std::getenv("DESMOE_FRONT_TSPLIT")) tsplit = std::atoi(ts);
  if (!front_plan(n, m, k, d, &a, &smem, tsplit) && !front_plan(n, m, k, d, &a, &smem, 0))
    return DESMOE_OK;
  if (std::getenv("DESMOE_DEBUG_PLAN"))
    std::fprintf(stderr, "front plan n=%d m=%d: chunk=%d stages=%d b_rows=%d vote_rows=%d smem=%zu\n",
                 n, m, a.chunk, a.stages, a.b_rows, a.vote_rows, smem);
  if (x != c->x_map_ptr || n != c->x_map_n || d != c->x_map_d) {
    int rc = make_box_maps(&c->x_maps, x, n, d);
    if (rc) return rc;
    c->x_map_ptr = x;
    c->x_map_n = n;
    c->x_map_d = d;
  }
  if (w_r != c->wr_map_ptr || m != c->wr_map_m || d != c->wr_map_d) {
    int rc = make_map(&c->wr_map, w_r, m, d, kBM);
    if (rc) return rc;
    c->wr_map_ptr = w_r;
    c->wr_map_m = m;
    c->wr_map_d = d;
  }
  a.n = n;
  a.m = m;
  a.k = k;
  a.act = cfg->activation;
  a.strategy = cfg->strategy;
  a.seq_k = cfg->seq_k;
  a.m_core = desmoe_vote_budget(cfg->vote_beta, m);
  a.raw = cfg->vote_source == DESMOE_VOTE_RAW_LOGITS;
  a.route_idx = c->route_idx;
  a.route_gate = c->route_gate;
  a.route_cnt = c->route_cnt;
  a.members = c->members;
  a.n_members = c->n_members;
  a.logits_out = c->logits32;
  a.seq = ex->ep_state;
  a.pub = ex->pub;
  a.route_words = ex->route_words;
  a.route_done = ex->route_done;
  a.err = c->err;
  a.trace = c->trace;
  a.trace_cap = c->trace_cap;
  if (const char* ff = std::getenv("DESMOE_FRONT_FLAGS")) a.flags = std::atoi(ff);
  if (a.tsplit == 3) {
    RouterArgs ra{};
    ra.n = n;
    ra.m = m;
    ra.d = d;
    ra.tc = kRouterTc;
    ra.mtiles = (m + kBM - 1) / kBM;
    ra.kb_cta = (d / kBK + kFrontCta - 1) / kFrontCta;  // most K blocks of a CTA (smem)
    ra.b_rows = b_rows_for(n < kRouterTc ? n : kRouterTc);
    int bi = 0;
    while ((16 << bi) < ra.b_rows) ++bi;
    ra.box_index = bi;
    ra.logits = c->logits32;
    cudaError_t re = launch_router_cluster(c->wr_map, c->x_maps, ra, st);
    if (re != cudaSuccess)
      return fail(DESMOE_ECUDA, std::string("router kernel: ") + cudaGetErrorString(re));
    c->launches += 1;
    a.logits_in = c->logits32;
    a.logits_out = nullptr;  // the router kernel wrote them
  }
  cudaError_t e = launch_front(c->wr_map, c->x_maps, a, smem, st);
  if (e != cudaSuccess) return fail(DESMOE_ECUDA, std::string("front kernel: ") + cudaGetErrorString(e));
  c->launches += 1;
  *used = true;
  return DESMOE_OK;
}

int layer_forward_impl(desmoe_ctx* c, const desmoe_experts* ex, const void* w_r, const void* x,
                       int n, const desmoe_route_cfg* cfg, float* y, int* stats,
                       cudaStream_t st, __nv_bfloat16* y_bf16 = nullptr, bool reset = true,
                       bool residual = false, bool ingress = false) {
  int rc;
  if (reset) {
    c->n_ev = 0;
    c->launches = 0;
  }
  // every FFN shape check before anything is launched: the front publishes
  // tagged words the next call's FFN would accept if no FFN + combine (which
  // advances the call sequence) ran behind it
  FfnPlan plan;
  rc = ffn_plan(ex, n, cfg->top_k, &plan);
  if (rc) return rc;
  if (ingress) {
    // host-buffer entry: the caller's pinned x comes in through its device
    // mapping (address in a host-mapped word), inside the graph
    const int n16 = n * ex->d / 8;
    const auto* word = reinterpret_cast<const unsigned long long*>(c->host_tail_dev + 8);
    auto* dst = static_cast<uint4*>(const_cast<void*>(x));
    const char* iv = std::getenv("DESMOE_INGRESS");
    if (iv && std::strcmp(iv, "ld") == 0) {
      x_ingress_kernel<<<std::max(1, (n16 + 1023) / 1024), 256, 0, st>>>(word, dst, n16);
    } else {
      int chunk = 32768;  // measured: 16 KB 11.0 us, >= 32 KB 8.1-8.5 us for 128 KB
      if (const char* cv = std::getenv("DESMOE_INGRESS_CHUNK"))
        chunk = std::max(256, std::min(kIngressChunk, std::atoi(cv))) & ~15;
      const size_t bytes = static_cast<size_t>(n16) * 16;
      if (static_cast<size_t>(chunk) > bytes) chunk = static_cast<int>(bytes);
      const int grid = static_cast<int>((bytes + chunk - 1) / chunk);
      x_ingress_bulk_kernel<<<grid, 32, chunk, st>>>(word, dst, n16, chunk);
    }
    DESMOE_LAUNCHED();
    c->launches += 1;
  }
  mark(c, st);
  bool zeroed = false;
  rc = front_impl(c, ex, x, w_r, n, cfg, st, &zeroed);
  if (rc) return rc;
  const bool front_used = zeroed;
  if (!zeroed) {
    // shapes outside the cluster kernel's envelope: split-K router + routing kernels
    int splits = 0;
    rc = router_impl(c, x, w_r, n, cfg->experts, ex->d, &splits, st);
    if (rc) return rc;
    c->launches += 1;
    mark(c, st);
    rc = route_impl<float>(c, nullptr, c->partials, splits, n, cfg, nullptr, st, ex->counters,
                           ffn_counter_words(ex->m, ex->f), &zeroed);
    if (rc) return rc;
    c->launches += zeroed ? 1 : (cfg->strategy == DESMOE_VANILLA ? 1 : 3);
  }
  mark(c, st);
  // dense FFN mode (every streamed expert x every token) for the DES
  // coresets; vanilla's union (~57 of 64 experts at C2) writes fewer rows in
  // the routed mode from N = 32 on. Measured (C2): vanilla N=32 131.6 routed
  // vs 133.0 dense, N=64 149.5 vs 153.6, but N=8 96.3 dense vs 100.3 routed;
  // DES-Seq k=2 at N=32 87.5 dense vs 89.4 routed.
  // Expert parallel (world > 1): always routed. Every output row a rank
  // computes is pushed to all G ranks over NVLink, and dense mode's U_own x N
  // rows (every owned expert x every token) would be ~U/K times the N x K
  // routed rows the combine actually reads: at C2 (U = 25, K = 8) 3.1x the
  // bytes per rank (DESMOE_EP_DENSE=1 restores dense for A/B).
  const bool prefer_dense = (cfg->strategy != DESMOE_VANILLA || n <= 16 ||
                             std::getenv("DESMOE_ALWAYS_DENSE")) &&
                            (ex->world <= 1 || std::getenv("DESMOE_EP_DENSE"));
  rc = ffn_impl(c, ex, x, n, cfg->top_k, c->route_idx, c->route_gate, c->route_cnt, y,
                cfg->strategy == DESMOE_VANILLA ? nullptr : c->n_members, stats, st, zeroed,
                front_used, y_bf16, residual ? x : nullptr, prefer_dense, true,
                stats != nullptr && stats == c->host_tail_dev);
  if (rc) return rc;
  return DESMOE_OK;
}

// Same launch sequence (kernels, grids, cluster shapes): only the buffers
// may differ, so an instantiated graph can be updated in place.
bool same_shape(const desmoe_ctx::Key& a, const desmoe_ctx::Key& b) {
  return a.ex == b.ex && a.ex_uid == b.ex_uid && a.n == b.n && a.prof == b.prof &&
         a.ingress == b.ingress && a.cfg.experts == b.cfg.experts &&
         a.cfg.top_k == b.cfg.top_k && a.cfg.activation == b.cfg.activation &&
         a.cfg.strategy == b.cfg.strategy && a.cfg.seq_k == b.cfg.seq_k &&
         a.cfg.vote_beta == b.cfg.vote_beta && a.cfg.vote_source == b.cfg.vote_source;
}

bool same_key(const desmoe_ctx::Key& a, const desmoe_ctx::Key& b) {
  return a.ex == b.ex && a.ex_uid == b.ex_uid && a.wr == b.wr && a.x == b.x && a.n == b.n &&
         a.y == b.y &&
         a.stats == b.stats && a.prof == b.prof && a.ingress == b.ingress &&
         a.cfg.experts == b.cfg.experts &&
         a.cfg.top_k == b.cfg.top_k && a.cfg.activation == b.cfg.activation &&
         a.cfg.strategy == b.cfg.strategy && a.cfg.seq_k == b.cfg.seq_k &&
         a.cfg.vote_beta == b.cfg.vote_beta && a.cfg.vote_source == b.cfg.vote_source;
}

}  // namespace

extern "C" {

}  // extern "C"

namespace {

// The layer's launch sequence as ONE CUDA graph, captured the first time a
// (experts, router, x, n, cfg, y, stats, ingress) tuple is seen and replayed
// afterwards (eager launches when graphs are off).
int layer_graph_launch(desmoe_ctx* c, const desmoe_experts* ex, const void* w_r, const void* x,
                       int n, const desmoe_route_cfg* cfg, float* y, int* stats, cudaStream_t st,
                       bool ingress) {
  int rc;
  if (!c->use_graphs)
    return layer_forward_impl(c, ex, w_r, x, n, cfg, y, stats, st, nullptr, true, false, ingress);
  desmoe_ctx::Key key{ex, w_r, x, ex->uid, n, *cfg, y, stats, c->profiling, ingress};
  if (!c->gexec || !same_key(key, c->gkey)) {
    // validate + capture the whole launch sequence on the context's capture
    // stream, then instantiate (or update) the executable graph
    cudaGraph_t g = nullptr;
    DESMOE_CUDA(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
    rc = layer_forward_impl(c, ex, w_r, x, n, cfg, y, stats, c->cap_stream, nullptr, true, false,
                            ingress);
    cudaError_t ce = cudaStreamEndCapture(c->cap_stream, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (ce != cudaSuccess) return fail(DESMOE_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    // In-place update only when the launch sequence is the same (new
    // buffers, same shapes / strategy / bank): cudaGraphExecUpdate accepted a
    // graph with the same node count but other kernels (in-envelope front
    // path -> split router/routing path for another shape) and kept the old
    // nodes' cluster launch attributes — the new routing kernels never wrote
    // the route (tests/test_gpu_ffn.py::test_recreated_expert_bank_...).
    bool updated = false;
    if (c->gexec && same_shape(key, c->gkey)) {
      cudaGraphExecUpdateResultInfo info;
      updated = cudaGraphExecUpdate(c->gexec, g, &info) == cudaSuccess;
      if (!updated) cudaGetLastError();
    }
    if (!updated) {
      if (c->gexec) {
        cudaGraphExecDestroy(c->gexec);
        c->gexec = nullptr;
      }
      cudaError_t ie = cudaGraphInstantiate(&c->gexec, g, 0);
      if (ie != cudaSuccess) {
        cudaGraphDestroy(g);
        c->gexec = nullptr;
        return fail(DESMOE_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ie));
      }
    }
    cudaGraphDestroy(g);
    c->gkey = key;
    c->g_n_ev = c->n_ev;
    c->g_launches = c->launches;
  }
  DESMOE_CUDA(cudaGraphLaunch(c->gexec, st));
  c->n_ev = c->g_n_ev;
  c->launches = c->g_launches;
  return DESMOE_OK;
}

// The host-buffer entry's graph: x = the context's device x (filled by the
// in-graph ingress kernel or a preceding copy), stats into host-mapped memory,
// completion published to the host.
int desmoe_layer_forward_host_graph(desmoe_ctx* c, const desmoe_experts* ex, const void* w_r, int n,
                                    const desmoe_route_cfg* cfg, float* y_dev, cudaStream_t st,
                                    bool ingress) {
  return layer_graph_launch(c, ex, w_r, c->x_dev, n, cfg, y_dev, c->host_tail_dev, st, ingress);
}

}  // namespace

extern "C" {

int desmoe_layer_forward(desmoe_ctx* c, const desmoe_experts* ex, const void* w_r, const void* x,
                         int n, const desmoe_route_cfg* cfg, float* y, int* stats, void* stream) {
  if (!c || !ex || !cfg) return fail(DESMOE_EINVAL, "null argument");
  if (cfg->experts != ex->m) return fail(DESMOE_EINVAL, "config experts differ from expert bank");
  int rc = check_block(c, n, cfg->experts);
  if (rc) return rc;
  return layer_graph_launch(c, ex, w_r, x, n, cfg, y, stats, S(stream), false);
}

int desmoe_layer_logits(desmoe_ctx* c, float* logits_dev, int n, int experts, void* stream) {
  int rc = check_block(c, n, experts);
  if (rc) return rc;
  DESMOE_CUDA(cudaMemcpyAsync(logits_dev, c->logits32, sizeof(float) * n * experts,
                              cudaMemcpyDeviceToDevice, S(stream)));
  return DESMOE_OK;
}

int desmoe_layer_route(desmoe_ctx* c, int* route_idx_dev, double* route_gate_dev,
                       int* route_cnt_dev, int* members_dev, int* n_members_dev, int n, int top_k,
                       int experts, void* stream) {
  int rc = check_block(c, n, experts);
  if (rc) return rc;
  if (top_k < 1 || top_k > c->max_k) return fail(DESMOE_EINVAL, "top_k out of range");
  cudaStream_t st = S(stream);
  const size_t nk = static_cast<size_t>(n) * top_k;
  if (route_idx_dev)
    DESMOE_CUDA(cudaMemcpyAsync(route_idx_dev, c->route_idx, nk * 4, cudaMemcpyDeviceToDevice, st));
  if (route_gate_dev)
    DESMOE_CUDA(cudaMemcpyAsync(route_gate_dev, c->route_gate, nk * 8, cudaMemcpyDeviceToDevice, st));
  if (route_cnt_dev)
    DESMOE_CUDA(cudaMemcpyAsync(route_cnt_dev, c->route_cnt, n * 4, cudaMemcpyDeviceToDevice, st));
  if (members_dev)
    DESMOE_CUDA(cudaMemcpyAsync(members_dev, c->members, static_cast<size_t>(experts) * 4,
                                cudaMemcpyDeviceToDevice, st));
  if (n_members_dev)
    DESMOE_CUDA(cudaMemcpyAsync(n_members_dev, c->n_members, 4, cudaMemcpyDeviceToDevice, st));
  return DESMOE_OK;
}

int desmoe_set_graphs(desmoe_ctx* c, int enable) {
  if (!c) return fail(DESMOE_EINVAL, "null context");
  c->use_graphs = enable != 0;
  return DESMOE_OK;
}

int desmoe_set_profiling(desmoe_ctx* c, int enable) {
  if (!c) return fail(DESMOE_EINVAL, "null context");
  c->profiling = enable != 0;
  c->gkey.ex = nullptr;  // force a re-capture
  return DESMOE_OK;
}

int desmoe_get_phase_ms(desmoe_ctx* c, float* ms, int max_phases) {
  if (!c || !ms) return -fail(DESMOE_EINVAL, "null argument");
  if (c->n_ev < 2) return 0;
  cudaError_t e = cudaEventSynchronize(c->ev[c->n_ev - 1]);
  int w = 0;
  for (int i = 0; e == cudaSuccess && i + 1 < c->n_ev && w < max_phases; ++i, ++w)
    e = cudaEventElapsedTime(&ms[w], c->ev[i], c->ev[i + 1]);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return -fail(DESMOE_ECUDA, std::string("phase timing: ") + cudaGetErrorString(e));
  }
  return w;
}

int desmoe_last_launch_count(desmoe_ctx* c) { return c ? c->launches : 0; }

int desmoe_set_trace(desmoe_ctx* c, uint64_t* buf_dev, int capacity) {
  if (!c) return fail(DESMOE_EINVAL, "null context");
  c->trace = capacity > 0 ? buf_dev : nullptr;
  c->trace_cap = capacity > 0 ? capacity : 0;
  c->gkey.ex = nullptr;  // force a re-capture
  return DESMOE_OK;
}

int desmoe_layer_forward_host(desmoe_ctx* c, const desmoe_experts* ex, const void* w_r,
                              const void* x_host, int n, const desmoe_route_cfg* cfg,
                              float* y_host, int* stats_host, void* stream) {
  if (!c || !ex || !cfg || !x_host || !y_host) return fail(DESMOE_EINVAL, "null argument");
  if (cfg->experts != ex->m) return fail(DESMOE_EINVAL, "config experts differ from expert bank");
  int rc = check_block(c, n, cfg->experts);
  if (rc) return rc;
  if (ex->d > c->max_d) return fail(DESMOE_EINVAL, "hidden exceeds context capacity");
  cudaStream_t st = S(stream);
  const size_t xb = static_cast<size_t>(n) * ex->d * 2, yb = static_cast<size_t>(n) * ex->d * 4;
  // pinned (device-mapped) buffers are used in place: x is copied in by the
  // graph's first kernel, y written by the combine straight into host memory
  // over the bus. Pageable buffers go through device copies.
  auto mapped = [](const void* p) -> const void* {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, p) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
        pa.devicePointer)
      return pa.devicePointer;
    cudaGetLastError();
    return nullptr;
  };
  if (x_host != c->last_x_host) {
    c->last_x_host = x_host;
    c->last_x_mapped = mapped(x_host);
  }
  if (y_host != c->last_y_host) {
    c->last_y_host = y_host;
    c->last_y_mapped = static_cast<float*>(const_cast<void*>(mapped(y_host)));
  }
  const bool ingress = c->last_x_mapped && !std::getenv("DESMOE_HOST_MEMCPY");
  float* y_dev = c->last_y_mapped ? c->last_y_mapped : c->y_dev;
  if (ingress) {
    const unsigned long long src = reinterpret_cast<unsigned long long>(c->last_x_mapped);
    std::memcpy(c->host_tail + 8, &src, sizeof(src));
  } else {
    DESMOE_CUDA(cudaMemcpyAsync(c->x_dev, x_host, xb, cudaMemcpyHostToDevice, st));
  }
  const int call = ++c->host_calls;
  reinterpret_cast<volatile int*>(c->host_tail)[5] = call;
  rc = desmoe_layer_forward_host_graph(c, ex, w_r, n, cfg, y_dev, st, ingress);
  if (rc) return rc;
  if (y_dev == c->y_dev)
    DESMOE_CUDA(cudaMemcpyAsync(y_host, c->y_dev, yb, cudaMemcpyDeviceToHost, st));
  if (y_dev != c->y_dev && !std::getenv("DESMOE_HOST_SYNC")) {
    // y, stats and the data-check word are host memory the kernels write; the
    // last combine CTA publishes the call number after a system fence. Spin on
    // it (the earliest the results are observable); the stream is polled now
    // and then so a failed launch reports its error instead of spinning.
    volatile int* done = c->host_tail + 6;
    for (unsigned spins = 1;; ++spins) {
      if (*done == call) break;
      if ((spins & 4095u) == 0) {
        const cudaError_t q = cudaStreamQuery(st);
        if (q == cudaSuccess) {
          if (*done == call) break;
          return fail(DESMOE_ECUDA, "layer finished without publishing its completion");
        }
        if (q != cudaErrorNotReady)
          return fail(DESMOE_ECUDA, std::string("layer: ") + cudaGetErrorString(q));
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    volatile int* fw = c->host_tail + 4;
    const int flag = *fw;
    rc = DESMOE_OK;
    if (flag) {
      *fw = 0;
      rc = flag == 2 ? fail(DESMOE_ECUDA, "expert-parallel exchange timed out (a peer rank stopped)")
                     : fail(DESMOE_EINVAL, "non-finite logit");
    }
  } else {
    rc = desmoe_check(c, stream);  // one synchronisation; stats and flag are host memory
  }
  if (stats_host) std::memcpy(stats_host, const_cast<const int*>(c->host_tail), 4 * sizeof(int));
  return rc;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// exact fp64 gating primitives of the reference API (gating_exact.cu)
// ---------------------------------------------------------------------------
extern "C" {

int desmoe_validate_params(const desmoe_route_cfg* cfg) {
  if (!cfg) return fail(DESMOE_EINVAL, "null config");
  return check_des_params(cfg);
}

int desmoe_select_top(desmoe_ctx* c, const double* values, int m, int k, const int* cand,
                      int n_cand, int* out, void* stream) {
  if (!c || !values || !out) return fail(DESMOE_EINVAL, "null argument");
  if (m < 1 || m > 16384) return fail(DESMOE_EINVAL, "gate count outside [1, 16384]");
  if (cand && (n_cand < 0 || n_cand > m))
    return fail(DESMOE_EINVAL, "candidate count outside [0, gate count]");
  if (k > (cand ? n_cand : m))
    return fail(DESMOE_EINVAL, cand ? "selection count exceeds candidate count"
                                    : "selection count exceeds gate count");
  if (k < 1) return DESMOE_OK;
  const size_t smem = static_cast<size_t>(m) * 9 + 33 * 4 + 16;
  if (smem > 48 * 1024)
    DESMOE_CUDA(cudaFuncSetAttribute(select_top_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
  const int threads = std::min(1024, round_up(std::max(cand ? n_cand : m, 32), 32));
  select_top_kernel<<<1, threads, smem, S(stream)>>>(values, m, k, cand, n_cand, out);
  DESMOE_LAUNCHED();
  return DESMOE_OK;
}

int desmoe_renormalize(desmoe_ctx* c, const double* values, const int* sel, int count,
                       double* out, void* stream) {
  if (!c || !values || !sel || !out) return fail(DESMOE_EINVAL, "null argument");
  if (count < 1) return DESMOE_OK;
  renormalize_kernel<<<1, 256, 0, S(stream)>>>(values, sel, count, out);
  DESMOE_LAUNCHED();
  return DESMOE_OK;
}

int desmoe_moe_forward_f64(desmoe_ctx* c, const double* w, const double* x, int n, int d, int m,
                           int k, const int* route_idx, const double* route_gate,
                           const int* route_cnt, double* y, void* stream) {
  if (!c || !w || !x || !y || !route_idx || !route_gate || !route_cnt)
    return fail(DESMOE_EINVAL, "null argument");
  if (n < 1) return fail(DESMOE_EINVAL, "block_size < 1");
  if (d < 1 || d > 16384) return fail(DESMOE_EINVAL, "hidden_dim outside [1, 16384]");
  if (m < 1 || k < 1) return fail(DESMOE_EINVAL, "experts and top_k must be >= 1");
  const int threads = std::min(256, round_up(d, 32));
  const size_t smem = static_cast<size_t>(d) * sizeof(double);
  if (smem > 48 * 1024)
    DESMOE_CUDA(cudaFuncSetAttribute(linear_expert_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
  dim3 grid((d + threads - 1) / threads, n);
  linear_expert_kernel<<<grid, threads, smem, S(stream)>>>(w, x, d, k, route_idx, route_gate,
                                                           route_cnt, y);
  DESMOE_LAUNCHED();
  return DESMOE_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// expert parallelism (EP): buffers and peer wiring
// ---------------------------------------------------------------------------
extern "C" {

int desmoe_ep_local_buffers(desmoe_experts* ex, void** slot_buf, size_t* slot_bytes,
                            void** flag_buf, size_t* flag_bytes) {
  if (!ex || !slot_buf || !slot_bytes || !flag_buf || !flag_bytes)
    return fail(DESMOE_EINVAL, "null argument");
  desmoe_ctx* c = ex->ctx;
  const size_t sb = 2 * static_cast<size_t>(c->max_n) * c->max_k * ex->d * sizeof(float);
  if (!ex->ep_slot) {
    // separate allocations, so each is the base of its own IPC handle
    DESMOE_CUDA(cudaMalloc(&ex->ep_slot, sb));
    DESMOE_CUDA(cudaMalloc(&ex->ep_flag, 256));
    DESMOE_CUDA(cudaMemset(ex->ep_flag, 0, 256));
    DESMOE_CUDA(cudaDeviceSynchronize());
  }
  *slot_buf = ex->ep_slot;
  *slot_bytes = sb;
  *flag_buf = ex->ep_flag;
  *flag_bytes = 256;
  return DESMOE_OK;
}

int desmoe_ep_connect(desmoe_experts* ex, int world, int rank, void* const* peer_slot_bufs,
                      void* const* peer_flag_bufs) {
  if (!ex) return fail(DESMOE_EINVAL, "null argument");
  if (world < 1 || world > kMaxWorld) return fail(DESMOE_EINVAL, "world outside [1, 8]");
  if (rank < 0 || rank >= world) return fail(DESMOE_EINVAL, "rank outside [0, world)");
  if (world > 1) {
    if (!peer_slot_bufs || !peer_flag_bufs) return fail(DESMOE_EINVAL, "missing peer buffers");
    if (!ex->ep_slot) return fail(DESMOE_EINVAL, "call desmoe_ep_local_buffers first");
    for (int r = 0; r < world; ++r)
      if (!peer_slot_bufs[r] || !peer_flag_bufs[r]) return fail(DESMOE_EINVAL, "null peer buffer");
    if (peer_slot_bufs[rank] != ex->ep_slot || peer_flag_bufs[rank] != ex->ep_flag)
      return fail(DESMOE_EINVAL, "own rank's entry must be the local buffers");
    for (int r = 0; r < world; ++r) {
      ex->peer_slot[r] = static_cast<float*>(peer_slot_bufs[r]);
      ex->peer_flag[r] = static_cast<unsigned long long*>(peer_flag_bufs[r]);
    }
  }
  ex->world = world;
  ex->uid = next_uid();  // graphs captured before this (re)connection are stale
  ex->rank = rank;
  ex->ctx->gkey.ex = nullptr;  // force a re-capture of the layer graph
  return DESMOE_OK;
}

int desmoe_ep_export(desmoe_experts* ex, void* handle_out) {
  if (!ex || !handle_out) return fail(DESMOE_EINVAL, "null argument");
  void *slot, *flag;
  size_t sb, fb;
  int rc = desmoe_ep_local_buffers(ex, &slot, &sb, &flag, &fb);
  if (rc) return rc;
  static_assert(sizeof(cudaIpcMemHandle_t) * 2 <= DESMOE_EP_HANDLE_BYTES, "handle size");
  cudaIpcMemHandle_t h[2];
  DESMOE_CUDA(cudaIpcGetMemHandle(&h[0], slot));
  DESMOE_CUDA(cudaIpcGetMemHandle(&h[1], flag));
  std::memset(handle_out, 0, DESMOE_EP_HANDLE_BYTES);
  std::memcpy(handle_out, h, sizeof(h));
  return DESMOE_OK;
}

int desmoe_ep_import(desmoe_experts* ex, int world, int rank, const void* handles) {
  if (!ex || !handles) return fail(DESMOE_EINVAL, "null argument");
  if (world < 1 || world > kMaxWorld) return fail(DESMOE_EINVAL, "world outside [1, 8]");
  if (rank < 0 || rank >= world) return fail(DESMOE_EINVAL, "rank outside [0, world)");
  void *slot, *flag;
  size_t sb, fb;
  int rc = desmoe_ep_local_buffers(ex, &slot, &sb, &flag, &fb);
  if (rc) return rc;
  void* slots[kMaxWorld] = {};
  void* flags[kMaxWorld] = {};
  const unsigned char* hb = static_cast<const unsigned char*>(handles);
  for (int r = 0; r < world; ++r) {
    if (r == rank) {
      slots[r] = slot;
      flags[r] = flag;
      continue;
    }
    cudaIpcMemHandle_t h[2];
    std::memcpy(h, hb + static_cast<size_t>(r) * DESMOE_EP_HANDLE_BYTES, sizeof(h));
    for (int b = 0; b < 2; ++b) {
      void* p = nullptr;
      DESMOE_CUDA(cudaIpcOpenMemHandle(&p, h[b], cudaIpcMemLazyEnablePeerAccess));
      ex->ipc_mapped[2 * r + b] = p;
      (b == 0 ? slots : flags)[r] = p;
    }
  }
  return desmoe_ep_connect(ex, world, rank, slots, flags);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// layer stacks: one block through `layers` DES MoE layers in one CUDA graph
// ---------------------------------------------------------------------------
extern "C" {

int desmoe_stack_forward(desmoe_ctx* c, desmoe_experts* const* experts, const void* const* w_router,
                         int layers, const void* x, int n, const desmoe_route_cfg* cfg, float* y,
                         int* stats, int residual, void* stream) {
  if (!c || !experts || !w_router || !x || !y || !cfg) return fail(DESMOE_EINVAL, "null argument");
  if (layers < 1) return fail(DESMOE_EINVAL, "layers < 1");
  const int d = experts[0]->d;
  for (int l = 0; l < layers; ++l) {
    if (!experts[l] || !w_router[l]) return fail(DESMOE_EINVAL, "null layer");
    if (experts[l]->d != d || experts[l]->m != cfg->experts)
      return fail(DESMOE_EINVAL, "layers differ in hidden size or expert count");
  }
  int rc = check_block(c, n, cfg->experts);
  if (rc) return rc;
  if (d > c->max_d) return fail(DESMOE_EINVAL, "hidden exceeds context capacity");
  for (auto*& b : c->stack_buf)
    if (!b) DESMOE_CUDA(cudaMalloc(&b, static_cast<size_t>(c->max_n) * c->max_d * 2));
  cudaStream_t st = S(stream);
  auto run = [&](cudaStream_t s) -> int {
    c->n_ev = 0;
    c->launches = 0;
    const void* xin = x;
    for (int l = 0; l < layers; ++l) {
      const bool last = l == layers - 1;
      __nv_bfloat16* out = last ? nullptr : c->stack_buf[l & 1];
      int r = layer_forward_impl(c, experts[l], w_router[l], xin, n, cfg, y,
                                 stats ? stats + 4 * l : nullptr, s, out, false, residual != 0);
      if (r) return r;
      xin = out;
    }
    return DESMOE_OK;
  };
  if (!c->use_graphs) return run(st);
  std::vector<const void*> key;
  key.reserve(2 * layers + 8);
  for (int l = 0; l < layers; ++l) {
    key.push_back(experts[l]);
    key.push_back(reinterpret_cast<const void*>(static_cast<uintptr_t>(experts[l]->uid)));
    key.push_back(w_router[l]);
  }
  key.push_back(x);
  key.push_back(y);
  key.push_back(stats);
  key.push_back(reinterpret_cast<const void*>(static_cast<intptr_t>(n)));
  const int cfgw[6] = {cfg->experts, cfg->top_k, cfg->activation, cfg->strategy, cfg->seq_k,
                       cfg->vote_source};
  for (int v : cfgw) key.push_back(reinterpret_cast<const void*>(static_cast<intptr_t>(v)));
  long long beta_bits;
  std::memcpy(&beta_bits, &cfg->vote_beta, 8);
  key.push_back(reinterpret_cast<const void*>(static_cast<intptr_t>(beta_bits)));
  key.push_back(reinterpret_cast<const void*>(static_cast<intptr_t>(c->profiling)));
  key.push_back(reinterpret_cast<const void*>(static_cast<intptr_t>(residual)));
  if (!c->sgexec || key != c->skey) {
    cudaGraph_t g = nullptr;
    DESMOE_CUDA(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
    rc = run(c->cap_stream);
    cudaError_t ce = cudaStreamEndCapture(c->cap_stream, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (ce != cudaSuccess) return fail(DESMOE_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    if (c->sgexec) cudaGraphExecDestroy(c->sgexec);
    c->sgexec = nullptr;
    cudaError_t ie = cudaGraphInstantiate(&c->sgexec, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) return fail(DESMOE_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ie));
    c->skey = key;
  }
  DESMOE_CUDA(cudaGraphLaunch(c->sgexec, st));
  return DESMOE_OK;
}

}  // extern "C"
