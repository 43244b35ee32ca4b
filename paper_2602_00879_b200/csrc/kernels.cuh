// Kernel argument blocks and kernel declarations shared by the C-ABI layer
// (capi.cu) and the kernel translation units.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace desmoe {

template <typename T>
struct GateTopkArgs {
  const T* logits;        // [n x m] (splits == 0)
  const float* partials;  // [splits x n x m_pad] router split-K partials (splits > 0)
  float* logits_out;      // optional fp32 logits written when reducing partials
  int splits, m_pad;
  int n, m, k, kmax, act, mode;  // mode 0 vanilla route, 1 DES top-K list
  double* probs;                 // [n x m] activated gates (optional in mode 0)
  int* topk_idx;                 // [n x k] rank order (mode 1)
  int* route_idx;                // [n x kmax] (mode 0)
  double* route_gate;
  float* route_gate32;
  int* route_cnt;
  int* err;
};

template <typename T>
struct FusedRouteArgs {
  const T* logits;        // [n x m] (splits == 0)
  const float* partials;  // [splits x n x m] router split-K partials (splits > 0)
  int splits;
  float* logits_out;      // fp32 logits written when reducing partials
  const T* raw_logits;    // raw-logit votes source
  int n, m, k, act, strategy, seq_k, m_core, raw;
  int* route_idx;      // [n x k]
  double* route_gate;  // [n x k]
  int* route_cnt;      // [n]
  int* members;        // [m] (optional)
  int* n_members;      // [1] (optional)
  uint8_t* member_flag;
  double* votes;       // [m] (optional)
  double* probs;       // [n x m] (optional)
  int* zero;           // words to zero for the next kernel (optional)
  int zero_words;
  int* err;
};

constexpr int kFusedRouteSmem = 200 * 1024;
constexpr int kMaxSplits = 32;  // router split-K factor bound
size_t fused_route_smem(int n, int m, int k);
template <typename T>
cudaError_t launch_fused_route(const FusedRouteArgs<T>& a, cudaStream_t st);
cudaError_t set_fused_route_smem_limit(int bytes);

// ---- front: router GEMM + routing in one thread-block cluster (front.cu) ----
constexpr int kFrontCta = 8;        // cluster size (portable maximum)
constexpr int kFrontThreads = 512;
constexpr int kDistRankMin = 64;  // DES-Vote pools above this size rank across the cluster
constexpr int kFrontSmemLimit = 223 * 1024;  // dynamic; + 4 KB static (exp table) = 227 KB

struct FrontArgs {
  int n, m, k, act, strategy, seq_k, m_core, raw;
  int b_rows, box_index, kb_per_cta, stages, tmem_cols;
  int chunk, own_max;  // token chunk of the split-K GEMM; own tokens per CTA bound
  int tsplit;          // 1/2: token-split router GEMM; 3: logits in (router_cluster_kernel)
  int vote_rows;       // token rows of the shared-memory vote matrix chunk
  int* route_idx;      // [n x k]
  double* route_gate;  // [n x k]
  int* route_cnt;      // [n]
  int* members;        // [m] (written by cluster rank 0)
  int* n_members;      // [1]
  double* votes;       // [m] optional
  float* logits_out;   // [n x m] optional fp32 logits
  const float* logits_in;  // [n x m] fp32 logits (tsplit == 3: router_cluster_kernel ran ahead)
  int* err;
  uint64_t* trace;     // optional timeline (events 40+)
  int trace_cap;
  // early hand-off to the expert-FFN kernel (no grid-completion wait): the
  // call sequence number, the published expert list and tagged route words
  const int* seq;          // [1] bumped by the combine kernel after every call
  uint32_t* pub;           // [1 + m] {tag | count}, {tag | expert} ...
  uint64_t* route_words;   // [n x k] {gate f32 | tag | expert}, expert kPadExpert = none
  uint32_t* route_done;    // [kFrontCta] tag, stored (release) once a CTA's route words are out
  int flags;               // experiments (DESMOE_FRONT_FLAGS)
};

// Router GEMM ahead of the front kernel for large blocks (front.cu,
// router_cluster_kernel): one 8-CTA cluster per (token tile, 128-expert tile),
// split-K over the cluster, partials summed by their owner CTA in fixed CTA
// order; logits [n x m] fp32 to global memory, read by the front in its
// logits-in mode (FrontArgs::tsplit == 3).
struct RouterArgs {
  int n, m, d;
  int tc;        // tokens per cluster
  int mtiles;    // 128-expert tiles (clusters per token tile)
  int kb_cta;    // 64-wide K blocks per CTA (d / 64 / 8)
  int b_rows;    // X box rows (>= tc)
  int box_index;
  float* logits;  // [n x m]
};
constexpr int kRouterTc = 32;  // tokens per router cluster

// Tagged hand-off words (front -> FFN). A word is valid for the current call
// when its 22-bit tag equals the call sequence number (mod 2^22); every word
// the FFN polls is rewritten by every call, so no flag, fence or reset is
// needed: the front's stores and the FFN's polling loads meet in L2.
constexpr uint32_t kTagBits = 22;
constexpr uint32_t kTagMask = (1u << kTagBits) - 1u;
constexpr int kPadExpert = 1023;
__host__ __device__ inline uint32_t hand_tag(int seq) {
  return static_cast<uint32_t>(seq) & kTagMask;
}
__host__ __device__ inline uint32_t pub_word(uint32_t tag, int v) {
  return (tag << 10) | static_cast<uint32_t>(v & 1023);
}
__host__ __device__ inline uint64_t route_word(uint32_t tag, int expert, float gate) {
  uint32_t g;
#ifdef __CUDA_ARCH__
  g = __float_as_uint(gate);
#else
  __builtin_memcpy(&g, &gate, 4);
#endif
  return (static_cast<uint64_t>(g) << 32) | (static_cast<uint64_t>(tag) << 10) |
         static_cast<uint64_t>(expert & 1023);
}

// Fills the plan fields of `a` (chunk, stages, boxes, TMEM) and the dynamic
// shared memory; false if the shape is outside the cluster kernel's envelope.
bool front_plan(int n, int m, int k, int d, FrontArgs* a, size_t* smem, int tsplit = 0);

struct CoresetArgs {
  int n, m, k, strategy, seq_k, m_core, raw;
  const int* topk_idx;  // [n x k] rank order
  const double* probs;  // [n x m]
  const double* logits64;
  const float* logits32;
  double* votes;         // [m] (optional)
  int* members;          // [m]
  int* n_members;        // [1]
  uint8_t* member_flag;  // [m]
};

struct RerouteArgs {
  int n, m, k;
  const double* probs;
  const int* topk_idx;  // optional fast path
  const uint8_t* member_flag;
  const int* n_members;
  int* route_idx;
  double* route_gate;
  float* route_gate32;
  int* route_cnt;
};

struct PermuteArgs {
  int n, m, k;
  const int* route_idx;
  const int* route_cnt;
  const double* route_gate;
  int* expert_count;   // [m]
  int* expert_offset;  // [m]
  int* slot_of;        // [n x k]
  int* slot_token;     // [n x k]
  float* slot_gate;    // [n x k]
  int* active;         // [m]
  int* n_active;       // [1]
  int* total;          // [1]
  int* zero;           // words zeroed for the FFN kernel's counters
  int zero_words;
};

// Host-side launcher of the K2a template (defined next to the kernel so the
// instantiations live in one translation unit).
template <typename T>
cudaError_t launch_gate_topk_kernel(const GateTopkArgs<T>& a, int grid, int block, size_t smem,
                                    cudaStream_t st);
__global__ void coreset_kernel(CoresetArgs a);
cudaError_t set_kernel_smem_limits();
__global__ void constrained_route_kernel(RerouteArgs a);
__global__ void set_members_kernel(const int* members, int nm, int m, uint8_t* flag,
                                   int* n_members);
__global__ void permute_kernel(PermuteArgs a);

// ---- tcgen05 swap-AB tiles (router GEMM / expert FFN) ----------------------
constexpr int kBM = 128;             // weight rows per tile (MMA M)
constexpr int kBK = 64;              // K elements per pipeline stage (128 B rows)
constexpr int kATile = kBM * kBK * 2;  // 16 KB
constexpr int kMaxBoxes = 5;         // activation box heights 16, 32, 64, 128, 256

struct BoxMaps {
  CUtensorMap map[kMaxBoxes];  // same tensor, box heights 16 << i
};

struct TileArgs {  // router GEMM (tile_gemm.cu)
  int n_tok;           // tokens in the block (rows of x)
  int kb_total;        // K blocks of the full contraction
  int splits;          // split-K factor
  int n_units_static;  // expert tiles * splits
  int stages;
  int b_rows;          // smem rows reserved for the activation tile
  int m_pad;           // experts (row stride of the partials)
  float* y_out;        // partials [split][token][expert]
};

constexpr int kMaxWorld = 8;  // expert-parallel ranks (one 8-GPU NVSwitch box)
constexpr int kDenseMaxTokens = 64;  // dense FFN mode up to this block size

struct FfnArgs {
  int mode;  // 0 = SwiGLU (phase A + B), 1 = linear expert (phase B on x)
  int n_tok, top_k, m, d, f, b_rows, stages;
  const int* route_idx;      // [n x k]
  const int* route_cnt;      // [n]
  const double* route_gate;  // [n x k]
  const __nv_bfloat16* x;    // [n x d]
  __nv_bfloat16* x_perm;     // [n*k x d]
  __nv_bfloat16* h_perm;     // [n*k x f]
  float* y_slot;             // [n*k x d]
  int* slot_of;              // [n x k] written by CTA 0 for the combine kernel
  int* counters;             // zeroed: sched, x_ready, h_ready[m][f/64]
  int* stats;                // optional [4]: U, coreset size, slots, 0
  const int* n_members;      // optional coreset size
  uint64_t* trace;           // optional timeline buffer ([0] cursor, then pairs)
  int trace_cap;
  // expert parallelism (world > 1): this rank owns experts [expert_lo,
  // expert_hi); packed weights hold only those. Phase-B epilogues push every
  // gate-scaled slot row into all ranks' slot buffers (peer_slot[r], NVLink
  // peer memory; parity (epoch & 1) selects one of two halves of
  // slot_stride floats) and each CTA signals every rank's arrival counter at
  // exit (system-scope release).
  int expert_lo, expert_hi;
  int world;
  float* peer_slot[kMaxWorld];
  unsigned long long* peer_flag[kMaxWorld];
  size_t slot_stride;        // floats per parity half
  const int* epoch;          // device call sequence number (= the hand-off seq)
  // early mode (behind the front kernel): the weight producer starts on the
  // published expert list and the prologue polls the tagged route words;
  // otherwise (standalone FFN) the route arrays after griddepcontrol.wait
  int early;
  const uint32_t* pub;
  const uint64_t* route_words;
  const uint32_t* route_done;  // [kFrontCta] the front CTAs' route-complete tags
  // host-buffer entry, dense mode, one rank: [m][d / 128] the call's tag,
  // stored (release) once the phase-B unit (expert, d tile) has stored its
  // rows, and the call's tag once the unit queue ran dry; the combine
  // streams on these (its y rows cross the bus while the last units finish)
  uint32_t* b_done;
  uint32_t* b_drained;
  const void* wa_base;       // packed gate/up tiles (L2 prefetch of the first unit)
  const void* wc_base;       // packed W_d / W_lin tiles
  int flags;                 // experiments: 1 = no L2 prefetch of the first unit
  int gather_ctas;           // CTAs that gather x rows (and the x_ready target)
  int dense;                 // every published expert x every token (small blocks)
  int kb;                    // 64-wide K blocks per ring stage: 4 when d, F allow, else 2
  int pair_b;                // dense mode: phase-B units of two d tiles sharing one H stream
  int split_b;               // the queue's last phase-B pairs run as single-tile units
  int pair_a, split_a;       // the same for phase A (two F tiles sharing one X stream)
};

// Ordered combine arguments (combine_slots_kernel).
struct CombineArgs {
  const float* y_slot;       // slot rows (world == 1) or the parity halves (EP)
  const int* slot_of;        // [n x k]
  const int* route_cnt;      // [n]
  int n, k, d;
  float* y;                  // [n x d]
  // EP: wait until flag >= (epoch + 1) * arrivals, read half (epoch & 1); the
  // last CTA to finish advances the epoch
  int world;
  const unsigned long long* flag;
  unsigned long long arrivals;  // world * FFN grid
  int* epoch;                // call sequence number: bumped by the last CTA
  int* done_ctas;
  size_t slot_stride;
  int* err;                  // set to 2 on an exchange timeout
  int* zero;                 // FFN counters, zeroed for the next call
  int zero_words;
  // dense mode (combine_dense_kernel)
  const uint64_t* route_words;  // [n x k] the front's tagged route (read before the FFN ends)
  const int* route_idx;      // [n x k]
  const double* route_gate;  // [n x k]
  const uint32_t* pub;       // published list (tagged words)
  int m, expert_lo, expert_hi;
  int* stats;                // optional [4]
  const uint32_t* b_done;    // FfnArgs::b_done (nullptr: wait for the FFN grid)
  const uint32_t* b_drained;
  int tiles_b;               // d / 128
  __nv_bfloat16* y_bf16;     // optional: write bf16 here instead of fp32 y (layer stacks)
  const __nv_bfloat16* resid;  // optional residual stream added before the store (stacks)
  uint64_t* trace;           // optional timeline (events 80 start, 81 end; CTA 0)
  int trace_cap;
  // host-buffer entry (desmoe_layer_forward_host): after every y row is
  // visible system-wide the last CTA copies *host_call (the host's call
  // number, host-mapped) into *host_done (host-mapped), which the host spins on
  const int* host_call;
  int* host_done;
};

// Host-buffer entry's x ingress, the first node of the layer graph: copies
// the caller's pinned x (its device-mapped address is read from the
// host-mapped word *src_word, written by the host before the launch, so the
// graph never changes with the caller's buffer) into the context's device x.
__global__ void x_ingress_kernel(const unsigned long long* src_word, uint4* dst, int n16);
constexpr int kIngressChunk = 128 * 1024;  // max bytes per ingress CTA (one bulk request)
__global__ void x_ingress_bulk_kernel(const unsigned long long* src_word, uint4* dst, int n16,
                                      int chunk);

// Comparison policies (baselines.cu): method 0 = top-k reduce, 1 = NAEE,
// 2 = MC-MoE (score 0 = max gate, 1 = -entropy).
template <typename T>
struct BaselineArgs {
  const T* logits;     // [n x m]
  int n, m, k, act;
  int method, k_reduced, score, important;
  double beta;
  double* probs;       // [n x m] workspace (activated rows)
  int* route_idx;      // [n x k]
  double* route_gate;  // [n x k]
  int* route_cnt;      // [n]
  int* err;            // bit 0: non-finite logit
};
template <typename T>
__global__ void baseline_route_kernel(BaselineArgs<T> a);

inline int ffn_counter_words(int m, int f) { return 2 + m * (f / 64); }

// KB = 64-wide K blocks per ring stage (2 or 4; compile-time so the stage
// loops unroll — a runtime count measured 2-3 us slower per block)
template <int KB>
__global__ void ffn_persistent_kernel(const __grid_constant__ CUtensorMap w_a,
                                      const __grid_constant__ CUtensorMap w_b,
                                      const __grid_constant__ CUtensorMap w_c,
                                      const __grid_constant__ BoxMaps xp_maps,
                                      const __grid_constant__ BoxMaps h_maps, FfnArgs a);
__global__ void pack_weights_kernel(const uint4* __restrict__ src, const uint4* __restrict__ src2,
                                    uint4* __restrict__ out, int experts, int rows_per_expert,
                                    int cols, int stacked);
__global__ void combine_slots_kernel(CombineArgs a);
__global__ void combine_dense_kernel(CombineArgs a);
__global__ void ep_wait_kernel(CombineArgs a);

cudaError_t launch_front(const CUtensorMap& wr_map, const BoxMaps& x_maps, const FrontArgs& a,
                         size_t smem, cudaStream_t st);
cudaError_t set_front_smem_limit();
cudaError_t launch_router_cluster(const CUtensorMap& wr_map, const BoxMaps& x_maps,
                                  const RouterArgs& a, cudaStream_t st);

// ---- exact fp64 gating primitives (gating_exact.cu) ----
__global__ void select_top_kernel(const double* __restrict__ values, int m, int k,
                                  const int* __restrict__ cand, int n_cand, int* __restrict__ out);
__global__ void renormalize_kernel(const double* __restrict__ values,
                                   const int* __restrict__ sel, int count,
                                   double* __restrict__ out);
__global__ void linear_expert_kernel(const double* __restrict__ w, const double* __restrict__ x,
                                     int d, int k, const int* __restrict__ route_idx,
                                     const double* __restrict__ route_gate,
                                     const int* __restrict__ route_cnt, double* __restrict__ y);

__global__ void tile_gemm_kernel(const __grid_constant__ CUtensorMap wa,
                                 const __grid_constant__ CUtensorMap wb,
                                 const __grid_constant__ BoxMaps acts, TileArgs a);

}  // namespace desmoe
