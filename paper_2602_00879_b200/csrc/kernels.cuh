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
__global__ void constrained_route_kernel(RerouteArgs a);
__global__ void set_members_kernel(const int* members, int nm, int m, uint8_t* flag,
                                   int* n_members);
__global__ void permute_kernel(PermuteArgs a);
__global__ void gather_rows_kernel(const uint4* __restrict__ x, const int* __restrict__ slot_token,
                                   const int* __restrict__ total, uint4* __restrict__ xp,
                                   int row_vec);
__global__ void combine_kernel(const float* __restrict__ y_slot, const int* __restrict__ slot_of,
                               const int* __restrict__ route_cnt, int n, int k, int d,
                               float* __restrict__ y);

// ---- tcgen05 swap-AB tile GEMM (router / expert FFN) -----------------------
constexpr int kBM = 128;             // weight rows per tile (MMA M)
constexpr int kBK = 64;              // K elements per pipeline stage (128 B rows)
constexpr int kATile = kBM * kBK * 2;  // 16 KB
constexpr int kMaxBoxes = 5;         // activation box heights 16, 32, 64, 128, 256

enum TileMode : int { kRouter = 0, kGateUp = 1, kDown = 2 };

struct BoxMaps {
  CUtensorMap map[kMaxBoxes];  // same tensor, box heights 16 << i
};

struct TileArgs {
  int mode;
  // schedule
  int n_tok;          // tokens in the block (router: rows of x)
  int tiles_per_unit_expert;  // weight tiles per expert (ffn/128 or hidden/128)
  int kb_total;       // K blocks of the full contraction
  int splits;         // router split-K factor (1 otherwise)
  int n_units_static; // router: expert tiles * splits
  const int* n_active;  // device U (ffn modes)
  const int* active;
  const int* expert_offset;
  const int* expert_count;
  int weight_rows_per_expert;  // rows of the 2-D weight view per expert
  int stages;
  int b_rows;         // smem rows reserved for the activation tile
  // epilogue
  int ld_out;         // leading dim (elements) of the output rows
  int m_pad;          // router: padded expert count of the partial rows
  const float* slot_gate;
  __nv_bfloat16* h_out;  // kGateUp: H [slots x ffn]
  float* y_out;          // kDown: y_slot [slots x hidden]; kRouter: partials
};

__global__ void tile_gemm_kernel(const __grid_constant__ CUtensorMap wa,
                                 const __grid_constant__ CUtensorMap wb,
                                 const __grid_constant__ BoxMaps acts, TileArgs a);

}  // namespace desmoe
