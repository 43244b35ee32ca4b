// K2 (gating + DES coreset + constrained re-route) and K3 (permutation)
// kernels for sm_100a.
//
// All routing arithmetic is fp64 in the reference's operation order so that
// selections, coresets and assignments are the reference's:
//   activation   gating.cpp:10-40   max (exact in any order), exp(x - max),
//                                   sum in ascending expert index, divide
//   selection    gating.cpp:42-71   k largest by (value desc, index asc),
//                                   emitted in ascending index
//   renormalise  gating.cpp:73-82   sum over the selection, ascending index
//   DES-Vote     des.cpp:65-95      model-K mask, votes summed over tokens in
//                                   ascending order, top floor(beta*M)
//   DES-Seq      des.cpp:33-45      union of per-token top-k
//   re-route     des.cpp:97-118     top-min(K,|C|) inside the coreset
// The sequential sums are the only serial chains; everything else is spread
// over one warp per token (K2a, K2c) or one thread per expert (K2b).
#include "common.cuh"
#include "kernels.cuh"

namespace desmoe {

namespace {

template <typename T>
__device__ inline double load_logit(const T* p) {
  return static_cast<double>(*p);
}

}  // namespace

// ---------------------------------------------------------------------------
// K2a: per-token activation + top-K (one warp per token).
//   mode 0 (VANILLA): writes the final route (ascending experts, renormalised
//                     gates) — topk_route(activate(block), K).
//   mode 1 (DES):     writes the rank-ordered top-K list for K2b/K2c.
// Input logits: T = double | float, or the router GEMM's split-K partials
// (splits > 0: logit = sum over s ascending of partial[s][n][e], fp32).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) gate_topk_kernel(GateTopkArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int n = blockIdx.x * nwarps + warp;
  const int m = a.m;
  double* row = reinterpret_cast<double*>(smem_raw) + static_cast<size_t>(warp) * m;
  int* sel = reinterpret_cast<int*>(reinterpret_cast<double*>(smem_raw) +
                                    static_cast<size_t>(nwarps) * m) +
             warp * 32;
  if (n >= a.n) return;

  // load (+ reduce split-K partials in fixed ascending split order)
  bool bad = false;
  double mx = -INFINITY;
  for (int i = lane; i < m; i += 32) {
    double x;
    if (a.splits > 0) {
      float v[kMaxSplits];
#pragma unroll
      for (int s = 0; s < kMaxSplits; ++s)
        v[s] = s < a.splits ? __ldcg(&a.partials[(static_cast<size_t>(s) * a.n + n) * a.m_pad + i])
                            : 0.0f;
      float acc = 0.0f;
#pragma unroll
      for (int s = 0; s < kMaxSplits; ++s)
        if (s < a.splits) acc += v[s];
      x = static_cast<double>(acc);
      if (a.logits_out) a.logits_out[static_cast<size_t>(n) * m + i] = acc;
    } else {
      x = load_logit(a.logits + static_cast<size_t>(n) * m + i);
    }
    bad |= !isfinite(x);
    row[i] = x;
    mx = fmax(mx, x);
  }
  if (__any_sync(0xffffffffu, bad)) {
    if (lane == 0) raise_flag(a.err, 1);
    return;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));

  if (a.act == 0) {  // softmax
    for (int i = lane; i < m; i += 32) row[i] = glibc_exp(row[i] - mx, kExpTab);
    __syncwarp();
    double s = 0.0;
    if (lane == 0) {
      for (int i = 0; i < m; ++i) s += row[i];
    }
    s = __shfl_sync(0xffffffffu, s, 0);
    for (int i = lane; i < m; i += 32) row[i] = row[i] / s;
  } else if (a.act == 1) {  // sigmoid
    for (int i = lane; i < m; i += 32) row[i] = 1.0 / (1.0 + glibc_exp(-row[i], kExpTab));
  }
  __syncwarp();
  if (a.probs) {
    for (int i = lane; i < m; i += 32) a.probs[static_cast<size_t>(n) * m + i] = row[i];
  }

  warp_select(row, m, a.k, nullptr, sel);
  if (a.mode == 1) {
    if (lane < a.k) a.topk_idx[static_cast<size_t>(n) * a.k + lane] = sel[lane];
    return;
  }
  // vanilla: ascending order + renormalisation over the selection
  int my = lane < a.k ? sel[lane] : 0x7fffffff;
  int pos = ascending_rank(my, lane, a.k);
  __syncwarp();
  if (lane < a.k) sel[pos] = my;
  __syncwarp();
  double ssum = 0.0;
  if (lane == 0) {
    for (int j = 0; j < a.k; ++j) ssum += row[sel[j]];
  }
  ssum = __shfl_sync(0xffffffffu, ssum, 0);
  if (lane < a.kmax) {
    size_t o = static_cast<size_t>(n) * a.kmax + lane;
    bool in = lane < a.k;
    int e = in ? sel[lane] : -1;
    double g = in ? row[e] / ssum : 0.0;
    a.route_idx[o] = e;
    a.route_gate[o] = g;
    if (a.route_gate32) a.route_gate32[o] = static_cast<float>(g);
  }
  if (lane == 0) a.route_cnt[n] = a.k;
}

template <typename T>
cudaError_t launch_gate_topk_kernel(const GateTopkArgs<T>& a, int grid, int block, size_t smem,
                                    cudaStream_t st) {
  gate_topk_kernel<T><<<grid, block, smem, st>>>(a);
  return cudaGetLastError();
}

template cudaError_t launch_gate_topk_kernel<double>(const GateTopkArgs<double>&, int, int,
                                                     size_t, cudaStream_t);
template cudaError_t launch_gate_topk_kernel<float>(const GateTopkArgs<float>&, int, int, size_t,
                                                    cudaStream_t);

// ---------------------------------------------------------------------------
// K2b: block-level coreset (single CTA, one thread per expert).
//   VOTE: V[i] = sum over tokens n ascending of masked p[n][i] (or the raw
//         logit), masked = outside token n's model-K top-K; coreset = the
//         floor(beta*M) largest V by (V desc, index asc).
//   SEQ:  union of each token's top-seq_k.
// Output: ascending member list, member flags, size.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) coreset_kernel(CoresetArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int m = a.m, n_tok = a.n, k = a.k;
  const int words = (m + 31) >> 5;
  uint32_t* bits = reinterpret_cast<uint32_t*>(smem_raw);                 // [n_tok][words]
  uint64_t* keys = reinterpret_cast<uint64_t*>(bits + static_cast<size_t>(n_tok) * words +
                                               ((n_tok * words) & 1));    // [m]
  int* flag = reinterpret_cast<int*>(keys + m);                           // [m]
  __shared__ int warp_tot[32];

  for (int i = threadIdx.x; i < n_tok * words; i += blockDim.x) bits[i] = 0;
  __syncthreads();
  const int depth = a.strategy == 0 ? a.seq_k : k;
  for (int e = threadIdx.x; e < n_tok * depth; e += blockDim.x) {
    int t = e / depth, r = e % depth;
    int x = a.topk_idx[static_cast<size_t>(t) * k + r];
    atomicOr(&bits[static_cast<size_t>(t) * words + (x >> 5)], 1u << (x & 31));
  }
  __syncthreads();

  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const uint32_t bit = 1u << (i & 31);
    const uint32_t* col = bits + (i >> 5);
    if (a.strategy == 0) {
      int in = 0;
      for (int t = 0; t < n_tok && !in; ++t) in = (col[static_cast<size_t>(t) * words] & bit) != 0;
      flag[i] = in;
    } else {
      double v = 0.0;
      for (int t = 0; t < n_tok; ++t) {
        if (col[static_cast<size_t>(t) * words] & bit) {
          size_t at = static_cast<size_t>(t) * m + i;
          v += a.raw ? (a.logits64 ? a.logits64[at] : static_cast<double>(a.logits32[at]))
                     : a.probs[at];
        }
      }
      if (a.votes) a.votes[i] = v;
      keys[i] = order_key(v);
    }
  }
  __syncthreads();
  if (a.strategy == 1) {
    // rank of expert i = #experts preceding it in (V desc, index asc)
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      const uint64_t ki = keys[i];
      int rank = 0;
      for (int j = 0; j < m; ++j) {
        uint64_t kj = keys[j];
        rank += (kj > ki) | ((kj == ki) & (j < i));
      }
      flag[i] = rank < a.m_core;
    }
    __syncthreads();
  }
  // ascending compaction of the flags (m <= blockDim.x: one pass of ballots)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = threadIdx.x;
  const int f = i < m ? flag[i] : 0;
  const uint32_t bal = __ballot_sync(0xffffffffu, f);
  if (lane == 0) warp_tot[warp] = __popc(bal);
  __syncthreads();
  if (threadIdx.x == 0) {
    int base = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      int t = warp_tot[w];
      warp_tot[w] = base;
      base += t;
    }
    *a.n_members = base;
  }
  __syncthreads();
  if (f) a.members[warp_tot[warp] + __popc(bal & ((1u << lane) - 1u))] = i;
  if (a.member_flag && i < m) a.member_flag[i] = static_cast<uint8_t>(f);
}

// ---------------------------------------------------------------------------
// K2c: constrained re-route (one warp per token): top-min(K,|C|) inside the
// coreset by the activated gate, renormalised (des.cpp:97-118). A token whose
// own top-K lies inside the coreset keeps it unchanged (the restricted
// selection is then provably the same set).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) constrained_route_kernel(RerouteArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int n = blockIdx.x * nwarps + warp;
  int* sel = reinterpret_cast<int*>(smem_raw) + warp * 32;
  if (n >= a.n) return;
  const int m = a.m, k = a.k;
  const int nm = *a.n_members;
  const int kk = k < nm ? k : nm;
  const double* p = a.probs + static_cast<size_t>(n) * m;

  bool covered = false;
  if (a.topk_idx && nm >= k) {
    int mine = lane < k ? a.topk_idx[static_cast<size_t>(n) * k + lane] : -1;
    bool ok = lane >= k || a.member_flag[mine];
    covered = __all_sync(0xffffffffu, ok);
    if (covered && lane < k) sel[lane] = mine;
    __syncwarp();
  }
  if (!covered) warp_select(p, m, kk, a.member_flag, sel);

  int my = lane < kk ? sel[lane] : 0x7fffffff;
  int pos = ascending_rank(my, lane, kk);
  __syncwarp();
  if (lane < kk) sel[pos] = my;
  __syncwarp();
  double ssum = 0.0;
  if (lane == 0) {
    for (int j = 0; j < kk; ++j) ssum += p[sel[j]];
  }
  ssum = __shfl_sync(0xffffffffu, ssum, 0);
  if (lane < k) {
    size_t o = static_cast<size_t>(n) * k + lane;
    bool in = lane < kk;
    int e = in ? sel[lane] : -1;
    double g = in ? p[e] / ssum : 0.0;
    a.route_idx[o] = e;
    a.route_gate[o] = g;
    if (a.route_gate32) a.route_gate32[o] = static_cast<float>(g);
  }
  if (lane == 0) a.route_cnt[n] = kk;
}

// Writes member flags from an explicit (host-provided, ascending) coreset.
__global__ void set_members_kernel(const int* members, int nm, int m, uint8_t* flag,
                                   int* n_members) {
  for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < m; i += blockDim.x * gridDim.x)
    flag[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < nm; i += blockDim.x) flag[members[i]] = 1;
  if (threadIdx.x == 0) *n_members = nm;
}

// ---------------------------------------------------------------------------
// K3: permutation (single CTA). Per-expert counts, ascending exclusive
// offsets, stable slot positions (tokens ascending inside an expert), the
// active-expert list and U; also zeroes the FFN kernel's counters.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) permute_kernel(PermuteArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int m = a.m, n_tok = a.n, k = a.k;
  const int tw = (n_tok + 31) >> 5;
  int* count = reinterpret_cast<int*>(smem_raw);              // [m]
  int* offset = count + m;                                     // [m]
  uint32_t* bits = reinterpret_cast<uint32_t*>(offset + m);    // [m][tw]
  __shared__ int warp_tot[32], warp_act[32];
  __shared__ int s_total, s_active;

  for (int i = threadIdx.x; i < m; i += blockDim.x) count[i] = 0;
  for (int i = threadIdx.x; i < m * tw; i += blockDim.x) bits[i] = 0;
  for (int i = threadIdx.x; i < a.zero_words; i += blockDim.x) a.zero[i] = 0;
  __syncthreads();
  for (int e = threadIdx.x; e < n_tok * k; e += blockDim.x) {
    int t = e / k, j = e % k;
    if (j >= a.route_cnt[t]) continue;
    int x = a.route_idx[e];
    atomicAdd(&count[x], 1);
    atomicOr(&bits[static_cast<size_t>(x) * tw + (t >> 5)], 1u << (t & 31));
  }
  __syncthreads();
  // exclusive scan over experts (ascending) + active compaction
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  {  // m <= blockDim.x: one pass
    const int i = threadIdx.x;
    const int c = i < m ? count[i] : 0;
    int incl = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      int o = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += o;
    }
    const uint32_t act = __ballot_sync(0xffffffffu, c > 0);
    if (lane == 31) warp_tot[warp] = incl;
    if (lane == 0) warp_act[warp] = __popc(act);
    __syncthreads();
    if (threadIdx.x == 0) {
      int base = 0, abase = 0;
      for (int w = 0; w < nw; ++w) {
        int t = warp_tot[w], u = warp_act[w];
        warp_tot[w] = base;
        warp_act[w] = abase;
        base += t;
        abase += u;
      }
      s_total = base;
      s_active = abase;
    }
    __syncthreads();
    if (i < m) offset[i] = warp_tot[warp] + incl - c;
    if (i < m && c > 0) a.active[warp_act[warp] + __popc(act & ((1u << lane) - 1u))] = i;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    if (a.expert_count) a.expert_count[i] = count[i];
    if (a.expert_offset) a.expert_offset[i] = offset[i];
  }
  for (int e = threadIdx.x; e < n_tok * k; e += blockDim.x) {
    int t = e / k, j = e % k;
    if (j >= a.route_cnt[t]) {
      if (a.slot_of) a.slot_of[e] = -1;
      continue;
    }
    int x = a.route_idx[e];
    const uint32_t* b = bits + static_cast<size_t>(x) * tw;
    int before = 0;
    for (int w = 0; w < (t >> 5); ++w) before += __popc(b[w]);
    before += __popc(b[t >> 5] & ((1u << (t & 31)) - 1u));
    int pos = offset[x] + before;
    if (a.slot_of) a.slot_of[e] = pos;
    if (a.slot_token) a.slot_token[pos] = t;
    if (a.slot_gate && a.route_gate) a.slot_gate[pos] = static_cast<float>(a.route_gate[e]);
  }
  if (threadIdx.x == 0) {
    if (a.n_active) *a.n_active = s_active;
    if (a.total) *a.total = s_total;
  }
}

// Raises every kernel's dynamic shared-memory ceiling once (context
// creation), so no attribute call happens inside a launch sequence / graph
// capture.
cudaError_t set_kernel_smem_limits() {
  cudaError_t e = cudaSuccess;
  auto set = [&](const void* fn, int bytes) {
    // dynamic + the kernel's static shared memory must stay within 227 KB
    cudaFuncAttributes fa{};
    cudaError_t r = cudaFuncGetAttributes(&fa, fn);
    const int cap = 227 * 1024 - static_cast<int>(fa.sharedSizeBytes);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               bytes < cap ? bytes : cap);
    if (e == cudaSuccess) e = r;
  };
  const int routing = 200 * 1024;  // leaves room for the kernels' static shared memory
  set(reinterpret_cast<const void*>(gate_topk_kernel<double>), routing);
  set(reinterpret_cast<const void*>(gate_topk_kernel<float>), routing);
  set(reinterpret_cast<const void*>(coreset_kernel), routing);
  set(reinterpret_cast<const void*>(constrained_route_kernel), routing);
  set(reinterpret_cast<const void*>(permute_kernel), routing);
  set(reinterpret_cast<const void*>(tile_gemm_kernel), 227 * 1024);
  set(reinterpret_cast<const void*>(ffn_persistent_kernel<2>), 227 * 1024);
  set(reinterpret_cast<const void*>(ffn_persistent_kernel<4>), 227 * 1024);
  set(reinterpret_cast<const void*>(x_ingress_bulk_kernel), kIngressChunk);
  const cudaError_t f = set_fused_route_smem_limit(kFusedRouteSmem);
  const cudaError_t g = set_front_smem_limit();
  return e != cudaSuccess ? e : (f != cudaSuccess ? f : g);
}

}  // namespace desmoe
