// Comparison expert-skipping policies of the reference (baselines.cpp) as one
// routing kernel, logits in -> route out, so the GPU path can run every
// method `dessim run` compares against DES:
//
//   TOPK_REDUCE  topk_route(activate(block), k_reduced)        baselines.cpp:10-16
//   NAEE         per token: rank the K selected gates (value desc, index asc);
//                drop ranks i..K for the smallest i >= 2 whose tail sum is
//                below beta x (sum of the selection in ascending index
//                order); renormalise the kept gates         baselines.cpp:23-76
//   MCMOE        the ceil(fraction x N) most important tokens (stable order
//                of the score, descending) keep their full top-K, the rest
//                get NAEE; score = max gate or -entropy      baselines.cpp:78-123
//
// One CTA (32 warps, one warp per token, tokens strided). Phase 1 activates
// every token row in fp64 in the reference's operation order (gating.cpp:
// 10-40) into `probs` and computes the MC-MoE score; phase 2 ranks the tokens
// by score (a stable rank count) and routes. Selection is exact on the fp64
// probabilities with the reference's comparator (warp_select), so ids equal
// the reference's; gates are the same fp64 quotients (modulo the last-bit
// freedom of exp / log).
#include "common.cuh"
#include "kernels.cuh"
#include "route_common.cuh"

namespace desmoe {

namespace {

// Kept experts of one token under the NAEE rule, rank order in sel[0..keep).
// sel holds the token's top-K in rank order (warp_select); p the row.
__device__ int naee_keep(const double* p, const int* sel, int k, double beta) {
  // total over the selection in ASCENDING index order (baselines.cpp:33-34)
  int asc[32];
  for (int j = 0; j < k; ++j) asc[j] = sel[j];
  for (int a = 1; a < k; ++a) {  // insertion sort, k <= 32
    const int v = asc[a];
    int b = a - 1;
    while (b >= 0 && asc[b] > v) {
      asc[b + 1] = asc[b];
      --b;
    }
    asc[b + 1] = v;
  }
  double total = 0.0;
  for (int j = 0; j < k; ++j) total = __dadd_rn(total, p[asc[j]]);
  // tails[u] = sum of ranks u..K accumulated from rank K down (:36-41)
  double tails[33];
  double tail = 0.0;
  for (int u = k; u >= 2; --u) {
    tail = __dadd_rn(tail, p[sel[u - 1]]);
    tails[u] = tail;
  }
  const double thr = __dmul_rn(beta, total);
  for (int i = 2; i <= k; ++i)
    if (tails[i] < thr) return i - 1;  // (:42-47)
  return k;
}

}  // namespace

template <typename T>
__global__ void __launch_bounds__(1024, 1) baseline_route_kernel(BaselineArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = a.n, m = a.m, k = a.k;
  double* score = reinterpret_cast<double*>(smem_raw);       // [n]
  int* sel_all = reinterpret_cast<int*>(score + n);          // [32 warps][32]
  __shared__ int s_bad;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  int* sel = sel_all + warp * 32;

  // ---- phase 1: activation (+ MC-MoE score) -----------------------------------
  for (int t = warp; t < n; t += 32) {
    double* row = a.probs + static_cast<size_t>(t) * m;
    bool bad = false;
    double mx = -INFINITY;
    for (int i = lane; i < m; i += 32) {
      const double x = static_cast<double>(a.logits[static_cast<size_t>(t) * m + i]);
      bad |= !isfinite(x);
      row[i] = x;
      mx = fmax(mx, x);
    }
    if (__any_sync(0xffffffffu, bad)) {
      if (lane == 0) s_bad = 1;
      continue;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    __syncwarp();
    const double s = token_activate(row, m, a.act, mx);
    // the row now holds p (softmax: numerators -> divide in place, gating.cpp:36-38)
    if (a.act == 0)
      for (int i = lane; i < m; i += 32) row[i] = div_f64(row[i], s);
    __syncwarp();
    if (a.method == 2) {
      double sc = 0.0;
      if (a.score == 0) {  // max gate (order-free)
        double v = -INFINITY;
        for (int i = lane; i < m; i += 32) v = fmax(v, row[i]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
        sc = v;
      } else if (lane == 0) {  // -entropy, ascending i, product then subtract (:96-101)
        double h = 0.0;
        for (int i = 0; i < m; ++i) {
          const double p = row[i];
          if (p > 0.0) h = __dsub_rn(h, __dmul_rn(p, log(p)));
        }
        sc = -h;
      }
      if (lane == 0) score[t] = sc;
    }
  }
  __syncthreads();
  if (s_bad) {
    if (tid == 0) raise_flag(a.err, 1);
    return;
  }

  // ---- phase 2: per-token selection + route ------------------------------------
  for (int t = warp; t < n; t += 32) {
    const double* row = a.probs + static_cast<size_t>(t) * m;
    bool full = a.method == 0 || a.method == 2;
    if (a.method == 2) {
      // stable rank by score descending (std::stable_sort, :106-108)
      const double st = score[t];
      int r = 0;
      for (int q = lane; q < n; q += 32) {
        const double sq = score[q];
        r += (sq > st) || (sq == st && q < t);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) r += __shfl_xor_sync(0xffffffffu, r, off);
      full = r < a.important;
    }
    const int want = a.method == 0 ? a.k_reduced : k;
    warp_select(row, m, want, nullptr, sel);  // rank order
    __syncwarp();
    int cnt = want;
    if (!full) {
      int keep = 0;
      if (lane == 0) keep = naee_keep(row, sel, k, a.beta);
      cnt = __shfl_sync(0xffffffffu, keep, 0);
    }
    token_write_route(row, 1.0, 2, sel, cnt, k, t, a.route_idx, a.route_gate, a.route_cnt);
  }
}

template __global__ void baseline_route_kernel<double>(BaselineArgs<double>);
template __global__ void baseline_route_kernel<float>(BaselineArgs<float>);

}  // namespace desmoe
