// K2 fused: the whole routing stage of a block in ONE single-CTA kernel
// (1024 threads, one warp per token, tokens strided over the 32 warps):
//   1. logits (fp64 / fp32, or the router's split-K partials reduced in fixed
//      split order) -> activation -> per-token top-K      (gating.cpp:10-71)
//   2. block coreset: DES-Vote votes summed over tokens in ascending order and
//      the top floor(beta*M) by (vote desc, index asc), or the DES-Seq union
//                                                          (des.cpp:33-95)
//   3. constrained re-route + renormalisation per token   (des.cpp:97-118)
//   VANILLA stops after 1 with topk_route's renormalised gates (gating.cpp:84-97).
// Every intermediate (activated rows, top-K lists, selection bitmaps, votes,
// coreset flags) stays in shared memory, so the stage costs one launch and no
// dependent global round trips. It also zeroes the expert-FFN kernel's
// scheduler counters for the launch that follows. Arithmetic is fp64 in the
// reference's operation order, identical to the multi-kernel path.
#include "common.cuh"
#include "kernels.cuh"

namespace desmoe {

template <typename T>
__global__ void __launch_bounds__(1024, 1) fused_route_kernel(FusedRouteArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = a.n, m = a.m, k = a.k;
  const int mw = (m + 31) >> 5;
  double* prow = reinterpret_cast<double*>(smem_raw);               // [n][m]
  double* vkey = prow + static_cast<size_t>(n) * m;                  // [m] votes
  int* topk = reinterpret_cast<int*>(vkey + m);                      // [n][k] rank order
  uint32_t* bits = reinterpret_cast<uint32_t*>(topk + n * k);        // [n][mw]
  int* sel = reinterpret_cast<int*>(bits + n * mw);                  // [32 warps][32]
  uint8_t* flag = reinterpret_cast<uint8_t*>(sel + 32 * 32);         // [m]
  __shared__ int warp_tot[33];
  __shared__ int s_bad;

  pdl_launch_dependents();  // the expert-FFN grid may start its own prologue
  pdl_wait();               // router partials / logits complete
  if (tid == 0) s_bad = 0;
  for (int i = tid; i < a.zero_words; i += blockDim.x) a.zero[i] = 0;
  for (int i = tid; i < n * mw; i += blockDim.x) bits[i] = 0;
  __syncthreads();
  const bool vanilla = a.strategy < 0;
  const int depth = a.strategy == 0 ? a.seq_k : k;  // selections feeding the coreset
  int* wsel = sel + warp * 32;

  // ---- 1. activation + per-token top-K ----------------------------------------
  for (int t = warp; t < n; t += 32) {
    double* row = prow + static_cast<size_t>(t) * m;
    bool bad = false;
    double mx = -INFINITY;
    for (int i = lane; i < m; i += 32) {
      double x;
      if (a.splits > 0) {
        // all split partials in flight at once, then summed in split order
        float v[kMaxSplits];
#pragma unroll
        for (int s = 0; s < kMaxSplits; ++s)
          v[s] = s < a.splits ? __ldcg(&a.partials[(static_cast<size_t>(s) * n + t) * m + i])
                              : 0.0f;
        float acc = 0.0f;
#pragma unroll
        for (int s = 0; s < kMaxSplits; ++s)
          if (s < a.splits) acc += v[s];
        if (a.logits_out) a.logits_out[static_cast<size_t>(t) * m + i] = acc;
        x = static_cast<double>(acc);
      } else {
        x = static_cast<double>(a.logits[static_cast<size_t>(t) * m + i]);
      }
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
    if (a.act == 0) {  // softmax: sum in ascending expert order (gating.cpp:30-34)
      for (int i = lane; i < m; i += 32) row[i] = glibc_exp(row[i] - mx, kExpTab);
      __syncwarp();
      double s = 0.0;
      if (lane == 0)
        for (int i = 0; i < m; ++i) s += row[i];
      s = __shfl_sync(0xffffffffu, s, 0);
      for (int i = lane; i < m; i += 32) row[i] = row[i] / s;
    } else if (a.act == 1) {
      for (int i = lane; i < m; i += 32) row[i] = 1.0 / (1.0 + glibc_exp(-row[i], kExpTab));
    }
    __syncwarp();
    if (a.probs)
      for (int i = lane; i < m; i += 32) a.probs[static_cast<size_t>(t) * m + i] = row[i];
    warp_select(row, m, k, nullptr, wsel);
    if (vanilla) {
      const int my = lane < k ? wsel[lane] : 0x7fffffff;
      const int pos = ascending_rank(my, lane, k);
      __syncwarp();
      if (lane < k) wsel[pos] = my;
      __syncwarp();
      double ssum = 0.0;
      if (lane == 0)
        for (int j = 0; j < k; ++j) ssum += row[wsel[j]];
      ssum = __shfl_sync(0xffffffffu, ssum, 0);
      if (lane < k) {
        const size_t o = static_cast<size_t>(t) * k + lane;
        a.route_idx[o] = wsel[lane];
        a.route_gate[o] = row[wsel[lane]] / ssum;
      }
      if (lane == 0) a.route_cnt[t] = k;
    } else {
      if (lane < k) topk[t * k + lane] = wsel[lane];
      if (lane < depth) atomicOr(&bits[t * mw + (wsel[lane] >> 5)], 1u << (wsel[lane] & 31));
    }
    __syncwarp();
  }
  __syncthreads();
  if (s_bad) {
    if (tid == 0) raise_flag(a.err, 1);
    return;
  }
  if (vanilla) return;

  // ---- 2. block coreset (thread per expert) ------------------------------------
  const int i = tid;
  if (i < m) {
    const uint32_t bit = 1u << (i & 31);
    const uint32_t* col = bits + (i >> 5);
    if (a.strategy == 0) {
      int in = 0;
      for (int t = 0; t < n && !in; ++t) in = (col[t * mw] & bit) != 0;
      flag[i] = static_cast<uint8_t>(in);
    } else {
      double v = 0.0;  // tokens in ascending order (des.cpp:86-91)
      for (int t = 0; t < n; ++t)
        if (col[t * mw] & bit)
          v += a.raw ? static_cast<double>(a.raw_logits[static_cast<size_t>(t) * m + i])
                     : prow[static_cast<size_t>(t) * m + i];
      if (a.votes) a.votes[i] = v;
      vkey[i] = v;
    }
  }
  __syncthreads();
  if (a.strategy == 1 && i < m) {
    const uint64_t ki = order_key(vkey[i]);
    int rank = 0;
    for (int j = 0; j < m; ++j) {
      const uint64_t kj = order_key(vkey[j]);
      rank += (kj > ki) | ((kj == ki) & (j < i));
    }
    flag[i] = static_cast<uint8_t>(rank < a.m_core);
  }
  __syncthreads();
  {  // ascending member list
    const int f = i < m ? flag[i] : 0;
    const uint32_t bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) warp_tot[warp] = __popc(bal);
    __syncthreads();
    if (tid == 0) {
      int acc = 0;
      for (int w = 0; w < 32; ++w) {
        const int c = warp_tot[w];
        warp_tot[w] = acc;
        acc += c;
      }
      warp_tot[32] = acc;
      if (a.n_members) *a.n_members = acc;
    }
    __syncthreads();
    if (f && a.members) a.members[warp_tot[warp] + __popc(bal & ((1u << lane) - 1u))] = i;
    if (a.member_flag && i < m) a.member_flag[i] = static_cast<uint8_t>(f);
  }
  const int nm = warp_tot[32];
  const int kk = k < nm ? k : nm;

  // ---- 3. constrained re-route (warp per token) --------------------------------
  for (int t = warp; t < n; t += 32) {
    const double* row = prow + static_cast<size_t>(t) * m;
    bool covered = false;
    if (nm >= k) {
      const int mine = lane < k ? topk[t * k + lane] : 0;
      covered = __all_sync(0xffffffffu, lane >= k || flag[mine]);
      if (covered && lane < k) wsel[lane] = mine;
      __syncwarp();
    }
    if (!covered) warp_select(row, m, kk, flag, wsel);
    const int my = lane < kk ? wsel[lane] : 0x7fffffff;
    const int pos = ascending_rank(my, lane, kk);
    __syncwarp();
    if (lane < kk) wsel[pos] = my;
    __syncwarp();
    double ssum = 0.0;
    if (lane == 0)
      for (int j = 0; j < kk; ++j) ssum += row[wsel[j]];
    ssum = __shfl_sync(0xffffffffu, ssum, 0);
    if (lane < k) {
      const size_t o = static_cast<size_t>(t) * k + lane;
      const bool in = lane < kk;
      a.route_idx[o] = in ? wsel[lane] : -1;
      a.route_gate[o] = in ? row[wsel[lane]] / ssum : 0.0;
    }
    if (lane == 0) a.route_cnt[t] = kk;
    __syncwarp();
  }
}

size_t fused_route_smem(int n, int m, int k) {
  const int mw = (m + 31) / 32;
  return static_cast<size_t>(n) * m * 8 + static_cast<size_t>(m) * 8 +
         static_cast<size_t>(n) * k * 4 + static_cast<size_t>(n) * mw * 4 + 32 * 32 * 4 +
         static_cast<size_t>(m) + 16;
}

template <typename T>
cudaError_t launch_fused_route(const FusedRouteArgs<T>& a, cudaStream_t st) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(1);
  lc.blockDim = dim3(1024);
  lc.dynamicSmemBytes = fused_route_smem(a.n, a.m, a.k);
  lc.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  return cudaLaunchKernelEx(&lc, fused_route_kernel<T>, a);
}

template cudaError_t launch_fused_route<double>(const FusedRouteArgs<double>&, cudaStream_t);
template cudaError_t launch_fused_route<float>(const FusedRouteArgs<float>&, cudaStream_t);

cudaError_t set_fused_route_smem_limit(int bytes) {
  cudaError_t e = cudaFuncSetAttribute(fused_route_kernel<double>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaError_t e2 = cudaFuncSetAttribute(fused_route_kernel<float>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  return e != cudaSuccess ? e : e2;
}

}  // namespace desmoe
