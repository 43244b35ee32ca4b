// K1 + K2 fused: router GEMM and the whole DES routing stage of one block in
// a single thread-block CLUSTER of kFrontCta CTAs (one per SM):
//
//   R  router GEMM, split-K over the cluster: CTA r multiplies W_r[:, K-slice r]
//      by X[:, K-slice r] on tcgen05 (swap-AB: 128 expert rows x N tokens per
//      M tile, TMA -> SWIZZLE_128B smem -> TMEM) and parks its fp32 partial
//      logits [N][M] in its own shared memory;
//   L  CTA r owns tokens [r*N/C, (r+1)*N/C): it sums each logit over the C
//      partials in fixed CTA order through distributed shared memory (so the
//      logits are deterministic), then activation + per-token top-K in fp64
//      (gating.cpp:10-71), one warp per token;
//   V  every CTA gathers all tokens' selections over DSMEM and computes the
//      block coreset redundantly — DES-Vote votes summed over tokens in
//      ascending order, top floor(beta*M) by (vote desc, index asc)
//      (des.cpp:65-95), or the DES-Seq union (des.cpp:33-45) — so no further
//      cluster round is needed;
//   RR constrained re-route + renormalisation of its own tokens
//      (des.cpp:97-118); VANILLA stops after L with topk_route's gates.
// Three cluster barriers in total; every intermediate stays on chip. The
// kernel also zeroes the expert-FFN scheduler counters and triggers the
// programmatic launch of the FFN kernel at its start.
#include "common.cuh"
#include "kernels.cuh"
#include "route_common.cuh"

namespace desmoe {

namespace {

__device__ inline uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ inline void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// address of the same shared-memory location in CTA `rank` of the cluster
__device__ inline uint32_t dsmem_addr(const void* local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(r)
               : "r"(smem_u32(local)), "r"(rank));
  return r;
}

__device__ inline float ld_dsmem_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}

__device__ inline int ld_dsmem_s32(uint32_t addr) {
  int v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}

__device__ inline double ld_dsmem_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}

}  // namespace

__global__ void __launch_bounds__(kFrontThreads, 1)
    front_kernel(const __grid_constant__ CUtensorMap wr_map, const __grid_constant__ BoxMaps x_maps,
                 FrontArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // align to 1024 B by offsetting the shared array itself, so the compiler
  // keeps the shared address space (LDS/STS instead of generic LD/ST)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const int C = kFrontCta;
  const int n = a.n, m = a.m, k = a.k;
  const int mt = (m + kBM - 1) / kBM;  // expert (M) tiles
  const int mw = (m + 31) >> 5;
  const int b_rows = a.b_rows;        // token box rows (>= n, multiple of 16)
  const int kb_cta = a.kb_per_cta;    // K blocks of this CTA
  // ---- shared memory -----------------------------------------------------------
  // [stage ring: per K block: mt weight tiles (16 KB) + token box] | barriers |
  // partial[n][m] f32 | prow[own][m] f64 | own topk/p | all topk/p | bits | flags
  const int stage_bytes = mt * kATile + b_rows * 128;
  const int S = a.stages;
  unsigned char* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + static_cast<size_t>(S) * stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* tdone = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tdone + 1);
  float* part = reinterpret_cast<float*>(tmem_slot + 4);                  // [n][m]
  const int t0 = (n * static_cast<int>(rank)) / C, t1 = (n * (static_cast<int>(rank) + 1)) / C;
  const int own = t1 - t0;
  const int own_max = (n + C - 1) / C;  // identical layout in every CTA (DSMEM offsets)
  const int nwarps = kFrontThreads / 32;
  double* prow = reinterpret_cast<double*>(part + static_cast<size_t>(n) * m +
                                           ((n * m) & 1));                // [own_max][m]
  double* psum = prow + static_cast<size_t>(own_max) * m;                 // [own_max] softmax s
  double* scratch_all = psum + own_max;                                   // [warps][m]
  double* otp = scratch_all + static_cast<size_t>(nwarps) * m;            // [own_max*k] vote vals
  double* atp = otp + own_max * k;                                        // [n*k] gathered vals
  double* slotv = atp + n * k;                                            // [n*k] expert-sorted
  double* votes = slotv + n * k;                                          // [m]
  uint64_t* wkey_all = reinterpret_cast<uint64_t*>(votes + m);            // [warps][64]
  int* otop = reinterpret_cast<int*>(wkey_all + nwarps * 64);             // [own_max*k] rank order
  int* atop = otop + own_max * k;                                         // [n*k] gathered ids
  int* ecount = atop + n * k;                                             // [m]
  int* eoff = ecount + m;                                                 // [m]
  const int tw = (n + 31) >> 5;
  uint32_t* ebits = reinterpret_cast<uint32_t*>(eoff + m);                // [m][tw]
  int* wsel_all = reinterpret_cast<int*>(ebits + m * tw);                 // [warps][64]
  uint8_t* flag = reinterpret_cast<uint8_t*>(wsel_all + nwarps * 64);     // [m]
  __shared__ int warp_tot[kFrontThreads / 32 + 1];
  __shared__ int s_bad;

  const bool vanilla = a.strategy < 0;
  const int depth = a.strategy == 0 ? a.seq_k : k;

  // ---- setup -------------------------------------------------------------------
  if (tid == 0) trace(a.trace, a.trace_cap, 10, static_cast<int>(rank));
  if (tid == 0) {
    tma_prefetch_desc(&wr_map);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tdone, 1);
    fence_mbar_init();
    s_bad = 0;
  }
  if (warp == 2) tmem_alloc(tmem_slot, a.tmem_cols);
  pdl_launch_dependents();
  pdl_wait();  // the previous kernel's outputs (x) are complete
  for (int i = tid + static_cast<int>(rank) * kFrontThreads; i < a.zero_words;
       i += kFrontThreads * C)
    a.zero[i] = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (tid == 0) trace(a.trace, a.trace_cap, 11, static_cast<int>(rank));
  const int box = a.box_index;
  const int n_mma = (n + 15) & ~15;
  const int kb0 = static_cast<int>(rank) * kb_cta;

  // ---- R: split-K router GEMM ---------------------------------------------------
  if (warp == 0 && lane == 0) {
    const uint64_t pol_w = l2_policy_evict_first();
    const uint64_t pol_x = l2_policy_evict_last();
    for (int i = 0; i < kb_cta; ++i) {
      const int s = i % S;
      mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
      unsigned char* st = ring + static_cast<size_t>(s) * stage_bytes;
      mbar_arrive_expect_tx(&full[s], mt * kATile + (16u << box) * 128u);
      for (int tl = 0; tl < mt; ++tl)
        tma_load_2d(st + tl * kATile, &wr_map, &full[s], (kb0 + i) * kBK, tl * kBM, pol_w);
      tma_load_2d(st + mt * kATile, &x_maps.map[box], &full[s], (kb0 + i) * kBK, 0, pol_x);
    }
  } else if (warp == 1) {
    const uint32_t idesc = idesc_bf16_f32(kBM, n_mma);
    for (int i = 0; i < kb_cta; ++i) {
      const int s = i % S;
      mbar_wait(&full[s], (i / S) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t a0 = smem_u32(ring + static_cast<size_t>(s) * stage_bytes);
        const uint32_t b0 = a0 + mt * kATile;
        for (int tl = 0; tl < mt; ++tl)
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk)
            tc_mma_bf16(tmem_base + tl * 256, sw128_kmajor_desc(a0 + tl * kATile + kk * 32),
                        sw128_kmajor_desc(b0 + kk * 32), idesc, (i > 0 || kk > 0) ? 1u : 0u);
        tc_commit(&empty[s]);
        if (i == kb_cta - 1) tc_commit(tdone);
      }
      __syncwarp();
    }
  } else if (warp >= 4 && warp < 8) {
    // drain TMEM: partial[t][e] for this CTA's K slice
    mbar_wait(tdone, 0);
    tc_fence_after();
    const int q = warp & 3;
    const int r = q * 32 + lane;
    for (int tl = 0; tl < mt; ++tl) {
      const int e = tl * kBM + r;
      const uint32_t lb = tmem_base + tl * 256 + (static_cast<uint32_t>(q * 32) << 16);
      for (int c0 = 0; c0 < n_mma; c0 += 16) {
        float v[16];
        tmem_ld16(lb + c0, v);
        if (e < m) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (c0 + j < n) part[(c0 + j) * m + e] = v[j];
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, a.tmem_cols);
  }
  if (tid == 0) trace(a.trace, a.trace_cap, 12, static_cast<int>(rank));
  cluster_sync();  // #1: all partials parked
  if (tid == 0) trace(a.trace, a.trace_cap, 13, static_cast<int>(rank));

  // ---- L: logit reduction over the cluster + activation + top-K (own tokens) -----
  uint32_t part_remote[kFrontCta];
#pragma unroll
  for (int c = 0; c < kFrontCta; ++c) part_remote[c] = dsmem_addr(part, c);
  int* wsel = wsel_all + warp * 64;
  uint64_t* wkey = wkey_all + warp * 64;
  double* scratch = scratch_all + static_cast<size_t>(warp) * m;
  for (int lt = warp; lt < own; lt += nwarps) {
    const int t = t0 + lt;
    double* row = prow + static_cast<size_t>(lt) * m;
    if (lt == 0 && lane == 0)
      trace(a.trace, a.trace_cap, 33, static_cast<int>(clock64() >> 4));
    bool bad = false;
    double mx = -INFINITY;
    for (int i = lane; i < m; i += 32) {
      float v[kFrontCta];
      const uint32_t off = static_cast<uint32_t>((t * m + i) * 4);
#pragma unroll
      for (int c = 0; c < kFrontCta; ++c) v[c] = ld_dsmem_f32(part_remote[c] + off);
      float acc = 0.0f;  // fixed cluster order: deterministic logits
#pragma unroll
      for (int c = 0; c < kFrontCta; ++c) acc += v[c];
      if (a.logits_out) a.logits_out[static_cast<size_t>(t) * m + i] = acc;
      const double x = static_cast<double>(acc);
      bad |= !isfinite(x);
      row[i] = x;
      mx = fmax(mx, x);
    }
    if (__any_sync(0xffffffffu, bad)) {
      if (lane == 0) s_bad = 1;
      continue;
    }
    const bool tr = lt == 0 && lane == 0;
    if (tr) trace(a.trace, a.trace_cap, 30, static_cast<int>(rank));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    const double ssum = token_activate(row, m, a.act, mx);
    if (tr) trace(a.trace, a.trace_cap, 31, static_cast<int>(rank));
    if (lane == 0) psum[lt] = ssum;
    const int cnt = token_select(row, ssum, a.act, m, k, vanilla ? 0 : depth, nullptr, m, wsel,
                                 wkey, scratch);
    if (tr) trace(a.trace, a.trace_cap, 32, static_cast<int>(clock64() >> 4));
    if (vanilla) {
      token_write_route(row, ssum, a.act, wsel, cnt, k, t, a.route_idx, a.route_gate,
                        a.route_cnt);
    } else if (lane < k) {
      const int e = wsel[lane];
      otop[lt * k + lane] = e;
      // vote value: the activated gate, or the raw logit (VoteSource::raw_logits)
      otp[lt * k + lane] = a.raw ? static_cast<double>(a.logits_out[static_cast<size_t>(t) * m + e])
                                 : p_of(row, ssum, a.act, e);
    }
    __syncwarp();
  }
  __syncthreads();
  if (s_bad && tid == 0) atomicOr(a.err, 1);
  if (tid == 0) trace(a.trace, a.trace_cap, 14, static_cast<int>(rank));
  cluster_sync();  // #2: every CTA's selections are visible
  if (tid == 0) trace(a.trace, a.trace_cap, 15, static_cast<int>(rank));
  if (vanilla) {
    cluster_sync();  // keep partials alive until every CTA finished reading them
    return;
  }

  // ---- V: block coreset, redundantly in every CTA ------------------------------------
  // gather every token's selections (token order) over DSMEM
  for (int e = tid; e < n * k; e += kFrontThreads) {
    const int t = e / k, j = e - t * k;
    int ow = C - 1;  // owner CTA: largest r with floor(n r / C) <= t
    while ((n * ow) / C > t) --ow;
    const int lt = t - (n * ow) / C;
    atop[e] = ld_dsmem_s32(dsmem_addr(otop + lt * k + j, ow));
    atp[e] = ld_dsmem_f64(dsmem_addr(otp + lt * k + j, ow));
  }
  for (int i = tid; i < m; i += kFrontThreads) ecount[i] = 0;
  for (int i = tid; i < m * tw; i += kFrontThreads) ebits[i] = 0;
  __syncthreads();
  if (tid == 0) trace(a.trace, a.trace_cap, 20, static_cast<int>(rank));
  // per-expert token sets of the first `depth` selections
  for (int e = tid; e < n * k; e += kFrontThreads) {
    const int t = e / k, j = e - t * k;
    if (j < depth) {
      atomicOr(&ebits[atop[e] * tw + (t >> 5)], 1u << (t & 31));
      atomicAdd(&ecount[atop[e]], 1);
    }
  }
  __syncthreads();
  if (a.strategy == 1) {
    // counting sort of the (token, expert) selections by expert, tokens kept
    // ascending inside each expert, then one ordered sum per expert
    for (int i = tid; i < m; i += kFrontThreads) eoff[i] = ecount[i];
    __syncthreads();
    if (warp == 0) {  // exclusive scan over experts (m <= 1024: 32 per lane)
      const int per = (m + 31) / 32;
      int loc = 0;
      for (int q = 0; q < per; ++q) {
        const int i = lane * per + q;
        if (i < m) loc += eoff[i];
      }
      int incl = loc;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
      }
      int base = incl - loc;
      for (int q = 0; q < per; ++q) {
        const int i = lane * per + q;
        if (i < m) {
          const int c = eoff[i];
          eoff[i] = base;
          base += c;
        }
      }
    }
    __syncthreads();
    for (int e = tid; e < n * k; e += kFrontThreads) {
      const int t = e / k, x = atop[e];
      const uint32_t* b = ebits + x * tw;
      int before = 0;
      for (int w = 0; w < (t >> 5); ++w) before += __popc(b[w]);
      before += __popc(b[t >> 5] & ((1u << (t & 31)) - 1u));
      slotv[eoff[x] + before] = atp[e];
    }
    __syncthreads();
    for (int i = tid; i < m; i += kFrontThreads) {
      double v = 0.0;  // tokens in ascending order (des.cpp:86-91)
      for (int q = eoff[i], qe = eoff[i] + ecount[i]; q < qe; ++q) v += slotv[q];
      votes[i] = v;
      if (a.votes && rank == 0) a.votes[i] = v;
    }
    __syncthreads();
    if (tid == 0) trace(a.trace, a.trace_cap, 21, static_cast<int>(rank));
    for (int i = tid; i < m; i += kFrontThreads) {
      const uint64_t ki = order_key(votes[i]);
      int rk = 0;
      for (int j = 0; j < m; ++j) {
        const uint64_t kj = order_key(votes[j]);
        rk += (kj > ki) | ((kj == ki) & (j < i));
      }
      flag[i] = static_cast<uint8_t>(rk < a.m_core);
    }
  } else {
    for (int i = tid; i < m; i += kFrontThreads) flag[i] = static_cast<uint8_t>(ecount[i] > 0);
  }
  __syncthreads();
  if (tid == 0) trace(a.trace, a.trace_cap, 22, static_cast<int>(rank));
  int nm = 0;
  {
    // ascending member list (block scan over chunks of kFrontThreads experts)
    int base = 0;
    for (int c0 = 0; c0 < m; c0 += kFrontThreads) {
      const int i = c0 + tid;
      const int f = i < m ? flag[i] : 0;
      const uint32_t bal = __ballot_sync(0xffffffffu, f);
      if (lane == 0) warp_tot[warp] = __popc(bal);
      __syncthreads();
      if (tid == 0) {
        int acc = 0;
        for (int w = 0; w < nwarps; ++w) {
          const int c = warp_tot[w];
          warp_tot[w] = acc;
          acc += c;
        }
        warp_tot[nwarps] = acc;
      }
      __syncthreads();
      if (f && rank == 0 && a.members)
        a.members[base + warp_tot[warp] + __popc(bal & ((1u << lane) - 1u))] = i;
      base += warp_tot[nwarps];
      __syncthreads();
    }
    nm = base;
    if (rank == 0 && tid == 0 && a.n_members) *a.n_members = nm;
  }
  if (tid == 0) trace(a.trace, a.trace_cap, 16, static_cast<int>(rank));

  // ---- RR: constrained re-route of own tokens -------------------------------------
  for (int lt = warp; lt < own; lt += nwarps) {
    const int t = t0 + lt;
    const double* row = prow + static_cast<size_t>(lt) * m;
    const double ssum = psum[lt];
    bool covered = false;
    if (nm >= k) {
      const int mine = lane < k ? otop[lt * k + lane] : 0;
      covered = __all_sync(0xffffffffu, lane >= k || flag[mine]);
      if (covered && lane < k) wsel[lane] = mine;
      __syncwarp();
    }
    int cnt = k < nm ? k : nm;
    if (!covered) cnt = token_select(row, ssum, a.act, m, k, 0, flag, nm, wsel, wkey, scratch);
    token_write_route(row, ssum, a.act, wsel, cnt, k, t, a.route_idx, a.route_gate, a.route_cnt);
  }
  if (tid == 0) trace(a.trace, a.trace_cap, 17, static_cast<int>(rank));
  cluster_sync();  // #3: no CTA exits while others may still read its shared memory
}

size_t front_smem_bytes(int n, int m, int k, int stages, int b_rows) {
  const int mt = (m + kBM - 1) / kBM;
  const int own = (n + kFrontCta - 1) / kFrontCta;  // own_max
  const int tw = (n + 31) / 32;
  const int nw = kFrontThreads / 32;
  size_t b = 1024;                                                     // alignment slack
  b += static_cast<size_t>(stages) * (mt * kATile + b_rows * 128);      // ring
  b += 8 * (2 * stages + 1) + 16;                                       // barriers, tmem slot
  b += static_cast<size_t>(n) * m * 4 + 4;                              // partials
  b += static_cast<size_t>(own) * m * 8 + own * 8;                      // own rows + sums
  b += static_cast<size_t>(nw) * m * 8;                                 // per-warp scratch rows
  b += static_cast<size_t>(own) * k * 8 + static_cast<size_t>(n) * k * 16;  // vote values
  b += static_cast<size_t>(m) * 8 + nw * 64 * 8;                        // votes, keys
  b += static_cast<size_t>(own) * k * 4 + static_cast<size_t>(n) * k * 4;   // selections
  b += static_cast<size_t>(m) * 8 + static_cast<size_t>(m) * tw * 4;   // counts, offsets, bitmaps
  b += nw * 64 * 4 + static_cast<size_t>(m) + 16;                       // warp sel, flags
  return b;
}

cudaError_t launch_front(const CUtensorMap& wr_map, const BoxMaps& x_maps, const FrontArgs& a,
                         size_t smem, cudaStream_t st) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(kFrontCta);
  lc.blockDim = dim3(kFrontThreads);
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kFrontCta;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = 2;
  return cudaLaunchKernelEx(&lc, front_kernel, wr_map, x_maps, a);
}

cudaError_t set_front_smem_limit() {
  return cudaFuncSetAttribute(front_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kFrontSmemLimit);
}

}  // namespace desmoe
