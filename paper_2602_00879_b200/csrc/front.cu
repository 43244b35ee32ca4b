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
  const int b_rows = a.b_rows;        // token box rows (>= n, multiple of 16)
  const int kb_cta = a.kb_per_cta;    // K blocks of this CTA
  const int nwarps = kFrontThreads / 32;
  const int npairs = nwarps / 2;      // one (main, helper) warp pair per token
  // ---- shared memory (identical layout in every CTA: DSMEM offsets) -------------
  const int stage_bytes = mt * kATile + b_rows * 128;
  const int S = a.stages;
  unsigned char* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + static_cast<size_t>(S) * stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* tdone = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tdone + 1);
  float* part = reinterpret_cast<float*>(tmem_slot + 4);                  // [n][m] f32 partial
  const int t0 = (n * static_cast<int>(rank)) / C, t1 = (n * (static_cast<int>(rank) + 1)) / C;
  const int own = t1 - t0;
  const int own_max = (n + C - 1) / C;
  double* xrow = reinterpret_cast<double*>(part + static_cast<size_t>(n) * m +
                                           ((n * m) & 1));                // [own_max][m] logits
  double* erow = xrow + static_cast<size_t>(own_max) * m;                 // [own_max][m] e or p
  double* psum = erow + static_cast<size_t>(own_max) * m;                 // [own_max] softmax s
  double* pmx = psum + own_max;                                           // [own_max] row max
  double* scratch_all = pmx + own_max;                                    // [pairs][m]
  double* otp = scratch_all + static_cast<size_t>(npairs) * m;            // [own_max*k]
  double* dense = otp + own_max * k;                                      // [n][m] vote values
  double* votes = dense + static_cast<size_t>(n) * m;                     // [m]
  uint64_t* wkey_all = reinterpret_cast<uint64_t*>(votes + m);            // [pairs][64]
  int* otop = reinterpret_cast<int*>(wkey_all + npairs * 64);             // [own_max*k]
  int* wsel_all = otop + own_max * k;                                     // [pairs][64]
  int* rankp = wsel_all + npairs * 64;                                    // [4][m] partial ranks
  uint8_t* flag = reinterpret_cast<uint8_t*>(rankp + 4 * m);              // [m]
  __shared__ int warp_tot[kFrontThreads / 32 + 1];
  __shared__ int s_bad;

  const bool vanilla = a.strategy < 0;
  const int depth = a.strategy == 0 ? a.seq_k : k;
  const int box = a.box_index;
  const int n_mma = (n + 15) & ~15;
  const int kb0 = static_cast<int>(rank) * kb_cta;
  const uint32_t xbytes = (16u << box) * 128u;

  // ---- setup: barriers, TMEM, router-weight prefetch (weights are static, so
  // they stream before the previous kernel's output is even waited for) ----------
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
    const uint64_t pol_w = l2_policy_evict_first();
    for (int i = 0; i < kb_cta && i < S; ++i) {
      unsigned char* st = ring + static_cast<size_t>(i) * stage_bytes;
      mbar_arrive_expect_tx(&full[i], mt * kATile + xbytes);
      for (int tl = 0; tl < mt; ++tl)
        tma_load_2d(st + tl * kATile, &wr_map, &full[i], (kb0 + i) * kBK, tl * kBM, pol_w);
    }
  }
  if (warp == 2) tmem_alloc(tmem_slot, a.tmem_cols);
  pdl_launch_dependents();
  pdl_wait();  // x (the previous kernel's output) is complete from here on
  for (int i = tid + static_cast<int>(rank) * kFrontThreads; i < a.zero_words;
       i += kFrontThreads * C)
    a.zero[i] = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (tid == 0) trace(a.trace, a.trace_cap, 11, static_cast<int>(rank));

  // ---- R: split-K router GEMM ---------------------------------------------------
  if (warp == 0 && lane == 0) {
    const uint64_t pol_w = l2_policy_evict_first();
    const uint64_t pol_x = l2_policy_evict_last();
    for (int i = 0; i < kb_cta; ++i) {
      const int s = i % S;
      unsigned char* st = ring + static_cast<size_t>(s) * stage_bytes;
      if (i >= S) {
        mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], mt * kATile + xbytes);
        for (int tl = 0; tl < mt; ++tl)
          tma_load_2d(st + tl * kATile, &wr_map, &full[s], (kb0 + i) * kBK, tl * kBM, pol_w);
      }
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
  // zero the dense vote matrix while the MMA drains (used only by DES)
  if (!vanilla)
    for (int i = tid; i < n * m; i += kFrontThreads) dense[i] = 0.0;
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, a.tmem_cols);
  }
  if (tid == 0) trace(a.trace, a.trace_cap, 12, static_cast<int>(rank));
  cluster_sync();  // #1: all partials parked
  if (tid == 0) trace(a.trace, a.trace_cap, 13, static_cast<int>(rank));

  // ---- L: logits (cluster reduction) -> activation -> top-K, own tokens ----------
  // Warp pair per token: the main warp reduces the logits and selects on the
  // logit order; the helper warp computes e = exp(x - max) and the ordered
  // softmax sum at the same time. Order by logit == order by probability
  // except for rounding ties; token_finish_selection() detects those and
  // re-selects exactly.
  const int pair = warp >> 1;
  const bool main_w = (warp & 1) == 0;
  int* wsel = wsel_all + pair * 64;
  uint64_t* wkey = wkey_all + pair * 64;
  double* scratch = scratch_all + static_cast<size_t>(pair) * m;
  uint32_t part_remote[kFrontCta];
#pragma unroll
  for (int c = 0; c < kFrontCta; ++c) part_remote[c] = dsmem_addr(part, c);
  for (int lt = pair; lt < own_max; lt += npairs) {
    const bool active = lt < own;  // uniform per pair
    const int t = t0 + lt;
    double* xr = xrow + static_cast<size_t>(lt) * m;
    double* er = erow + static_cast<size_t>(lt) * m;
    if (active && main_w) {
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
        xr[i] = x;
        mx = fmax(mx, x);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      if (__any_sync(0xffffffffu, bad) && lane == 0) s_bad = 1;
      if (lane == 0) pmx[lt] = mx;
    }
    named_bar_sync(1 + pair, 64);  // x row + max published to the helper
    if (active && !main_w) {
      const double mx = pmx[lt];
      double ssum = 1.0;
      if (a.act == 0) {
        for (int i = lane; i < m; i += 32) er[i] = exp_f64(xr[i] - mx);
        __syncwarp();
        ssum = 0.0;
        if (lane == 0)
          for (int i = 0; i < m; ++i) ssum += er[i];  // ascending index (gating.cpp:31-33)
      } else if (a.act == 1) {
        for (int i = lane; i < m; i += 32) er[i] = sigmoid_f64(xr[i]);
      } else {
        for (int i = lane; i < m; i += 32) er[i] = xr[i];
      }
      if (lane == 0) psum[lt] = ssum;
    } else if (active && main_w) {
      // softmax: order by logit; sigmoid/identity: order by the probability
      // itself (the main warp computes it — saturation ties are value ties)
      const double* key_src = xr;
      if (a.act != 0) {
        for (int i = lane; i < m; i += 32)
          scratch[i] = a.act == 1 ? sigmoid_f64(xr[i]) : xr[i];
        __syncwarp();
        key_src = scratch;
      }
      const int rounds = k < m ? k + 1 : k;
      warp_topk_fast(key_src, m, rounds, nullptr, wsel, wkey);
    }
    named_bar_sync(1 + pair, 64);  // e row + sum ready
    if (active && main_w) {
      const double ssum = psum[lt];
      const int cnt = token_finish_selection(xr, er, ssum, pmx[lt], a.act, m, k,
                                             vanilla ? 0 : depth, nullptr, m, wsel, scratch);
      if (vanilla) {
        token_write_route(er, ssum, a.act, wsel, cnt, k, t, a.route_idx, a.route_gate,
                          a.route_cnt);
      } else if (lane < k) {
        const int e = wsel[lane];
        otop[lt * k + lane] = e;
        // vote value: the activated gate, or the raw logit (VoteSource::raw_logits)
        otp[lt * k + lane] = a.raw ? xr[e] : p_of(er, ssum, a.act, e);
      }
      __syncwarp();
    }
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
  // scatter every token's selections into the dense [token][expert] vote matrix
  for (int e = tid; e < n * k; e += kFrontThreads) {
    const int t = e / k, j = e - t * k;
    if (j >= depth) continue;
    int ow = C - 1;  // owner CTA: largest r with floor(n r / C) <= t
    while ((n * ow) / C > t) --ow;
    const int lt = t - (n * ow) / C;
    const int x = ld_dsmem_s32(dsmem_addr(otop + lt * k + j, ow));
    dense[t * m + x] = a.strategy == 1 ? ld_dsmem_f64(dsmem_addr(otp + lt * k + j, ow)) : 1.0;
  }
  __syncthreads();
  if (tid == 0) trace(a.trace, a.trace_cap, 20, static_cast<int>(rank));
  for (int i = tid; i < m; i += kFrontThreads) {
    double v = 0.0;  // every token in ascending order (des.cpp:86-91); +0 is exact
    for (int t = 0; t < n; ++t) v += dense[t * m + i];
    votes[i] = v;
    if (a.votes && rank == 0 && a.strategy == 1) a.votes[i] = v;
  }
  __syncthreads();
  if (tid == 0) trace(a.trace, a.trace_cap, 21, static_cast<int>(rank));
  if (a.strategy == 1) {
    // rank of expert i = #experts before it in (vote desc, index asc); four
    // threads per expert each count a quarter of the pool
    for (int w = tid; w < 4 * m; w += kFrontThreads) {
      const int i = w % m, part4 = w / m;
      const uint64_t ki = order_key(votes[i]);
      int rk = 0;
      const int j0 = (m * part4) / 4, j1 = (m * (part4 + 1)) / 4;
      for (int j = j0; j < j1; ++j) {
        const uint64_t kj = order_key(votes[j]);
        rk += (kj > ki) | ((kj == ki) & (j < i));
      }
      rankp[part4 * m + i] = rk;
    }
    __syncthreads();
    for (int i = tid; i < m; i += kFrontThreads)
      flag[i] = static_cast<uint8_t>(rankp[i] + rankp[m + i] + rankp[2 * m + i] + rankp[3 * m + i] <
                                     a.m_core);
  } else {
    for (int i = tid; i < m; i += kFrontThreads) flag[i] = static_cast<uint8_t>(votes[i] > 0.0);
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

  // ---- RR: constrained re-route of own tokens (main warps) ------------------------
  if (main_w) {
    for (int lt = pair; lt < own; lt += npairs) {
      const int t = t0 + lt;
      const double* xr = xrow + static_cast<size_t>(lt) * m;
      const double* er = erow + static_cast<size_t>(lt) * m;
      const double ssum = psum[lt];
      bool covered = false;
      if (nm >= k) {
        const int mine = lane < k ? otop[lt * k + lane] : 0;
        covered = __all_sync(0xffffffffu, lane >= k || flag[mine]);
        if (covered && lane < k) wsel[lane] = mine;
        __syncwarp();
      }
      int cnt = k < nm ? k : nm;
      if (!covered) {
        const double* key_src = xr;
        if (a.act != 0) {
          for (int i = lane; i < m; i += 32) scratch[i] = er[i];
          __syncwarp();
          key_src = scratch;
        }
        const int rounds = cnt < nm ? cnt + 1 : cnt;
        warp_topk_fast(key_src, m, rounds, flag, wsel, wkey);
        cnt = token_finish_selection(xr, er, ssum, pmx[lt], a.act, m, k, 0, flag, nm, wsel,
                                     scratch);
      }
      token_write_route(er, ssum, a.act, wsel, cnt, k, t, a.route_idx, a.route_gate,
                        a.route_cnt);
    }
  }
  if (tid == 0) trace(a.trace, a.trace_cap, 17, static_cast<int>(rank));
  cluster_sync();  // #3: no CTA exits while others may still read its shared memory
}

size_t front_smem_bytes(int n, int m, int k, int stages, int b_rows) {
  const int mt = (m + kBM - 1) / kBM;
  const int own = (n + kFrontCta - 1) / kFrontCta;  // own_max
  const int pairs = kFrontThreads / 64;
  size_t b = 1024;                                                     // alignment slack
  b += static_cast<size_t>(stages) * (mt * kATile + b_rows * 128);      // ring
  b += 8 * (2 * stages + 1) + 16;                                       // barriers, tmem slot
  b += static_cast<size_t>(n) * m * 4 + 4;                              // partials
  b += static_cast<size_t>(own) * m * 16 + own * 16;                    // x/e rows, sums, max
  b += static_cast<size_t>(pairs) * m * 8;                              // scratch rows
  b += static_cast<size_t>(own) * k * 8;                                // own vote values
  b += static_cast<size_t>(n) * m * 8 + static_cast<size_t>(m) * 8;    // dense votes, votes
  b += pairs * 64 * 8 + static_cast<size_t>(own) * k * 4 + pairs * 64 * 4;  // keys, sels
  b += static_cast<size_t>(m) * 16 + static_cast<size_t>(m) + 16;      // partial ranks, flags
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
