// K1 + K2 fused: router GEMM and the whole DES routing stage of one block in
// a single 8-CTA thread-block CLUSTER (one CTA per SM, 16 warps each), for
// every block size N <= 256 and pool size M <= 256.
//
//   R  router GEMM, split-K over the cluster, token-chunked so the partials
//      fit in shared memory: for each chunk of Tc tokens, CTA r multiplies
//      W_r[:, K-slice r] by X[chunk, K-slice r] on tcgen05 (swap-AB: 128
//      expert rows x Tc tokens per M tile, TMA -> SWIZZLE_128B smem -> TMEM)
//      and parks its fp32 partial [Tc][M] in shared memory;
//   L  CTA r owns tokens [r*Tc/8, (r+1)*Tc/8) of every chunk: it sums each
//      logit over the 8 partials in fixed CTA order through distributed
//      shared memory (deterministic logits). Then, data-parallel over the
//      CTA's (token, expert) pairs, the reference's activation in fp64
//      (gating.cpp:10-40): e = exp(x - max) (or the sigmoid); one LANE per
//      token accumulates the softmax sum in ascending expert order
//      (gating.cpp:31-33) while the other warps select each token's top-K on
//      exact (fp32 logit, index) keys (one warp per token, register-resident
//      keys, two REDUX per round); a boundary that exp/division rounding
//      could flip (gap <= 2^-40, or underflow) re-selects exactly on the fp64
//      probabilities with the reference's comparator;
//   V  every CTA gathers all tokens' (expert, weight) selections over DSMEM
//      and computes the coreset redundantly: DES-Vote sums each expert's
//      votes over its tokens in ascending token order (des.cpp:86-91) via a
//      stable counting sort (no dense N x M matrix), then keeps the top
//      floor(beta*M) by (vote desc, index asc) with a rank count
//      (des.cpp:93); DES-Seq takes the union of the top-seq_k (des.cpp:33-45);
//   RR constrained re-route + renormalisation of own tokens (des.cpp:97-118);
//      VANILLA writes topk_route's gates right after L.
// Every intermediate stays on chip. The kernel also zeroes the expert-FFN
// scheduler counters and triggers the programmatic launch of the FFN kernel
// at its start. Rare exact fallbacks live in out-of-line functions so the
// common path's code (and its instruction fetch after an L2 flush) is small.
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

// order-preserving u32 key of an fp32 value (-0 folded onto +0)
__device__ inline uint32_t fkey(float f) {
  uint32_t u = __float_as_uint(f);
  if (u == 0x80000000u) u = 0;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Out-of-line fp64 exp / division (IEEE, as the reference's std::exp and
// operator/): ONE copy of each in the kernel. After the L2 flush every cold
// 128-byte instruction line costs ~0.15 us on this path, so the routing code
// is written for the smallest executed footprint (rolled loops, no sorting
// networks), not for the fewest instructions.
__device__ __noinline__ double f_exp(double x) { return exp(x); }
__device__ __noinline__ double f_div(double a, double b) { return a / b; }

// ---------------------------------------------------------------------------
// Warp selection: the first `rounds` entries of (value desc, index asc) order
// among i < m (m <= 256) allowed by `allow` (nullptr = all). Softmax keys
// are (fp32 logit, index) — exact; sigmoid/identity keys pack the fp64
// activation with the index in its 10 low bits (near-ties re-checked by the
// caller). Each lane keeps its 8 keys in registers; a round is a local max,
// two REDUX and a predicated clear of the winner. sel[r] (shared) = index,
// or -1 once the candidates run out.
// ---------------------------------------------------------------------------
__device__ __noinline__ void warp_rank_select(const float* x, const double* e, int m, int act,
                                              int rounds, const uint8_t* allow, int* sel) {
  const int lane = threadIdx.x & 31;
  uint64_t k[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int i = lane + 32 * s;
    uint64_t key = 0;
    if (i < m && (!allow || allow[i]))
      key = act == 0 ? ((static_cast<uint64_t>(fkey(x[i])) << 32) | static_cast<uint64_t>(1023 - i))
                     : packed_key(e[i], i);
    k[s] = key;
  }
#pragma unroll 1
  for (int r = 0; r < rounds; ++r) {
    uint64_t best = k[0];
#pragma unroll
    for (int s = 1; s < 8; ++s) best = k[s] > best ? k[s] : best;
    const uint32_t hi = __reduce_max_sync(0xffffffffu, static_cast<uint32_t>(best >> 32));
    const uint32_t lo = __reduce_max_sync(
        0xffffffffu, static_cast<uint32_t>(best >> 32) == hi ? static_cast<uint32_t>(best) : 0u);
    const uint64_t win = (static_cast<uint64_t>(hi) << 32) | lo;
    if (lane == 0) sel[r] = win ? 1023 - static_cast<int>(lo & 0x3FFu) : -1;
#pragma unroll
    for (int s = 0; s < 8; ++s) k[s] = k[s] == win ? 0ull : k[s];
  }
  __syncwarp();
}

// Writes a token's route from a rank-ordered selection: experts ascending,
// gates = p / (sum of the selection's p in ascending index order)
// (gating.cpp:73-82, des.cpp:113-116), -1 / 0 padding to k.
// wp: 32 doubles of per-warp scratch.
__device__ __noinline__ void write_route(const double* e, double s, int act, const int* selr,
                                         int cnt, int k, int t, double* wp, int* route_idx,
                                         double* route_gate, int* route_cnt) {
  const int lane = threadIdx.x & 31;
  const int my = lane < cnt ? selr[lane] : 0x7fffffff;
  int pos = 0;  // ascending position among the selected (indices are distinct)
#pragma unroll 1
  for (int j = 0; j < cnt; ++j) pos += __shfl_sync(0xffffffffu, my, j) < my;
  if (lane >= cnt) pos = lane;  // padding slots cnt .. k-1
  double p = 0.0;
  if (lane < cnt) {
    p = act == 0 ? f_div(e[my], s) : e[my];
    wp[pos] = p;
  }
  __syncwarp();
  double tot = 0.0;
  if (lane == 0) {
#pragma unroll 1
    for (int j = 0; j < cnt; ++j) tot += wp[j];
  }
  tot = __shfl_sync(0xffffffffu, tot, 0);
  if (lane < k) {
    const size_t o = static_cast<size_t>(t) * k + pos;
    route_idx[o] = lane < cnt ? my : -1;
    route_gate[o] = lane < cnt ? f_div(p, tot) : 0.0;
  }
  if (lane == 0) route_cnt[t] = cnt;
  __syncwarp();
}

// True if the boundary between ranks b-1 and b of `sel` could order
// differently on the reference's fp64 probabilities (gating.cpp:49-52).
__device__ inline bool risky_boundary(const float* x, const double* e, int act, const int* sel,
                                      int b) {
  const int hi = sel[b - 1], lo = sel[b];
  if (act == 0) {
    const double gap = static_cast<double>(x[hi]) - static_cast<double>(x[lo]);
    return !(gap > 0x1.0p-40) || !(e[lo] > 0x1.0p-960);
  }
  return near_tie(e[hi], e[lo]);
}

// Exact re-selection on the reference's probabilities p = e / s (softmax) or
// p = e (sigmoid/identity) with its comparator. Rare (near-ties only).
__device__ __noinline__ void exact_reselect(const double* e, double s, int act, int m, int want,
                                            const uint8_t* allow, double* scratch, int* sel) {
  const int lane = threadIdx.x & 31;
#pragma unroll 1
  for (int i = lane; i < m; i += 32) scratch[i] = act == 0 ? f_div(e[i], s) : e[i];
  __syncwarp();
  warp_select(scratch, m, want, allow, sel);
}

// timeline marks 0..count-1 of this CTA -> trace buffer as events 40 + i
__device__ __noinline__ void front_dump_marks(const FrontArgs& a, const uint64_t* ts, int tid,
                                              int count) {
  if (!a.trace || tid != 0) return;
  unsigned long long* cur = reinterpret_cast<unsigned long long*>(a.trace);
  const unsigned long long i0 = atomicAdd(cur, static_cast<unsigned long long>(count));
#pragma unroll 1
  for (int i = 0; i < count; ++i)
    if (i0 + i < static_cast<unsigned long long>(a.trace_cap)) {
      a.trace[2 + 2 * (i0 + i)] = (static_cast<uint64_t>(blockIdx.x) << 8) | (40 + i);
      a.trace[3 + 2 * (i0 + i)] = ts[i];
    }
}

}  // namespace

// Shared-memory plan (host and device agree on it).
struct FrontSmem {
  size_t ring, erow, dreg, scratch, partial, xrow, mx, ssum, sel, psel, wsel, wp, own_tok, flag,
      total;
};

__host__ __device__ inline size_t fr_align(size_t v, size_t a) { return (v + a - 1) / a * a; }

__host__ __device__ inline FrontSmem front_smem_plan(int n, int m, int k, int chunk, int own_max,
                                                      int stages, int b_rows) {
  FrontSmem p{};
  const int mt = (m + kBM - 1) / kBM;
  const size_t ring = static_cast<size_t>(stages) * (mt * kATile + b_rows * 128);
  const int words = (n + 31) / 32;
  // region A: GEMM ring, later the fp64 activations + the vote workspace
  p.ring = 0;
  p.erow = 0;
  const size_t erow_b = fr_align(static_cast<size_t>(own_max) * (m + 1) * 8, 16);
  p.dreg = erow_b;
  const size_t nk = static_cast<size_t>(n) * k;
  size_t dreg_b = nk * 4 + nk * 8 + static_cast<size_t>(m) * words * 4 + 2 * m * 4 + 8 + nk * 8 +
                  m * 8 + 4 * m * 4 + 64;
  p.scratch = p.dreg;  // per-warp fallback scratch aliases the vote workspace
  const size_t scr_b = static_cast<size_t>(kFrontThreads / 32) * m * 8;
  if (scr_b > dreg_b) dreg_b = scr_b;
  size_t a_end = erow_b + fr_align(dreg_b, 16);
  if (ring > a_end) a_end = ring;
  // region B: partial logits of the current chunk (read remotely)
  p.partial = fr_align(a_end, 1024);
  size_t o = p.partial + fr_align(static_cast<size_t>(chunk) * m * 4, 16);
  // region C: own tokens' rows and selections (read remotely after L)
  p.xrow = o;
  o += fr_align(static_cast<size_t>(own_max) * m * 4, 16);
  p.mx = o;
  o += fr_align(static_cast<size_t>(own_max) * 4, 16);
  p.ssum = o;
  o += fr_align(static_cast<size_t>(own_max) * 8, 16);
  p.sel = o;
  o += fr_align(static_cast<size_t>(own_max) * 33 * 4, 16);
  p.psel = o;
  o += fr_align(static_cast<size_t>(own_max) * 32 * 8, 16);
  p.wsel = o;
  o += fr_align(static_cast<size_t>(kFrontThreads / 32) * 33 * 4, 16);
  p.wp = o;
  o += static_cast<size_t>(kFrontThreads / 32) * 32 * 8;
  p.own_tok = o;
  o += fr_align(static_cast<size_t>(own_max) * 4, 16);
  p.flag = o;
  o += fr_align(static_cast<size_t>(m) + own_max, 16);
  p.total = o + 1024;  // alignment slack of the dynamic base
  return p;
}

__global__ void __launch_bounds__(kFrontThreads, 1)
    front_kernel(const __grid_constant__ CUtensorMap wr_map, const __grid_constant__ BoxMaps x_maps,
                 FrontArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // align to 1024 B by offsetting the shared array itself, so the compiler
  // keeps the shared address space (LDS/STS instead of generic LD/ST)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bars[2 * 4 + 1];
  __shared__ uint32_t tmem_slot[2];
  __shared__ int s_bad, s_nm;
  __shared__ int warp_tot[kFrontThreads / 32 + 1];
  __shared__ uint64_t s_ts[16];  // timeline marks (trace buffer only)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool tracing = a.trace != nullptr;
#define FRONT_MARK(ev)                          \
  do {                                          \
    if (tracing && tid == 0) s_ts[ev] = gtime(); \
  } while (0)
  FRONT_MARK(0);
  constexpr int C = kFrontCta, NW = kFrontThreads / 32;
  const int rk = static_cast<int>(cluster_rank());
  const int n = a.n, m = a.m, k = a.k, act = a.act;
  const int mt = (m + kBM - 1) / kBM;
  const int Tc = a.chunk, nch = (n + Tc - 1) / Tc;
  const int opc = (Tc * (rk + 1)) / C - (Tc * rk) / C;  // own tokens per full chunk
  const FrontSmem P = front_smem_plan(n, m, k, Tc, a.own_max, a.stages, a.b_rows);
  unsigned char* ring = smem + P.ring;
  double* erow = reinterpret_cast<double*>(smem + P.erow);  // [own][m + 1]
  float* part = reinterpret_cast<float*>(smem + P.partial);  // [Tc][m]
  float* xrow = reinterpret_cast<float*>(smem + P.xrow);     // [own][m]
  float* mxv = reinterpret_cast<float*>(smem + P.mx);
  double* ssum = reinterpret_cast<double*>(smem + P.ssum);
  int* sel = reinterpret_cast<int*>(smem + P.sel);           // [own][33] rank order
  double* psel = reinterpret_cast<double*>(smem + P.psel);   // [own][32]
  int* wsel_all = reinterpret_cast<int*>(smem + P.wsel);     // [NW][33]
  int* own_tok = reinterpret_cast<int*>(smem + P.own_tok);
  uint8_t* flag = smem + P.flag;                             // [m] coreset members
  uint8_t* risky = flag + m;                                 // [own]
  const int ew = m + 1;                                      // erow row stride
  uint64_t* full = bars;
  uint64_t* empty = bars + 4;
  uint64_t* tdone = bars + 8;
  const int S = a.stages;
  const int stage_bytes = mt * kATile + a.b_rows * 128;
  const int kb_cta = a.kb_per_cta;
  const int kb0 = rk * kb_cta;
  const uint32_t xbytes = static_cast<uint32_t>(a.b_rows) * 128u;
  const bool vanilla = a.strategy < 0;
  const int depth = a.strategy == 0 ? a.seq_k : k;

  // ---- setup: barriers, TMEM, router-weight prefetch (weights are static, so
  // they stream before the previous kernel's output is even waited for) ----------
  if (tid == 0) {
    tma_prefetch_desc(&wr_map);
#pragma unroll 1
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tdone, 1);
    fence_mbar_init();
    s_bad = 0;
    const uint64_t pol = l2_policy_evict_first();
#pragma unroll 1
    for (int i = 0; i < kb_cta && i < S; ++i) {
      unsigned char* st = ring + static_cast<size_t>(i) * stage_bytes;
      mbar_arrive_expect_tx(&full[i], mt * kATile + xbytes);
#pragma unroll 1
      for (int tl = 0; tl < mt; ++tl)
        tma_load_2d(st + tl * kATile, &wr_map, &full[i], (kb0 + i) * kBK, tl * kBM, pol);
    }
  }
  if (warp == 2) tmem_alloc(tmem_slot, a.tmem_cols);
  pdl_launch_dependents();
  pdl_wait();  // x (the previous kernel's output) is complete from here on
#pragma unroll 1
  for (int i = tid + rk * kFrontThreads; i < a.zero_words; i += kFrontThreads * C) a.zero[i] = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_slot[0];
  FRONT_MARK(1);

  // ---- R + L1: per token chunk, split-K GEMM, then the owners' logit sums ----------
  int own = 0;
#pragma unroll 1
  for (int c = 0; c < nch; ++c) {
    const int c0 = c * Tc;
    const int nc = n - c0 < Tc ? n - c0 : Tc;
    const int n_mma = (nc + 15) & ~15;
    if (warp == 0 && lane == 0) {
      const uint64_t pol_w = l2_policy_evict_first();
      const uint64_t pol_x = l2_policy_evict_last();
#pragma unroll 1
      for (int i = 0; i < kb_cta; ++i) {
        const int it = c * kb_cta + i, s = it % S;
        unsigned char* st = ring + static_cast<size_t>(s) * stage_bytes;
        if (it >= S) {
          mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], mt * kATile + xbytes);
#pragma unroll 1
          for (int tl = 0; tl < mt; ++tl)
            tma_load_2d(st + tl * kATile, &wr_map, &full[s], (kb0 + i) * kBK, tl * kBM, pol_w);
        }
        tma_load_2d(st + mt * kATile, &x_maps.map[a.box_index], &full[s], (kb0 + i) * kBK, c0,
                    pol_x);
      }
    } else if (warp == 1) {
      const uint32_t idesc = idesc_bf16_f32(kBM, n_mma);
#pragma unroll 1
      for (int i = 0; i < kb_cta; ++i) {
        const int it = c * kb_cta + i, s = it % S;
        mbar_wait(&full[s], (it / S) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a0 = smem_u32(ring + static_cast<size_t>(s) * stage_bytes);
          const uint32_t b0 = a0 + mt * kATile;
#pragma unroll 1
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
      // drain TMEM: partial[t][e] of this CTA's K slice
      mbar_wait(tdone, c & 1);
      tc_fence_after();
      const int q = warp & 3;
      const int r = q * 32 + lane;
#pragma unroll 1
      for (int tl = 0; tl < mt; ++tl) {
        const int e = tl * kBM + r;
        const uint32_t lb = tmem_base + tl * 256 + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll 1
        for (int cc = 0; cc < n_mma; cc += 16) {
          float v[16];
          tmem_ld16(lb + cc, v);
          if (e < m) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (cc + j < nc) part[(cc + j) * m + e] = v[j];
          }
        }
      }
      tc_fence_before();
    }
    __syncthreads();
    FRONT_MARK(2);
    cluster_sync();  // this chunk's partials are parked in every CTA
    FRONT_MARK(3);
    // owners: logits = sum of the 8 partials in fixed CTA order (deterministic)
    const int lo = (nc * rk) / C, hi = (nc * (rk + 1)) / C;
    const int ob = c * opc;
    const int cnt = (hi - lo) * m;
    const uint32_t pbase = smem_u32(part);
#pragma unroll 1
    for (int w = tid; w < cnt; w += kFrontThreads) {
      const int j = w / m, e = w - j * m;
      const uint32_t off = pbase + static_cast<uint32_t>(((lo + j) * m + e) * 4);
      float v[C];
#pragma unroll
      for (int r = 0; r < C; ++r) {
        uint32_t ad;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ad) : "r"(off), "r"(r));
        v[r] = ld_dsmem_f32(ad);
      }
      float acc = 0.0f;
#pragma unroll
      for (int r = 0; r < C; ++r) acc += v[r];
      xrow[(ob + j) * m + e] = acc;
      if (a.logits_out) a.logits_out[static_cast<size_t>(c0 + lo + j) * m + e] = acc;
    }
    if (tid < hi - lo) own_tok[ob + tid] = c0 + lo + tid;
    own = ob + (hi - lo);
    if (c + 1 < nch) cluster_sync();  // partials consumed before the next chunk's drain
  }
  __syncthreads();
  FRONT_MARK(4);
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, a.tmem_cols);
  }

  // ---- L2: row max + finiteness (warp per token) ----------------------------------
#pragma unroll 1
  for (int j = warp; j < own; j += NW) {
    uint32_t best = 0;
    bool bad = false;
#pragma unroll 1
    for (int i = lane; i < m; i += 32) {
      const float v = xrow[j * m + i];
      bad |= !isfinite(v);
      const uint32_t kk = fkey(v);
      best = kk > best ? kk : best;
    }
    best = __reduce_max_sync(0xffffffffu, best);
    if (__any_sync(0xffffffffu, bad) && lane == 0) s_bad = 1;
    if (lane == 0) mxv[j] = __uint_as_float((best & 0x80000000u) ? (best & 0x7fffffffu) : ~best);
  }
  __syncthreads();
  FRONT_MARK(5);
  // ---- L3: activation in fp64, data-parallel over (own token, expert) ----------
#pragma unroll 1
  for (int w = tid; w < own * m; w += kFrontThreads) {
    const int j = w / m, i = w - j * m;
    const double x = static_cast<double>(xrow[w]);
    double e = x;
    if (act < 2) {
      const double ex = f_exp(act == 0 ? x - static_cast<double>(mxv[j]) : -x);
      e = act == 0 ? ex : f_div(1.0, 1.0 + ex);  // softmax numerator / sigmoid
    }
    erow[j * ew + i] = e;
  }
  __syncthreads();
  FRONT_MARK(6);
  // ---- L4: ordered softmax sums (one lane per token, last warp) || top-K (others)
  if (warp == NW - 1) {
#pragma unroll 1
    for (int j = lane; j < own; j += 32) {
      double s = 1.0;
      if (act == 0) {
        s = 0.0;
        const double* er = erow + j * ew;
#pragma unroll 1
        for (int i = 0; i < m; ++i) s += er[i];  // ascending index (gating.cpp:31-33)
      }
      ssum[j] = s;
    }
  } else {
    const int want = k < m ? k : m;
    const int rounds = want < m ? want + 1 : want;
#pragma unroll 1
    for (int j = warp; j < own; j += NW - 1) {
      int* sj = sel + j * 33;
      const float* xr = xrow + j * m;
      const double* er = erow + j * ew;
      warp_rank_select(xr, er, m, act, rounds, nullptr, sj);
      if (lane == 0) {
        bool r = want < m && risky_boundary(xr, er, act, sj, want);
        if (!vanilla && depth < want) r |= risky_boundary(xr, er, act, sj, depth);
        risky[j] = r;
      }
    }
  }
  __syncthreads();
  FRONT_MARK(7);
  if (s_bad && tid == 0) atomicOr(a.err, 1);
  // ---- L5: exact fallback for near-ties; vote weights / vanilla routes ---------------
  {
    const int want = k < m ? k : m;
    int* wsel = wsel_all + warp * 33;
    double* wp = reinterpret_cast<double*>(smem + P.wp) + warp * 32;
    double* scratch = reinterpret_cast<double*>(smem + P.scratch) + warp * m;
#pragma unroll 1
    for (int j = warp; j < own; j += NW) {
      int* sj = sel + j * 33;
      const double* er = erow + j * ew;
      const double s = ssum[j];
      if (risky[j]) exact_reselect(er, s, act, m, want, nullptr, scratch, sj);  // rare
      if (vanilla) {
        write_route(er, s, act, sj, want, k, own_tok[j], wp, a.route_idx, a.route_gate,
                    a.route_cnt);
      } else if (lane < want) {
        const int e = sj[lane];
        psel[j * 32 + lane] = a.raw ? static_cast<double>(xrow[j * m + e])
                                    : (act == 0 ? f_div(er[e], s) : er[e]);
      }
      __syncwarp();
    }
  }
  __syncthreads();
  FRONT_MARK(8);
  cluster_sync();  // #2: every CTA's selections are visible
  FRONT_MARK(9);
  if (vanilla) {  // every remote read (partials) happened before #2
    front_dump_marks(a, s_ts, tid, 10);
    return;
  }

  // ---- V: block coreset, redundantly in every CTA ------------------------------------
  const int words = (n + 31) / 32;
  const int nk = n * k;
  int* tri_e = reinterpret_cast<int*>(smem + P.dreg);                          // [n][k]
  double* tri_p = reinterpret_cast<double*>(smem + P.dreg + fr_align(nk * 4, 8));  // [n][k]
  uint32_t* bits = reinterpret_cast<uint32_t*>(tri_p + nk);                    // [m][words]
  int* ecnt = reinterpret_cast<int*>(bits + m * words);                        // [m]
  int* eoff = ecnt + m;                                                        // [m]
  double* val = reinterpret_cast<double*>(
      smem + fr_align(static_cast<size_t>(reinterpret_cast<unsigned char*>(eoff + m) - smem), 8));
  double* votes = val + nk;                                                    // [m]
  int* rankp = reinterpret_cast<int*>(votes + m);                              // [4][m]
#pragma unroll 1
  for (int i = tid; i < m; i += kFrontThreads) {
    flag[i] = 0;
    ecnt[i] = 0;
  }
#pragma unroll 1
  for (int i = tid; i < m * words; i += kFrontThreads) bits[i] = 0;
  __syncthreads();
  FRONT_MARK(10);
  // gather every token's top-`depth` from its owner CTA (DSMEM)
#pragma unroll 1
  for (int w = tid; w < n * depth; w += kFrontThreads) {
    const int t = w / depth, j = w - t * depth;
    const int c = t / Tc, l = t - c * Tc;
    const int nc = n - c * Tc < Tc ? n - c * Tc : Tc;
    int ow = C - 1;  // owner: largest r with floor(nc r / C) <= l
    while ((nc * ow) / C > l) --ow;
    const int lt = c * ((Tc * (ow + 1)) / C - (Tc * ow) / C) + (l - (nc * ow) / C);
    const int e = ld_dsmem_s32(dsmem_addr(sel + lt * 33 + j, ow));
    if (a.strategy == 1) {
      tri_e[t * k + j] = e;
      tri_p[t * k + j] = ld_dsmem_f64(dsmem_addr(psel + lt * 32 + j, ow));
      atomicAdd(&ecnt[e], 1);
      atomicOr(&bits[e * words + (t >> 5)], 1u << (t & 31));
    } else {
      flag[e] = 1;  // DES-Seq: union of the top-seq_k
    }
  }
  __syncthreads();
  FRONT_MARK(11);
  if (a.strategy == 1) {
    // stable counting sort by expert (ascending token within an expert)
    if (warp == 0) {
      int base = 0;
#pragma unroll 1
      for (int b0 = 0; b0 < m; b0 += 32) {
        const int i = b0 + lane;
        const int v = i < m ? ecnt[i] : 0;
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        if (i < m) eoff[i] = base + incl - v;
        base += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    __syncthreads();
#pragma unroll 1
    for (int w = tid; w < nk; w += kFrontThreads) {
      const int t = w / k;
      const int e = tri_e[w];
      const uint32_t* b = bits + e * words;
      int before = 0;
#pragma unroll 1
      for (int q = 0; q < (t >> 5); ++q) before += __popc(b[q]);
      before += __popc(b[t >> 5] & ((1u << (t & 31)) - 1u));
      val[eoff[e] + before] = tri_p[w];
    }
    __syncthreads();
#pragma unroll 1
    for (int i = tid; i < m; i += kFrontThreads) {
      double v = 0.0;  // every token in ascending order (des.cpp:86-91)
      const double* vv = val + eoff[i];
#pragma unroll 1
      for (int q = 0; q < ecnt[i]; ++q) v += vv[q];
      votes[i] = v;
      if (a.votes && rk == 0) a.votes[i] = v;
    }
    __syncthreads();
    // rank of expert i = #experts before it in (vote desc, index asc)
#pragma unroll 1
    for (int w = tid; w < 4 * m; w += kFrontThreads) {
      const int i = w % m, part4 = w / m;
      const uint64_t ki = order_key(votes[i]);
      int r = 0;
      const int j0 = (m * part4) / 4, j1 = (m * (part4 + 1)) / 4;
#pragma unroll 1
      for (int j = j0; j < j1; ++j) {
        const uint64_t kj = order_key(votes[j]);
        r += (kj > ki) | ((kj == ki) & (j < i));
      }
      rankp[part4 * m + i] = r;
    }
    __syncthreads();
#pragma unroll 1
    for (int i = tid; i < m; i += kFrontThreads)
      flag[i] = static_cast<uint8_t>(rankp[i] + rankp[m + i] + rankp[2 * m + i] + rankp[3 * m + i] <
                                     a.m_core);
    __syncthreads();
  }
  // ascending member list (block scan over chunks of kFrontThreads experts)
  {
    int base = 0;
#pragma unroll 1
    for (int b0 = 0; b0 < m; b0 += kFrontThreads) {
      const int i = b0 + tid;
      const int f = i < m ? flag[i] : 0;
      const uint32_t bal = __ballot_sync(0xffffffffu, f);
      if (lane == 0) warp_tot[warp] = __popc(bal);
      __syncthreads();
      if (tid == 0) {
        int acc = 0;
#pragma unroll 1
        for (int w = 0; w < NW; ++w) {
          const int cc = warp_tot[w];
          warp_tot[w] = acc;
          acc += cc;
        }
        warp_tot[NW] = acc;
      }
      __syncthreads();
      if (f && rk == 0 && a.members)
        a.members[base + warp_tot[warp] + __popc(bal & ((1u << lane) - 1u))] = i;
      base += warp_tot[NW];
      __syncthreads();
    }
    if (tid == 0) {
      s_nm = base;
      if (rk == 0 && a.n_members) *a.n_members = base;
    }
    __syncthreads();
  }
  const int nm = s_nm;
  FRONT_MARK(12);

  // ---- RR: constrained re-route of own tokens (warp per token) ----------------------
  {
    int* wsel = wsel_all + warp * 33;
    double* wp = reinterpret_cast<double*>(smem + P.wp) + warp * 32;
    double* scratch = reinterpret_cast<double*>(smem + P.scratch) + warp * m;
#pragma unroll 1
    for (int j = warp; j < own; j += NW) {
      const int* sj = sel + j * 33;
      const float* xr = xrow + j * m;
      const double* er = erow + j * ew;
      const double s = ssum[j];
      bool covered = false;
      if (nm >= k) {
        const int mine = lane < k ? sj[lane] : 0;
        covered = __all_sync(0xffffffffu, lane >= k || flag[mine]);
        if (covered && lane < k) wsel[lane] = mine;
        __syncwarp();
      }
      const int cnt = k < nm ? k : nm;
      if (!covered) {
        const int rounds = cnt < nm ? cnt + 1 : cnt;
        warp_rank_select(xr, er, m, act, rounds, flag, wsel);  // rank order
        const bool r = cnt < nm && risky_boundary(xr, er, act, wsel, cnt);
        if (r) exact_reselect(er, s, act, m, cnt, flag, scratch, wsel);  // rare
      }
      write_route(er, s, act, wsel, cnt, k, own_tok[j], wp, a.route_idx, a.route_gate,
                  a.route_cnt);
    }
  }
  FRONT_MARK(13);
  cluster_sync();  // #3: no CTA exits while others may still read its shared memory
  FRONT_MARK(14);
  front_dump_marks(a, s_ts, tid, 15);
#undef FRONT_MARK
}

// Host plan: token chunk, pipeline depth, shared memory. Returns false when
// the shape is outside the kernel's envelope.
bool front_plan(int n, int m, int k, int d, FrontArgs* a, size_t* smem) {
  if (n < 1 || n > 256 || m < 1 || m > 256 || k < 1 || k > 32 || k > m) return false;
  if (d % (kBK * kFrontCta)) return false;
  const int mt = (m + kBM - 1) / kBM;
  const int kb_cta = (d / kBK) / kFrontCta;
  int chunk = n;
  for (;;) {
    int b_rows = 16;
    while (b_rows < chunk) b_rows <<= 1;
    const int nch = (n + chunk - 1) / chunk;
    const int own_max = nch * ((chunk + kFrontCta - 1) / kFrontCta);
    int stages = kb_cta < 4 ? kb_cta : 4;
    FrontSmem p{};
    for (; stages >= 1; --stages) {
      p = front_smem_plan(n, m, k, chunk, own_max, stages, b_rows);
      if (p.total <= static_cast<size_t>(kFrontSmemLimit)) break;
    }
    const bool deep_enough = stages >= 2 || kb_cta == 1;
    if (stages >= 1 && p.total <= static_cast<size_t>(kFrontSmemLimit) && deep_enough) {
      int bi = 0;
      while ((16 << bi) < b_rows) ++bi;
      a->chunk = chunk;
      a->own_max = own_max;
      a->stages = stages;
      a->b_rows = b_rows;
      a->box_index = bi;
      a->kb_per_cta = kb_cta;
      a->tmem_cols = mt * 256;
      *smem = p.total;
      return true;
    }
    if (chunk <= 16) return false;
    chunk = ((chunk / 2) + 15) & ~15;
  }
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
