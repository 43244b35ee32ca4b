// K1 + K2 fused: router GEMM and the whole DES routing stage of one block in
// a single 8-CTA thread-block CLUSTER (one CTA per SM, 16 warps each), for
// every block size N <= 256 and pool size M <= 256.
//
//   (blocks > 32 tokens or pools > 128 experts: R runs ahead in
//      router_cluster_kernel, one cluster per 32 tokens x 128 experts, and
//      this kernel reads the logits: FrontArgs::tsplit == 3)
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
//   V  every token's owner pushes its top-`depth` (ids, weights) to every CTA
//      over DSMEM; every CTA computes the votes redundantly: the reference
//      sums each column of its masked N x M matrix (des.cpp:73-91) in
//      ascending token order, zeros included; zeros leave an fp64 sum
//      unchanged, so the (token, expert) pairs are bucketed by expert with a
//      stable counting sort and each expert sums its own bucket in token
//      order — the same additions, no N x M matrix. The coreset = top
//      floor(beta*M) by (vote desc, index asc) via a rank count (des.cpp:93),
//      split over the cluster for pools > 64 (membership words exchanged
//      over DSMEM); DES-Seq takes the union of the top-seq_k (des.cpp:33-45);
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

// split cluster barrier: arrive (release: this thread's shared writes become
// visible cluster-wide; relaxed: nothing to publish) ... wait (acquire)
__device__ inline void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ inline void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ inline void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
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

// Asynchronous remote shared-memory stores that complete_tx on the
// destination CTA's mbarrier: data is pushed to its consumer and signalled
// without any cluster-scope release fence (those compile to a gpu-scope
// MEMBAR, measured at ~2.5 us right after the router GEMM's bulk copies).
__device__ inline void st_async_b32(uint32_t raddr, uint32_t v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                   raddr),
               "r"(v), "r"(rbar)
               : "memory");
}
__device__ inline void st_async_b64(uint32_t raddr, uint64_t v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(
                   raddr),
               "l"(v), "r"(rbar)
               : "memory");
}
// bulk copy of `bytes` (multiple of 16) from this CTA's shared memory to
// another CTA's (TMA engine), completing tx on that CTA's mbarrier
__device__ inline void bulk_s2cluster(uint32_t rdst, uint32_t src, uint32_t bytes, uint32_t rbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(rdst),
      "r"(src), "r"(bytes), "r"(rbar)
      : "memory");
}

__device__ inline uint32_t mapa_u32(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ inline void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
}
// chunk-local token t's owner CTA (largest r with floor(nc r / C) <= t)
__device__ inline int token_owner(int t, int nc) {
  int r = kFrontCta - 1;
#pragma unroll 1
  while ((nc * r) / kFrontCta > t) --r;
  return r;
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
__device__ __noinline__ double f_exp(double x, const unsigned long long* tab) {
  return glibc_exp(x, tab);  // bit-identical to the reference's std::exp (libm_exp.cuh)
}
__device__ __noinline__ double f_div(double a, double b) { return a / b; }

// ---------------------------------------------------------------------------
// Warp selection: the first `rounds` entries of (logit desc, index asc) order
// among i < m (m <= 512) allowed by `allow` (nullptr = all). Every
// activation is monotone in the logit, so the logit order is the order of
// the reference's gate values except where rounding makes gates tie — the
// caller's boundary check (risky_boundary) sends those to the exact path.
// One 32-bit key per candidate: the order key of the fp32 logit with its 8
// low bits replaced by (255 - index) (9 bits, 511 - index, for pools of
// 257-512), so ONE REDUX per round picks (logit desc, index asc) — exact
// unless two logits agree in their top 24 (23) key bits, which the boundary
// check also catches. P keys per lane (m <= 32 P).
// sel[r] (shared) = index, or -1 once the candidates run out.
// ---------------------------------------------------------------------------
__device__ inline uint32_t sel_key(float x, int i) {
  return (fkey(x) & 0xFFFFFF00u) | static_cast<uint32_t>(255 - i);
}
// pools of 257-512 experts (logits-in front): 9 index bits, 23 key bits
__device__ inline int key_ibits(int m) { return m > 256 ? 9 : 8; }
__device__ inline uint32_t sel_key_b(float x, int i, int ib) {
  const uint32_t lo = (1u << ib) - 1u;
  return (fkey(x) & ~lo) | (lo - static_cast<uint32_t>(i));
}

template <int P>
__device__ __noinline__ void warp_rank_select_p(const float* x, int m, int rounds,
                                                const uint8_t* allow, int* sel) {
  const int lane = threadIdx.x & 31;
  const int ib = P > 8 ? 9 : 8;  // index bits of the key (m <= 32 P)
  const uint32_t lo = (1u << ib) - 1u;
  uint32_t k[P];
#pragma unroll
  for (int s = 0; s < P; ++s) {
    const int i = lane + 32 * s;
    k[s] = (i < m && (!allow || allow[i])) ? sel_key_b(x[i], i, ib) : 0u;
  }
#pragma unroll 1
  for (int r = 0; r < rounds; ++r) {
    uint32_t best = k[0];
#pragma unroll
    for (int s = 1; s < P; ++s) best = k[s] > best ? k[s] : best;
    const uint32_t win = __reduce_max_sync(0xffffffffu, best);
    if (lane == 0) sel[r] = win ? static_cast<int>(lo - (win & lo)) : -1;
#pragma unroll
    for (int s = 0; s < P; ++s) k[s] = k[s] == win ? 0u : k[s];
  }
  __syncwarp();
}

__device__ inline void warp_rank_select(const float* x, int m, int rounds, const uint8_t* allow,
                                        int* sel) {
  if (m <= 64)
    warp_rank_select_p<2>(x, m, rounds, allow, sel);
  else if (m <= 128)
    warp_rank_select_p<4>(x, m, rounds, allow, sel);
  else if (m <= 256)
    warp_rank_select_p<8>(x, m, rounds, allow, sel);
  else
    warp_rank_select_p<16>(x, m, rounds, allow, sel);
}

// Writes a token's route from a rank-ordered selection: experts ascending,
// gates = p / (sum of the selection's p in ascending index order)
// (gating.cpp:73-82, des.cpp:113-116), -1 / 0 padding to k.
// wp: 32 doubles of per-warp scratch.
__device__ __noinline__ void write_route(const double* e, double s, int act, const int* selr,
                                         int cnt, int k, int t, double* wp, int* route_idx,
                                         double* route_gate, int* route_cnt,
                                         uint64_t* route_words, uint32_t tag) {
  const int lane = threadIdx.x & 31;
  const int my = lane < cnt ? selr[lane] : 0x7fffffff;
  int pos = 0;  // ascending position among the selected (indices are distinct)
#pragma unroll 1
  for (int j = 0; j < cnt; ++j) pos += __shfl_sync(0xffffffffu, my, j) < my;  // (cnt <= 32)
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
    const double g = lane < cnt ? f_div(p, tot) : 0.0;
    route_idx[o] = lane < cnt ? my : -1;
    route_gate[o] = g;
    // the FFN kernel polls these (tagged with the call number) instead of
    // waiting for this kernel to complete
    if (route_words)
      route_words[o] = route_word(tag, lane < cnt ? my : kPadExpert, static_cast<float>(g));
  }
  if (lane == 0) route_cnt[t] = cnt;
  __syncwarp();
}

// True if the boundary between ranks b-1 and b of `sel` could order
// differently on the reference's fp64 gate values (gating.cpp:49-52): a
// logit gap exp/division rounding could close (<= 2^-40) or an underflowing
// rejected gate (softmax), or gates within 2^-40 relative of each other
// (sigmoid/identity).
__device__ inline bool fp64_risky(const float* x, const double* e, int act, const int* sel, int b) {
  const int hi = sel[b - 1], lo = sel[b];
  if (act == 0) {
    const double gap = static_cast<double>(x[hi]) - static_cast<double>(x[lo]);
    return !(gap > 0x1.0p-40) || !(e[lo] > 0x1.0p-960);
  }
  return near_tie(e[hi], e[lo]);
}
// ... or, for the fast selection's keys, equal truncated keys (index-ordered
// by the fast path).
__device__ inline bool risky_boundary(const float* x, const double* e, int act, const int* sel,
                                      int b, int m) {
  const int hi = sel[b - 1], lo = sel[b];
  // (the fast keys keep the top 32 - key_ibits(m) bits of the fp32 order key)
  if (((fkey(x[hi]) ^ fkey(x[lo])) >> key_ibits(m)) == 0) return true;
  return fp64_risky(x, e, act, sel, b);
}

// The first `rounds` entries of (fp32 logit desc, index asc) order, exactly:
// full 32-bit logit keys, then the lowest index among the keys that won —
// two REDUX per round. For boundaries the truncated keys cannot order.
__device__ __noinline__ void warp_rank_select_exact32(const float* x, int m, int rounds,
                                                      const uint8_t* allow, int* sel) {
  const int lane = threadIdx.x & 31;
  uint32_t k[16];  // m <= 512
#pragma unroll
  for (int s = 0; s < 16; ++s) {
    const int i = lane + 32 * s;
    k[s] = (i < m && (!allow || allow[i])) ? fkey(x[i]) : 0u;  // fkey > 0 for every float
  }
#pragma unroll 1
  for (int r = 0; r < rounds; ++r) {
    uint32_t best = k[0];
#pragma unroll
    for (int s = 1; s < 16; ++s) best = k[s] > best ? k[s] : best;
    const uint32_t win = __reduce_max_sync(0xffffffffu, best);
    uint32_t idx = 0xffffffffu;
#pragma unroll
    for (int s = 15; s >= 0; --s)
      if (win && k[s] == win) idx = static_cast<uint32_t>(lane + 32 * s);
    const uint32_t wi = __reduce_min_sync(0xffffffffu, idx);
    if (lane == 0) sel[r] = win ? static_cast<int>(wi) : -1;
#pragma unroll
    for (int s = 0; s < 16; ++s)
      if (win && static_cast<uint32_t>(lane + 32 * s) == wi) k[s] = 0u;
  }
  __syncwarp();
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

// A boundary the fast selection could not order (risky_boundary): re-select
// on exact fp32 logit keys first (m <= 512); only a boundary that is still
// ambiguous on the fp64 gates (equal logits, gap <= 2^-40, underflow) pays
// for the full fp64 re-selection (measured ~13 us for one token at M = 256,
// where the fp32 re-selection costs ~1 us). `b2` < want: a second boundary
// (DES-Seq's seq_k) that must be exact too.
__device__ __noinline__ void fix_boundary(const float* x, const double* e, double s, int act,
                                          int m, int want, int b2, const uint8_t* allow,
                                          double* scratch, int* sel) {
  warp_rank_select_exact32(x, m, want < m ? want + 1 : want, allow, sel);
  bool r = false;
  if (want < m && sel[want] >= 0) r = fp64_risky(x, e, act, sel, want);
  if (b2 > 0 && b2 < want) r |= fp64_risky(x, e, act, sel, b2);
  if (r) exact_reselect(e, s, act, m, want, allow, scratch, sel);
}

// timeline marks 0..count-1 of this CTA -> trace buffer as events 100 + i
__device__ __noinline__ void front_dump_marks(uint64_t* trace, int cap, const uint64_t* ts,
                                              int tid, int count) {
  if (!trace || tid != 0) return;
  unsigned long long* cur = reinterpret_cast<unsigned long long*>(trace);
  const unsigned long long i0 = atomicAdd(cur, static_cast<unsigned long long>(count));
  for (int i = 0; i < count; ++i)
    if (i0 + i < static_cast<unsigned long long>(cap)) {
      trace[2 + 2 * (i0 + i)] = (static_cast<uint64_t>(blockIdx.x) << 8) | (100 + i);
      trace[3 + 2 * (i0 + i)] = ts[i];
    }
}

// Publishes the ascending list of flagged experts (coreset / union): the
// tagged words the expert-FFN kernel polls to start streaming weights, plus
// the C-ABI outputs members / n_members. One warp.
__device__ __noinline__ void publish_list(const uint8_t* flag, int m, uint32_t tag, uint32_t* pub,
                                          int* members, int* n_members) {
  const int lane = threadIdx.x & 31;
  int base = 0;
#pragma unroll 1
  for (int b0 = 0; b0 < m; b0 += 32) {
    const int i = b0 + lane;
    const bool f = i < m && flag[i];
    const uint32_t bal = __ballot_sync(0xffffffffu, f);
    const int pos = base + __popc(bal & ((1u << lane) - 1u));
    if (f) {
      if (pub) pub[1 + pos] = pub_word(tag, i);
      if (members) members[pos] = i;
    }
    base += __popc(bal);
  }
  if (lane == 0) {
    if (pub) pub[0] = pub_word(tag, base);
    if (n_members) *n_members = base;
  }
  __syncwarp();
}

// Global writes nobody in the cluster reads, issued after the last cluster
// barrier so no release has to wait for them: the fp32 logits (for
// desmoe_layer_logits) and the zeroed expert-FFN counters.
__device__ __noinline__ void front_tail(float* logits_out, const float* xrow, const int* own_tok,
                                        int own, int m, int tid) {
  if (!logits_out) return;
#pragma unroll 1
  for (int w = tid; w < own * m; w += kFrontThreads) {
    const int j = w / m, e = w - j * m;
    logits_out[static_cast<size_t>(own_tok[j]) * m + e] = xrow[w];
  }
}

}  // namespace

// L3 activation over the CTA's (own token, expert) pairs, threads t0, t0 +
// stride, ...: softmax numerators exp(x - max) (gating.cpp:24-38) four per
// thread in flight and inlined (an out-of-line call per element serialised
// its latency chain: C3 N=256 -1.4 us), sigmoid / identity through the
// out-of-line helpers; the reference's fp64 operations either way.
// (kUnroll: the large-block path. Small blocks run a few exps per thread
// once, where the 4-wide inlined body's instruction fetch cost more than it
// saved: C3 N = 32 / 64 activation +1.4 / +1.0 us.)
template <bool kUnroll>
__device__ __forceinline__ void activate_rows(const float* xrow, const float* mxv, double* erow,
                                              int ew, int own, int m, int act,
                                              const unsigned long long* tab, int t0, int stride) {
  int w0 = t0;
  if (kUnroll && act == 0) {
#pragma unroll 1
    for (; w0 + 3 * stride < own * m; w0 += 4 * stride) {
      double ex[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int w = w0 + u * stride;
        ex[u] = glibc_exp(static_cast<double>(xrow[w]) - static_cast<double>(mxv[w / m]), tab);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int w = w0 + u * stride;
        const int j = w / m, i = w - j * m;
        erow[j * ew + i] = ex[u];
      }
    }
  }
#pragma unroll 1
  for (int w = w0; w < own * m; w += stride) {
    const int j = w / m, i = w - j * m;
    const double x = static_cast<double>(xrow[w]);
    double e = x;
    if (act < 2) {
      const double ex = f_exp(act == 0 ? x - static_cast<double>(mxv[j]) : -x, tab);
      e = act == 0 ? ex : f_div(1.0, 1.0 + ex);  // softmax numerator / sigmoid
    }
    erow[j * ew + i] = e;
  }
}

// Shared-memory plan (host and device agree on it).
struct FrontSmem {
  size_t ring, erow, dreg, scratch, partial, xrow, mx, ssum, sel, wsel, wp, own_tok, flag,
      allsel, allp, stage, total;
};

__host__ __device__ inline size_t fr_align(size_t v, size_t a) { return (v + a - 1) / a * a; }

__host__ __device__ inline FrontSmem front_smem_plan(int n, int m, int k, int chunk, int own_max,
                                                      int stages, int b_rows, int vote_rows,
                                                      int tsplit) {
  FrontSmem p{};
  const int mt = (m + kBM - 1) / kBM;
  const size_t ring = static_cast<size_t>(stages) * (mt * kATile + b_rows * 128);
  // region A: GEMM ring, later the fp64 activations + the vote workspace
  p.ring = 0;
  p.erow = 0;
  const size_t erow_b = fr_align(static_cast<size_t>(own_max) * (m + 1) * 8, 16);
  p.dreg = erow_b;
  // vote buckets: token bitmask per expert [m][ceil(n/32)] + offsets [m+1] +
  // the bucketed weights [n][k] f64; later votes + keys + rank parts
  (void)vote_rows;
  size_t dreg_b = fr_align(static_cast<size_t>(m * ((n + 31) / 32) + m + 1) * 4, 16) +
                  static_cast<size_t>(n) * k * 8;
  const size_t rank_b = static_cast<size_t>(m) * (8 + 8 + 16 * 4) + 64;
  if (rank_b > dreg_b) dreg_b = rank_b;
  p.scratch = p.dreg;  // per-warp fallback scratch aliases the vote workspace
  const size_t scr_b = static_cast<size_t>(kFrontThreads / 32) * m * 8;
  if (scr_b > dreg_b) dreg_b = scr_b;
  size_t a_end = erow_b + fr_align(dreg_b, 16);
  if (ring > a_end) a_end = ring;
  // region B: the partial logits pushed to this CTA for its own tokens of the
  // current chunk: [sender][own][m]
  p.partial = fr_align(a_end, 1024);
  // (token split: no partials are exchanged)
  const int ocm = tsplit ? 0 : (chunk + kFrontCta - 1) / kFrontCta;
  const int m4 = (m + 3) & ~3;
  size_t o = p.partial + fr_align(static_cast<size_t>(kFrontCta) * ocm * m4 * 4, 16);
  p.stage = o;  // this CTA's own partial [chunk][m4], copied out in owner blocks
  o += tsplit ? 0 : fr_align(static_cast<size_t>(chunk) * m4 * 4, 16);
  // every token's selection pushed by its owner: [n][k] ids + weights
  p.allsel = o;
  o += fr_align(static_cast<size_t>(n) * k * 4, 16);
  p.allp = o;
  o += fr_align(static_cast<size_t>(n) * k * 8, 16);
  // region C: own tokens' rows and selections (read remotely after L)
  p.xrow = o;
  o += fr_align(static_cast<size_t>(own_max) * m * 4, 16);
  p.mx = o;
  o += fr_align(static_cast<size_t>(own_max) * 4, 16);
  p.ssum = o;
  o += fr_align(static_cast<size_t>(own_max) * 8, 16);
  p.sel = o;
  o += fr_align(static_cast<size_t>(own_max) * 33 * 4, 16);
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

// Compile-time specialised on the routing strategy (kStrat: -1 vanilla, 0
// DES-Seq, 1 DES-Vote), the router-GEMM shape (kG: 0 split-K over the
// cluster, 1 token split, 2 logits in from router_cluster_kernel) and the
// small-block L stage (kSmall: at most one own token per warp of a group):
// each instantiation executes one contiguous code path, so the instruction
// fetch (cold after the FFN streamed hundreds of MB) follows it sequentially
// instead of jumping over the other variants.
template <int kStrat, int kG, bool kSmall>
__global__ void __launch_bounds__(kFrontThreads, 1)
    front_kernel(const __grid_constant__ CUtensorMap wr_map, const __grid_constant__ BoxMaps x_maps,
                 const __grid_constant__ FrontArgs a_param) {
  // The arguments are copied to shared memory once, all words in flight
  // together: first touches of kernel-parameter (constant-bank) lines later
  // in the kernel each stalled the critical path for ~1 us.
  __shared__ FrontArgs a;
  {
    constexpr int kWords = static_cast<int>(sizeof(FrontArgs) / 4);
    static_assert(sizeof(FrontArgs) % 4 == 0, "FrontArgs size");
    if (threadIdx.x < kWords)
      reinterpret_cast<int*>(&a)[threadIdx.x] = reinterpret_cast<const int*>(&a_param)[threadIdx.x];
    __syncthreads();
  }
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // align to 1024 B by offsetting the shared array itself, so the compiler
  // keeps the shared address space (LDS/STS instead of generic LD/ST)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int kMaxStages = 12;  // ring stages (the token-split GEMM runs deep rings)
  __shared__ uint64_t bars[2 * kMaxStages + 4];  // full[], empty[], tdone, recv, selx, mask
  __shared__ uint64_t s_mask[kFrontCta];         // coreset slices (distributed rank)
  __shared__ uint32_t s_tag;                     // this call's hand-off tag
  __shared__ uint32_t tmem_slot[2];
  __shared__ int s_bad, s_nm;
  __shared__ int warp_tot[kFrontThreads / 32 + 1];
  __shared__ uint64_t s_ts[48];  // timeline marks (trace buffer only)
  __shared__ uint64_t s_pw[96];  // instruction-cache prewarm scratch
  // glibc exp's 2^(k/128) table, staged while the router GEMM runs
  __shared__ __align__(16) unsigned long long s_exptab[256];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr bool kTs = kG == 1;   // token-split GEMM
  constexpr bool kLin = kG == 2;  // logits in (router_cluster_kernel ran ahead)
  const bool tracing = a.trace != nullptr;
  if (tracing && tid == 0) s_ts[24] = clock64();
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
  const FrontSmem P =
      front_smem_plan(n, m, k, Tc, a.own_max, a.stages, a.b_rows, a.vote_rows, a.tsplit);
  unsigned char* ring = smem + P.ring;
  double* erow = reinterpret_cast<double*>(smem + P.erow);  // [own][m + 1]
  float* recv = reinterpret_cast<float*>(smem + P.partial);  // [C][ocm][m4]
  float* stage = reinterpret_cast<float*>(smem + P.stage);   // [Tc][m4]
  const int m4 = (m + 3) & ~3;
  float* xrow = reinterpret_cast<float*>(smem + P.xrow);     // [own][m]
  float* mxv = reinterpret_cast<float*>(smem + P.mx);
  double* ssum = reinterpret_cast<double*>(smem + P.ssum);
  int* sel = reinterpret_cast<int*>(smem + P.sel);           // [own][33] rank order
  int* wsel_all = reinterpret_cast<int*>(smem + P.wsel);     // [NW][33]
  int* own_tok = reinterpret_cast<int*>(smem + P.own_tok);
  uint8_t* flag = smem + P.flag;                             // [m] coreset members
  uint8_t* risky = flag + m;                                 // [own]
  const int ew = m + 1;                                      // erow row stride
  uint64_t* full = bars;
  uint64_t* empty = bars + kMaxStages;
  uint64_t* tdone = bars + 2 * kMaxStages;
  uint64_t* bar_recv = bars + 2 * kMaxStages + 1;  // partials pushed to this CTA (one phase per chunk)
  uint64_t* bar_selx = bars + 2 * kMaxStages + 2;  // every token's selection pushed to this CTA
  uint64_t* bar_mask = bars + 2 * kMaxStages + 3;  // every CTA's coreset slice pushed to this CTA
  // DES-Vote over a large pool: the O(m^2) rank count is split over the
  // cluster (CTA r ranks experts [r*ms, (r+1)*ms) against all m votes) and the
  // slices' membership masks are exchanged; small pools rank redundantly
  const int ms = (m + C - 1) / C;
  const bool dist_rank = kStrat == 1 && m > kDistRankMin && !(a.flags & 4);  // bit 2: A/B off
  int* allsel = reinterpret_cast<int*>(smem + P.allsel);       // [n][k]
  double* allp = reinterpret_cast<double*>(smem + P.allp);     // [n][k]
  const int ocm = (Tc + C - 1) / C;                            // recv rows per sender
  const int S = a.stages;
  const int stage_bytes = mt * kATile + a.b_rows * 128;
  const int kb_cta = a.kb_per_cta;
  const int kb0 = rk * kb_cta;
  const uint32_t xbytes = static_cast<uint32_t>(a.b_rows) * 128u;
  constexpr bool vanilla = kStrat < 0;
  const int depth = kStrat == 0 ? a.seq_k : k;

  // ---- setup: barriers, TMEM, router-weight prefetch (weights are static, so
  // they stream before the previous kernel's output is even waited for) ----------
  if (tid == 0) {
    tma_prefetch_desc(&wr_map);
    tma_prefetch_desc(&x_maps.map[a.box_index]);
#pragma unroll 1
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      // token split with multicast W_r: every CTA's MMA frees a slot
      mbar_init(&empty[s], a.tsplit == 1 ? C : 1);
    }
    mbar_init(tdone, 1);
    mbar_init(bar_recv, 1);
    mbar_init(bar_selx, 1);
    mbar_init(bar_mask, 1);
    fence_mbar_init();
    if (dist_rank) mbar_arrive_expect_tx(bar_mask, static_cast<uint32_t>(C * 8));
    s_bad = 0;
    // arm: chunk 0's partials for this CTA's own tokens from all C senders,
    // and (DES) every token's top-`depth` selection
    const int nc0 = n < Tc ? n : Tc;
    const int own0 = (nc0 * (rk + 1)) / C - (nc0 * rk) / C;
    if constexpr (kG == 0) mbar_arrive_expect_tx(bar_recv, static_cast<uint32_t>(C * own0 * m4 * 4));
    if constexpr (kStrat >= 0)  // every token's top-depth ids (+ weights, DES-Vote)
      mbar_arrive_expect_tx(bar_selx, static_cast<uint32_t>(n * depth * (kStrat == 1 ? 12 : 4)));
    else if (rk == 0 && a.pub)
      mbar_arrive_expect_tx(bar_selx, static_cast<uint32_t>(n * k * 4));  // union of top-K
    const uint64_t pol = l2_policy_evict_last();  // W_r: small, read every call
    if (kTs && a.tsplit == 2) {
      // token split, local W_r: the first S K-blocks stream before the
      // previous kernel is waited for (the X rows follow after pdl_wait)
#pragma unroll 1
      for (int i = 0; i < kb_cta * C && i < S; ++i) {
        unsigned char* st = ring + static_cast<size_t>(i) * stage_bytes;
        mbar_arrive_expect_tx(&full[i], mt * kATile + xbytes);
#pragma unroll 1
        for (int tl = 0; tl < mt; ++tl)
          tma_load_2d(st + tl * kATile, &wr_map, &full[i], i * kBK, tl * kBM, pol);
      }
    }
    if constexpr (kG == 0) {
#pragma unroll 1
      for (int i = 0; i < kb_cta && i < S; ++i) {
        unsigned char* st = ring + static_cast<size_t>(i) * stage_bytes;
        mbar_arrive_expect_tx(&full[i], mt * kATile + xbytes);
#pragma unroll 1
        for (int tl = 0; tl < mt; ++tl)
          tma_load_2d(st + tl * kATile, &wr_map, &full[i], (kb0 + i) * kBK, tl * kBM, pol);
      }
    }
    FRONT_MARK(45);
  }
  if (warp == 2 && !kLin) {
    tmem_alloc(tmem_slot, a.tmem_cols);
    if (tracing && lane == 0) s_ts[46] = gtime();
  }
  // the exp table: asynchronous copies (nobody waits for them until the
  // activation stage, cp.async.wait_all before the barrier that precedes it)
  if (tid < 128)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s_exptab + 2 * tid)),
                 "l"(kExpTab + 2 * tid)
                 : "memory");
  // instruction-cache prewarm: the layer's FFN streams hundreds of MB
  // between two calls, so this kernel's code comes back from far memory and
  // every new code region costs a miss chain (~2 µs measured at the top-K
  // entry). Four idle warps each run one later phase's code once on scratch
  // (s_pw; 32 dummy experts), in parallel so the misses overlap: during the
  // router GEMM, or in logits-in mode before griddepcontrol.wait, while
  // router_cluster_kernel still runs (DESMOE_FRONT_FLAGS=1 disables)
  auto prewarm = [&]() {
    uint8_t* df = reinterpret_cast<uint8_t*>(s_pw + 48);      // [32] flags; pub words at +52
    int* ds = wsel_all + warp * 33;
    if (warp == 8) {
      warp_rank_select(reinterpret_cast<const float*>(erow), m, k < m ? k + 1 : k, nullptr, ds);
    } else if (warp == 9) {
      if (lane == 0) {
        // (the global table: the shared copy may still be in flight here)
        volatile double sink = f_exp(-1.5, kExpTab) + f_div(1.0, 2.0);
        (void)sink;
      }
    } else if (warp == 10) {
      df[lane] = static_cast<uint8_t>(lane & 1);
      __syncwarp();
      publish_list(df, 32, 0u, reinterpret_cast<uint32_t*>(s_pw + 52), nullptr, nullptr);
    } else {
      write_route(erow, 1.0, 2, ds, 0, 0, 0, reinterpret_cast<double*>(s_pw + 64), nullptr,
                  nullptr, ds, nullptr, 0u);
    }
    // (The exact near-tie path is not prewarmed: a fifth prewarm warp running
    // it cost the coreset 2-2.7 us at C2/C3 N = 32 — that warp joins the
    // activation late — more than its rare cold misses.)
  };
  if (kLin && !(a.flags & 1) && warp >= 8 && warp < 12) prewarm();
  pdl_wait();  // x (the previous kernel's output) is complete from here on
  // the expert-FFN kernel may launch now — not earlier: it reads the call
  // sequence word the previous call's combine advances, and that combine
  // lets the next kernels launch at ITS start (cross-layer overlap in a
  // stack), so only this wait orders the FFN behind it
  pdl_launch_dependents();
  // the first ring stages' X boxes go out at once (their W_r halves and the
  // stages' transaction counts were armed in the setup): no CTA barrier or
  // cluster barrier on the way to the router GEMM's inputs
  const int x_pre = kLin ? 0 : (!kTs || a.tsplit == 2) ? (kTs ? (kb_cta * C < S ? kb_cta * C : S)
                                                   : (kb_cta < S ? kb_cta : S))
                                             : 0;
  if (tid == 0) {
    const uint64_t pol_x = l2_policy_evict_last();
    const int x_row0 = kTs ? (n * rk) / C : 0;
#pragma unroll 1
    for (int i = 0; i < x_pre; ++i)
      tma_load_2d(ring + static_cast<size_t>(i) * stage_bytes + mt * kATile,
                  &x_maps.map[a.box_index], &full[i], (kTs ? i : kb0 + i) * kBK, x_row0, pol_x);
  }
  FRONT_MARK(47);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  FRONT_MARK(41);
  const uint32_t tmem_base = tmem_slot[0];
  // every CTA's barriers are initialised and armed before anyone pushes
  cluster_arrive_relaxed();
  cluster_wait();
  FRONT_MARK(1);
  // this call's hand-off tag: an L2 round trip (the sequence word the last
  // combine advanced), taken by a warp idle during the router GEMM and read
  // from shared memory after the GEMM's barrier (loaded by every thread at
  // this point, it stalled all 16 warps, the MMA issuer included, ~1 us)
  if (tid == 96) s_tag = a.seq ? hand_tag(*a.seq) : 0u;
  if (!kLin && !(a.flags & 1) && warp >= 8 && warp < 12) prewarm();

  // ---- R + L1: per token chunk, split-K GEMM, then the owners' logit sums ----------
  int own = 0;
  if constexpr (kTs) {
    // token split: this CTA owns tokens [tlo, thi) and computes their logits
    // over the whole hidden dimension. K-block `it` of W_r is loaded once per
    // cluster by CTA (it mod C) and multicast into every CTA's ring slot;
    // each CTA adds its own X rows. A slot is refilled once all C CTAs'
    // MMAs have released it (each commits to every CTA's empty barrier).
    const int tlo = (n * rk) / C, thi = (n * (rk + 1)) / C;
    own = thi - tlo;
    const int KB = kb_cta * C;
    const int n_mma = a.b_rows;
    if (warp == 0 && lane == 0) {
      const uint64_t pol_w = l2_policy_evict_last();
      const uint64_t pol_x = l2_policy_evict_last();
#pragma unroll 1
      for (int it = 0; it < KB; ++it) {
        const int s = it % S;
        unsigned char* st = ring + static_cast<size_t>(s) * stage_bytes;
        if (it >= S) mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
        const bool pre = a.tsplit == 2 && it < S;  // W_r already issued in the setup
        if (!pre) mbar_arrive_expect_tx(&full[s], mt * kATile + xbytes);
        if (pre) {
        } else if (a.tsplit == 2) {  // every CTA streams all of W_r itself (no cluster lockstep)
#pragma unroll 1
          for (int tl = 0; tl < mt; ++tl)
            tma_load_2d(st + tl * kATile, &wr_map, &full[s], it * kBK, tl * kBM, pol_w);
        } else if (it % C == rk) {
#pragma unroll 1
          for (int tl = 0; tl < mt; ++tl)
            tma_load_2d_mc(st + tl * kATile, &wr_map, &full[s], it * kBK, tl * kBM,
                           static_cast<uint16_t>((1u << C) - 1u), pol_w);
        }
        if (it >= x_pre)
          tma_load_2d(st + mt * kATile, &x_maps.map[a.box_index], &full[s], it * kBK, tlo, pol_x);
      }
    } else if (warp == 1) {
      const uint32_t idesc = idesc_bf16_f32(kBM, n_mma);
#pragma unroll 1
      for (int it = 0; it < KB; ++it) {
        const int s = it % S;
        mbar_wait(&full[s], (it / S) & 1);
        if (tracing && lane == 0 && (it & 7) == 0 && it < 40) s_ts[26 + it / 8] = gtime();
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a0 = smem_u32(ring + static_cast<size_t>(s) * stage_bytes);
          const uint32_t b0 = a0 + mt * kATile;
#pragma unroll 1
          for (int tl = 0; tl < mt; ++tl)
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              tc_mma_bf16(tmem_base + tl * 256, sw128_kmajor_desc(a0 + tl * kATile + kk * 32),
                          sw128_kmajor_desc(b0 + kk * 32), idesc, (it > 0 || kk > 0) ? 1u : 0u);
          if (a.tsplit == 1)
            tc_commit_mc(&empty[s], static_cast<uint16_t>((1u << C) - 1u));
          else
            tc_commit(&empty[s]);
          if (it == KB - 1) tc_commit(tdone);
        }
        __syncwarp();
      }
    } else if (warp >= 4 && warp < 8) {
      // drain TMEM: the own tokens' logits straight into xrow
      mbar_wait(tdone, 0);
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
              if (cc + j < own) xrow[(cc + j) * m + e] = v[j];
          }
        }
      }
      tc_fence_before();
    }
    if (tid < own) own_tok[tid] = tlo + tid;
    FRONT_MARK(2);
    FRONT_MARK(3);
  }
#pragma unroll 1
  if constexpr (kLin) {
    // logits from router_cluster_kernel (complete since griddepcontrol.wait):
    // this CTA owns tokens [n rk / C, n (rk + 1) / C), as in the token split
    const int tlo = (n * rk) / C, thi = (n * (rk + 1)) / C;
    own = thi - tlo;
    const float* src = a.logits_in + static_cast<size_t>(tlo) * m;
    if ((m & 3) == 0) {
      const int cnt4 = own * m / 4;
#pragma unroll 1
      for (int w = tid; w < cnt4; w += kFrontThreads)
        reinterpret_cast<float4*>(xrow)[w] = __ldcg(reinterpret_cast<const float4*>(src) + w);
    } else {
#pragma unroll 1
      for (int w = tid; w < own * m; w += kFrontThreads) xrow[w] = __ldcg(src + w);
    }
    if (tid < own) own_tok[tid] = tlo + tid;
    FRONT_MARK(2);
    FRONT_MARK(3);
  }
#pragma unroll 1
  for (int c = 0; c < nch && kG == 0; ++c) {
    const int c0 = c * Tc;
    const int nc = n - c0 < Tc ? n - c0 : Tc;
    const int n_mma = (nc + 15) & ~15;
    if (warp == 0 && lane == 0) {
      const uint64_t pol_w = l2_policy_evict_last();
      const uint64_t pol_x = l2_policy_evict_last();
      // a ring with one stage per K block holds this CTA's whole W_r slice:
      // it stays resident over the token chunks, which reload only their X
      // boxes (C3 N=64: the second chunk re-streamed 128 KB of W_r, ~4 us)
      const bool w_resident = S == kb_cta;
#pragma unroll 1
      for (int i = 0; i < kb_cta; ++i) {
        const int it = c * kb_cta + i, s = it % S;
        unsigned char* st = ring + static_cast<size_t>(s) * stage_bytes;
        if (it >= S) {
          mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], w_resident ? xbytes : mt * kATile + xbytes);
          if (!w_resident) {
#pragma unroll 1
            for (int tl = 0; tl < mt; ++tl)
              tma_load_2d(st + tl * kATile, &wr_map, &full[s], (kb0 + i) * kBK, tl * kBM, pol_w);
          }
        }
        if (it >= x_pre)
          tma_load_2d(st + mt * kATile, &x_maps.map[a.box_index], &full[s], (kb0 + i) * kBK, c0,
                      pol_x);
      }
      if (tracing && c == 0) s_ts[44] = gtime();
    } else if (warp == 1) {
      const uint32_t idesc = idesc_bf16_f32(kBM, n_mma);
#pragma unroll 1
      for (int i = 0; i < kb_cta; ++i) {
        const int it = c * kb_cta + i, s = it % S;
        mbar_wait(&full[s], (it / S) & 1);
        if (tracing && lane == 0 && c == 0 && (i == 0 || i == kb_cta - 1))
          s_ts[i == 0 ? 42 : 43] = gtime();
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
      if (tracing && warp == 4 && lane == 0 && c == 0) s_ts[18] = gtime();
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
              if (cc + j < nc) stage[(cc + j) * m4 + e] = v[j];
          }
        }
      }
      tc_fence_before();
      if (tracing && warp == 4 && lane == 0 && c == 0) s_ts[19] = gtime();
      // generic-proxy writes -> visible to the bulk-copy (async) proxy
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      named_bar_sync(1, 128);
      if (warp == 4 && lane < C) {
        // one bulk copy per owner: its contiguous token rows -> recv[rk] there
        const int ow = lane;
        const int lo_q = (nc * ow) / C, hi_q = (nc * (ow + 1)) / C;
        const uint32_t bytes = static_cast<uint32_t>((hi_q - lo_q) * m4 * 4);
        if (bytes)
          bulk_s2cluster(mapa_u32(smem_u32(recv + rk * ocm * m4), ow),
                         smem_u32(stage + lo_q * m4), bytes, mapa_u32(smem_u32(bar_recv), ow));
        if (tracing && lane == 0 && c == 0) s_ts[20] = gtime();
      }
    }
    FRONT_MARK(2);
    mbar_wait_cluster(bar_recv, c & 1);  // all C partials of this CTA's tokens arrived
    FRONT_MARK(3);
    // owners: logits = sum of the C partials in fixed CTA order (deterministic)
    const int lo = (nc * rk) / C, hi = (nc * (rk + 1)) / C;
    const int ob = c * opc;
    const int cnt = (hi - lo) * m;
#pragma unroll 1
    for (int w = tid; w < cnt; w += kFrontThreads) {
      const int j = w / m, e = w - j * m;
      float acc = 0.0f;
#pragma unroll
      for (int r = 0; r < C; ++r) acc += recv[(r * ocm + j) * m4 + e];
      xrow[(ob + j) * m + e] = acc;
    }
    if (tid < hi - lo) own_tok[ob + tid] = c0 + lo + tid;
    own = ob + (hi - lo);
    if (tracing && tid == 0 && c < 8) s_ts[26 + c] = gtime();
    if (c + 1 < nch) {
      // re-arm for the next chunk, then a (relaxed) cluster barrier: every
      // owner consumed this chunk before anyone pushes the next one
      __syncthreads();
      if (tid == 0) {
        const int c1 = c + 1;
        const int nc1 = n - c1 * Tc < Tc ? n - c1 * Tc : Tc;
        const int own1 = (nc1 * (rk + 1)) / C - (nc1 * rk) / C;
        mbar_arrive_expect_tx(bar_recv, static_cast<uint32_t>(C * own1 * m4 * 4));
      }
      cluster_arrive_relaxed();
      cluster_wait();
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");  // the exp table (issued in the setup)
  __syncthreads();
  FRONT_MARK(4);
  const uint32_t tag = s_tag;
  if (warp == 2 && !kLin) {
    tc_fence_after();
    tmem_dealloc(tmem_base, a.tmem_cols);
  }

  // ---- L2-L4 in two warp groups (small blocks: at most one token per warp) ------
  // The top-K selection keys on the fp32 logits (every activation is monotone
  // in the logit), so warps 0-7 select while warps 8-15 compute the row max,
  // the fp64 activation and the ordered sums; the selectors then wait (named
  // barrier 2) for the activation to check their boundaries.
  constexpr int kGW = NW / 2;  // warps per group
  if constexpr (kSmall) {  // (host: own tokens <= kGW; DESMOE_FRONT_FLAGS bit 2 forces the sequence)
    if (warp < kGW) {
      const int want = k < m ? k : m;
      const int rounds = want < m ? want + 1 : want;
      if (tracing && warp == 0 && lane == 0) s_ts[34] = gtime();
#pragma unroll 1
      for (int j = warp; j < own; j += kGW) {
        long long c0 = clock64();
        if (tracing && warp == 0 && lane == 0 && j == 0) s_ts[35] = gtime();
        warp_rank_select(xrow + j * m, m, rounds, nullptr, sel + j * 33);
        if (tracing && warp == 0 && lane == 0 && j == 0) {
          s_ts[23] = clock64() - c0;
          s_ts[36] = gtime();
        }
      }
      named_bar_sync(2, kFrontThreads);  // the activation (erow) is written
#pragma unroll 1
      for (int j = warp; j < own; j += kGW) {
        if (lane == 0) {
          const int* sj = sel + j * 33;
          const float* xr = xrow + j * m;
          const double* er = erow + j * ew;
          bool r = want < m && risky_boundary(xr, er, act, sj, want, m);
          if (!vanilla && depth < want) r |= risky_boundary(xr, er, act, sj, depth, m);
          risky[j] = r;
        }
      }
      if (tracing && warp == 0 && lane == 0) s_ts[37] = gtime();
      if (tracing && warp == 0 && lane == 0) s_ts[22] = gtime();
  } else {
      const int gw = warp - kGW, gt = tid - kGW * 32;
      // L2: row max + finiteness (warp per token)
#pragma unroll 1
      for (int j = gw; j < own; j += kGW) {
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
      named_bar_sync(3, kFrontThreads / 2);
      if (tracing && gt == 0) s_ts[5] = gtime();
      // L3: activation in fp64, data-parallel over (own token, expert)
      activate_rows<false>(xrow, mxv, erow, ew, own, m, act, s_exptab, gt, kFrontThreads / 2);
      named_bar_sync(3, kFrontThreads / 2);
      named_bar_arrive(2, kFrontThreads);  // hand the activation to the selectors
      if (tracing && gt == 0) s_ts[6] = gtime();
      // L4: ordered softmax sums, one lane per token (ascending index, gating.cpp:31-33)
      if (warp == NW - 1) {
#pragma unroll 1
        for (int j = lane; j < own; j += 32) {
          double s = 1.0;
          if (act == 0) {
            s = 0.0;
            const double* er = erow + j * ew;
            int i = 0;
#pragma unroll 4
            for (; i + 8 <= m; i += 8) {  // (unrolled: the next batch's loads overlap the adds)
              double v[8];
#pragma unroll
              for (int q = 0; q < 8; ++q) v[q] = er[i + q];
#pragma unroll
              for (int q = 0; q < 8; ++q) s += v[q];
            }
#pragma unroll 1
            for (; i < m; ++i) s += er[i];
          }
          ssum[j] = s;
        }
        if (tracing && lane == 0) s_ts[21] = gtime();
      }
    }
    } else {
    // large blocks: the phases in sequence over all warps
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
    activate_rows<true>(xrow, mxv, erow, ew, own, m, act, s_exptab, tid, kFrontThreads);
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
          int i = 0;
#pragma unroll 4
          for (; i + 8 <= m; i += 8) {  // ascending index (gating.cpp:31-33)
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = er[i + q];
#pragma unroll
            for (int q = 0; q < 8; ++q) s += v[q];
          }
#pragma unroll 1
          for (; i < m; ++i) s += er[i];
        }
        ssum[j] = s;
      }
      if (tracing && lane == 0) s_ts[21] = gtime();
    } else {
      const int want = k < m ? k : m;
      const int rounds = want < m ? want + 1 : want;
      if (tracing && warp == 0 && lane == 0) s_ts[34] = gtime();
#pragma unroll 1
      for (int j = warp; j < own; j += NW - 1) {
        int* sj = sel + j * 33;
        const float* xr = xrow + j * m;
        const double* er = erow + j * ew;
        long long c0 = clock64();
        if (tracing && warp == 0 && lane == 0 && j == 0) s_ts[35] = gtime();
        warp_rank_select(xr, m, rounds, nullptr, sj);
        if (tracing && warp == 0 && lane == 0 && j == 0) {
          s_ts[23] = clock64() - c0;
          s_ts[36] = gtime();
        }
        if (lane == 0) {
          bool r = want < m && risky_boundary(xr, er, act, sj, want, m);
          if (!vanilla && depth < want) r |= risky_boundary(xr, er, act, sj, depth, m);
          risky[j] = r;
        }
        if (tracing && warp == 0 && lane == 0 && j == 0) s_ts[37] = gtime();
      }
      if (tracing && warp == 0 && lane == 0) s_ts[22] = gtime();
    }
  }
  __syncthreads();
  FRONT_MARK(7);
  if (s_bad && tid == 0) raise_flag(a.err, 1);
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
      if (risky[j])  // rare
        fix_boundary(xrow + j * m, er, s, act, m, want, vanilla ? 0 : depth, nullptr, scratch, sj);
      if constexpr (vanilla) {
        write_route(er, s, act, sj, want, k, own_tok[j], wp, a.route_idx, a.route_gate,
                    a.route_cnt, a.route_words, tag);
        if (a.pub && lane < k)  // the union (unique experts) is published by rank 0
          st_async_b32(mapa_u32(smem_u32(allsel + own_tok[j] * k + lane), 0),
                       static_cast<uint32_t>(sj[lane]), mapa_u32(smem_u32(bar_selx), 0));
      } else if (lane < depth) {
        // broadcast the token's top-`depth` (ids, weights) to every CTA
        const int e = sj[lane];
        const int t = own_tok[j];
        const uint32_t ea = smem_u32(allsel + t * k + lane);
        const uint32_t ba = smem_u32(bar_selx);
        double pv = 0.0;
        if constexpr (kStrat == 1)
          pv = a.raw ? static_cast<double>(xrow[j * m + e]) : (act == 0 ? f_div(er[e], s) : er[e]);
        const uint32_t pa = smem_u32(allp + t * k + lane);
#pragma unroll 1
        for (int r = 0; r < C; ++r) {
          const uint32_t rb = mapa_u32(ba, r);
          st_async_b32(mapa_u32(ea, r), static_cast<uint32_t>(e), rb);
          if constexpr (kStrat == 1)
            st_async_b64(mapa_u32(pa, r), static_cast<uint64_t>(__double_as_longlong(pv)), rb);
        }
      }
      __syncwarp();
    }
  }
  __syncthreads();
  FRONT_MARK(8);
  if constexpr (vanilla) {
    if (tid == 0 && a.route_done)  // route words out (a hint: see the DES path's RR)
      st_relaxed_u32(a.route_done + rk, tag);
    if (rk == 0 && a.pub) {
      // union of every token's top-K = the experts the FFN will stream
      mbar_wait_cluster(bar_selx, 0);
#pragma unroll 1
      for (int i = tid; i < m; i += kFrontThreads) flag[i] = 0;
      __syncthreads();
#pragma unroll 1
      for (int i = tid; i < n * k; i += kFrontThreads) flag[allsel[i]] = 1;
      __syncthreads();
      if (warp == 0) publish_list(flag, m, tag, a.pub, nullptr, nullptr);
    }
    // every remote access (partials, ids) is done once all CTAs reach this barrier
    cluster_arrive_relaxed();
    cluster_wait();
    FRONT_MARK(9);
    if (a.logits_out) front_tail(a.logits_out, xrow, own_tok, own, m, tid);
    if (tracing) front_dump_marks(a.trace, a.trace_cap, s_ts, tid, 48);
    return;
  }
  mbar_wait_cluster(bar_selx, 0);       // every token's selection has arrived
  cluster_arrive_relaxed();             // exit barrier (#3): all pushes landed; wait at the end
  FRONT_MARK(9);

  // ---- V: block coreset, redundantly in every CTA ------------------------------------
  // DES-Vote: V_e = the reference's column sum of the masked matrix over the
  // tokens in ascending order, zeros included (des.cpp:73-91). Adding +0.0
  // leaves an fp64 sum unchanged, so each expert sums only the tokens that
  // selected it, in token order: the (token, expert) pairs are bucketed by
  // expert with a stable counting sort (a token bitmask per expert, its
  // popcounts as counts and ranks), then thread e walks its own list — the
  // same fp64 additions in the same order as the dense N x M matrix.
  double vsum = 0.0;
#pragma unroll 1
  for (int i = tid; i < m; i += kFrontThreads) flag[i] = 0;
  FRONT_MARK(10);
  if constexpr (kStrat == 1) {
    const int nw = (n + 31) >> 5;                                        // token words
    uint32_t* vbits = reinterpret_cast<uint32_t*>(smem + P.dreg);        // [m][nw]
    int* voff = reinterpret_cast<int*>(vbits + m * nw);                  // [m + 1]
    double* vlist = reinterpret_cast<double*>(smem + P.dreg + fr_align(
        static_cast<size_t>(m * nw + m + 1) * 4, 16));                   // [n * depth]
#pragma unroll 1
    for (int i = tid; i < m * nw; i += kFrontThreads) vbits[i] = 0u;
    __syncthreads();
#pragma unroll 1
    for (int w = tid; w < n * depth; w += kFrontThreads) {
      const int t = w / depth, j = w - t * depth;
      const int e = allsel[t * k + j];
      atomicOr(&vbits[e * nw + (t >> 5)], 1u << (t & 31));
    }
    __syncthreads();
    // counts -> exclusive offsets (m <= 256 <= kFrontThreads: one expert per thread)
    int cnt_e = 0;
    if (tid < m)
#pragma unroll 1
      for (int q = 0; q < nw; ++q) cnt_e += __popc(vbits[tid * nw + q]);
    int inc = cnt_e;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    if (tid < m) {
      int base = 0;
#pragma unroll 1
      for (int q = 0; q < warp; ++q) base += warp_tot[q];
      voff[tid] = base + inc - cnt_e;
      if (tid == m - 1) voff[m] = base + inc;
    }
    __syncthreads();
    // scatter: (t, e) -> e's list at its rank among e's tokens (token order)
#pragma unroll 1
    for (int w = tid; w < n * depth; w += kFrontThreads) {
      const int t = w / depth, j = w - t * depth;
      const int e = allsel[t * k + j];
      const uint32_t* b = vbits + e * nw;
      int pos = voff[e] + __popc(b[t >> 5] & ((1u << (t & 31)) - 1u));
#pragma unroll 1
      for (int q = 0; q < (t >> 5); ++q) pos += __popc(b[q]);
      vlist[pos] = allp[t * k + j];
    }
    __syncthreads();
    if (tid < m) {
      const int i1 = voff[tid + 1];
      int i = voff[tid];
#pragma unroll 1
      for (; i + 8 <= i1; i += 8) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = vlist[i + q];
#pragma unroll
        for (int q = 0; q < 8; ++q) vsum += v[q];
      }
#pragma unroll 1
      for (; i < i1; ++i) vsum += vlist[i];
    }
    __syncthreads();  // list reads done before votes / keys reuse the region
  } else {
    // DES-Seq: the union of every token's top-seq_k. (The barrier orders the
    // zeroing above before any thread's set: without it a late zero could
    // erase another thread's member — a rare wrong coreset / re-route, ~1 in
    // 1500 calls of one criterion-6 instance.)
    __syncthreads();
#pragma unroll 1
    for (int w = tid; w < n * depth; w += kFrontThreads) {
      const int t = w / depth, j = w - t * depth;
      flag[allsel[t * k + j]] = 1;
    }
    __syncthreads();
  }
  FRONT_MARK(11);
  if (kStrat == 1) {
    double* votes = reinterpret_cast<double*>(smem + P.dreg);      // [m] (aliases the buckets)
    uint64_t* vkey = reinterpret_cast<uint64_t*>(votes + m);        // [m]
    int* rankp = reinterpret_cast<int*>(vkey + m);                  // [parts][m]
    if (tid < m) {
      votes[tid] = vsum;
      vkey[tid] = order_key(vsum);
      if (a.votes && rk == 0) a.votes[tid] = vsum;
    }
    __syncthreads();
    FRONT_MARK(15);
    // rank of expert e = #experts before it in (vote desc, index asc), the
    // pool split into `parts` key ranges counted by different threads —
    // inline and with one division per thread (the out-of-line helper with
    // its per-call divisions measured 1300 vs 440 cycles, tools/micro/phase.cu)
    const int e0 = dist_rank ? rk * ms : 0;
    const int me = dist_rank ? (m - e0 < ms ? (m - e0 > 0 ? m - e0 : 0) : ms) : m;
    const int span_e = dist_rank ? ms : m;  // experts ranked by this CTA (stride of rankp)
    const int pmax = kFrontThreads / span_e < 16 ? kFrontThreads / span_e : 16;
    const int parts = dist_rank ? kFrontThreads / span_e : pmax;
    if (tid < parts * span_e) {
      const int part = tid / span_e, el = tid - part * span_e;
      const int e = e0 + el;
      const int span = (m + parts - 1) / parts;
      const int j0 = part * span, j1 = j0 + span < m ? j0 + span : m;
      int r = 0;
      if (el < me) {
        const uint64_t ki = vkey[e];
#pragma unroll 4
        for (int j = j0; j < j1; ++j) {
          const uint64_t kj = vkey[j];
          r += (kj > ki) | ((kj == ki) & (j < e));
        }
      }
      rankp[part * span_e + el] = r;
    }
    __syncthreads();
    FRONT_MARK(16);
    if (!dist_rank) {
      if (tid < m) {
        int r = 0;
#pragma unroll 1
        for (int q = 0; q < parts; ++q) r += rankp[q * m + tid];
        flag[tid] = static_cast<uint8_t>(r < a.m_core);
      }
    } else {
      // this CTA's slice -> one 64-bit membership word pushed to every CTA
      // (ms <= 64: pools of up to 512 experts)
      if (warp == 0) {
        int r0 = 0, r1 = 0;
#pragma unroll 1
        for (int q = 0; q < parts; ++q) {
          if (lane < me) r0 += rankp[q * ms + lane];
          if (lane + 32 < me) r1 += rankp[q * ms + lane + 32];
        }
        const uint32_t w0 = __ballot_sync(0xffffffffu, lane < me && r0 < a.m_core);
        const uint32_t w1 = __ballot_sync(0xffffffffu, lane + 32 < me && r1 < a.m_core);
        const uint64_t word = (static_cast<uint64_t>(w1) << 32) | w0;
        if (lane < C)
          st_async_b64(mapa_u32(smem_u32(s_mask + rk), lane), word,
                       mapa_u32(smem_u32(bar_mask), lane));
      }
      mbar_wait_cluster(bar_mask, 0);
      if (tid < m) flag[tid] = static_cast<uint8_t>((s_mask[tid / ms] >> (tid % ms)) & 1ull);
    }
  }
  const int nm = __syncthreads_count(tid < m && flag[tid]);  // m <= 256 < kFrontThreads
  if (rk == 0 && warp == 0) publish_list(flag, m, tag, a.pub, a.members, a.n_members);
  FRONT_MARK(12);

  // ---- RR: constrained re-route of own tokens (warp per token) ----------------------
  {
    int* wsel = wsel_all + warp * 33;
    double* wp = reinterpret_cast<double*>(smem + P.wp) + warp * 32;
    double* scratch = reinterpret_cast<double*>(smem + P.scratch) + warp * m;
    if (tracing && tid < 3) s_ts[38 + tid] = 0;
    __syncthreads();
#pragma unroll 1
    for (int j = warp; j < own; j += NW) {
      const long long rr0 = clock64();
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
      bool r = false;
      if (!covered) {
        const int rounds = cnt < nm ? cnt + 1 : cnt;
        warp_rank_select(xr, m, rounds, flag, wsel);  // rank order
        r = cnt < nm && risky_boundary(xr, er, act, wsel, cnt, m);
        if (r) fix_boundary(xr, er, s, act, m, cnt, 0, flag, scratch, wsel);  // rare
      }
      write_route(er, s, act, wsel, cnt, k, own_tok[j], wp, a.route_idx, a.route_gate,
                  a.route_cnt, a.route_words, tag);
      if (tracing && lane == 0) {  // (timeline: slowest token, uncovered / exact masks)
        atomicMax(reinterpret_cast<unsigned long long*>(&s_ts[38]),
                  static_cast<unsigned long long>(clock64() - rr0));
        if (!covered) atomicOr(reinterpret_cast<unsigned long long*>(&s_ts[39]), 1ull << j);
        if (r) atomicOr(reinterpret_cast<unsigned long long*>(&s_ts[40]), 1ull << j);
      }
    }
  }
  // this CTA's route words are all out: one release word for the expert-FFN
  // kernel (routed mode), which polls these 8 words, not the N*K route words
  // (140 CTAs re-reading the same 2-16 KB of route words flooded their L2
  // lines: the routed prologue took 11-20 us after the front had finished)
  // (No fence: a GPU-scope MEMBAR here cost one CTA up to 10 us. The word is
  // only a hint — the route words carry the tag themselves and the FFN
  // re-polls any word whose tag is not yet this call's.)
  __syncthreads();
  if (tid == 0 && a.route_done) st_relaxed_u32(a.route_done + rk, tag);
  FRONT_MARK(13);
  if (tracing && tid == 0) s_ts[25] = clock64();
  cluster_wait();  // #3: no CTA exits while others may still read its shared memory
  FRONT_MARK(14);
  // (guarded here: a call into an out-of-line function fetches its code even
  // when it returns at once — measured as 5 % of the kernel's warp samples)
  if (a.logits_out) front_tail(a.logits_out, xrow, own_tok, own, m, tid);
  if (tracing) front_dump_marks(a.trace, a.trace_cap, s_ts, tid, 48);
#undef FRONT_MARK
}

// ---------------------------------------------------------------------------
// Router GEMM for large blocks, ahead of the front kernel (logits-in mode).
// In the front, large blocks either re-stream W_r per token chunk (split-K)
// or stream all of W_r into each of the 8 SMs (token split): ~12-17 us at
// M = 256, N >= 64, bound by per-SM ingress. Here one 8-CTA cluster per
// (32-token tile, 128-expert tile) splits K over its CTAs (each loads a 1/8
// slice of one W_r tile, <= 64 KB, plus its X boxes), drains TMEM into a
// stage and pushes each owner CTA its token rows with one bulk DSMEM copy;
// the owner sums the 8 partials in fixed CTA order (deterministic logits)
// and writes them to global memory. C3 N = 256: 16 clusters on 128 SMs.
// The front (programmatic launch) sets up meanwhile and reads the logits
// after griddepcontrol.wait.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 1)
    router_cluster_kernel(const __grid_constant__ CUtensorMap wr_map,
                          const __grid_constant__ BoxMaps x_maps, const RouterArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bars[8 + 2];  // full[kb_cta <= 8], tdone, recv
  __shared__ uint32_t tmem_slot[2];
  constexpr int C = kFrontCta;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rk = static_cast<int>(cluster_rank());
  const int cl = static_cast<int>(blockIdx.x) / C;
  const int tt = cl / a.mtiles, mtile = cl - tt * a.mtiles;
  const int t0 = tt * a.tc;
  const int nt = a.n - t0 < a.tc ? a.n - t0 : a.tc;  // tokens of this cluster
  const int e0 = mtile * kBM;
  const int me = a.m - e0 < kBM ? a.m - e0 : kBM;     // experts of this tile
  // K blocks of this CTA: an even split of d / 64 over the cluster (any
  // hidden size that is a multiple of 64; a CTA may get none)
  const int kbt = a.d / kBK;
  const int kb0 = (kbt * rk) / C, kb = (kbt * (rk + 1)) / C - kb0;
  const int ocm = (a.tc + C - 1) / C;                 // owner rows per sender
  const uint32_t xbytes = static_cast<uint32_t>(a.b_rows) * 128u;
  const int stage_bytes = kATile + a.b_rows * 128;
  unsigned char* ring = smem;                                                   // [kb][W tile | X box]
  // (laid out for the largest K share, a.kb_cta: every CTA's stage / recv at
  // the same offset, since peers address them through mapa)
  float* stage = reinterpret_cast<float*>(smem + static_cast<size_t>(a.kb_cta) * stage_bytes);  // [tc][128]
  float* recv = stage + a.tc * kBM;                                             // [C][ocm][128]
  uint64_t* full = bars;
  uint64_t* tdone = bars + 8;
  uint64_t* bar_recv = bars + 9;
  const int lo = (nt * rk) / C, hi = (nt * (rk + 1)) / C;  // this CTA's owner rows
  if (tid == 0) {
    tma_prefetch_desc(&wr_map);
    tma_prefetch_desc(&x_maps.map[a.box_index]);
    for (int i = 0; i < kb; ++i) mbar_init(&full[i], 1);
    mbar_init(tdone, 1);
    mbar_init(bar_recv, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(bar_recv, static_cast<uint32_t>(C * (hi - lo) * kBM * 4));
    const uint64_t pol = l2_policy_evict_last();  // W_r: re-read by every token tile
    for (int i = 0; i < kb; ++i) {  // static weights: before the previous kernel is waited for
      mbar_arrive_expect_tx(&full[i], kATile + xbytes);
      tma_load_2d(ring + static_cast<size_t>(i) * stage_bytes, &wr_map, &full[i], (kb0 + i) * kBK,
                  e0, pol);
    }
  }
  if (warp == 2) tmem_alloc(tmem_slot, 32u < static_cast<uint32_t>(a.b_rows) ? a.b_rows : 32u);
  pdl_launch_dependents();
  pdl_wait();  // x is complete from here on
  if (tid == 0) {
    const uint64_t pol_x = l2_policy_evict_last();
    for (int i = 0; i < kb; ++i)
      tma_load_2d(ring + static_cast<size_t>(i) * stage_bytes + kATile, &x_maps.map[a.box_index],
                  &full[i], (kb0 + i) * kBK, t0, pol_x);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_slot[0];
  // every CTA's recv barrier is armed before anyone pushes
  cluster_arrive_relaxed();
  cluster_wait();
  const int n_mma = (nt + 15) & ~15;
  if (warp == 1 && kb > 0) {
    const uint32_t idesc = idesc_bf16_f32(kBM, n_mma);
    for (int i = 0; i < kb; ++i) {
      mbar_wait(&full[i], 0);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t a0 = smem_u32(ring + static_cast<size_t>(i) * stage_bytes);
        const uint32_t b0 = a0 + kATile;
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk)
          tc_mma_bf16(tmem_base, sw128_kmajor_desc(a0 + kk * 32), sw128_kmajor_desc(b0 + kk * 32),
                      idesc, (i > 0 || kk > 0) ? 1u : 0u);
        if (i == kb - 1) tc_commit(tdone);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    // drain: partial[token][expert] of this CTA's K slice (zeros without one)
    const int q = warp & 3;
    const int r = q * 32 + lane;
    if (kb > 0) {
      mbar_wait(tdone, 0);
      tc_fence_after();
      const uint32_t lb = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
      for (int cc = 0; cc < n_mma; cc += 16) {
        float v[16];
        tmem_ld16(lb + cc, v);
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (cc + j < nt) stage[(cc + j) * kBM + r] = v[j];
      }
    } else {
      for (int t = 0; t < nt; ++t) stage[t * kBM + r] = 0.0f;
    }
    tc_fence_before();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    named_bar_sync(1, 128);
    if (warp == 4 && lane < C) {
      // one bulk copy per owner: its token rows -> recv[rk] there
      const int lo_q = (nt * lane) / C, hi_q = (nt * (lane + 1)) / C;
      const uint32_t bytes = static_cast<uint32_t>((hi_q - lo_q) * kBM * 4);
      if (bytes)
        bulk_s2cluster(mapa_u32(smem_u32(recv + rk * ocm * kBM), lane),
                       smem_u32(stage + lo_q * kBM), bytes, mapa_u32(smem_u32(bar_recv), lane));
    }
  }
  mbar_wait_cluster(bar_recv, 0);  // all C partials of this CTA's rows arrived
  // owner sums in fixed CTA order -> logits
  const int cnt = (hi - lo) * me;
  for (int w = tid; w < cnt; w += blockDim.x) {
    const int j = w / me, e = w - j * me;
    float acc = 0.0f;
#pragma unroll
    for (int r = 0; r < C; ++r) acc += recv[(r * ocm + j) * kBM + e];
    a.logits[static_cast<size_t>(t0 + lo + j) * a.m + e0 + e] = acc;
  }
  // no CTA exits while a peer's bulk copy may still read its stage
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 32u < static_cast<uint32_t>(a.b_rows) ? a.b_rows : 32u);
  }
}

size_t router_cluster_smem(const RouterArgs& a) {
  return 1024 + static_cast<size_t>(a.kb_cta) * (kATile + a.b_rows * 128) +
         static_cast<size_t>(a.tc) * kBM * 4 +
         static_cast<size_t>(kFrontCta) * ((a.tc + kFrontCta - 1) / kFrontCta) * kBM * 4;
}

cudaError_t launch_router_cluster(const CUtensorMap& wr_map, const BoxMaps& x_maps,
                                  const RouterArgs& a, cudaStream_t st) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(kFrontCta * a.mtiles * ((a.n + a.tc - 1) / a.tc));
  lc.blockDim = dim3(256);
  lc.dynamicSmemBytes = router_cluster_smem(a);
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
  return cudaLaunchKernelEx(&lc, router_cluster_kernel, wr_map, x_maps, a);
}

// Host plan: token chunk, pipeline depth, shared memory. Returns false when
// the shape is outside the kernel's envelope.
bool front_plan(int n, int m, int k, int d, FrontArgs* a, size_t* smem, int tsplit) {
  // pools of 257-512 experts only with the router GEMM ahead (logits in)
  if (n < 1 || n > 256 || m < 1 || m > (tsplit == 3 ? 512 : 256) || k < 1 || k > 32 || k > m)
    return false;
  if (tsplit == 3) {
    // logits in (router_cluster_kernel): no ring, no partial exchange
    const int own_max = (n + kFrontCta - 1) / kFrontCta;
    const FrontSmem p = front_smem_plan(n, m, k, n, own_max, 0, 0, n, 3);
    if (p.total > static_cast<size_t>(kFrontSmemLimit)) return false;
    a->tsplit = 3;
    a->chunk = n;
    a->own_max = own_max;
    a->stages = 0;
    a->b_rows = 16;
    a->box_index = 0;
    a->kb_per_cta = (d / kBK) / kFrontCta;
    a->tmem_cols = 0;
    a->vote_rows = n;
    *smem = p.total;
    return true;
  }
  if (d % (kBK * kFrontCta)) return false;
  const int mt = (m + kBM - 1) / kBM;
  const int kb_cta = (d / kBK) / kFrontCta;
  if (tsplit) {
    // token split: one "chunk", own = ceil(n / C) rows per CTA, X boxes of
    // b_rows >= own rows, up to 4 ring stages over all d / 64 K-blocks
    const int own_max = (n + kFrontCta - 1) / kFrontCta;
    int b_rows = 16;
    while (b_rows < own_max) b_rows <<= 1;
    for (int vr = n;; vr = vr > 16 ? (vr + 1) / 2 : 0) {
      if (vr == 0) return false;
      const int kb_total = kb_cta * kFrontCta;
      for (int stages = kb_total < 12 ? kb_total : 12; stages >= 2; --stages) {
        const FrontSmem p = front_smem_plan(n, m, k, n, own_max, stages, b_rows, vr, 1);
        if (p.total > static_cast<size_t>(kFrontSmemLimit)) continue;
        int bi = 0;
        while ((16 << bi) < b_rows) ++bi;
        a->tsplit = tsplit;
        a->chunk = n;
        a->own_max = own_max;
        a->stages = stages;
        a->b_rows = b_rows;
        a->box_index = bi;
        a->kb_per_cta = kb_cta;
        a->tmem_cols = mt * 256;
        a->vote_rows = vr;
        *smem = p.total;
        return true;
      }
    }
  }
  const int max_stages = kb_cta < 4 ? kb_cta : 4;
  // prefer: whole block in one GEMM chunk, >= 2 pipeline stages, the whole
  // vote matrix on chip; shrink the vote chunk first, then the token chunk
  for (int chunk = n;;) {
    int b_rows = 16;
    while (b_rows < chunk) b_rows <<= 1;
    const int nch = (n + chunk - 1) / chunk;
    const int own_max = nch * ((chunk + kFrontCta - 1) / kFrontCta);
    for (int vr = n;; vr = vr > 16 ? (vr + 1) / 2 : 0) {
      if (vr == 0) break;
      for (int stages = max_stages; stages >= 1; --stages) {
        if (stages < 2 && kb_cta > 1) break;
        const FrontSmem p = front_smem_plan(n, m, k, chunk, own_max, stages, b_rows, vr, 0);
        if (p.total > static_cast<size_t>(kFrontSmemLimit)) continue;
        int bi = 0;
        while ((16 << bi) < b_rows) ++bi;
        a->chunk = chunk;
        a->own_max = own_max;
        a->stages = stages;
        a->b_rows = b_rows;
        a->box_index = bi;
        a->kb_per_cta = kb_cta;
        a->tmem_cols = mt * 256;
        a->vote_rows = vr;
        *smem = p.total;
        return true;
      }
    }
    if (chunk <= 16) return false;
    chunk = ((chunk / 2) + 15) & ~15;
  }
}

using FrontFn = void (*)(const CUtensorMap, const BoxMaps, const FrontArgs);

// The instantiation for (strategy, token split, small block).
// kG: 0 split-K, 1 token split, 2 logits in (FrontArgs::tsplit 0 / 1-2 / 3)
static FrontFn front_variant(int strategy, int kg, bool small) {
#define DESMOE_FRONT_ROW(S)                                                      \
  {front_kernel<S, 0, false>, front_kernel<S, 0, true>, front_kernel<S, 1, false>, \
   front_kernel<S, 1, true>, front_kernel<S, 2, false>, front_kernel<S, 2, true>}
  static const FrontFn table[3][6] = {DESMOE_FRONT_ROW(-1), DESMOE_FRONT_ROW(0),
                                      DESMOE_FRONT_ROW(1)};
#undef DESMOE_FRONT_ROW
  const int si = strategy < 0 ? 0 : (strategy == 0 ? 1 : 2);
  return table[si][2 * kg + (small ? 1 : 0)];
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
  // small block: at most one own token per warp of a 8-warp group, so the
  // selection and the activation run side by side (DESMOE_FRONT_FLAGS bit 2
  // forces the sequential L stage, for A/B runs)
  const bool small = a.own_max <= kFrontThreads / 64 && !(a.flags & 2);
  const int kg = a.tsplit == 3 ? 2 : (a.tsplit != 0 ? 1 : 0);
  return cudaLaunchKernelEx(&lc, front_variant(a.strategy, kg, small), wr_map, x_maps, a);
}

cudaError_t set_front_smem_limit() {
  cudaError_t e = cudaSuccess;
  for (int strategy = -1; strategy <= 1; ++strategy)
    for (int v = 0; v < 6; ++v) {
      const cudaError_t r = cudaFuncSetAttribute(
          reinterpret_cast<const void*>(front_variant(strategy, v / 2, v & 1)),
          cudaFuncAttributeMaxDynamicSharedMemorySize, kFrontSmemLimit);
      if (e == cudaSuccess) e = r;
    }
  const cudaError_t r = cudaFuncSetAttribute(reinterpret_cast<const void*>(router_cluster_kernel),
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             200 * 1024);
  return e == cudaSuccess ? r : e;
}

}  // namespace desmoe
