// Shared device helpers for the sm_100a DES MoE kernels: mbarrier, TMA
// (cp.async.bulk.tensor), tcgen05 (MMA / TMEM alloc / TMEM load) and warp
// selection primitives. Inline PTX only; compiled for sm_100a exclusively.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include "libm_exp.cuh"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "desmoe kernels target sm_100a only"
#endif

namespace desmoe {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// Ordering keys. Every selection in the reference orders by (value desc,
// index asc) (gating.cpp:49-52, des.cpp:143-146, des.cpp:210-213). For fp64
// values we map the IEEE bits to an order-preserving u64 so one integer
// compare decides the value part; the index breaks exact ties.
// ---------------------------------------------------------------------------
__host__ __device__ inline uint64_t order_key(double v) {
  uint64_t u;
#ifdef __CUDA_ARCH__
  u = static_cast<uint64_t>(__double_as_longlong(v));
#else
  __builtin_memcpy(&u, &v, 8);
#endif
  // -0.0 and +0.0 compare equal in the reference's `!=`; fold -0 onto +0.
  if (u == 0x8000000000000000ull) u = 0;
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

// (ka, ia) precedes (kb, ib) in (value desc, index asc) order
__host__ __device__ inline bool key_precedes(uint64_t ka, int ia, uint64_t kb, int ib) {
  return ka != kb ? ka > kb : ia < ib;
}

// Warp-wide arg-best under key_precedes; every lane gets the winner.
__device__ inline void warp_argbest(uint64_t& key, int& idx) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    uint64_t ok = __shfl_xor_sync(0xffffffffu, key, off);
    int oi = __shfl_xor_sync(0xffffffffu, idx, off);
    if (key_precedes(ok, oi, key, idx)) {
      key = ok;
      idx = oi;
    }
  }
}

// Returns, for lane j < cnt, the ascending position of `my` among the cnt
// values held by lanes 0..cnt-1 (values distinct).
__device__ inline int ascending_rank(int my, int lane, int cnt) {
  int pos = 0;
  for (int j = 0; j < cnt; ++j) {
    int o = __shfl_sync(0xffffffffu, my, j);
    if (lane < cnt && (o < my)) ++pos;
  }
  return pos;
}

// Per-warp selection of `k` entries of row p[0..m) restricted to `allow`
// (nullptr = all) in (p desc, index asc) order — the reference's
// select_top_gates order (gating.cpp:42-71). Rank-ordered result in sel[0..k)
// (written by every lane). Lane l owns elements l, l+32, ... (m <= 1024).
static __device__ __noinline__ void warp_select(const double* p, int m, int k,
                                                const uint8_t* allow, int* sel) {
  const int lane = threadIdx.x & 31;
  uint32_t taken = 0;
  uint64_t bk = 0;
  int bi = 0x7fffffff;
  auto rescan = [&]() {
    bk = 0;
    bi = 0x7fffffff;
    for (int s = 0, i = lane; i < m; ++s, i += 32) {
      if ((taken >> s) & 1u) continue;
      if (allow && !allow[i]) continue;
      const uint64_t kk = order_key(p[i]);
      if (bi == 0x7fffffff || key_precedes(kk, i, bk, bi)) {
        bk = kk;
        bi = i;
      }
    }
  };
  rescan();
  for (int r = 0; r < k; ++r) {
    uint64_t wk = bk;
    int wi = bi;
    // lanes without a candidate carry (0, INT_MAX), which never beats a real
    // candidate (order_key of a finite double is never 0)
    warp_argbest(wk, wi);
    sel[r] = wi;
    if ((wi & 31) == lane) {
      taken |= 1u << (wi >> 5);
      rescan();
    }
  }
  __syncwarp();
}

// Fast warp top-k for the routing hot path. Candidates carry a packed 64-bit
// key: the order-preserving key of the value with its 10 lowest bits replaced
// by (1023 - index), so ONE unsigned max picks (value desc, index asc) —
// exactly the reference's order unless two distinct values agree in all but
// those 10 bits (relative gap < 2^-42). Each round is two 32-bit warp
// reductions (REDUX) instead of a 5-level 64-bit shuffle tree. Rounds run to
// `rounds` (>= k; one past a boundary lets the caller see the next key).
// sel[r] = index of round r (all lanes), keys[r] = its packed key.
// m <= 1024, rounds <= 32. Lanes own elements lane, lane+32, ...
__device__ inline uint64_t packed_key(double v, int i) {
  return (order_key(v) & ~0x3FFull) | static_cast<uint64_t>(1023 - i);
}

static __device__ __noinline__ void warp_topk_packed(const double* val, int m, int rounds,
                                                     const uint8_t* allow, int* sel,
                                                     uint64_t* keys) {
  const int lane = threadIdx.x & 31;
  uint32_t taken = 0;
  auto local_best = [&]() -> uint64_t {
    uint64_t b = 0;
    for (int s = 0, i = lane; i < m; ++s, i += 32) {
      if (((taken >> s) & 1u) || (allow && !allow[i])) continue;
      const uint64_t kk = packed_key(val[i], i);
      b = kk > b ? kk : b;
    }
    return b;
  };
  uint64_t best = local_best();
  for (int r = 0; r < rounds; ++r) {
    const uint32_t hi = __reduce_max_sync(0xffffffffu, static_cast<uint32_t>(best >> 32));
    const uint32_t lo = __reduce_max_sync(
        0xffffffffu, static_cast<uint32_t>(best >> 32) == hi ? static_cast<uint32_t>(best) : 0u);
    const uint64_t win = (static_cast<uint64_t>(hi) << 32) | lo;
    const int idx = 1023 - static_cast<int>(lo & 0x3FFu);
    if (lane == 0) {
      sel[r] = win ? idx : -1;
      keys[r] = win;
    }
    if (win && (idx & 31) == lane) {
      taken |= 1u << (idx >> 5);
      best = local_best();
    }
  }
  __syncwarp();
}

// Out-of-line fp64 exp and division (as the reference's std::exp /
// operator/): the routing kernels execute these once per element
// from many sites; one shared copy keeps their code (and instruction fetch
// after an L2 flush) small.
// exp is glibc's, restated bit for bit (libm_exp.cuh).
static __device__ __noinline__ double exp_f64(double x) { return glibc_exp(x, kExpTab); }
static __device__ __noinline__ double div_f64(double a, double b) { return a / b; }
static __device__ __noinline__ double sigmoid_f64(double x) {
  return 1.0 / (1.0 + glibc_exp(-x, kExpTab));
}

// Truncated key of a packed key (drops the index bits).
__device__ inline uint64_t key_value_part(uint64_t pk) { return pk >> 10; }

// ---------------------------------------------------------------------------
// shared-memory addressing / mbarrier
// ---------------------------------------------------------------------------
__device__ inline uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ inline void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ inline void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ inline void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ inline void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ inline bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ inline void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// ---------------------------------------------------------------------------
// TMA (tensor-map bulk copies, async proxy)
// ---------------------------------------------------------------------------
__device__ inline void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ inline uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ inline uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 2-D tile load: coords (c0 = innermost / K element, c1 = row)
__device__ inline void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                   int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}

// 2-D tile load multicast to the CTAs of `mask` in the cluster: the tile lands
// at the same shared-memory offset in each and completes the transaction
// bytes on the mbarrier at `bar`'s offset in each
__device__ inline void tma_load_2d_mc(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                      int c1, uint16_t mask, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5, %6;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask),
      "l"(policy)
      : "memory");
}

// 3-D tile load (packed weight tiles): coords (c0, c1, c2)
__device__ inline void tma_load_3d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                   int c1, int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "l"(policy)
      : "memory");
}

// L2 prefetch of a contiguous global range (one bulk instruction)
__device__ inline void bulk_prefetch_l2(const void* gaddr, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gaddr), "r"(bytes) : "memory");
}

// L2 prefetch of a 3-D tile (no shared memory, no completion tracking)
__device__ inline void tma_prefetch_l2_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

// Orders this thread's generic-proxy view (e.g. an acquire of a flag set by a
// producer CTA) before its subsequent async-proxy (TMA) global reads.
__device__ inline void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ inline void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------------------
// tcgen05: TMEM allocation, MMA, commit, TMEM -> register loads
// ---------------------------------------------------------------------------
__device__ inline void tmem_alloc(uint32_t* slot_smem, uint32_t ncols) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ inline void tmem_dealloc(uint32_t taddr, uint32_t ncols) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

__device__ inline void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ inline void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// Shared-memory matrix descriptor for a K-major operand tile stored in the
// canonical SWIZZLE_128B layout that TMA writes: rows of 128 B (64 bf16),
// 8-row / 1024 B swizzle atoms. LBO unused (1), SBO = 1024 B, version 1,
// layout type 2 (SWIZZLE_128B).
__device__ inline uint64_t sw128_kmajor_desc(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;
  d |= static_cast<uint64_t>(1024u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}

// Instruction descriptor, kind::f16: BF16 A/B, F32 accumulate, both K-major.
__host__ __device__ inline uint32_t idesc_bf16_f32(int m, int n) {
  return (1u << 4)                                   // D format F32
         | (1u << 7)                                 // A format BF16
         | (1u << 10)                                // B format BF16
         | (static_cast<uint32_t>(n >> 3) << 17)     // N / 8
         | (static_cast<uint32_t>(m >> 4) << 24);    // M / 16
}

// D[tmem] (+)= A[smem] * B[smem]^T, single elected thread.
__device__ inline void tc_mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                   uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrives on `bar` when every previously issued tcgen05.mma of this thread
// has completed (implicitly fences before_thread_sync).
__device__ inline void tc_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// arrive (once) on the mbarrier at `bar`'s offset in every CTA of `mask` when
// this thread's prior tcgen05 operations complete
__device__ inline void tc_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

// 32 lanes x 32-bit, 16 consecutive columns: thread t of warp (w % 4) gets
// TMEM lane 32*(w%4)+t, columns [col, col+16).
__device__ inline void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ inline uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Optional timeline trace: records {unit<<32 | cta<<8 | event, globaltimer ns}.
__device__ inline void trace(uint64_t* buf, int cap, int event, int unit) {
  if (!buf) return;
  // timestamp first: the cursor atomic can take microseconds when many CTAs
  // trace at once (same-address atomics serialise in L2)
  const uint64_t ts = gtime();
  unsigned long long* cur = reinterpret_cast<unsigned long long*>(buf);
  const unsigned long long i = atomicAdd(cur, 1ull);
  if (i < static_cast<unsigned long long>(cap)) {
    buf[2 + 2 * i] = (static_cast<uint64_t>(static_cast<uint32_t>(unit)) << 32) |
                     (static_cast<uint64_t>(blockIdx.x) << 8) | static_cast<uint64_t>(event);
    buf[3 + 2 * i] = ts;
  }
}

// Atomic-free per-thread trace cursor: one emitting thread claims `slots`
// records at its start (when the memory system is idle) and then only stores
// into them, so tracing does not stall the traced code on a contended atomic.
// Unused records are written as event 255 (ignored by the decoders).
struct TraceCursor {
  uint64_t* p;
  int n, cap;
};

__device__ inline TraceCursor trace_open(uint64_t* buf, int cap, int slots) {
  TraceCursor c{nullptr, 0, 0};
  if (!buf) return c;
  const unsigned long long i0 =
      atomicAdd(reinterpret_cast<unsigned long long*>(buf), static_cast<unsigned long long>(slots));
  const long long room = static_cast<long long>(cap) - static_cast<long long>(i0);
  c.p = buf + 2 + 2 * i0;
  c.cap = room <= 0 ? 0 : (room < slots ? static_cast<int>(room) : slots);
  return c;
}

__device__ inline void trace_put(TraceCursor& c, int event, int unit) {
  if (c.n >= c.cap) return;
  const uint64_t ts = gtime();
  c.p[2 * c.n] = (static_cast<uint64_t>(static_cast<uint32_t>(unit)) << 32) |
                 (static_cast<uint64_t>(blockIdx.x) << 8) | static_cast<uint64_t>(event);
  c.p[2 * c.n + 1] = ts;
  ++c.n;
}

__device__ inline void trace_close(TraceCursor& c) {
  for (; c.n < c.cap; ++c.n) c.p[2 * c.n] = 255;
}

// Programmatic dependent launch: let the next kernel in the stream start its
// prologue now / wait until the previous kernel's results are visible.
__device__ inline void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ inline void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ inline bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// gpu-scope acquire load / release add for cross-CTA flags
__device__ inline unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ inline void atomic_add_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ inline uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ inline uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Data-check flags (c->err) live in host-mapped pinned memory: a plain
// (volatile) store, no atomics (PCIe may lack native host atomics).
__device__ inline void raise_flag(int* p, int v) { *reinterpret_cast<volatile int*>(p) = v; }

__device__ inline uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ inline void st_relaxed_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ inline void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ inline int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// release increment without a returned value: the thread does not wait for
// the atomic's response (under a full TMA ring every response to an SM
// queues behind the weights in flight, ~3-4 us)
__device__ inline void red_add_release(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ inline int atomic_add_release(int* p, int v) {
  int old;
  asm volatile("atom.add.release.gpu.global.s32 %0, [%1], %2;"
               : "=r"(old)
               : "l"(p), "r"(v)
               : "memory");
  return old;
}

__device__ inline int atomic_add_acq_rel(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;"
               : "=r"(old)
               : "l"(p), "r"(v)
               : "memory");
  return old;
}

__device__ inline void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Arrive on a named barrier without waiting (producer side of a hand-off:
// the threads that bar.sync on it see this thread's earlier shared writes).
__device__ inline void named_bar_arrive(int id, int threads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

}  // namespace desmoe
