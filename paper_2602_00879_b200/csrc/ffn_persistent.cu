// K3 + K4: persistent grouped expert FFN for sm_100a, one CTA per SM.
//
// One launch does the whole post-routing half of the DES MoE layer:
//   prologue  every CTA rebuilds the permutation from the route (per-expert
//             counts, ascending offsets, stable token order, active experts —
//             the count route of moe_latency, analysis.cpp:16-30) in shared
//             memory, then gathers its share of token rows into the
//             expert-grouped activation buffer x_perm;
//   phase A   (SwiGLU) units (expert, 128-row F tile): G = W_g.X_e^T and
//             U = W_u.X_e^T in two TMEM accumulators, H = bf16(silu(G) * U)
//             written to h_perm; per-expert readiness counter bumped;
//   phase B   units (expert, 128-row d tile): Y = W_d.H_e^T (or the linear
//             expert W.X_e^T), scaled by each slot's gate into y_slot; the
//             last unit to finish a (token, d tile) sums that token's slots in
//             ascending expert order (moe_forward's order, gating.cpp:141-155)
//             into y — a deterministic fused combine.
// Units are handed out by a global atomic counter (phase A before phase B,
// expert-major), so every SM streams weights until the queue drains; each
// active expert's weights are read from HBM exactly once.
//
// Warp roles (256 threads): warp 0 = scheduler + TMA producer, warp 1 = MMA
// issuer (one elected lane, tcgen05.mma kind::f16, swap-AB: 128 weight rows
// x N tokens, N = tokens of the expert rounded to 16), warp 2 = TMEM
// allocator, then gather, then combine worker; warp 3 = combine worker;
// warps 4-7 = epilogue (tcgen05.ld of TMEM lane quarters 0-3). The gather and
// the combine run on their own warps so neither delays the weight stream nor
// the TMEM drain.
// Shared-memory ring stages hold two 128x64 bf16 weight tiles (32 KB: gate +
// up in phase A, two consecutive K blocks of W_d in phase B) and two
// activation boxes, all SWIZZLE_128B as TMA writes them.
#include "common.cuh"
#include "kernels.cuh"

namespace desmoe {

namespace {

constexpr int kThreads = 256;
constexpr int kQ = 4;  // unit queue depth
constexpr int kC = 8;  // combine queue depth

struct Tables {
  int* count;      // [m]
  int* offset;     // [m]
  int* active;     // [m]
  int* slot_token; // [S]
  float* slot_gate;// [S]
  int* slot_of;    // [n*k]
  int* scalars;    // [0] U, [1] S, [2] list size (combine), [3..] token list
};

struct UnitInfo {
  int phase;  // 0 = A (gate/up), 1 = B (down / linear)
  int expert, tile, brow, count;
};

__device__ inline UnitInfo decode(int u, int nA, int tilesA, int tilesB, const Tables& t) {
  UnitInfo r;
  if (u < nA) {
    r.phase = 0;
    int ei = u / tilesA;
    r.tile = u - ei * tilesA;
    r.expert = t.active[ei];
  } else {
    u -= nA;
    r.phase = 1;
    int ei = u / tilesB;
    r.tile = u - ei * tilesB;
    r.expert = t.active[ei];
  }
  r.brow = t.offset[r.expert];
  r.count = t.count[r.expert];
  return r;
}

__device__ inline int box_for(int count) {
  int b = 0;
  while ((16 << b) < count && b < kMaxBoxes - 1) ++b;
  return b;
}

__device__ inline float silu(float g) { return g / (1.0f + expf(-g)); }

__device__ inline uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Optional timeline trace: records {unit<<32 | cta<<8 | event, globaltimer ns}.
__device__ inline void trace(uint64_t* buf, int cap, int event, int unit) {
  if (!buf) return;
  unsigned long long* cur = reinterpret_cast<unsigned long long*>(buf);
  const unsigned long long i = atomicAdd(cur, 1ull);
  if (i < static_cast<unsigned long long>(cap)) {
    buf[2 + 2 * i] = (static_cast<uint64_t>(static_cast<uint32_t>(unit)) << 32) |
                     (static_cast<uint64_t>(blockIdx.x) << 8) | static_cast<uint64_t>(event);
    buf[3 + 2 * i] = gtime();
  }
}

// Block-wide exclusive scan of v[0..n) (n <= 4 * kThreads) in place; returns total.
__device__ int block_exclusive_scan(int* v, int n, int* warp_sums) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int loc[4];
  int sum = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int idx = tid * 4 + i;
    loc[i] = idx < n ? v[idx] : 0;
    sum += loc[i];
  }
  int incl = sum;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
      int t = warp_sums[w];
      warp_sums[w] = acc;
      acc += t;
    }
    warp_sums[kThreads / 32] = acc;
  }
  __syncthreads();
  int base = warp_sums[warp] + incl - sum;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int idx = tid * 4 + i;
    if (idx < n) v[idx] = base;
    base += loc[i];
  }
  int total = warp_sums[kThreads / 32];
  __syncthreads();
  return total;
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 1)
    ffn_persistent_kernel(const __grid_constant__ CUtensorMap w_a,   // W_g (A) or W_d / W_lin (B)
                          const __grid_constant__ CUtensorMap w_b,   // W_u (A)
                          const __grid_constant__ CUtensorMap w_c,   // W_d (B, SwiGLU)
                          const __grid_constant__ BoxMaps xp_maps,   // x_perm boxes
                          const __grid_constant__ BoxMaps h_maps,    // h_perm boxes
                          FfnArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_tok = a.n_tok, k = a.top_k, m = a.m, d = a.d, f = a.f;
  if (tid == 0) trace(a.trace, a.trace_cap, 0, -1);
  const bool swiglu = a.mode == 0;
  const int S = a.stages;
  const int b_box_bytes = a.b_rows * 128;
  const int stage_bytes = 2 * kATile + 2 * b_box_bytes;

  // ---- shared-memory carve-up --------------------------------------------
  unsigned char* ring = smem;
  unsigned char* p = ring + static_cast<size_t>(S) * stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(p);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;   // [2]
  uint64_t* tempty = tfull + 2;  // [2]
  uint64_t* qfull = tempty + 2;  // [kQ]
  uint64_t* qempty = qfull + kQ; // [kQ]
  uint64_t* cfull = qempty + kQ; // [kC] combine queue
  uint64_t* cempty = cfull + kC; // [kC]
  int* unit_q = reinterpret_cast<int*>(cempty + kC);
  int* comb_q = unit_q + kQ;     // [kC]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(comb_q + kC);
  int* warp_sums = reinterpret_cast<int*>(tmem_slot + 4);  // [9]
  Tables t;
  t.scalars = warp_sums + 12;  // [4 + n_tok]
  t.count = t.scalars + 4 + n_tok;
  t.offset = t.count + m;
  t.active = t.offset + m;
  t.slot_of = t.active + m;
  t.slot_token = t.slot_of + n_tok * k;
  t.slot_gate = reinterpret_cast<float*>(t.slot_token + n_tok * k);
  // prologue scratch aliases the ring (unused until the roles start)
  const int tw = (n_tok + 31) >> 5;
  uint32_t* bits = reinterpret_cast<uint32_t*>(ring);  // [m][tw]

  int* sched = a.counters;
  int* x_ready = a.counters + 1;
  int* h_ready = a.counters + 2;             // [m]
  int* tok_done = a.counters + 2 + m;        // [n_tok][d/128]

  // ---- prologue: permutation (redundantly per CTA) ------------------------
  for (int i = tid; i < m; i += kThreads) t.count[i] = 0;
  for (int i = tid; i < m * tw; i += kThreads) bits[i] = 0;
  __syncthreads();
  for (int e = tid; e < n_tok * k; e += kThreads) {
    const int tok = e / k, j = e - tok * k;
    if (j >= a.route_cnt[tok]) continue;
    const int x = a.route_idx[e];
    atomicAdd(&t.count[x], 1);
    atomicOr(&bits[x * tw + (tok >> 5)], 1u << (tok & 31));
  }
  __syncthreads();
  for (int i = tid; i < m; i += kThreads) t.offset[i] = t.count[i];
  __syncthreads();
  const int total_slots = block_exclusive_scan(t.offset, m, warp_sums);
  // active list (ascending)
  for (int i = tid; i < m; i += kThreads) t.active[i] = t.count[i] > 0 ? 1 : 0;
  __syncthreads();
  int* act_pos = reinterpret_cast<int*>(bits + m * tw);  // ring scratch
  for (int i = tid; i < m; i += kThreads) act_pos[i] = t.active[i];
  __syncthreads();
  const int U = block_exclusive_scan(act_pos, m, warp_sums);
  int my_act[4];
  for (int r = 0; r < 4; ++r) {
    int i = tid + r * kThreads;
    my_act[r] = (i < m && t.count[i] > 0) ? act_pos[i] : -1;
  }
  __syncthreads();
  for (int r = 0; r < 4; ++r) {
    int i = tid + r * kThreads;
    if (my_act[r] >= 0) t.active[my_act[r]] = i;
  }
  for (int e = tid; e < n_tok * k; e += kThreads) {
    const int tok = e / k, j = e - tok * k;
    if (j >= a.route_cnt[tok]) {
      t.slot_of[e] = -1;
      continue;
    }
    const int x = a.route_idx[e];
    const uint32_t* b = bits + x * tw;
    int before = 0;
    for (int w = 0; w < (tok >> 5); ++w) before += __popc(b[w]);
    before += __popc(b[tok >> 5] & ((1u << (tok & 31)) - 1u));
    const int slot = t.offset[x] + before;
    t.slot_of[e] = slot;
    t.slot_token[slot] = tok;
    t.slot_gate[slot] = static_cast<float>(a.route_gate[e]);
  }
  if (tid == 0) {
    t.scalars[0] = U;
    t.scalars[1] = total_slots;
  }
  __syncthreads();
  if (blockIdx.x == 0 && tid == 0 && a.stats) {
    a.stats[0] = U;
    a.stats[1] = a.n_members ? *a.n_members : U;
    a.stats[2] = total_slots;
    a.stats[3] = 0;
  }
  // ---- barriers / TMEM ---------------------------------------------------
  const int tilesA = f / kBM, tilesB = d / kBM;
  const int nA = swiglu ? U * tilesA : 0;
  const int n_units = nA + U * tilesB;
  const int ksA = d / kBK;                          // phase A k-steps (1 K block each)
  const int ksB = (swiglu ? f : d) / (2 * kBK);     // phase B k-steps (2 K blocks each)
  const bool dbuf = a.b_rows <= 128;
  const uint32_t buf_cols = dbuf ? 256u : 512u;
  const uint32_t up_off = dbuf ? static_cast<uint32_t>(a.b_rows) : 256u;

  if (tid == 0) {
    tma_prefetch_desc(&w_a);
    if (swiglu) {
      tma_prefetch_desc(&w_b);
      tma_prefetch_desc(&w_c);
    }
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);  // one arrival per epilogue warp
    }
    for (int q = 0; q < kQ; ++q) {
      mbar_init(&qfull[q], 1);
      mbar_init(&qempty[q], 2);  // MMA lane + epilogue
    }
    for (int q = 0; q < kC; ++q) {
      mbar_init(&cfull[q], 1);
      mbar_init(&cempty[q], 2);  // both combine warps
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ============ scheduler + TMA producer ============
    if (lane == 0) {
      const uint64_t pol_w = l2_policy_evict_first();
      const uint64_t pol_x = l2_policy_evict_last();
      uint32_t it = 0;
      bool x_seen = false;
      for (int qi = 0;; ++qi) {
        const int q = qi % kQ;
        const int u = atomicAdd(sched, 1);
        const int uu = u < n_units ? u : -1;
        mbar_wait(&qempty[q], ((qi / kQ) & 1) ^ 1);
        unit_q[q] = uu;
        mbar_arrive(&qfull[q]);
        if (uu < 0) break;
        trace(a.trace, a.trace_cap, 2, uu);
        const UnitInfo ui = decode(uu, nA, tilesA, tilesB, t);
        const int bi = box_for(ui.count);
        const int box_bytes = (16 << bi) * 128;
        const bool phaseA = ui.phase == 0;
        const BoxMaps& acts = (phaseA || !swiglu) ? xp_maps : h_maps;
        const CUtensorMap* wmap = phaseA ? &w_a : (swiglu ? &w_c : &w_a);
        const int wrow = phaseA ? ui.expert * f + ui.tile * kBM : ui.expert * d + ui.tile * kBM;
        const int ksteps = phaseA ? ksA : ksB;
        const uint32_t bytes = 2 * kATile + (phaseA ? 1 : 2) * box_bytes;
        for (int ks = 0; ks < ksteps; ++ks, ++it) {
          const int s = it % S;
          mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
          unsigned char* st = ring + static_cast<size_t>(s) * stage_bytes;
          mbar_arrive_expect_tx(&full[s], bytes);
          if (phaseA) {
            tma_load_2d(st, &w_a, &full[s], ks * kBK, wrow, pol_w);
            tma_load_2d(st + kATile, &w_b, &full[s], ks * kBK, wrow, pol_w);
          } else {
            tma_load_2d(st, wmap, &full[s], 2 * ks * kBK, wrow, pol_w);
            tma_load_2d(st + kATile, wmap, &full[s], (2 * ks + 1) * kBK, wrow, pol_w);
          }
          if (ks == 0) {
            // activations must be complete before their first TMA read
            if (phaseA || !swiglu) {
              if (!x_seen) {
                while (ld_acquire(x_ready) < static_cast<int>(gridDim.x)) {
                }
                x_seen = true;
                trace(a.trace, a.trace_cap, 6, uu);
              }
            } else {
              while (ld_acquire(&h_ready[ui.expert]) < tilesA) {
              }
              trace(a.trace, a.trace_cap, 7, uu);
            }
            fence_proxy_async_global();
          }
          if (phaseA) {
            tma_load_2d(st + 2 * kATile, &acts.map[bi], &full[s], ks * kBK, ui.brow, pol_x);
          } else {
            tma_load_2d(st + 2 * kATile, &acts.map[bi], &full[s], 2 * ks * kBK, ui.brow, pol_x);
            tma_load_2d(st + 2 * kATile + b_box_bytes, &acts.map[bi], &full[s],
                        (2 * ks + 1) * kBK, ui.brow, pol_x);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ============ MMA issuer ============
    uint32_t it = 0, nunit = 0;
    for (int qi = 0;; ++qi) {
      const int q = qi % kQ;
      mbar_wait(&qfull[q], (qi / kQ) & 1);
      const int uu = unit_q[q];
      __syncwarp();
      if (lane == 0) mbar_arrive(&qempty[q]);
      if (uu < 0) break;
      const UnitInfo ui = decode(uu, nA, tilesA, tilesB, t);
      const bool phaseA = ui.phase == 0;
      const int n_mma = (ui.count + 15) & ~15;
      const uint32_t idesc = idesc_bf16_f32(kBM, n_mma);
      const uint32_t buf = dbuf ? (nunit & 1u) : 0u;
      const uint32_t use = dbuf ? (nunit >> 1) : nunit;
      mbar_wait(&tempty[buf], (use & 1u) ^ 1u);
      tc_fence_after();
      const uint32_t d_acc = tmem_base + buf * buf_cols;
      const int ksteps = phaseA ? ksA : ksB;
      for (int ks = 0; ks < ksteps; ++ks, ++it) {
        const int s = it % S;
        mbar_wait(&full[s], (it / S) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a0 = smem_u32(ring + static_cast<size_t>(s) * stage_bytes);
          const uint32_t a1 = a0 + kATile;
          const uint32_t b0 = a0 + 2 * kATile;
          const uint32_t b1 = b0 + b_box_bytes;
          if (phaseA) {
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk) {
              const uint32_t acc = (ks > 0 || kk > 0) ? 1u : 0u;
              const uint64_t bd = sw128_kmajor_desc(b0 + kk * 32);
              tc_mma_bf16(d_acc, sw128_kmajor_desc(a0 + kk * 32), bd, idesc, acc);
              tc_mma_bf16(d_acc + up_off, sw128_kmajor_desc(a1 + kk * 32), bd, idesc, acc);
            }
          } else {
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              tc_mma_bf16(d_acc, sw128_kmajor_desc(a0 + kk * 32), sw128_kmajor_desc(b0 + kk * 32),
                          idesc, (ks > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              tc_mma_bf16(d_acc, sw128_kmajor_desc(a1 + kk * 32), sw128_kmajor_desc(b1 + kk * 32),
                          idesc, 1u);
          }
          tc_commit(&empty[s]);
          if (ks == ksteps - 1) tc_commit(&tfull[buf]);
        }
        __syncwarp();
      }
      ++nunit;
    }
  } else if (warp == 2 || warp == 3) {
    // ============ gather (warp 2), then combine workers (warps 2-3) ============
    if (warp == 2) {
      const int vec = d / 8;
      const uint4* src = reinterpret_cast<const uint4*>(a.x);
      uint4* dst = reinterpret_cast<uint4*>(a.x_perm);
      const int total_slots = t.scalars[1];
      for (int s2 = blockIdx.x; s2 < total_slots; s2 += gridDim.x) {
        const uint4* rs = src + static_cast<size_t>(t.slot_token[s2]) * vec;
        uint4* rd = dst + static_cast<size_t>(s2) * vec;
        for (int i = lane; i < vec; i += 32) rd[i] = rs[i];
      }
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        atomic_add_release(x_ready, 1);
        trace(a.trace, a.trace_cap, 1, -1);
      }
    }
    const int ctid = tid - 64;  // 0..63
    const int dtiles = d / kBM;
    int* list_n = t.scalars + 2;
    int* list = t.scalars + 4;
    for (int ci = 0;; ++ci) {
      const int q = ci % kC;
      mbar_wait(&cfull[q], (ci / kC) & 1);
      const int uu = comb_q[q];
      named_bar_sync(2, 64);
      if (lane == 0) mbar_arrive(&cempty[q]);
      if (uu < 0) break;
      const UnitInfo ui = decode(uu, nA, tilesA, tilesB, t);
      if (ctid == 0) *list_n = 0;
      named_bar_sync(2, 64);
      for (int c = ctid; c < ui.count; c += 64) {
        const int tok = t.slot_token[ui.brow + c];
        const int old = atomic_add_acq_rel(&tok_done[tok * dtiles + ui.tile], 1);
        if (old + 1 == a.route_cnt[tok]) list[atomicAdd(list_n, 1)] = tok;
      }
      named_bar_sync(2, 64);
      const int nl = *list_n;
      // each thread owns rows ctid and ctid+64 of the d tile; all slot loads
      // of a token are independent and issued together
      for (int li = 0; li < nl; ++li) {
        const int tok = list[li];
        const int cnt = a.route_cnt[tok];
        const float* base = a.y_slot + ui.tile * kBM + ctid;
        float acc0 = 0.0f, acc1 = 0.0f;
        float v0[8], v1[8];
        for (int j0 = 0; j0 < cnt; j0 += 8) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int jj = j0 + j;
            if (jj < cnt) {
              const float* row = base + static_cast<size_t>(t.slot_of[tok * k + jj]) * d;
              v0[j] = __ldcg(row);
              v1[j] = __ldcg(row + 64);
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (j0 + j < cnt) {
              acc0 += v0[j];
              acc1 += v1[j];
            }
          }
        }
        float* out = a.y + static_cast<size_t>(tok) * d + ui.tile * kBM + ctid;
        out[0] = acc0;
        out[64] = acc1;
      }
      named_bar_sync(2, 64);
    }
  } else if (warp >= 4) {
    // ============ epilogue ============
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;  // accumulator row = weight row within the tile
    const int etid = tid - 128;    // 0..127
    uint32_t nunit = 0, ncomb = 0;
    for (int qi = 0;; ++qi) {
      const int q = qi % kQ;
      mbar_wait(&qfull[q], (qi / kQ) & 1);
      const int uu = unit_q[q];
      named_bar_sync(1, 128);
      if (etid == 0) mbar_arrive(&qempty[q]);
      if (uu < 0) {
        if (etid == 0) {
          const int cq = ncomb % kC;
          mbar_wait(&cempty[cq], ((ncomb / kC) & 1) ^ 1);
          comb_q[cq] = -1;
          mbar_arrive(&cfull[cq]);
        }
        break;
      }
      const UnitInfo ui = decode(uu, nA, tilesA, tilesB, t);
      const bool phaseA = ui.phase == 0;
      const int n_mma = (ui.count + 15) & ~15;
      const uint32_t buf = dbuf ? (nunit & 1u) : 0u;
      const uint32_t use = dbuf ? (nunit >> 1) : nunit;
      mbar_wait(&tfull[buf], use & 1u);
      tc_fence_after();
      const uint32_t lane_base =
          tmem_base + buf * buf_cols + (static_cast<uint32_t>(q4 * 32) << 16);
      if (phaseA) {
        __nv_bfloat16* hrow = a.h_perm + static_cast<size_t>(ui.brow) * f + ui.tile * kBM + r;
        for (int c0 = 0; c0 < n_mma; c0 += 16) {
          float g[16], uacc[16];
          tmem_ld16(lane_base + c0, g);
          tmem_ld16(lane_base + up_off + c0, uacc);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int col = c0 + j;
            if (col < ui.count)
              hrow[static_cast<size_t>(col) * f] = __float2bfloat16_rn(silu(g[j]) * uacc[j]);
          }
        }
      } else {
        float* yrow = a.y_slot + static_cast<size_t>(ui.brow) * d + ui.tile * kBM + r;
        for (int c0 = 0; c0 < n_mma; c0 += 16) {
          float v[16];
          tmem_ld16(lane_base + c0, v);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int col = c0 + j;
            if (col < ui.count)
              yrow[static_cast<size_t>(col) * d] = v[j] * t.slot_gate[ui.brow + col];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      named_bar_sync(1, 128);
      if (etid == 0) {
        __threadfence();  // all epilogue stores (ordered by the barrier) -> gpu scope
        if (phaseA) {
          atomic_add_release(&h_ready[ui.expert], 1);
        } else {
          const int q = ncomb % kC;
          mbar_wait(&cempty[q], ((ncomb / kC) & 1) ^ 1);
          comb_q[q] = uu;
          mbar_arrive(&cfull[q]);
        }
        trace(a.trace, a.trace_cap, 3, uu);
      }
      if (!phaseA) ++ncomb;
      ++nunit;
    }
  }
  __syncthreads();
  if (tid == 0) trace(a.trace, a.trace_cap, 5, -1);
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace desmoe
