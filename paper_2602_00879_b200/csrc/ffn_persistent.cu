// K3 + K4: persistent grouped expert FFN for sm_100a, one CTA per SM.
//
// One launch does the post-routing half of the DES MoE layer except the final
// ordered combine (combine_slots_kernel):
//   prologue  every CTA rebuilds the permutation from the route (per-expert
//             counts, ascending offsets, stable token order, active experts —
//             the count route of moe_latency, analysis.cpp:16-30) in shared
//             memory and gathers its share of token rows into the
//             expert-grouped activation buffer x_perm;
//   phase A   (SwiGLU) units (expert, 64-row F tile): one 128-row MMA tile
//             stacks 64 rows of W_g over the matching 64 rows of W_u, so one
//             accumulator holds G (TMEM lanes 0-63) and U (lanes 64-127) of
//             the same 64 F outputs; the epilogue pairs them through shared
//             memory: H = bf16(silu(G) * U) -> h_perm; one readiness flag per
//             (expert, F tile). 512 KB units keep the phase-A waves short;
//   phase B   units (expert, 128-row d tile): Y = W_d.H_e^T (or the linear
//             expert W.X_e^T) scaled by each slot's gate into y_slot. The
//             k-loop of a phase-B unit walks F in 128-wide chunks (= two
//             phase-A tiles) and waits only for the chunk it is about to read.
// Units are handed out by a global atomic counter (phase A before phase B,
// expert-major), so every SM streams weights until the queue drains; each
// active expert's weights are read from HBM exactly once.
//
// Weights are pre-packed at registration (pack_weights_kernel) into
// tile-contiguous 16 KB blocks [128 rows x 64 K] in (expert, row tile, K block)
// order — phase-A blocks stack 64 gate rows over the matching 64 up rows — so
// every unit streams one contiguous HBM region.
//
// Warp roles (256 threads):
//   warp 0  scheduler + weight producer: TMA of the two 16 KB weight blocks of
//           every stage; never waits for activations, so the HBM stream runs
//           ahead as far as the ring allows;
//   warp 1  MMA issuer (one elected lane, tcgen05.mma kind::f16, swap-AB:
//           128 weight rows x N tokens, N = the expert's tokens rounded to 16);
//   warp 2  TMEM allocator;
//   warp 3  activation producer: TMA of the x_perm / h_perm boxes once they
//           are ready (gather handshake / per-chunk H flags);
//   warps 4-7 epilogue (tcgen05.ld of TMEM lane quarters 0-3).
// Ring stages (both phases): two consecutive 64-wide K blocks of a 128-row
// weight tile (32 KB) + the two matching activation boxes, SWIZZLE_128B as TMA
// writes them; each stage's full barrier takes one arrival per producer.
#include "common.cuh"
#include "kernels.cuh"

namespace desmoe {

namespace {

constexpr int kThreads = 256;
constexpr int kQ = 4;      // unit queue depth
constexpr int kHalf = 64;  // F rows per phase-A tile (gate and up halves)

struct Tables {
  int* count;       // [m]
  int* offset;      // [m]
  int* active;      // [m]
  int* slot_token;  // [S]
  float* slot_gate; // [S]
  int* slot_of;     // [n*k]
  int* scalars;     // [0] U, [1] S
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
    ffn_persistent_kernel(const __grid_constant__ CUtensorMap w_a,   // packed gate/up tiles
                          const __grid_constant__ CUtensorMap w_b,   // (unused)
                          const __grid_constant__ CUtensorMap w_c,   // packed W_d / W_lin tiles
                          const __grid_constant__ BoxMaps xp_maps,   // x_perm boxes
                          const __grid_constant__ BoxMaps h_maps,    // h_perm boxes
                          FfnArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // align to 1024 B by offsetting the shared array itself, so the compiler
  // keeps the shared address space (LDS/STS instead of generic LD/ST)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
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
  uint64_t* tfull = empty + S;    // [2]
  uint64_t* tempty = tfull + 2;   // [2]
  uint64_t* qfull = tempty + 2;   // [kQ]
  uint64_t* qempty = qfull + kQ;  // [kQ]
  int* unit_q = reinterpret_cast<int*>(qempty + kQ);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(unit_q + kQ);
  int* warp_sums = reinterpret_cast<int*>(tmem_slot + 4);  // [9]
  Tables t;
  t.scalars = warp_sums + 12;  // [4]
  t.count = t.scalars + 4;
  t.offset = t.count + m;
  t.active = t.offset + m;
  t.slot_of = t.active + m;
  t.slot_token = t.slot_of + n_tok * k;
  t.slot_gate = reinterpret_cast<float*>(t.slot_token + n_tok * k);
  // prologue scratch aliases the ring (unused until the roles start)
  const int tw = (n_tok + 31) >> 5;
  uint32_t* bits = reinterpret_cast<uint32_t*>(ring);      // [m][tw]
  int* act_pos = reinterpret_cast<int*>(bits + m * tw);    // [m]

  int* sched = a.counters;
  int* x_ready = a.counters + 1;
  const int tilesA = f / kHalf, tilesB = d / kBM;
  int* h_ready = a.counters + 2;  // [m][tilesA]

  // ---- barrier init / TMEM allocation (independent of the route) ----------
  if (tid == 0) {
    if (swiglu) tma_prefetch_desc(&w_a);
    tma_prefetch_desc(&w_c);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 2);  // weight producer + activation producer
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);  // one arrival per epilogue warp
    }
    for (int q = 0; q < kQ; ++q) {
      mbar_init(&qfull[q], 1);
      mbar_init(&qempty[q], 3);  // MMA lane + activation producer + epilogue
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  pdl_launch_dependents();  // the combine kernel may launch; it waits for us
  pdl_wait();               // route + zeroed counters from the routing kernel
  const size_t ep_half = a.world > 1 ? (static_cast<size_t>(*a.epoch) & 1u) * a.slot_stride : 0;

  // ---- prologue: permutation (redundantly per CTA) ------------------------
  for (int i = tid; i < m; i += kThreads) t.count[i] = 0;
  for (int i = tid; i < m * tw; i += kThreads) bits[i] = 0;
  if (tid == 0) t.scalars[2] = 0;
  __syncthreads();
  for (int e = tid; e < n_tok * k; e += kThreads) {
    const int tok = e / k, j = e - tok * k;
    if (j >= a.route_cnt[tok]) continue;
    const int x = a.route_idx[e];
    atomicAdd(&t.count[x], 1);
    atomicOr(&bits[x * tw + (tok >> 5)], 1u << (tok & 31));
  }
  __syncthreads();
  // active experts = the owned ones (all of them unless expert-parallel)
  const int lo = a.expert_lo, hi = a.expert_hi;
  int u_all = 0;
  for (int i = tid; i < m; i += kThreads) {
    t.offset[i] = t.count[i];
    act_pos[i] = (t.count[i] > 0 && i >= lo && i < hi) ? 1 : 0;
    u_all += t.count[i] > 0;
  }
  u_all = __reduce_add_sync(0xffffffffu, u_all);
  if (lane == 0) atomicAdd(&t.scalars[2], u_all);
  __syncthreads();
  const int total_slots = block_exclusive_scan(t.offset, m, warp_sums);
  const int U = block_exclusive_scan(act_pos, m, warp_sums);
  for (int i = tid; i < m; i += kThreads)
    if (t.count[i] > 0 && i >= lo && i < hi) t.active[act_pos[i]] = i;
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
  if (blockIdx.x == 0) {  // products the combine kernel and the caller read
    for (int e = tid; e < n_tok * k; e += kThreads) a.slot_of[e] = t.slot_of[e];
    if (tid == 0 && a.stats) {
      a.stats[0] = t.scalars[2];  // unique experts of the block (all ranks)
      a.stats[1] = a.n_members ? *a.n_members : t.scalars[2];
      a.stats[2] = total_slots;
      a.stats[3] = U;             // experts this rank streams
    }
  }
  // gather this CTA's share of token rows into x_perm: every thread issues
  // its 16-byte loads before its stores (one memory round trip)
  {
    const int vec = d / 8;
    const uint4* src = reinterpret_cast<const uint4*>(a.x);
    uint4* dst = reinterpret_cast<uint4*>(a.x_perm);
    // only the owned experts' slot rows (a contiguous slot range)
    const int row0 = lo < m ? (lo > 0 ? t.offset[lo] : 0) : total_slots;
    const int row1 = hi < m ? t.offset[hi] : total_slots;
    const int nrows = row1 - row0;
    const int my_rows = nrows > static_cast<int>(blockIdx.x)
                            ? (nrows - 1 - static_cast<int>(blockIdx.x)) / gridDim.x + 1
                            : 0;
    const int items = my_rows * vec;
    constexpr int kU = 4;
    for (int i0 = tid; i0 < items; i0 += kThreads * kU) {
      uint4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = i0 + u * kThreads;
        if (i < items) {
          const int row = row0 + blockIdx.x + (i / vec) * gridDim.x;
          v[u] = src[static_cast<size_t>(t.slot_token[row]) * vec + (i % vec)];
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = i0 + u * kThreads;
        if (i < items) {
          const int row = row0 + blockIdx.x + (i / vec) * gridDim.x;
          dst[static_cast<size_t>(row) * vec + (i % vec)] = v[u];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    __threadfence();
    atomic_add_release(x_ready, 1);
    trace(a.trace, a.trace_cap, 1, -1);
  }
  const uint32_t tmem_base = *tmem_slot;

  const int nA = swiglu ? U * tilesA : 0;
  const int n_units = nA + U * tilesB;
  const int ksA = d / (2 * kBK);                 // k-steps: 2 K blocks each
  const int ksB = (swiglu ? f : d) / (2 * kBK);
  float* xchg = reinterpret_cast<float*>(t.slot_gate + n_tok * k);  // [16][64] U exchange

  if (warp == 0) {
    // ============ scheduler + weight producer ============
    if (lane == 0) {
      const uint64_t pol_w = l2_policy_evict_first();  // streamed once
      uint32_t it = 0;
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
        const bool phaseA = ui.phase == 0;
        const int ksteps = phaseA ? ksA : ksB;
        for (int ks = 0; ks < ksteps; ++ks, ++it) {
          const int s = it % S;
          mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
          unsigned char* st = ring + static_cast<size_t>(s) * stage_bytes;
          mbar_arrive_expect_tx(&full[s], 2 * kATile);
          // packed weights: tile-contiguous 16 KB blocks in (expert, row tile,
          // K block) order, so a unit streams one contiguous region
          const int el = ui.expert - lo;  // packed weights hold the owned experts only
          const int tile0 = phaseA ? (el * tilesA + ui.tile) * (2 * ksA) + 2 * ks
                                   : (el * tilesB + ui.tile) * (2 * ksB) + 2 * ks;
          const CUtensorMap* wmap = phaseA ? &w_a : &w_c;
          tma_load_3d(st, wmap, &full[s], 0, 0, tile0, pol_w);
          tma_load_3d(st + kATile, wmap, &full[s], 0, 0, tile0 + 1, pol_w);
        }
      }
    }
  } else if (warp == 3) {
    // ============ activation producer ============
    if (lane == 0) {
      const uint64_t pol_x = l2_policy_evict_last();  // re-read by every tile
      uint32_t it = 0;
      bool x_seen = false;
      for (int qi = 0;; ++qi) {
        const int q = qi % kQ;
        mbar_wait(&qfull[q], (qi / kQ) & 1);
        const int uu = unit_q[q];
        mbar_arrive(&qempty[q]);
        if (uu < 0) break;
        const UnitInfo ui = decode(uu, nA, tilesA, tilesB, t);
        const bool phaseA = ui.phase == 0;
        const bool from_x = phaseA || !swiglu;
        const int bi = box_for(ui.count);
        const uint32_t box_bytes = (16u << bi) * 128u;
        const BoxMaps& acts = from_x ? xp_maps : h_maps;
        const int ksteps = phaseA ? ksA : ksB;
        if (from_x && !x_seen) {
          while (ld_acquire(x_ready) < static_cast<int>(gridDim.x)) {
          }
          fence_proxy_async_global();
          x_seen = true;
          trace(a.trace, a.trace_cap, 6, uu);
        }
        for (int ks = 0; ks < ksteps; ++ks, ++it) {
          const int s = it % S;
          mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
          if (!from_x) {
            // H columns [128 ks, 128 ks + 128) = phase-A tiles 2ks, 2ks+1
            for (int h = 0; h < 2; ++h) {
              const int* flag = &h_ready[ui.expert * tilesA + 2 * ks + h];
              if (ld_acquire(flag) == 0) {
                while (ld_acquire(flag) == 0) {
                }
                trace(a.trace, a.trace_cap, 7, uu);
              }
            }
            fence_proxy_async_global();
          }
          unsigned char* st = ring + static_cast<size_t>(s) * stage_bytes + 2 * kATile;
          mbar_arrive_expect_tx(&full[s], 2 * box_bytes);
          tma_load_2d(st, &acts.map[bi], &full[s], 2 * ks * kBK, ui.brow, pol_x);
          tma_load_2d(st + b_box_bytes, &acts.map[bi], &full[s], (2 * ks + 1) * kBK, ui.brow,
                      pol_x);
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
      const uint32_t buf = nunit & 1u;
      const uint32_t use = nunit >> 1;
      mbar_wait(&tempty[buf], (use & 1u) ^ 1u);
      tc_fence_after();
      const uint32_t d_acc = tmem_base + buf * 256u;
      const int ksteps = phaseA ? ksA : ksB;
      for (int ks = 0; ks < ksteps; ++ks, ++it) {
        const int s = it % S;
        mbar_wait(&full[s], (it / S) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a0 = smem_u32(ring + static_cast<size_t>(s) * stage_bytes);
          const uint32_t b0 = a0 + 2 * kATile;
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              tc_mma_bf16(d_acc, sw128_kmajor_desc(a0 + h * kATile + kk * 32),
                          sw128_kmajor_desc(b0 + h * b_box_bytes + kk * 32), idesc,
                          (ks > 0 || h > 0 || kk > 0) ? 1u : 0u);
          tc_commit(&empty[s]);
          if (ks == ksteps - 1) tc_commit(&tfull[buf]);
        }
        __syncwarp();
      }
      ++nunit;
    }
  } else if (warp >= 4) {
    // ============ epilogue ============
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;  // accumulator row = weight row within the tile
    const int etid = tid - 128;    // 0..127
    uint32_t nunit = 0;
    for (int qi = 0;; ++qi) {
      const int q = qi % kQ;
      mbar_wait(&qfull[q], (qi / kQ) & 1);
      const int uu = unit_q[q];
      named_bar_sync(1, 128);
      if (etid == 0) mbar_arrive(&qempty[q]);
      if (uu < 0) break;
      const UnitInfo ui = decode(uu, nA, tilesA, tilesB, t);
      const bool phaseA = ui.phase == 0;
      const int n_mma = (ui.count + 15) & ~15;
      const uint32_t buf = nunit & 1u;
      const uint32_t use = nunit >> 1;
      mbar_wait(&tfull[buf], use & 1u);
      tc_fence_after();
      const uint32_t lane_base = tmem_base + buf * 256u + (static_cast<uint32_t>(q4 * 32) << 16);
      if (phaseA) {
        // lanes 0-63: G, lanes 64-127: U of F columns tile*64 + (r mod 64)
        const bool is_g = r < kHalf;
        const int rr = r & (kHalf - 1);
        __nv_bfloat16* hrow =
            a.h_perm + static_cast<size_t>(ui.brow) * f + ui.tile * kHalf + rr;
        for (int c0 = 0; c0 < n_mma; c0 += 16) {
          float v[16];
          tmem_ld16(lane_base + c0, v);
          if (!is_g) {
#pragma unroll
            for (int j = 0; j < 16; ++j) xchg[j * kHalf + rr] = v[j];
          }
          named_bar_sync(1, 128);
          if (is_g) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int col = c0 + j;
              if (col < ui.count)
                hrow[static_cast<size_t>(col) * f] =
                    __float2bfloat16_rn(silu(v[j]) * xchg[j * kHalf + rr]);
            }
          }
          named_bar_sync(1, 128);
        }
      } else if (a.world <= 1) {
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
      } else {
        // expert parallel: push the gate-scaled rows straight into every
        // rank's slot buffer (own + NVLink peers) while later tiles stream
        const size_t off = ep_half + static_cast<size_t>(ui.brow) * d + ui.tile * kBM + r;
        for (int c0 = 0; c0 < n_mma; c0 += 16) {
          float v[16];
          tmem_ld16(lane_base + c0, v);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int col = c0 + j;
            if (col < ui.count) {
              const float val = v[j] * t.slot_gate[ui.brow + col];
              for (int p = 0; p < a.world; ++p)
                __stcg(a.peer_slot[p] + off + static_cast<size_t>(col) * d, val);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      if (phaseA) {
        named_bar_sync(1, 128);
        if (etid == 0) {
          __threadfence();  // all epilogue stores (ordered by the barrier) -> gpu scope
          atomic_add_release(&h_ready[ui.expert * tilesA + ui.tile], 1);
        }
      }
      if (etid == 0) trace(a.trace, a.trace_cap, 3, uu);
      ++nunit;
    }
  }
  __syncthreads();
  if (a.world > 1 && tid == 0) {
    // every slot row this CTA pushed is visible system-wide before the
    // arrival (fence cumulativity over the CTA barrier above)
    __threadfence_system();
    for (int p = 0; p < a.world; ++p) atomic_add_release_sys(a.peer_flag[p], 1ull);
  }
  if (tid == 0) trace(a.trace, a.trace_cap, 5, -1);
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

// Packs row-major bf16 weights into tile-contiguous blocks:
//   out[((e * row_tiles + rt) * kblocks + kb)][r][c] = src(e, rt, r)[kb * 64 + c]
// with src row = e * rows_per_expert + rt * rows_per_tile + r for r < rows_per_tile
// (stacked = 0), or, when stacked, rows 0-63 from src (gate) and 64-127 from
// src2 (up) at row e * rows_per_expert + rt * 64 + (r mod 64). One thread per
// 16-byte vector.
__global__ void pack_weights_kernel(const uint4* __restrict__ src, const uint4* __restrict__ src2,
                                    uint4* __restrict__ out, int experts, int rows_per_expert,
                                    int cols, int stacked) {
  const int row_tiles = stacked ? rows_per_expert / 64 : rows_per_expert / 128;
  const int kblocks = cols / 64;
  const size_t total = static_cast<size_t>(experts) * row_tiles * kblocks * 128 * 8;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int c8 = static_cast<int>(i & 7);
    const int r = static_cast<int>((i >> 3) & 127);
    const size_t tile = i >> 10;
    const int kb = static_cast<int>(tile % kblocks);
    const size_t et = tile / kblocks;
    const int rt = static_cast<int>(et % row_tiles);
    const int e = static_cast<int>(et / row_tiles);
    const uint4* base = src;
    int row;
    if (stacked) {
      base = r < 64 ? src : src2;
      row = e * rows_per_expert + rt * 64 + (r & 63);
    } else {
      row = e * rows_per_expert + rt * 128 + r;
    }
    out[i] = base[static_cast<size_t>(row) * (cols / 8) + kb * 8 + c8];
  }
}

// Ordered combine (moe_forward's order, gating.cpp:141-155): y[t][c] = sum
// over j ascending (= ascending expert) of y_slot[slot_of[t][j]][c]. Launched
// with programmatic stream serialisation behind the FFN kernel. Expert
// parallel: every rank holds every slot row (pushed by the owners), so the
// sum is the same sequence of fp32 adds as on one GPU — bit-identical.
// Expert-parallel arrival wait: ONE 32-thread CTA per rank spins (system-
// scope acquire) until every rank's FFN CTAs signalled this call's epoch,
// then lets the combine run. Kept out of the combine so a waiting rank holds
// almost no SM resources (several simulated ranks can share one GPU).
__global__ void __launch_bounds__(32) ep_wait_kernel(CombineArgs a) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    const unsigned long long want =
        (static_cast<unsigned long long>(*a.epoch) + 1ull) * a.arrivals;
    const uint64_t t0 = gtime();
    while (ld_acquire_sys(a.flag) < want) {
      if (gtime() - t0 > 4000000000ull) {  // 4 s: a peer is gone; fail, never hang
        atomicExch(a.err, 2);
        break;
      }
      __nanosleep(100);
    }
  }
  __syncwarp();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__global__ void __launch_bounds__(256) combine_slots_kernel(CombineArgs a) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ int s_epoch;
  const float* y_slot = a.y_slot;
  if (a.world > 1) {
    // ep_wait_kernel established (acquire) that all slot rows arrived
    if (threadIdx.x == 0) s_epoch = *a.epoch;
    __syncthreads();
    y_slot += (static_cast<size_t>(s_epoch) & 1u) * a.slot_stride;
  }
  const int vec = a.d / 4;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < a.n * vec) {
    const int tok = i / vec, c = (i - tok * vec) * 4;
    const int cnt = a.route_cnt[tok];
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 v[8];
    for (int j0 = 0; j0 < cnt; j0 += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j0 + j < cnt)
          v[j] = __ldcg(reinterpret_cast<const float4*>(
              y_slot + static_cast<size_t>(a.slot_of[tok * a.k + j0 + j]) * a.d + c));
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j0 + j < cnt) {
          acc.x += v[j].x;
          acc.y += v[j].y;
          acc.z += v[j].z;
          acc.w += v[j].w;
        }
    }
    *reinterpret_cast<float4*>(a.y + static_cast<size_t>(tok) * a.d + c) = acc;
  }
  if (a.world > 1) {
    // the last CTA to finish advances the epoch (every CTA read it above)
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(a.done_ctas, 1) == static_cast<int>(gridDim.x) - 1) {
        *a.done_ctas = 0;
        __threadfence();
        atomicAdd(a.epoch, 1);
      }
    }
  }
}

}  // namespace desmoe
