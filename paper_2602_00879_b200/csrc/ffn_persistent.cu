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
  int nt;     // row tiles: 2 = a phase-B pair (tiles tile, tile + 1) sharing the activations
};

// Queue position -> (phase, list index, first tile, tiles). Phase A units
// first (expert-major), then phase B: pw tiles per unit (pw = 2: pairs that
// read the expert's H once for both tiles), the last nBs pairs split into
// single tiles so the queue drains on small units.
struct UnitPos {
  int phase, ei, tile, nt;
};
// Phase A the same way: pa tiles per unit (two F tiles sharing the X stream),
// the last A pairs split; nA = phase-A units, nAp of them pairs.
struct UnitMap {
  int nA, nAp, pa, nBp, pw, total;
};
__device__ inline UnitPos unit_pos(int u, const UnitMap& q, int tilesA, int tilesB) {
  const int nA = q.nA, nBp = q.nBp, pw = q.pw;
  UnitPos r;
  r.nt = 1;
  if (u < nA) {
    int ta;
    if (u < q.nAp) {
      ta = u * q.pa;
      r.nt = q.pa;
    } else {
      ta = q.nAp * q.pa + (u - q.nAp);
    }
    r.phase = 0;
    r.ei = ta / tilesA;
    r.tile = ta - r.ei * tilesA;
    return r;
  }
  const int b = u - nA;
  int tb;  // first tile in the flat phase-B tile order
  if (b < nBp) {
    tb = b * pw;
    r.nt = pw;
  } else {
    tb = nBp * pw + (b - nBp);
  }
  r.phase = 1;
  r.ei = tb / tilesB;
  r.tile = tb - r.ei * tilesB;
  return r;
}

// dense: every unit covers all n_tok tokens; row block = expert id x n_tok
// (t.offset holds the expert id)
__device__ inline UnitInfo decode(int u, const UnitMap& q, int tilesA, int tilesB,
                                  const Tables& t, bool dense, int n_tok) {
  UnitInfo r;
  const UnitPos p = unit_pos(u, q, tilesA, tilesB);
  const int ei = p.ei;
  r.phase = p.phase;
  r.tile = p.tile;
  r.nt = p.nt;
  r.expert = t.active[ei];
  if (dense) {
    r.brow = t.offset[ei] * n_tok;
    r.count = n_tok;
  } else {
    r.brow = t.offset[r.expert];
    r.count = t.count[r.expert];
  }
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

// Routed mode: one batch of 256 tagged route words (8 per lane, all in
// flight at once), re-polled until every word carries this call's tag, then
// staged as (expert or -1, gate). Out of line: the dense path's code stays
// compact (its instruction fetches are cold after an L2 flush).
__device__ __noinline__ void poll_route_batch(const uint64_t* route_words, int total, int b0,
                                              uint32_t tag, int* rexp, float* gate_tmp) {
  const int lane = threadIdx.x & 31;
  uint64_t w[8];
  bool ok;
  do {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int e = b0 + j * 32 + lane;
      w[j] = e < total ? ld_relaxed_u64(route_words + e) : 0ull;
    }
    ok = true;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int e = b0 + j * 32 + lane;
      ok &= e >= total || ((static_cast<uint32_t>(w[j]) >> 10) & kTagMask) == tag;
    }
    ok = __all_sync(0xffffffffu, ok);
  } while (!ok);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int e = b0 + j * 32 + lane;
    if (e < total) {
      const int x = static_cast<int>(w[j] & 1023u);
      rexp[e] = x == kPadExpert ? -1 : x;
      gate_tmp[e] = __uint_as_float(static_cast<uint32_t>(w[j] >> 32));
    }
  }
}

}  // namespace

template <int KB>
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
  // timeline (desmoe_set_trace): tid 0 = prologue + scheduler, 96 = activation
  // producer, 128 = epilogue; atomic-free after the claim here
  TraceCursor tc{nullptr, 0, 0};
  if (a.trace && (tid == 0 || tid == 32 || tid == 96 || tid == 128))
    tc = trace_open(a.trace, a.trace_cap, 96);
  if (tid == 0) trace_put(tc, 0, -1);
  const bool swiglu = a.mode == 0;
  const bool dense = a.dense != 0;
  const int S = a.stages;
  const int b_box_bytes = a.b_rows * 128;
  const int stage_bytes = KB * kATile + KB * b_box_bytes;

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
  float* xchg = reinterpret_cast<float*>(t.slot_gate + n_tok * k);  // [16][64] U exchange
  // prologue scratch in the LAST ring stage: the early weight prefetch fills
  // at most stages 0..S-2 before the prologue is done
  const int tw = (n_tok + 31) >> 5;
  uint32_t* bits = reinterpret_cast<uint32_t*>(ring + static_cast<size_t>(S - 1) * stage_bytes);
  int* act_pos = reinterpret_cast<int*>(bits + m * tw);             // [m]
  int* pubm = act_pos + m;                                          // [m] published experts
  int* pubidx = pubm + m;                                           // [m] their list index
  float* gate_tmp = reinterpret_cast<float*>(pubidx + m);           // [n*k] staged gates

  int* sched = a.counters;
  int* x_ready = a.counters + 1;
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
  __shared__ uint64_t s_pts[8];  // prologue timeline (trace buffer only)
  if (a.trace && tid < 8) s_pts[tid] = 0;
  __shared__ int s_upub;         // early mode: owned published experts
  __shared__ int s_pcnt;         // early mode: published list length
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  pdl_launch_dependents();  // the combine kernel may launch; it waits for us
  // standalone: route + zeroed counters from the previous kernel. Behind the
  // front kernel (early mode) nothing waits for its completion: the expert
  // list and the route arrive as tagged words (see kernels.cuh).
  if (!a.early) pdl_wait();
  const int seq = *a.epoch;
  const uint32_t tag = hand_tag(seq);
  const int lo = a.expert_lo, hi = a.expert_hi;
  const int tilesA = f / kHalf, tilesB = d / kBM;
  const int ksA = d / (KB * kBK);               // k-steps: KB K blocks each
  const int ksB = (swiglu ? f : d) / (KB * kBK);
  constexpr int KH = KB / 2;  // a phase-B pair stage: KH K blocks of each tile (+ KH boxes)
  const int pw = a.pair_b ? 2 : 1;
  const int pa = a.pair_a && swiglu ? 2 : 1;
  // the unit list for U owned experts
  auto unit_map = [&](int u_) {
    UnitMap q;
    const int nAs = pa == 2 ? min(a.split_a, u_ * (tilesA / 2)) : 0;
    q.pa = pa;
    q.nAp = swiglu ? u_ * (tilesA / pa) - nAs : 0;
    q.nA = q.nAp + pa * nAs;
    const int nBs = pw == 2 ? min(a.split_b, u_ * (tilesB / 2)) : 0;
    q.pw = pw;
    q.nBp = u_ * (tilesB / pw) - nBs;
    q.total = q.nA + q.nBp + pw * nBs;
    return q;
  };
  int pre_u = -1, pre_ks = 0;  // early mode: unit claimed and k-steps issued before the prologue
  if (a.early && warp == 0) {
    // the published expert list (coreset / union) -> the unit list; claim
    // the first unit and start streaming its weights while the route is
    // still being computed (one warp polls the list in parallel)
    // claim the first unit at once: this kernel launched behind the front's
    // griddepcontrol.wait, so the last call's combine (which zeroes the
    // counter) is complete; the claim's round trip overlaps the list's
    int u0 = 0;
    if (lane == 0) u0 = atomicAdd(sched, 1);
    // the count word and the first 32 list words in ONE round trip per poll
    // (each word carries the call's tag): every lane loads both
    uint32_t w0, w1;
    bool ok;
    do {
      w0 = ld_relaxed_u32(a.pub);
      w1 = ld_relaxed_u32(a.pub + 1 + lane);
      const int c0 = static_cast<int>(w0 & 1023u);
      ok = (w0 >> 10) == tag && (lane >= c0 || (w1 >> 10) == tag);
    } while (!__all_sync(0xffffffffu, ok));
    if (a.trace && lane == 0) s_pts[5] = gtime();  // list count seen
    const int cnt = static_cast<int>(w0 & 1023u);
    if (lane == 0) s_pcnt = cnt;
    int u = 0;
    for (int i0 = 0; i0 < cnt; i0 += 32) {
      const int i = i0 + lane;
      int e = -1;
      if (i < cnt) {
        uint32_t w = w1;
        if (i0 > 0) {
          do {
            w = ld_relaxed_u32(a.pub + 1 + i);
          } while ((w >> 10) != tag);
        }
        e = static_cast<int>(w & 1023u);
      }
      const bool own = e >= lo && e < hi;
      const uint32_t bal = __ballot_sync(0xffffffffu, own);
      if (own) {
        const int pos = u + __popc(bal & ((1u << lane) - 1u));
        pubm[pos] = e;
        pubidx[pos] = i;  // global list index: the dense row block (same on every rank)
      }
      u += __popc(bal);
    }
    __syncwarp();
    if (lane == 0) {
      if (a.trace) s_pts[6] = gtime();  // list words loaded
      s_upub = u;
      const UnitMap q0 = unit_map(u);
      const int n_units0 = q0.total;
      if (u0 < n_units0) pre_u = u0;
      const UnitPos p0 = unit_pos(u0, q0, tilesA, tilesB);
      if (u0 < n_units0 && p0.nt == 1) {  // (a first pair streams from the main loop)
        const bool phaseA = p0.phase == 0;
        const int tile = p0.tile;
        const int el = pubm[p0.ei] - lo;
        const int ksteps = phaseA ? ksA : ksB;
        const uint64_t pol_w = l2_policy_evict_first();
        const CUtensorMap* wmap = phaseA ? &w_a : &w_c;
        for (; pre_ks < ksteps && pre_ks < S - 1; ++pre_ks) {
          unsigned char* st = ring + static_cast<size_t>(pre_ks) * stage_bytes;
          mbar_arrive_expect_tx(&full[pre_ks], KB * kATile);
          const int tile0 = phaseA ? (el * tilesA + tile) * (KB * ksA) + KB * pre_ks
                                   : (el * tilesB + tile) * (KB * ksB) + KB * pre_ks;
#pragma unroll
          for (int j = 0; j < KB; ++j)
            tma_load_3d(st + j * kATile, wmap, &full[pre_ks], 0, 0, tile0 + j, pol_w);
        }
        // the rest of the unit (one contiguous packed region) goes to L2 now,
        // so HBM keeps streaming while the prologue waits for the route
        if (pre_ks < ksteps && !(a.flags & 1)) {
          const int tile0 = phaseA ? (el * tilesA + tile) * (KB * ksA) + KB * pre_ks
                                   : (el * tilesB + tile) * (KB * ksB) + KB * pre_ks;
          const unsigned char* base =
              static_cast<const unsigned char*>(phaseA ? a.wa_base : a.wc_base);
          bulk_prefetch_l2(base + static_cast<size_t>(tile0) * kATile,
                           static_cast<uint32_t>((ksteps - pre_ks) * KB * kATile));
        }
      }
    }
  }
  if (a.trace && tid == 0) s_pts[0] = gtime();
  const size_t ep_half = a.world > 1 ? (static_cast<size_t>(seq) & 1u) * a.slot_stride : 0;

  int U = 0, total_slots = 0;
  if (dense) {
    // dense mode: units over the published list, all tokens each; no route,
    // permutation, gather or handshake (X itself is the activation source)
    __syncthreads();  // s_upub / pubm from the early block
    U = s_upub;
    for (int i = tid; i < U; i += kThreads) {
      t.active[i] = pubm[i];
      t.offset[i] = pubm[i];  // rows [expert][token]: the combine needs no list
    }
    if (blockIdx.x == 0 && tid == 0 && a.stats) {
      a.stats[1] = s_pcnt;  // published list (coreset / union) length
      a.stats[3] = U;       // experts this rank streams
    }
    __syncthreads();
  } else {
  // ---- prologue: permutation (redundantly per CTA) ------------------------
  for (int i = tid; i < m; i += kThreads) t.count[i] = 0;
  for (int i = tid; i < m * tw; i += kThreads) bits[i] = 0;
  if (tid == 0) t.scalars[2] = 0;
  __syncthreads();
  // route slot e: expert (-1 = none) and gate, staged in shared memory; early
  // mode: ONE warp per CTA polls the tagged words until the first batch is
  // valid (all threads polling would flood L2 while the front is still
  // writing them), then every warp loads its share of the rest
  int* rexp = t.slot_of;           // staged here until the slot pass rewrites it
  if (a.early) {
    // batches of 8 words per lane with every load of a batch in flight at
    // once; re-poll until the whole batch carries this call's tag. Warp 1
    // polls the first batch alone; once it is valid the front is finishing,
    // and all 8 warps load the remaining batches in parallel (one round trip
    // instead of one per batch)
    const int total = n_tok * k;
    auto poll_batch = [&](int b0) {
      poll_route_batch(a.route_words, total, b0, tag, rexp, gate_tmp);
    };
    if (a.flags & 2) {  // (A/B runs: warp 1 alone, one batch per round trip)
      if (warp == 1)
        for (int b0 = 0; b0 < total; b0 += 256) poll_batch(b0);
    } else if (a.route_done && !(a.flags & 4)) {
      // one lane waits for the 8 front CTAs' route-complete words
      // — one 32-byte sector, polled with a short back-off — then every
      // warp loads its share of the route words once (their tags are
      // re-checked, so a stale word can never be taken)
      if (tid == 32) {
#pragma unroll 1
        for (;;) {
          bool all = true;
#pragma unroll
          for (int r = 0; r < kFrontCta; ++r)
            all &= ld_relaxed_u32(a.route_done + r) == tag;
          if (all) break;
          __nanosleep(64);
        }
      }
      __syncthreads();
      for (int b = warp; b * 256 < total; b += kThreads / 32) poll_batch(b * 256);
    } else {
      if (warp == 1) poll_batch(0);
      __syncthreads();
      for (int b = 1 + warp; b * 256 < total; b += kThreads / 32) poll_batch(b * 256);
    }
  } else {
    for (int e = tid; e < n_tok * k; e += kThreads) {
      const int tok = e / k, j = e - tok * k;
      const int x = j < a.route_cnt[tok] ? a.route_idx[e] : -1;
      rexp[e] = x;
      gate_tmp[e] = x >= 0 ? static_cast<float>(a.route_gate[e]) : 0.0f;
    }
  }
  __syncthreads();
  for (int e = tid; e < n_tok * k; e += kThreads) {
    const int x = rexp[e];
    if (x < 0) continue;
    const int tok = e / k;
    atomicAdd(&t.count[x], 1);
    atomicOr(&bits[x * tw + (tok >> 5)], 1u << (tok & 31));
  }
  __syncthreads();
  if (a.trace && tid == 0) s_pts[1] = gtime();
  // active experts = the owned ones (all of them unless expert-parallel)
  int u_all = 0;
  for (int i = tid; i < m; i += kThreads) {
    t.offset[i] = t.count[i];
    act_pos[i] = (t.count[i] > 0 && i >= lo && i < hi) ? 1 : 0;
    u_all += t.count[i] > 0;
  }
  u_all = __reduce_add_sync(0xffffffffu, u_all);
  if (lane == 0) atomicAdd(&t.scalars[2], u_all);
  __syncthreads();
  total_slots = block_exclusive_scan(t.offset, m, warp_sums);
  U = block_exclusive_scan(act_pos, m, warp_sums);
  if (a.early) {
    // units run over the published list (a listed expert may get no token
    // after re-routing: its units stream nothing useful but stay consistent
    // with the weights already in flight)
    U = s_upub;
    for (int i = tid; i < U; i += kThreads) t.active[i] = pubm[i];
  } else {
    for (int i = tid; i < m; i += kThreads)
      if (t.count[i] > 0 && i >= lo && i < hi) t.active[act_pos[i]] = i;
  }
  // (each thread rewrites only its own entries e of rexp / slot_of)
  for (int e = tid; e < n_tok * k; e += kThreads) {
    const int tok = e / k;
    const int x = rexp[e];
    if (x < 0) {
      t.slot_of[e] = -1;
      continue;
    }
    const uint32_t* b = bits + x * tw;
    int before = 0;
    for (int w = 0; w < (tok >> 5); ++w) before += __popc(b[w]);
    before += __popc(b[tok >> 5] & ((1u << (tok & 31)) - 1u));
    const int slot = t.offset[x] + before;
    t.slot_of[e] = slot;
    t.slot_token[slot] = tok;
    t.slot_gate[slot] = gate_tmp[e];
  }
  if (tid == 0) {
    t.scalars[0] = U;
    t.scalars[1] = total_slots;
  }
  __syncthreads();
  if (a.trace && tid == 0) s_pts[2] = gtime();
  if (blockIdx.x == 0) {  // products the combine kernel and the caller read
    for (int e = tid; e < n_tok * k; e += kThreads) a.slot_of[e] = t.slot_of[e];
    if (tid == 0 && a.stats) {
      a.stats[0] = t.scalars[2];  // unique experts of the block (all ranks)
      a.stats[1] = a.early ? s_pcnt : (a.n_members ? *a.n_members : t.scalars[2]);
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
    // gather duty: the first a.gather_ctas CTAs (behind the front kernel the
    // last ones start only when its SMs free up)
    const int gcta = a.gather_ctas;
    const int my_rows = static_cast<int>(blockIdx.x) < gcta && nrows > static_cast<int>(blockIdx.x)
                            ? (nrows - 1 - static_cast<int>(blockIdx.x)) / gcta + 1
                            : 0;
    const int items = my_rows * vec;
    constexpr int kU = 4;
    for (int i0 = tid; i0 < items; i0 += kThreads * kU) {
      uint4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = i0 + u * kThreads;
        if (i < items) {
          const int row = row0 + blockIdx.x + (i / vec) * gcta;
          v[u] = src[static_cast<size_t>(t.slot_token[row]) * vec + (i % vec)];
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = i0 + u * kThreads;
        if (i < items) {
          const int row = row0 + blockIdx.x + (i / vec) * gcta;
          dst[static_cast<size_t>(row) * vec + (i % vec)] = v[u];
        }
      }
    }
  }
  }  // !dense
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (!dense && tid == 0 && static_cast<int>(blockIdx.x) < a.gather_ctas) {
    if (a.trace) s_pts[3] = gtime();
    __threadfence();
    red_add_release(x_ready, 1);
    if (a.trace) s_pts[4] = gtime();
    trace_put(tc, 1, -1);
  }
  const uint32_t tmem_base = *tmem_slot;

  const UnitMap qm = unit_map(U);
  const int n_units = qm.total;

  if (warp == 0) {
    // ============ scheduler + weight producer ============
    if (lane == 0) {
      const uint64_t pol_w = l2_policy_evict_first();  // streamed once
      uint32_t it = 0;
      for (int qi = 0;; ++qi) {
        const int q = qi % kQ;
        const bool pre = qi == 0 && a.early;  // claimed (and started) before the prologue
        const int u = pre ? (pre_u >= 0 ? pre_u : n_units) : atomicAdd(sched, 1);
        const int uu = u < n_units ? u : -1;
        // the first claim past the end: every unit is out (streamed combine)
        if (u == n_units && a.b_drained) st_relaxed_u32(a.b_drained, tag);
        mbar_wait(&qempty[q], ((qi / kQ) & 1) ^ 1);
        unit_q[q] = uu;
        mbar_arrive(&qfull[q]);
        if (uu < 0) break;
        trace_put(tc, 2, uu);
        const UnitInfo ui = decode(uu, qm, tilesA, tilesB, t, dense, n_tok);
        const bool phaseA = ui.phase == 0;
        const bool pair = ui.nt == 2;
        const int ksteps = (phaseA ? ksA : ksB) * ui.nt;
        const int ks0 = pre ? pre_ks : 0;
        it += ks0;
        for (int ks = ks0; ks < ksteps; ++ks, ++it) {
          const int s = it % S;
          mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
          unsigned char* st = ring + static_cast<size_t>(s) * stage_bytes;
          mbar_arrive_expect_tx(&full[s], KB * kATile);
          // packed weights: tile-contiguous 16 KB blocks in (expert, row tile,
          // K block) order, so a unit streams one contiguous region
          const int el = ui.expert - lo;  // packed weights hold the owned experts only
          if (pair) {  // KH blocks of each of the two tiles
            const CUtensorMap* pmap = phaseA ? &w_a : &w_c;
#pragma unroll
            for (int tt = 0; tt < 2; ++tt) {
              const int tile0 = phaseA ? (el * tilesA + ui.tile + tt) * (KB * ksA) + KH * ks
                                       : (el * tilesB + ui.tile + tt) * (KB * ksB) + KH * ks;
#pragma unroll
              for (int j = 0; j < KH; ++j)
                tma_load_3d(st + (tt * KH + j) * kATile, pmap, &full[s], 0, 0, tile0 + j, pol_w);
            }
            continue;
          }
          const int tile0 = phaseA ? (el * tilesA + ui.tile) * (KB * ksA) + KB * ks
                                   : (el * tilesB + ui.tile) * (KB * ksB) + KB * ks;
          const CUtensorMap* wmap = phaseA ? &w_a : &w_c;
#pragma unroll
          for (int j = 0; j < KB; ++j)
            tma_load_3d(st + j * kATile, wmap, &full[s], 0, 0, tile0 + j, pol_w);
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
        const UnitInfo ui = decode(uu, qm, tilesA, tilesB, t, dense, n_tok);
        const bool phaseA = ui.phase == 0;
        const bool from_x = phaseA || !swiglu;
        const int bi = box_for(ui.count);
        const uint32_t box_bytes = (16u << bi) * 128u;
        const BoxMaps& acts = from_x ? xp_maps : h_maps;
        const int nb = ui.nt == 2 ? KH : KB;  // activation boxes per k-step
        const int ksteps = (phaseA ? ksA : ksB) * ui.nt;
        if (from_x && !x_seen && ui.count > 0 && !dense) {
          while (ld_acquire(x_ready) < a.gather_ctas) {
          }
          fence_proxy_async_global();
          x_seen = true;
          trace_put(tc, 6, uu);
        }
        for (int ks = 0; ks < ksteps; ++ks, ++it) {
          const int s = it % S;
          mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
          if (ui.count == 0) {  // a published expert without tokens: no activations
            mbar_arrive(&full[s]);
            continue;
          }
          if (!from_x) {
            // H columns [128 ks, 128 ks + 128) = phase-A tiles 2ks, 2ks+1
            for (int h = 0; h < nb; ++h) {
              const int* flag = &h_ready[ui.expert * tilesA + nb * ks + h];
              if (ld_acquire(flag) == 0) {
                while (ld_acquire(flag) == 0) {
                }
                trace_put(tc, 7, uu);
              }
            }
            fence_proxy_async_global();
          }
          unsigned char* st = ring + static_cast<size_t>(s) * stage_bytes + KB * kATile;
          mbar_arrive_expect_tx(&full[s], nb * box_bytes);
          const int row = dense && from_x ? 0 : ui.brow;  // dense: X itself (all tokens)
#pragma unroll
          for (int j = 0; j < KB; ++j)
            if (j < nb)
              tma_load_2d(st + j * b_box_bytes, &acts.map[bi], &full[s], (nb * ks + j) * kBK, row,
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
      const UnitInfo ui = decode(uu, qm, tilesA, tilesB, t, dense, n_tok);
      const bool phaseA = ui.phase == 0;
      const int n_mma = (ui.count + 15) & ~15;
      const uint32_t idesc = idesc_bf16_f32(kBM, n_mma);
      const uint32_t buf = nunit & 1u;
      const uint32_t use = nunit >> 1;
      mbar_wait(&tempty[buf], (use & 1u) ^ 1u);
      tc_fence_after();
      if (lane == 0) trace_put(tc, 9, uu);  // accumulator free: the unit's MMAs may start
      const uint32_t d_acc = tmem_base + buf * 256u;
      const bool pair = ui.nt == 2;
      const int ksteps = (phaseA ? ksA : ksB) * ui.nt;
      for (int ks = 0; ks < ksteps; ++ks, ++it) {
        const int s = it % S;
        mbar_wait(&full[s], (it / S) & 1);
        tc_fence_after();
        if (n_mma == 0) {  // no tokens: release the stage (and the accumulator)
          if (lane == 0) {
            mbar_arrive(&empty[s]);
            if (ks == ksteps - 1) mbar_arrive(&tfull[buf]);
          }
        } else if (elect_one()) {
          const uint32_t a0 = smem_u32(ring + static_cast<size_t>(s) * stage_bytes);
          const uint32_t b0 = a0 + KB * kATile;
          if (pair) {
            // tile tt: its KH blocks x the KH shared boxes -> columns [128 tt, 128 tt + n_mma)
            // of accumulator buffer `buf` (256 columns). Pairs run in dense mode
            // (n_mma <= 64) and in routed mode for blocks of n <= 128 tokens, so
            // n_mma <= 128 and tile 1 ends at column 256 of the buffer: buffer 1
            // spans TMEM columns 256-511, tile 1 of it 384-511
#pragma unroll
            for (int tt = 0; tt < 2; ++tt)
#pragma unroll
              for (int h = 0; h < KH; ++h)
#pragma unroll
                for (int kk = 0; kk < kBK / 16; ++kk)
                  tc_mma_bf16(d_acc + tt * 128u,
                              sw128_kmajor_desc(a0 + (tt * KH + h) * kATile + kk * 32),
                              sw128_kmajor_desc(b0 + h * b_box_bytes + kk * 32), idesc,
                              (ks > 0 || h > 0 || kk > 0) ? 1u : 0u);
          } else {
#pragma unroll
            for (int h = 0; h < KB; ++h)
#pragma unroll
              for (int kk = 0; kk < kBK / 16; ++kk)
                tc_mma_bf16(d_acc, sw128_kmajor_desc(a0 + h * kATile + kk * 32),
                            sw128_kmajor_desc(b0 + h * b_box_bytes + kk * 32), idesc,
                            (ks > 0 || h > 0 || kk > 0) ? 1u : 0u);
          }
          tc_commit(&empty[s]);
          if (ks == ksteps - 1) tc_commit(&tfull[buf]);
        }
        __syncwarp();
      }
      if (lane == 0) trace_put(tc, 10, uu);  // the unit's last MMA issued
      ++nunit;
    }
  } else if (warp == 2) {
    // ============ (idle after the TMEM allocation) ============
    if (dense && blockIdx.x == 0 && a.stats) {
      // the route stats (unique experts of the route, analysis.cpp:16-30, and
      // the selections) off the combine's critical path; t.count is unused in
      // dense mode and marks the experts seen
      int* seen = t.count;
      for (int i = lane; i < m; i += 32) seen[i] = 0;
      __syncwarp();
      int sel = 0;
      for (int o = lane; o < n_tok * k; o += 32) {
        uint64_t w;
        do {
          w = ld_relaxed_u64(a.route_words + o);
        } while (((static_cast<uint32_t>(w) >> 10) & kTagMask) != tag);
        const int x = static_cast<int>(w & 1023u);
        if (x != kPadExpert) {
          ++sel;
          seen[x] = 1;
        }
      }
      __syncwarp();
      int u = 0;
      for (int i = lane; i < m; i += 32) u += seen[i];
      u = __reduce_add_sync(0xffffffffu, u);
      sel = __reduce_add_sync(0xffffffffu, sel);
      if (lane == 0) {
        a.stats[0] = u;
        a.stats[2] = sel;
      }
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
      const UnitInfo ui = decode(uu, qm, tilesA, tilesB, t, dense, n_tok);
      const bool phaseA = ui.phase == 0;
      const int n_mma = (ui.count + 15) & ~15;
      const uint32_t buf = nunit & 1u;
      const uint32_t use = nunit >> 1;
      mbar_wait(&tfull[buf], use & 1u);
      tc_fence_after();
      if (etid == 0) trace_put(tc, 8, uu);  // accumulator ready
      const uint32_t lane_base = tmem_base + buf * 256u + (static_cast<uint32_t>(q4 * 32) << 16);
      if (phaseA) {
        // lanes 0-63: G, lanes 64-127: U of F columns tile*64 + (r mod 64)
        const bool is_g = r < kHalf;
        const int rr = r & (kHalf - 1);
        for (int tt = 0; tt < ui.nt; ++tt) {
        __nv_bfloat16* hrow =
            a.h_perm + static_cast<size_t>(ui.brow) * f + (ui.tile + tt) * kHalf + rr;
        for (int c0 = 0; c0 < n_mma; c0 += 16) {
          float v[16];
          tmem_ld16(lane_base + tt * 128u + c0, v);
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
        }  // tiles of the unit
      } else if (a.world <= 1) {
        for (int tt = 0; tt < ui.nt; ++tt) {
        float* yrow = a.y_slot + static_cast<size_t>(ui.brow) * d + (ui.tile + tt) * kBM + r;
        for (int c0 = 0; c0 < n_mma; c0 += 16) {
          float v[16];
          tmem_ld16(lane_base + tt * 128u + c0, v);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int col = c0 + j;
            if (col < ui.count)
              yrow[static_cast<size_t>(col) * d] =
                  dense ? v[j] : v[j] * t.slot_gate[ui.brow + col];
          }
        }
        }  // tiles of the unit
        if (a.b_done) {
          // (streamed combine) the barrier orders every epilogue thread's row
          // stores before the cumulative release the combine acquires
          named_bar_sync(1, 128);
          if (etid == 0)
            for (int tt = 0; tt < ui.nt; ++tt)
              st_release_u32(&a.b_done[ui.expert * tilesB + ui.tile + tt], tag);
        }
      } else {
        // expert parallel: push the gate-scaled rows straight into every
        // rank's slot buffer (own + NVLink peers) while later tiles stream
        for (int tt = 0; tt < ui.nt; ++tt) {
        const size_t off =
            ep_half + static_cast<size_t>(ui.brow) * d + (ui.tile + tt) * kBM + r;
        for (int c0 = 0; c0 < n_mma; c0 += 16) {
          float v[16];
          tmem_ld16(lane_base + tt * 128u + c0, v);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int col = c0 + j;
            if (col < ui.count) {
              const float val = dense ? v[j] : v[j] * t.slot_gate[ui.brow + col];
              for (int p = 0; p < a.world; ++p)
                __stcg(a.peer_slot[p] + off + static_cast<size_t>(col) * d, val);
            }
          }
        }
        }  // tiles of the unit
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      if (etid == 0) trace_put(tc, 11, uu);  // accumulator drained
      if (phaseA) {
        named_bar_sync(1, 128);
        // the barrier orders every epilogue thread's H stores before this
        if (etid == 0)
          for (int tt = 0; tt < ui.nt; ++tt)  // cumulative release
            red_add_release(&h_ready[ui.expert * tilesA + ui.tile + tt], 1);
      }
      if (etid == 0) trace_put(tc, 3, uu);
      ++nunit;
    }
  }
  __syncthreads();
  if (a.trace && tid == 0) {
    unsigned long long* cur = reinterpret_cast<unsigned long long*>(a.trace);
    const unsigned long long i0 = atomicAdd(cur, 7ull);
    for (int i = 0; i < 7; ++i)
      if (i0 + i < static_cast<unsigned long long>(a.trace_cap)) {
        a.trace[2 + 2 * (i0 + i)] = (static_cast<uint64_t>(blockIdx.x) << 8) | (90 + i);
        a.trace[3 + 2 * (i0 + i)] = s_pts[i];
      }
  }
  if (a.world > 1 && tid == 0) {
    // every slot row this CTA pushed is visible system-wide before the
    // arrival (fence cumulativity over the CTA barrier above)
    __threadfence_system();
    for (int p = 0; p < a.world; ++p) atomic_add_release_sys(a.peer_flag[p], 1ull);
  }
  if (tid == 0) trace_put(tc, 5, -1);
  trace_close(tc);
  // early mode never waited for the front kernel: do it before completing, so
  // the FFN's completion (which the combine waits for) implies the front's
  if (a.early && tid == 0) pdl_wait();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

template __global__ void ffn_persistent_kernel<2>(const __grid_constant__ CUtensorMap,
                                                   const __grid_constant__ CUtensorMap,
                                                   const __grid_constant__ CUtensorMap,
                                                   const __grid_constant__ BoxMaps,
                                                   const __grid_constant__ BoxMaps, FfnArgs);
template __global__ void ffn_persistent_kernel<4>(const __grid_constant__ CUtensorMap,
                                                   const __grid_constant__ CUtensorMap,
                                                   const __grid_constant__ CUtensorMap,
                                                   const __grid_constant__ BoxMaps,
                                                   const __grid_constant__ BoxMaps, FfnArgs);

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
        raise_flag(a.err, 2);
        break;
      }
      __nanosleep(100);
    }
  }
  __syncwarp();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ inline void store_row4(const CombineArgs& a, size_t off, float4 v) {
  if (a.resid) {  // h + MoE(h): the residual stream of a layer stack
    const uint2 r = *reinterpret_cast<const uint2*>(a.resid + off);
    const float2 r0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.x));
    const float2 r1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.y));
    v.x += r0.x;
    v.y += r0.y;
    v.z += r1.x;
    v.w += r1.y;
  }
  if (a.y_bf16) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&lo);
    u.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(a.y_bf16 + off) = u;
  } else {
    *reinterpret_cast<float4*>(a.y + off) = v;
  }
}

// Dense-mode combine: the FFN computed every published expert for every
// token (rows [list index][token]); y[t] = sum over the token's routed
// experts in ascending order of gate * row (gating.cpp:141-155) — the same
// fp32 products and sums as the routed path. CTA 0 also writes the block's
// stats (unique experts of the route, published list length, selections,
// experts this rank streamed).
// Ordered combine of 4 columns [c, c+4) of token tok over 8 route entries
// (moe_forward's order, gating.cpp:141-155): ascending slot order (=
// ascending expert), dense rows [expert][token], y += gate * row as a product
// then an add (no contraction) — the routed path's epilogue product followed
// by its combine add. All 8 rows are in flight at once.
__device__ __forceinline__ float4 combine4_rows(const float* ys, const int* e, const float* g,
                                                int n, int d, int tok, int c, float4 acc) {
  float4 v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (e[j] >= 0)
      v[j] = __ldcg(
          reinterpret_cast<const float4*>(ys + (static_cast<size_t>(e[j]) * n + tok) * d + c));
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (e[j] >= 0) {
      acc.x = __fadd_rn(acc.x, __fmul_rn(v[j].x, g[j]));
      acc.y = __fadd_rn(acc.y, __fmul_rn(v[j].y, g[j]));
      acc.z = __fadd_rn(acc.z, __fmul_rn(v[j].z, g[j]));
      acc.w = __fadd_rn(acc.w, __fmul_rn(v[j].w, g[j]));
    }
  return acc;
}

// End of a combine CTA (thread 0, after the CTA barrier that follows its y
// stores): the last CTA advances the call sequence and, for the host-buffer
// entry, publishes the host's call number once every CTA's y rows are visible
// system-wide (each CTA fences before it counts itself; fence cumulativity
// over the barrier covers its other threads' stores).
__device__ __forceinline__ void combine_retire(const CombineArgs& a) {
  if (a.host_done) __threadfence_system();
  if (atomicAdd(a.done_ctas, 1) == static_cast<int>(gridDim.x) - 1) {
    *a.done_ctas = 0;
    atomicAdd(a.epoch, 1);
    if (a.host_done) {
      __threadfence_system();
      *reinterpret_cast<volatile int*>(a.host_done) = *reinterpret_cast<const volatile int*>(a.host_call);
    }
  }
}

__global__ void __launch_bounds__(256) combine_dense_kernel(CombineArgs a) {
  // the next layer's router / front may launch at once: they prefetch their
  // static router weights and set up under this kernel, and their own
  // griddepcontrol.wait orders every read of this kernel's output
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // before the FFN grid completes: the call's tag and this thread's route
  // (the front's tagged words; the previous call's sequence bump completed
  // before this call's front started), so after the wait only the rows'
  // round trip remains. The FFN computed the route stats.
  __shared__ int s_epoch;
  const int tid = threadIdx.x;
  if (tid == 0) s_epoch = *a.epoch;
  __syncthreads();
  const uint32_t tag = hand_tag(s_epoch);
  const int vec = a.d / 4;
  const int i = blockIdx.x * blockDim.x + tid;
  const bool mine = i < a.n * vec;
  const int tok = mine ? i / vec : 0, c = mine ? (i - tok * vec) * 4 : 0;
  constexpr int kMaxK = 32;
  int e[kMaxK];
  float g[kMaxK];
#pragma unroll
  for (int j = 0; j < kMaxK; ++j) {
    e[j] = -1;
    g[j] = 0.f;
  }
  if (mine) {
#pragma unroll
    for (int j0 = 0; j0 < kMaxK; j0 += 8) {
      if (j0 >= a.k) break;
      uint64_t w[8];
      bool ok;
      do {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          w[j] = j0 + j < a.k ? ld_relaxed_u64(a.route_words + static_cast<size_t>(tok) * a.k + j0 + j)
                              : route_word(tag, kPadExpert, 0.f);
        ok = true;
#pragma unroll
        for (int j = 0; j < 8; ++j) ok &= ((static_cast<uint32_t>(w[j]) >> 10) & kTagMask) == tag;
      } while (!ok);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int x = static_cast<int>(w[j] & 1023u);
        e[j0 + j] = x == kPadExpert ? -1 : x;
        g[j0 + j] = __uint_as_float(static_cast<uint32_t>(w[j] >> 32));
      }
    }
  }
  // streamed (host-buffer entry): wait only for the phase-B units (expert,
  // d tile) of this thread's experts and columns — their tags are released
  // after the rows' stores — so the sums and y's bus writes overlap the
  // FFN's last units. One thread per CTA first waits (slow polls) until the
  // unit queue ran dry; then every warp polls its flags, all in flight at
  // once (relaxed), followed by one fence. A 2 s bound falls back to the
  // grid wait (never a hang).
  bool ready = false;
  if (a.b_done) {
    if (tid == 0) {
      const uint64_t t0 = gtime();
      while (ld_relaxed_u32(a.b_drained) != tag && gtime() - t0 < 2000000000ull) __nanosleep(512);
    }
    __syncthreads();
  }
  if (a.b_done && mine) {
    const uint32_t* bd = a.b_done + c / kBM;
    const uint64_t t0 = gtime();
    ready = true;
    bool ok;
    do {
      ok = true;
#pragma unroll
      for (int j = 0; j < kMaxK; ++j)
        if (j < a.k && e[j] >= 0) ok &= ld_relaxed_u32(bd + e[j] * a.tiles_b) == tag;
      if (!ok) {
        if (gtime() - t0 > 2000000000ull) {
          ready = false;
          break;
        }
        __nanosleep(256);
      }
    } while (!ok);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  if (!ready) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (blockIdx.x == 0 && tid == 0) trace(a.trace, a.trace_cap, 80, -1);
  const float* y_slot = a.y_slot;
  if (a.world > 1) y_slot += (static_cast<size_t>(s_epoch) & 1u) * a.slot_stride;
  if (mine) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int j0 = 0; j0 < kMaxK; j0 += 8) {
      if (j0 >= a.k) break;
      acc = combine4_rows(y_slot, e + j0, g + j0, a.n, a.d, tok, c, acc);
    }
    store_row4(a, static_cast<size_t>(tok) * a.d + c, acc);
  }
  // the FFN grid is complete before its counters are zeroed and the call
  // sequence advances (a no-op for the threads that already waited)
  if (ready || !mine) asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int w = i; w < a.zero_words; w += gridDim.x * blockDim.x) a.zero[w] = 0;
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) trace(a.trace, a.trace_cap, 81, -1);
  if (tid == 0) combine_retire(a);
}

__global__ void __launch_bounds__(256) combine_slots_kernel(CombineArgs a) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // (as combine_dense_kernel)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (blockIdx.x == 0 && threadIdx.x == 0) trace(a.trace, a.trace_cap, 80, -1);
  __shared__ int s_epoch;
  if (threadIdx.x == 0) s_epoch = *a.epoch;
  __syncthreads();
  const float* y_slot = a.y_slot;
  // expert parallel: ep_wait_kernel established (acquire) that every slot row arrived
  if (a.world > 1) y_slot += (static_cast<size_t>(s_epoch) & 1u) * a.slot_stride;
  const int vec = a.d / 4;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < a.n * vec) {
    const int tok = i / vec, c = (i - tok * vec) * 4;
    const int* so = a.slot_of + tok * a.k;  // ascending experts, -1 padded
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 v[8];
    for (int j0 = 0; j0 < a.k; j0 += 8) {
      int sl[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) sl[j] = j0 + j < a.k ? so[j0 + j] : -1;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (sl[j] >= 0)
          v[j] = __ldcg(reinterpret_cast<const float4*>(y_slot + static_cast<size_t>(sl[j]) * a.d + c));
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (sl[j] >= 0) {
          acc.x += v[j].x;
          acc.y += v[j].y;
          acc.z += v[j].z;
          acc.w += v[j].w;
        }
    }
    store_row4(a, static_cast<size_t>(tok) * a.d + c, acc);
  }
  // the FFN is complete: zero its counters for the next call
  for (int w = i; w < a.zero_words; w += gridDim.x * blockDim.x) a.zero[w] = 0;
  // the last CTA to finish advances the call sequence number (every CTA read it above)
  __syncthreads();
  // (relaxed atomics suffice: each CTA's epoch read completed before its
  // increment; the bump is published by the kernel's completion)
  if (blockIdx.x == 0 && threadIdx.x == 0) trace(a.trace, a.trace_cap, 81, -1);
  if (threadIdx.x == 0) combine_retire(a);
}

// x ingress of the host-buffer entry: 16-byte loads from the caller's pinned
// x over the bus, all of a thread's loads in flight at once, then the stores.
// The front kernel (programmatic launch) prefetches its router weights and
// sets up meanwhile; its griddepcontrol.wait orders it behind this copy.
__global__ void __launch_bounds__(256) x_ingress_kernel(const unsigned long long* src_word,
                                                        uint4* dst, int n16) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint4* src =
      reinterpret_cast<const uint4*>(*reinterpret_cast<const volatile unsigned long long*>(src_word));
  constexpr int kU = 4;
  uint4 v[kU];
  const int stride = gridDim.x * blockDim.x;
  const int i0 = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
  for (int u = 0; u < kU; ++u)
    if (i0 + u * stride < n16) v[u] = __ldcv(src + i0 + u * stride);
#pragma unroll
  for (int u = 0; u < kU; ++u)
    if (i0 + u * stride < n16) dst[i0 + u * stride] = v[u];
}

// The same copy through the TMA engine: each CTA moves one chunk of
// kIngressChunk bytes host -> shared (one bulk request, large bus reads) and
// shared -> device x (one bulk store).
__global__ void __launch_bounds__(32) x_ingress_bulk_kernel(const unsigned long long* src_word,
                                                            uint4* dst, int n16, int chunk) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(128) unsigned char buf[];  // [chunk]
  __shared__ __align__(8) uint64_t bar;
  const size_t off = static_cast<size_t>(blockIdx.x) * chunk;
  const size_t total = static_cast<size_t>(n16) * 16;
  if (threadIdx.x != 0 || off >= total) return;
  const uint32_t bytes = static_cast<uint32_t>(total - off < static_cast<size_t>(chunk) ? total - off : chunk);
  const unsigned char* src =
      reinterpret_cast<const unsigned char*>(*reinterpret_cast<const volatile unsigned long long*>(src_word));
  mbar_init(&bar, 1);
  fence_mbar_init();
  mbar_arrive_expect_tx(&bar, bytes);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(buf)),
      "l"(src + off), "r"(bytes), "r"(smem_u32(&bar))
      : "memory");
  mbar_wait(&bar, 0);
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                   reinterpret_cast<unsigned char*>(dst) + off),
               "r"(smem_u32(buf)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace desmoe
