// K1: router GEMM as a split-K swap-AB tcgen05 tile GEMM.
//
// logits^T tile = W_r[128 experts x K-slice] . X^T: the router weights are the
// MMA's A operand (M = 128 expert rows, K-major), the block's tokens the B
// operand (N = tokens rounded to 16). Both arrive by TMA (SWIZZLE_128B, 64-wide
// K blocks) into a shared-memory ring guarded by mbarriers; one elected thread
// issues tcgen05.mma into a TMEM accumulator; four epilogue warps drain TMEM
// with tcgen05.ld and write fp32 partials [split][token][expert]. The K range
// is split over up to 32 CTAs so the (<= 1 MiB) router weights stream from
// all SMs at once; the partials are reduced in fixed split order by the gating
// kernel, so logits are deterministic.
//
// Roles (256 threads): warp 0 = TMA producer, warp 1 = MMA issuer,
// warp 2 = TMEM allocator, warps 4-7 = epilogue (TMEM lane quarters 0-3).
#include "common.cuh"
#include "kernels.cuh"

namespace desmoe {

namespace {

struct Unit {
  bool valid;
  int wrow;      // first weight row of the tile (2-D weight view)
  int brow;      // first activation row (token / slot)
  int count;     // tokens in the tile
  int kb0, kb1;  // K-block range
  int out_col;   // first output column (f / d / expert index)
  int split;
};

__device__ inline Unit decode_unit(const TileArgs& a, int u) {
  Unit t{};
  if (u >= a.n_units_static) return t;
  const int et = u / a.splits, s = u % a.splits;
  const int kbs = (a.kb_total + a.splits - 1) / a.splits;
  t.wrow = et * kBM;
  t.brow = 0;
  t.count = a.n_tok;
  t.kb0 = s * kbs;
  t.kb1 = min(a.kb_total, t.kb0 + kbs);
  t.out_col = et * kBM;
  t.split = s;
  t.valid = t.kb0 < t.kb1;
  return t;
}

__device__ inline int box_index(int count) {
  int b = 0;
  while ((16 << b) < count && b < kMaxBoxes - 1) ++b;
  return b;
}

}  // namespace

__global__ void __launch_bounds__(256, 1)
    tile_gemm_kernel(const __grid_constant__ CUtensorMap wa, const __grid_constant__ CUtensorMap wb,
                     const __grid_constant__ BoxMaps acts, TileArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment for SWIZZLE_128B atoms
  // align to 1024 B by offsetting the shared array itself, so the compiler
  // keeps the shared address space (LDS/STS instead of generic LD/ST)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const Unit unit = decode_unit(a, blockIdx.x);
  if (!unit.valid) return;

  const int b_bytes_max = a.b_rows * 128;
  const int stage_bytes = kATile + b_bytes_max;
  const int S = a.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(S) * stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* tmem_full = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int bi = box_index(unit.count);
  const int box_rows = 16 << bi;
  const int n_mma = (unit.count + 15) & ~15;
  const uint32_t tmem_cols_needed = a.b_rows;
  uint32_t tmem_cols = 32;
  while (tmem_cols < tmem_cols_needed) tmem_cols <<= 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&wa);
    tma_prefetch_desc(&acts.map[bi]);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int nkb = unit.kb1 - unit.kb0;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      const uint64_t pol_w = l2_policy_evict_first();  // weights: streamed once
      const uint64_t pol_x = l2_policy_evict_last();   // activations: re-read per tile
      const uint32_t bytes = kATile + box_rows * 128;
      for (int i = 0; i < nkb; ++i) {
        const int s = i % S;
        const uint32_t ph = (i / S) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        unsigned char* st = smem + static_cast<size_t>(s) * stage_bytes;
        const int kc = (unit.kb0 + i) * kBK;
        mbar_arrive_expect_tx(&full[s], bytes);
        tma_load_2d(st, &wa, &full[s], kc, unit.wrow, pol_w);
        tma_load_2d(st + kATile, &acts.map[bi], &full[s], kc, unit.brow, pol_x);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = idesc_bf16_f32(kBM, n_mma);
    const uint32_t d_acc = tmem_base;
    for (int i = 0; i < nkb; ++i) {
      const int s = i % S;
      const uint32_t ph = (i / S) & 1;
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (elect_one()) {
        unsigned char* st = smem + static_cast<size_t>(s) * stage_bytes;
        const uint32_t a0 = smem_u32(st);
        const uint32_t b0 = a0 + kATile;
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {
          const uint32_t acc = (i > 0 || k > 0) ? 1u : 0u;
          const uint64_t bdesc = sw128_kmajor_desc(b0 + k * 32);
          tc_mma_bf16(d_acc, sw128_kmajor_desc(a0 + k * 32), bdesc, idesc, acc);
        }
        tc_commit(&empty[s]);
        if (i == nkb - 1) tc_commit(tmem_full);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const int q = warp & 3;
    const int r = q * 32 + lane;  // accumulator row = weight row within the tile
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    for (int c0 = 0; c0 < n_mma; c0 += 16) {
      float v[16];
      tmem_ld16(lane_base + c0, v);
      {  // router partials [split][token][expert]
        const int e = unit.out_col + r;
        if (e < a.m_pad) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int col = c0 + j;
            if (col < unit.count)
              a.y_out[(static_cast<size_t>(unit.split) * a.n_tok + col) * a.m_pad + e] = v[j];
          }
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, tmem_cols);
  }
}

}  // namespace desmoe
