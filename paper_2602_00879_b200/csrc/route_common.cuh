// Per-token routing steps shared by the fused routing kernels (front.cu,
// route_fused.cu). One warp per token; the token's row lives in shared memory.
//
// Row contents after token_activate(): softmax -> e_i = exp(x_i - max) (the
// reference's numerators, gating.cpp:30-33), sigmoid -> p_i, identity -> p_i.
// The softmax probabilities are p_i = e_i / s with s the ascending-index sum
// (gating.cpp:34-38); p_of() recomputes exactly that quotient wherever a
// probability is needed, so values equal the reference's bit for bit (modulo
// the last-bit freedom of exp).
//
// Selection: p and e order the same way except where a division rounds two
// distinct e to one p. The fast path selects on e with packed keys
// (warp_topk_packed, two REDUX per round) and inspects the boundary element;
// if the last selected and the first rejected value are within 2^-40
// relative of each other (a near-tie the division or the key truncation could
// flip), the token is re-selected exactly on the fp64 probabilities with the
// reference's comparator (warp_select). Otherwise the selected SET provably
// equals the reference's top-k.
#pragma once

#include "common.cuh"

namespace desmoe {

__device__ inline double p_of(const double* row, double s, int act, int i) {
  return act == 0 ? div_f64(row[i], s) : row[i];
}

// Activation of one token row in place; returns the softmax sum (1 otherwise).
__device__ inline double token_activate(double* row, int m, int act, double mx) {
  const int lane = threadIdx.x & 31;
  if (act == 0) {
    for (int i = lane; i < m; i += 32) row[i] = exp_f64(row[i] - mx);
  } else if (act == 1) {
    for (int i = lane; i < m; i += 32) row[i] = sigmoid_f64(row[i]);
  }
  __syncwarp();
  double s = 1.0;
  if (act == 0) {
    s = 0.0;
    if (lane == 0)
      for (int i = 0; i < m; ++i) s += row[i];
    s = __shfl_sync(0xffffffffu, s, 0);
  }
  return s;
}

__device__ inline bool near_tie(double a, double b) {
  // a should be >= b (selected before rejected); treat reversed order or a
  // relative gap below 2^-40 as ambiguous
  return !(a - b > b * 0x1.0p-40) || a < b;
}

// Top-`k` (rank order) of the token's probabilities restricted to `allow`
// (nullptr = all), exactly in the reference's order for the set and for the
// prefix of length `k2` (0 = no second boundary). `navail` = number of
// allowed candidates. scratch: m doubles. Returns the number selected.
static __device__ __noinline__ int token_select(const double* row, double s, int act, int m, int k, int k2,
                                   const uint8_t* allow, int navail, int* sel, uint64_t* keys,
                                   double* scratch) {
  const int lane = threadIdx.x & 31;
  const int want = k < navail ? k : navail;
  const int rounds = want < navail ? want + 1 : want;
  warp_topk_packed(row, m, rounds, allow, sel, keys);
  bool amb = false;
  if (want < navail) amb |= near_tie(row[sel[want - 1]], row[sel[want]]);
  if (k2 > 0 && k2 < want) amb |= near_tie(row[sel[k2 - 1]], row[sel[k2]]);
  if (amb) {
    for (int i = lane; i < m; i += 32) scratch[i] = p_of(row, s, act, i);
    __syncwarp();
    warp_select(scratch, m, want, allow, sel);
  }
  return want;
}

// Sorts sel[0..cnt) ascending (distinct indices) in place.
__device__ inline void sort_selection(int* sel, int cnt) {
  const int lane = threadIdx.x & 31;
  const int my = lane < cnt ? sel[lane] : 0x7fffffff;
  const int pos = ascending_rank(my, lane, cnt);
  __syncwarp();
  if (lane < cnt) sel[pos] = my;
  __syncwarp();
}

// Writes the token's route: experts ascending, gates renormalised over the
// selection in ascending index order (gating.cpp:73-82), -1/0 padding.
static __device__ __noinline__ void token_write_route(const double* row, double s, int act, int* sel, int cnt,
                                         int k, int t, int* route_idx, double* route_gate,
                                         int* route_cnt) {
  const int lane = threadIdx.x & 31;
  sort_selection(sel, cnt);
  double ssum = 0.0;
  if (lane == 0)
    for (int j = 0; j < cnt; ++j) ssum += p_of(row, s, act, sel[j]);
  ssum = __shfl_sync(0xffffffffu, ssum, 0);
  if (lane < k) {
    const size_t o = static_cast<size_t>(t) * k + lane;
    const bool in = lane < cnt;
    route_idx[o] = in ? sel[lane] : -1;
    route_gate[o] = in ? div_f64(p_of(row, s, act, sel[lane]), ssum) : 0.0;
  }
  if (lane == 0) route_cnt[t] = cnt;
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Register-resident top-k: each lane keeps its (up to P) packed candidate
// keys sorted descending in registers, so a round is two REDUX (~28 cycles
// each) plus predicated register shifts in the owner lane — no shared-memory
// traffic or divergent rescans on the critical path.
// ---------------------------------------------------------------------------
template <int P>
struct LaneKeys {
  uint64_t k[P];
};

template <int P>
__device__ inline void lane_sort_desc(LaneKeys<P>& L) {
#pragma unroll
  for (int i = 0; i < P; ++i)
#pragma unroll
    for (int j = 0; j + 1 < P - i; ++j) {
      const uint64_t a = L.k[j], b = L.k[j + 1];
      const bool sw = b > a;
      L.k[j] = sw ? b : a;
      L.k[j + 1] = sw ? a : b;
    }
}

// rounds <= 64; sel[r]/keys[r] written by lane 0 (sel = -1 once exhausted).
template <int P>
__device__ inline void warp_topk_regs(LaneKeys<P>& L, int rounds, int* sel, uint64_t* keys) {
  const int lane = threadIdx.x & 31;
  lane_sort_desc<P>(L);
  for (int r = 0; r < rounds; ++r) {
    const uint64_t best = L.k[0];
    const uint32_t hi = __reduce_max_sync(0xffffffffu, static_cast<uint32_t>(best >> 32));
    const uint32_t lo = __reduce_max_sync(
        0xffffffffu, static_cast<uint32_t>(best >> 32) == hi ? static_cast<uint32_t>(best) : 0u);
    const uint64_t win = (static_cast<uint64_t>(hi) << 32) | lo;
    const int idx = 1023 - static_cast<int>(lo & 0x3FFu);
    if (lane == 0) {
      sel[r] = win ? idx : -1;
      keys[r] = win;
    }
    const bool own = win != 0 && best == win;
#pragma unroll
    for (int j = 0; j + 1 < P; ++j) L.k[j] = own ? L.k[j + 1] : L.k[j];
    L.k[P - 1] = own ? 0ull : L.k[P - 1];
  }
  __syncwarp();
}

// Loads the lane's candidates of `val` (allow == nullptr -> all) as packed keys.
template <int P>
__device__ inline void lane_load_keys(LaneKeys<P>& L, const double* val, int m,
                                      const uint8_t* allow) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 0; s < P; ++s) {
    const int i = lane + 32 * s;
    L.k[s] = (i < m && (!allow || allow[i])) ? packed_key(val[i], i) : 0ull;
  }
}

// Top-`want` of `val` (restricted to allow) in (value desc, index asc) order
// of the packed keys, for any m <= 32 * 32 (dispatches on candidates/lane).
// Runs `rounds` >= want rounds so the caller can inspect the boundary.
static __device__ __noinline__ void warp_topk_fast(const double* val, int m, int rounds, const uint8_t* allow,
                                      int* sel, uint64_t* keys) {
  if (m <= 64) {
    LaneKeys<2> L;
    lane_load_keys<2>(L, val, m, allow);
    warp_topk_regs<2>(L, rounds, sel, keys);
  } else if (m <= 128) {
    LaneKeys<4> L;
    lane_load_keys<4>(L, val, m, allow);
    warp_topk_regs<4>(L, rounds, sel, keys);
  } else if (m <= 256) {
    LaneKeys<8> L;
    lane_load_keys<8>(L, val, m, allow);
    warp_topk_regs<8>(L, rounds, sel, keys);
  } else {
    warp_topk_packed(val, m, rounds, allow, sel, keys);
  }
}

// Completes a fast selection made on packed keys of the logits (softmax) or of
// the probabilities (sigmoid / identity). `sel` holds the fast rounds
// (want + 1 when a boundary element exists). The selected SET (and the prefix
// of length k2) is exactly the reference's unless a boundary is a near-tie:
//   softmax  x gap <= 2^-40 (exp / division could merge the two values) or the
//            rejected e is tiny (exp underflow ties, p subnormal);
//   else     relative p gap <= 2^-40.
// Near-ties re-select exactly on the fp64 probabilities with the reference's
// comparator. Returns the number selected.
static __device__ __noinline__ int token_finish_selection(const double* xr, const double* er, double s,
                                             double mx, int act, int m, int k, int k2,
                                             const uint8_t* allow, int navail, int* sel,
                                             double* scratch) {
  const int lane = threadIdx.x & 31;
  const int want = k < navail ? k : navail;
  auto risky = [&](int b) -> bool {  // boundary between ranks b-1 and b
    const int hi = sel[b - 1], lo = sel[b];
    if (act == 0) {
      const double gap = xr[hi] - xr[lo];
      return !(gap > 0x1.0p-40) || !(er[lo] > 0x1.0p-960);
    }
    return near_tie(er[hi], er[lo]);
  };
  bool amb = false;
  if (want < navail) amb |= risky(want);
  if (k2 > 0 && k2 < want) amb |= risky(k2);
  if (amb) {
    for (int i = lane; i < m; i += 32) scratch[i] = p_of(er, s, act, i);
    __syncwarp();
    warp_select(scratch, m, want, allow, sel);
  }
  __syncwarp();
  return want;
}

}  // namespace desmoe
