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
  return act == 0 ? row[i] / s : row[i];
}

// Activation of one token row in place; returns the softmax sum (1 otherwise).
__device__ inline double token_activate(double* row, int m, int act, double mx) {
  const int lane = threadIdx.x & 31;
  if (act == 0) {
    for (int i = lane; i < m; i += 32) row[i] = exp(row[i] - mx);
  } else if (act == 1) {
    for (int i = lane; i < m; i += 32) row[i] = 1.0 / (1.0 + exp(-row[i]));
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
__device__ inline int token_select(const double* row, double s, int act, int m, int k, int k2,
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
__device__ inline void token_write_route(const double* row, double s, int act, int* sel, int cnt,
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
    route_gate[o] = in ? p_of(row, s, act, sel[lane]) / ssum : 0.0;
  }
  if (lane == 0) route_cnt[t] = cnt;
  __syncwarp();
}

}  // namespace desmoe
