// Exact fp64 gating primitives of the reference's public API that the fused
// layer kernels do not cover on their own:
//
//   select_top_kernel      select_top_gates (gating.cpp:42-71), both overloads,
//                          any k: a rank count per candidate under the
//                          reference's comparator (value desc, index asc; -0 ==
//                          +0 as in `gates[a] != gates[b]`), then an ascending
//                          compaction of the selected indices;
//   renormalize_kernel     renormalize_over (gating.cpp:73-82): the sum runs
//                          over `selected` in the given order, then divides;
//   linear_expert_kernel   moe_forward / expert_output (gating.cpp:122-157) on
//                          the reference's linear D x D experts in fp64 with
//                          the reference's exact operation order and no FMA
//                          contraction (__dmul_rn / __dadd_rn), so outputs are
//                          bit-identical to the CPU library's.
#include "common.cuh"
#include "kernels.cuh"

namespace desmoe {

namespace {

__device__ inline bool ref_before(double va, int a, double vb, int b) {
  // gating.cpp:49-52: if (g[a] != g[b]) return g[a] > g[b]; return a < b;
  return va != vb ? va > vb : a < b;
}

}  // namespace

// One CTA (blockDim multiple of 32, <= 1024). values [m]; cand [n_cand]
// (nullptr = all m). Dynamic smem: m doubles + m bytes of flags + 33 ints.
__global__ void select_top_kernel(const double* __restrict__ values, int m, int k,
                                  const int* __restrict__ cand, int n_cand, int* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* v = reinterpret_cast<double*>(smem);
  int* warp_tot = reinterpret_cast<int*>(v + m);
  uint8_t* flag = reinterpret_cast<uint8_t*>(warp_tot + 33);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int i = tid; i < m; i += blockDim.x) {
    v[i] = values[i];
    flag[i] = 0;
  }
  __syncthreads();
  const int nc = cand ? n_cand : m;
  for (int p = tid; p < nc; p += blockDim.x) {
    const int i = cand ? cand[p] : p;
    const double vi = v[i];
    int rank = 0;
    for (int q = 0; q < nc; ++q) {
      const int j = cand ? cand[q] : q;
      rank += ref_before(v[j], j, vi, i);
    }
    if (rank < k) flag[i] = 1;
  }
  __syncthreads();
  // ascending compaction (std::sort of the selection, gating.cpp:55)
  int base = 0;
  for (int c0 = 0; c0 < m; c0 += blockDim.x) {
    const int i = c0 + tid;
    const int f = i < m ? flag[i] : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) warp_tot[warp] = __popc(bal);
    __syncthreads();
    if (tid == 0) {
      int acc = 0;
      for (int w = 0; w < nw; ++w) {
        const int c = warp_tot[w];
        warp_tot[w] = acc;
        acc += c;
      }
      warp_tot[32] = acc;
    }
    __syncthreads();
    if (f) out[base + warp_tot[warp] + __popc(bal & ((1u << lane) - 1u))] = i;
    base += warp_tot[32];
    __syncthreads();
  }
}

__global__ void renormalize_kernel(const double* __restrict__ values,
                                   const int* __restrict__ sel, int count,
                                   double* __restrict__ out) {
  __shared__ double s_sum;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int j = 0; j < count; ++j) s = __dadd_rn(s, values[sel[j]]);
    s_sum = s;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < count; j += blockDim.x) out[j] = __ddiv_rn(values[sel[j]], s_sum);
}

// grid (ceil(d / blockDim.x), n); thread = one output row r of token t.
// y[t][r] = sum_j (in stored order) g_j * (sum_c W_{e_j}[r][c] * x[t][c]).
// Dynamic smem: the token's input row (d doubles).
__global__ void linear_expert_kernel(const double* __restrict__ w, const double* __restrict__ x,
                                     int d, int k, const int* __restrict__ route_idx,
                                     const double* __restrict__ route_gate,
                                     const int* __restrict__ route_cnt, double* __restrict__ y) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* xs = reinterpret_cast<double*>(smem);
  const int t = blockIdx.y;
  for (int c = threadIdx.x; c < d; c += blockDim.x) xs[c] = x[static_cast<size_t>(t) * d + c];
  __syncthreads();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= d) return;
  const int cnt = route_cnt[t];
  double acc_y = 0.0;
  for (int j = 0; j < cnt; ++j) {
    const int e = route_idx[static_cast<size_t>(t) * k + j];
    const double g = route_gate[static_cast<size_t>(t) * k + j];
    const double* wr = w + (static_cast<size_t>(e) * d + r) * d;
    double acc = 0.0;
    for (int c = 0; c < d; ++c) acc = __dadd_rn(acc, __dmul_rn(wr[c], xs[c]));
    acc_y = __dadd_rn(acc_y, __dmul_rn(g, acc));
  }
  y[static_cast<size_t>(t) * d + r] = acc_y;
}

}  // namespace desmoe
