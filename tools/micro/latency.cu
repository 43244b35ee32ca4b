// Microbenchmarks (clock64 cycles, one warp) of the routing stage's building
// blocks on sm_100a: serial fp64 sum, exp(double), fp64 division, warp
// top-K selection, shuffles, and shared-memory round trips.
#include <cstdio>
#include <cstdint>
#include "../../paper_2602_00879_b200/csrc/common.cuh"

using namespace desmoe;

__global__ void probe(const double* in, long long* out, int m, int k) {
  __shared__ double row[1024];
  __shared__ int sel[64];
  const int lane = threadIdx.x;
  for (int i = lane; i < m; i += 32) row[i] = in[i];
  __syncwarp();
  long long t0 = clock64();
  double s = 0.0;
  if (lane == 0)
    for (int i = 0; i < m; ++i) s += row[i];
  s = __shfl_sync(0xffffffffu, s, 0);
  long long t1 = clock64();
  double e = 0.0;
  for (int i = lane; i < m; i += 32) e += exp(row[i] - 1.0);
  e = __shfl_sync(0xffffffffu, e, 0);
  long long t2 = clock64();
  double q = 0.0;
  for (int i = lane; i < m; i += 32) q += row[i] / (s + 3.0);
  q = __shfl_sync(0xffffffffu, q, 0);
  long long t3 = clock64();
  warp_select(row, m, k, nullptr, sel);
  long long t4 = clock64();
  uint64_t kk = order_key(row[lane]);
  int ii = lane;
  warp_argbest(kk, ii);
  long long t5 = clock64();
  float f = 0.f;
  for (int i = lane; i < m; i += 32) f += expf(static_cast<float>(row[i]));
  f = __shfl_sync(0xffffffffu, f, 0);
  long long t6 = clock64();
  uint64_t pk[40];
  warp_topk_packed(row, m, 9, nullptr, sel, pk);
  long long t7 = clock64();
  uint32_t rv = static_cast<uint32_t>(row[lane] * 1000.0);
  for (int r = 0; r < 8; ++r) rv = __reduce_max_sync(0xffffffffu, rv + r);
  long long t8 = clock64();
  uint32_t sv = rv;
  for (int r = 0; r < 8; ++r) sv = __shfl_xor_sync(0xffffffffu, sv, 1) + r;
  long long t9 = clock64();
  if (lane == 0) {
    out[7] = t7 - t6;
    out[8] = (t8 - t7) / 8;
    out[9] = (t9 - t8) / 8;
    out[10] = static_cast<long long>(sv + pk[0]);
    out[0] = t1 - t0;
    out[1] = t2 - t1;
    out[2] = t3 - t2;
    out[3] = t4 - t3;
    out[4] = t5 - t4;
    out[5] = t6 - t5;
    out[6] = static_cast<long long>(s + e + q + sel[0] + ii + f);
  }
}

int main2();
int main() {
  main2();
  const int ms[] = {64, 256};
  double* in;
  long long* out;
  cudaMalloc(&in, 1024 * 8);
  cudaMalloc(&out, 16 * 8);
  double h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = 0.001 * ((i * 7919) % 1000) - 0.5;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int m : ms) {
    for (int rep = 0; rep < 3; ++rep) probe<<<1, 32>>>(in, out, m, 8);
    long long r[12];
    cudaMemcpy(r, out, sizeof(r), cudaMemcpyDeviceToHost);
    printf("m=%d cycles: serial_dadd_sum=%lld exp_f64=%lld div_f64=%lld warp_select_k8=%lld "
           "warp_argbest=%lld expf_f32=%lld topk_packed_9=%lld redux=%lld shfl=%lld\n",
           m, r[0], r[1], r[2], r[3], r[4], r[5], r[7], r[8], r[9]);
  }
  return 0;
}

// CTA-level probes: barrier, smem atomics, global atomic round trip, globaltimer.
__global__ void probe_cta(unsigned long long* gcnt, long long* out) {
  __shared__ uint32_t words[64];
  __shared__ int cnt[64];
  const int tid = threadIdx.x;
  if (tid < 64) { words[tid] = 0; cnt[tid] = 0; }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < 10; ++i) __syncthreads();
  long long t1 = clock64();
  atomicOr(&words[(tid * 7) & 63], 1u << (tid & 31));
  atomicAdd(&cnt[(tid * 7) & 63], 1);
  __syncthreads();
  long long t2 = clock64();
  if (tid == 0) atomicAdd(gcnt, 1ull);
  __syncthreads();
  long long t3 = clock64();
  uint64_t g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  long long t4 = clock64();
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1)); } while (g1 == g0);
  long long t5 = clock64();
  if (tid == 0) {
    out[0] = (t1 - t0) / 10;
    out[1] = t2 - t1;
    out[2] = t3 - t2;
    out[3] = t5 - t4;
    out[4] = static_cast<long long>(g1 - g0);
    out[5] = words[0] + cnt[0];
  }
}

int main2() {
  unsigned long long* g;
  long long* out;
  cudaMalloc(&g, 8);
  cudaMalloc(&out, 64);
  for (int rep = 0; rep < 3; ++rep) probe_cta<<<1, 256>>>(g, out);
  long long r[6];
  cudaMemcpy(r, out, sizeof(r), cudaMemcpyDeviceToHost);
  printf("cta: syncthreads=%lld smem_atomics+sync=%lld global_atomic+sync=%lld "
         "globaltimer_tick_cycles=%lld tick_ns=%lld\n", r[0], r[1], r[2], r[3], r[4]);
  return 0;
}
