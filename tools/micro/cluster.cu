// Cluster-barrier and DSMEM latency probe (8-CTA cluster, 512 threads/CTA):
// globaltimer stamps around the first (cold) and subsequent cluster barriers
// and a remote shared-memory load round trip.
#include <cstdio>
#include <cstdint>

__device__ inline uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ inline void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ inline void csync_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(512, 1) probe(uint64_t* out) {
  __shared__ float buf[1024];
  for (int i = threadIdx.x; i < 1024; i += 512) buf[i] = i;
  __syncthreads();
  uint64_t t[10];
  t[0] = gt();
  csync();
  t[1] = gt();
  csync();
  t[2] = gt();
  csync_relaxed();
  t[3] = gt();
  __syncthreads();
  t[4] = gt();
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  uint32_t la = static_cast<uint32_t>(__cvta_generic_to_shared(&buf[threadIdx.x & 1023])), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"((rank + 1) & 7));
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ra) : "memory");
  asm volatile("" ::"f"(v));
  t[5] = gt();
  float acc = 0;
  for (int r = 0; r < 8; ++r) {
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(r));
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ra) : "memory");
    acc += v;
  }
  asm volatile("" ::"f"(acc));
  t[6] = gt();
  csync();
  t[7] = gt();
  if (threadIdx.x == 0)
    for (int i = 0; i < 8; ++i) out[blockIdx.x * 8 + i] = t[i];
}

int main() {
  uint64_t* d;
  cudaMalloc(&d, 8 * 8 * 8 * 4);
  uint64_t h[64];
  for (int rep = 0; rep < 4; ++rep) {
    probe<<<8, 512>>>(d);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("rep %d (ns, CTA0): sync1 %llu sync2 %llu relaxed %llu syncthreads %llu dsmem1 %llu dsmem8 %llu sync4 %llu\n", rep,
           (unsigned long long)(h[1] - h[0]), (unsigned long long)(h[2] - h[1]), (unsigned long long)(h[3] - h[2]),
           (unsigned long long)(h[4] - h[3]), (unsigned long long)(h[5] - h[4]), (unsigned long long)(h[6] - h[5]),
           (unsigned long long)(h[7] - h[6]));
  }
  return 0;
}
