// Pure-read HBM streaming ceiling on this GPU: every CTA (one per SM) pulls a
// contiguous slice of a large buffer into a shared-memory ring with 1-D bulk
// copies (cp.async.bulk, mbarrier complete_tx) and does nothing else — the
// best the expert-weight stream could do. Also plain vectorised loads.
// Usage: ./stream  (prints GB/s per configuration)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ inline uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(128, 1) tma_stream(const char* src, size_t per_cta, int chunk, int stages, int* sink) {
  extern __shared__ __align__(128) char ring[];
  __shared__ __align__(8) uint64_t bar[16];
  const char* base = src + per_cta * blockIdx.x;
  const int n = static_cast<int>(per_cta / chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      if (i >= stages) {  // wait for the stage's previous fill
        const uint32_t ph = ((i / stages) - 1) & 1;
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                       : "=r"(ok) : "r"(su32(&bar[s])), "r"(ph));
      }
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(chunk));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(ring + static_cast<size_t>(s) * chunk)), "l"(base + static_cast<size_t>(i) * chunk),
                   "r"(chunk), "r"(su32(&bar[s])) : "memory");
    }
    for (int i = n; i < n + stages; ++i) {  // drain
      const int s = i % stages;
      const uint32_t ph = ((i / stages) - 1) & 1;
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(su32(&bar[s])), "r"(ph));
    }
    sink[blockIdx.x] = ring[5];
  }
}

__global__ void ld_stream(const int4* src, size_t n, int* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    int4 v = __ldcs(src + i);
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345) sink[0] = 1;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = size_t(2) << 30;  // 2 GiB
  char* buf;
  int* sink;
  cudaMalloc(&buf, total);
  cudaMalloc(&sink, 4096 * 4);
  cudaMemset(buf, 1, total);
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int chunks[] = {16384, 32768};
  for (int chunk : chunks)
    for (int stages = 2; stages <= 6; ++stages) {
      if ((size_t)chunk * stages > (200u << 10)) continue;
      const size_t per = (total / sms) / chunk * chunk;
      float best = 1e9f;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        tma_stream<<<sms, 128, chunk * stages>>>(buf, per, chunk, stages, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
      }
      printf("bulk chunk=%6d stages=%d in-flight=%4d KB: %.0f GB/s\n", chunk, stages, chunk * stages / 1024,
             per * sms / (best * 1e6));
    }
  for (int bpsm = 1; bpsm <= 8; bpsm *= 2) {
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      ld_stream<<<sms * bpsm, 512>>>(reinterpret_cast<int4*>(buf), total / 16, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    printf("ld.cs %d x 512 thr/SM: %.0f GB/s\n", bpsm, total / (best * 1e6));
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
