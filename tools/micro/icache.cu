// Does straight-line code executed once per launch run at instruction-fetch
// speed? Times (clock64) a fully unrolled block of ~N independent FFMAs:
// first launch after a code-thrashing kernel vs immediate relaunch.
#include <cstdio>

template <int N>
__global__ void straight(float* out, long long* cyc, float a) {
  float x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3;
  long long t0;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0)::"memory");
  asm volatile("" : "+f"(x0), "+f"(x1), "+f"(x2), "+f"(x3)::"memory");
#pragma unroll
  for (int i = 0; i < N; ++i) {
    x0 = x0 * 1.0001f + 0.5f;
    x1 = x1 * 0.9999f + 0.25f;
    x2 = x2 * 1.0002f - 0.5f;
    x3 = x3 * 0.9998f - 0.25f;
  }
  asm volatile("" : "+f"(x0), "+f"(x1), "+f"(x2), "+f"(x3)::"memory");
  long long t1;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1)::"memory");
  if (threadIdx.x == 0) {
    out[blockIdx.x] = x0 + x1 + x2 + x3;
    cyc[0] = t1 - t0;
  }
}

template <int N>
__global__ void thrash(float* out, float a) {  // different large code body
  float x0 = a;
#pragma unroll
  for (int i = 0; i < N; ++i) x0 = x0 * 1.0003f + 0.125f * i;
  if (threadIdx.x == 0) out[blockIdx.x + 1] = x0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4096);
  cudaMalloc(&cyc, 64);
  long long c;
  for (int rep = 0; rep < 3; ++rep) {
    thrash<8000><<<148, 32>>>(out, 1.f);
    straight<1000><<<1, 32>>>(out, cyc, 1.f);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("after thrash: 4000 FFMA straight-line: %lld cycles\n", c);
    straight<1000><<<1, 32>>>(out, cyc, 1.f);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("relaunch    : 4000 FFMA straight-line: %lld cycles\n", c);
  }
  return 0;
}
