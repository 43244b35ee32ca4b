// Cost of reading %globaltimer (the timeline marks' clock) vs %clock64.
#include <cstdint>
#include <cstdio>
__global__ void k(long long* out, int n) {
  uint64_t acc = 0, g;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    acc += g;
  }
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) {
    long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    acc += c;
  }
  long long t2 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = acc; }
}
int main() {
  long long* d; cudaMalloc(&d, 64); long long h[3];
  for (int r = 0; r < 2; ++r) {
    k<<<1, 32>>>(d, 256);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("cycles per read: globaltimer %.1f, clock64 %.1f\n", h[0] / 256.0, h[1] / 256.0);
  }
}
