// Dependent-chain latencies on sm_100a: DADD, DFMA, FADD, LDS.32 pointer
// chase, and a warp's throughput of broadcast LDS.64 (clock64, one warp).
#include <cstdint>
#include <cstdio>

__global__ void lat(long long* out, double a, float b, int n) {
  __shared__ int nxt[1024];
  __shared__ uint64_t keys[256];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) nxt[i] = (i * 37 + 11) & 1023;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) keys[i] = i * 0x9E3779B97F4A7C15ull;
  __syncthreads();
  if (threadIdx.x >= 32) return;
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + a;  // DADD chain
  long long t1 = clock64();
  double y = a;
  for (int i = 0; i < n; ++i) y = fma(y, a, a);  // DFMA chain
  long long t2 = clock64();
  float f = b;
  for (int i = 0; i < n; ++i) f = f + b;  // FADD chain
  long long t3 = clock64();
  int p = threadIdx.x;
  for (int i = 0; i < n; ++i) p = nxt[p];  // LDS chase
  long long t4 = clock64();
  uint64_t acc = 0;
#pragma unroll 8
  for (int i = 0; i < n; ++i) acc += keys[i & 255] > 12345u;  // broadcast LDS.64 + compare
  long long t5 = clock64();
  if (threadIdx.x == 0) {
    out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4;
    out[5] = (long long)(x + y + f + p + acc);
  }
}

int main() {
  long long* d; cudaMalloc(&d, 64);
  long long h[8];
  const int n = 1024;
  for (int r = 0; r < 2; ++r) {
    lat<<<1, 128>>>(d, 1.0000001, 1.0001f, n);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 48, cudaMemcpyDeviceToHost);
    printf("per op (cycles): DADD %.1f DFMA %.1f FADD %.1f LDS-chase %.1f LDS64-bcast-tput %.1f\n",
           (double)h[0] / n, (double)h[1] / n, (double)h[2] / n, (double)h[3] / n, (double)h[4] / n);
  }
  return 0;
}
