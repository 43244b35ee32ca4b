// Cost of executing code that is not in the SM's instruction caches:
// a chain of NF distinct noinline functions (each ~40 instructions, called
// once) vs the same chain re-run (warm), after a thrash kernel that evicts
// the instruction caches. Prints cycles per cold call.
#include <cstdio>
#include <cstdint>

#define FN(i)                                                              \
  __device__ __noinline__ float f##i(float x) {                            \
    _Pragma("unroll") for (int k = 0; k < 10; ++k) x = x * 1.0001f + 0.5f * (i + 1); \
    return x;                                                              \
  }
FN(0) FN(1) FN(2) FN(3) FN(4) FN(5) FN(6) FN(7) FN(8) FN(9) FN(10) FN(11) FN(12) FN(13) FN(14) FN(15)
FN(16) FN(17) FN(18) FN(19) FN(20) FN(21) FN(22) FN(23) FN(24) FN(25) FN(26) FN(27) FN(28) FN(29) FN(30) FN(31)

__device__ __noinline__ float chain(float x) {
  x = f0(x); x = f1(x); x = f2(x); x = f3(x); x = f4(x); x = f5(x); x = f6(x); x = f7(x);
  x = f8(x); x = f9(x); x = f10(x); x = f11(x); x = f12(x); x = f13(x); x = f14(x); x = f15(x);
  x = f16(x); x = f17(x); x = f18(x); x = f19(x); x = f20(x); x = f21(x); x = f22(x); x = f23(x);
  x = f24(x); x = f25(x); x = f26(x); x = f27(x); x = f28(x); x = f29(x); x = f30(x); x = f31(x);
  return x;
}

__global__ void probe(float* out, long long* cyc, float a) {
  float x = a;
  long long t0, t1, t2;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0)::"memory");
  asm volatile("" : "+f"(x)::"memory");
  x = chain(x);
  asm volatile("" : "+f"(x)::"memory");
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1)::"memory");
  x = chain(x);
  asm volatile("" : "+f"(x)::"memory");
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t2)::"memory");
  if (threadIdx.x == 0) {
    out[blockIdx.x] = x;
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
  }
}

template <int N>
__global__ void thrash(float* out, float a) {
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
  char* big;
  cudaMalloc(&big, 256 << 20);
  long long c[2];
  for (int rep = 0; rep < 3; ++rep) {
    thrash<8000><<<148, 32>>>(out, 1.f);
    probe<<<1, 32>>>(out, cyc, 1.f);
    cudaMemcpy(c, cyc, 16, cudaMemcpyDeviceToHost);
    printf("after I$ thrash : cold chain %lld cyc (%.0f/call), warm chain %lld cyc (%.0f/call)\n",
           c[0], c[0] / 32.0, c[1], c[1] / 32.0);
    cudaMemset(big, rep, 256 << 20);  // evict L2 too
    thrash<8000><<<148, 32>>>(out, 1.f);
    probe<<<1, 32>>>(out, cyc, 1.f);
    cudaMemcpy(c, cyc, 16, cudaMemcpyDeviceToHost);
    printf("after L2 flush  : cold chain %lld cyc (%.0f/call), warm chain %lld cyc (%.0f/call)\n",
           c[0], c[0] / 32.0, c[1], c[1] / 32.0);
  }
  return 0;
}
