// Host <-> device activation transfer options for the host-buffer entry
// (128 KB of bf16 x in, 256 KB of fp32 y out, C2 shape), timed with CUDA
// events behind a spin kernel (device time only):
//   in : bulk copies (G CTAs x one request of C bytes, or several in flight),
//        16-byte loads (G CTAs x T threads x U loads in flight), cudaMemcpyAsync
//   out: 16-byte stores from G CTAs, bulk smem -> host stores, cudaMemcpyAsync
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hostio hostio.cu
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

__global__ void spin(long long cyc) {
  long long t0 = clock64();
  while (clock64() - t0 < cyc) {
  }
}

__device__ inline uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// G CTAs; CTA b copies [b*chunk, (b+1)*chunk) as `sub`-byte bulk requests all in flight
__global__ void bulk_in(const unsigned char* src, unsigned char* dst, int total, int chunk, int sub) {
  extern __shared__ __align__(128) unsigned char buf[];
  __shared__ __align__(8) uint64_t bar;
  const int off = blockIdx.x * chunk;
  if (threadIdx.x != 0 || off >= total) return;
  const int bytes = min(chunk, total - off);
  asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bar)));
  asm volatile("fence.mbarrier_init.release.cluster;");
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes));
  for (int o = 0; o < bytes; o += sub) {
    const int b = min(sub, bytes - o);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            su32(buf + o)),
        "l"(src + off + o), "r"(b), "r"(su32(&bar))
        : "memory");
  }
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(
          su32(&bar)));
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off),
               "r"(su32(buf)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;");
  asm volatile("cp.async.bulk.wait_group 0;");
}

template <int U>
__global__ void ld_in(const uint4* src, uint4* dst, int n16) {
  const int stride = gridDim.x * blockDim.x;
  const int i0 = blockIdx.x * blockDim.x + threadIdx.x;
  uint4 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (i0 + u * stride < n16) v[u] = __ldcv(src + i0 + u * stride);
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (i0 + u * stride < n16) dst[i0 + u * stride] = v[u];
}

// contiguous per-thread runs (adjacent 16 B pieces of one 64..256 B line per thread)
template <int U>
__global__ void ld_in_run(const uint4* src, uint4* dst, int n16) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int i0 = t * U;
  uint4 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (i0 + u < n16) v[u] = __ldcv(src + i0 + u);
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (i0 + u < n16) dst[i0 + u] = v[u];
}

__global__ void st_out(const uint4* src, uint4* dst, int n16) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x)
    __stcs(dst + i, src[i]);
}

__global__ void bulk_out(const unsigned char* src, unsigned char* dst, int total, int chunk) {
  extern __shared__ __align__(128) unsigned char buf[];
  const int off = blockIdx.x * chunk;
  if (off >= total) return;
  const int bytes = min(chunk, total - off);
  for (int i = threadIdx.x * 16; i < bytes; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(buf + i) = *reinterpret_cast<const uint4*>(src + off + i);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off),
                 "r"(su32(buf)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;");
    asm volatile("cp.async.bulk.wait_group 0;");
  }
}

template <class F>
static float timeit(cudaStream_t st, F launch, int reps = 200) {
  std::vector<float> t;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int r = 0; r < reps + 10; ++r) {
    spin<<<1, 1, 0, st>>>(40000);
    cudaEventRecord(e0, st);
    launch();
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 10) t.push_back(ms * 1e3f);
  }
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}

int main() {
  const int xin = 32 * 2048 * 2, yout = 32 * 2048 * 4;
  unsigned char *hx, *hy, *dx, *dy, *hxd, *hyd;
  cudaHostAlloc(&hx, xin, cudaHostAllocMapped);
  cudaHostAlloc(&hy, yout, cudaHostAllocMapped);
  cudaHostGetDevicePointer(reinterpret_cast<void**>(&hxd), hx, 0);
  cudaHostGetDevicePointer(reinterpret_cast<void**>(&hyd), hy, 0);
  cudaMalloc(&dx, xin);
  cudaMalloc(&dy, yout);
  for (int i = 0; i < xin; ++i) hx[i] = static_cast<unsigned char>(i * 7);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaFuncSetAttribute(bulk_in, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(bulk_out, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  printf("empty kernel: %.2f us\n", timeit(st, [&] { spin<<<1, 1, 0, st>>>(0); }));
  printf("memcpy H2D 128K: %.2f us\n",
         timeit(st, [&] { cudaMemcpyAsync(dx, hx, xin, cudaMemcpyHostToDevice, st); }));
  printf("memcpy D2H 256K: %.2f us\n",
         timeit(st, [&] { cudaMemcpyAsync(hy, dy, yout, cudaMemcpyDeviceToHost, st); }));
  for (int chunk : {2048, 4096, 8192, 16384, 32768, 65536, 131072})
    for (int sub : {1024, 4096, 16384, 131072}) {
      if (sub > chunk && sub != 131072) continue;
      const int g = (xin + chunk - 1) / chunk;
      const int s = std::min(sub, chunk);
      printf("bulk_in chunk %6d sub %6d (G=%3d): %.2f us\n", chunk, s, g,
             timeit(st, [&] { bulk_in<<<g, 32, chunk, st>>>(hxd, dx, xin, chunk, s); }));
    }
  const int n16 = xin / 16;
  for (int g : {8, 32, 64, 148}) {
    for (int t : {64, 256}) {
      printf("ld_in U=1 G=%3d T=%3d: %.2f us\n", g, t,
             timeit(st, [&] { ld_in<1><<<g, t, 0, st>>>(reinterpret_cast<uint4*>(hxd),
                                                         reinterpret_cast<uint4*>(dx), n16); }));
      printf("ld_in U=4 G=%3d T=%3d: %.2f us\n", g, t,
             timeit(st, [&] { ld_in<4><<<g, t, 0, st>>>(reinterpret_cast<uint4*>(hxd),
                                                         reinterpret_cast<uint4*>(dx), n16); }));
    }
  }
  for (int u : {4, 8, 16}) {
    const int threads = (n16 + u - 1) / u;
    for (int t : {32, 128}) {
      const int g = (threads + t - 1) / t;
      if (u == 4)
        printf("ld_in_run U=%d G=%d T=%d: %.2f us\n", u, g, t,
               timeit(st, [&] { ld_in_run<4><<<g, t, 0, st>>>(reinterpret_cast<uint4*>(hxd),
                                                               reinterpret_cast<uint4*>(dx), n16); }));
      if (u == 8)
        printf("ld_in_run U=%d G=%d T=%d: %.2f us\n", u, g, t,
               timeit(st, [&] { ld_in_run<8><<<g, t, 0, st>>>(reinterpret_cast<uint4*>(hxd),
                                                               reinterpret_cast<uint4*>(dx), n16); }));
      if (u == 16)
        printf("ld_in_run U=%d G=%d T=%d: %.2f us\n", u, g, t,
               timeit(st, [&] { ld_in_run<16><<<g, t, 0, st>>>(reinterpret_cast<uint4*>(hxd),
                                                                reinterpret_cast<uint4*>(dx), n16); }));
    }
  }
  const int y16 = yout / 16;
  for (int g : {16, 64, 148, 296})
    printf("st_out G=%3d T=256: %.2f us\n", g,
           timeit(st, [&] { st_out<<<g, 256, 0, st>>>(reinterpret_cast<uint4*>(dy),
                                                       reinterpret_cast<uint4*>(hyd), y16); }));
  for (int chunk : {4096, 16384, 65536}) {
    const int g = (yout + chunk - 1) / chunk;
    printf("bulk_out chunk %6d (G=%3d): %.2f us\n", chunk, g,
           timeit(st, [&] { bulk_out<<<g, 256, chunk, st>>>(dy, hyd, yout, chunk); }));
  }
  printf("check %d\n", static_cast<int>(cudaGetLastError()));
  return 0;
}
