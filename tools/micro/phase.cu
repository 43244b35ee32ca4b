// Cost of the front kernel's vote-rank phase in isolation (512 threads, M=64
// u64 keys in shared memory, 8 parts): rank count + barrier, timed with
// clock64 by thread 0, in a plain CTA and in an 8-CTA cluster, first and
// second execution in the same launch.
#include <cstdio>
#include <cstdint>

__device__ __noinline__ void rank_part(const uint64_t* vkey, int m, int parts, int idx, int* rankp) {
  const int i = idx % m, part = idx / m;
  const uint64_t ki = vkey[i];
  int r = 0;
  const int j0 = (m * part) / parts, j1 = (m * (part + 1)) / parts;
#pragma unroll 4
  for (int j = j0; j < j1; ++j) {
    const uint64_t kj = vkey[j];
    r += (kj > ki) | ((kj == ki) & (j < i));
  }
  rankp[part * m + i] = r;
}

__global__ void __launch_bounds__(512, 1) phase(long long* out, int m) {
  __shared__ uint64_t vkey[256];
  __shared__ int rankp[16 * 256];
  __shared__ uint8_t flag[256];
  const int tid = threadIdx.x;
  if (tid < m) vkey[tid] = (uint64_t)((tid * 2654435761u) & 0xffff) << 20 | tid;
  __syncthreads();
  for (int rep = 0; rep < 3; ++rep) {
    long long t0 = clock64();
    const int parts = 512 / m < 16 ? 512 / m : 16;
    if (tid < parts * m) rank_part(vkey, m, parts, tid, rankp);
    long long t1 = clock64();
    __syncthreads();
    long long t2 = clock64();
    // inline, division-free (m = 64, 8 parts of 8)
    if (tid < 512) {
      const int e = tid & 63, part = tid >> 6;
      const uint64_t ki = vkey[e];
      int r = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = part * 8 + q;
        const uint64_t kj = vkey[j];
        r += (kj > ki) | ((kj == ki) & (j < e));
      }
      rankp[part * 64 + e] = r;
    }
    long long t3 = clock64();
    __syncthreads();
    long long t4 = clock64();
    if (tid == 0 && blockIdx.x == 0) {
      out[rep * 4 + 0] = t1 - t0;
      out[rep * 4 + 1] = t2 - t1;
      out[rep * 4 + 2] = t3 - t2;
      out[rep * 4 + 3] = t4 - t3;
    }
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 64 * 8);
  long long h[16];
  for (int cl = 0; cl < 2; ++cl) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(8);
    lc.blockDim = dim3(512);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl ? 8 : 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    for (int it = 0; it < 2; ++it) {
      cudaLaunchKernelEx(&lc, phase, d, 64);
      cudaDeviceSynchronize();
      cudaMemcpy(h, d, 12 * 8, cudaMemcpyDeviceToHost);
      printf("cluster=%d: rank_part %lld + bar %lld | inline %lld + bar %lld (rep 2: %lld + %lld | %lld + %lld)\n",
             cl ? 8 : 1, h[0], h[1], h[2], h[3], h[8], h[9], h[10], h[11]);
    }
  }
  return 0;
}
