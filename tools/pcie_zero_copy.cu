// PCIe microbenchmark (nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/pcie_zero_copy.cu): kernels reading / writing pinned host rows vs cudaMemcpy. Measured on B200: memcpy 55 GB/s each way, zero-copy row reads 26 GB/s, row writes 18.5 GB/s -> host batches go through copy engines on their own streams (host-async mode), not zero-copy.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
// one warp per 32 rows; row = C floats; lanes = channels -> coalesced row access
__global__ void rd(const float* __restrict__ src, const int* __restrict__ perm, int64_t q, int C, float* sink) {
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; int lane = threadIdx.x & 31;
  float acc = 0;
  for (int r = 0; r < 32; ++r) {
    int64_t s = w * 32 + r; if (s >= q) break;
    int64_t qi = perm ? perm[s] : s;
    for (int c = lane; c < C; c += 32) acc += src[qi * C + c];
  }
  if (acc == 1234.5f) sink[0] = acc;
}
__global__ void wr(float* __restrict__ dst, const int* __restrict__ perm, int64_t q, int C) {
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; int lane = threadIdx.x & 31;
  for (int r = 0; r < 32; ++r) {
    int64_t s = w * 32 + r; if (s >= q) break;
    int64_t qi = perm ? perm[s] : s;
    for (int c = lane; c < C; c += 32) dst[qi * C + c] = (float)c;
  }
}
// lane-per-row scattered 4B writes (what the current kernels do)
__global__ void wr_lane(float* __restrict__ dst, const int* __restrict__ perm, int64_t q, int C) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; if (s >= q) return;
  int64_t qi = perm ? perm[s] : s;
  for (int c = 0; c < C; ++c) dst[qi * C + c] = (float)c;
}
int main() {
  const int64_t q = 4000000; const int C = 49; size_t bytes = q * C * 4;
  float *h, *d, *sink; int *perm;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocDefault));
  CK(cudaMalloc(&d, bytes)); CK(cudaMalloc(&sink, 4)); CK(cudaMalloc(&perm, q * 4));
  std::vector<int> p(q); for (int64_t i = 0; i < q; ++i) p[i] = i; std::shuffle(p.begin(), p.end(), std::mt19937(1));
  CK(cudaMemcpy(perm, p.data(), q * 4, cudaMemcpyHostToDevice));
  memset(h, 0, bytes);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int it = 0; it < 2; ++it) {
    cudaEventRecord(a); CK(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice)); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("memcpy H2D %.2f ms %.1f GB/s\n", ms, bytes / ms / 1e6);
    cudaEventRecord(a); CK(cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost)); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("memcpy D2H %.2f ms %.1f GB/s\n", ms, bytes / ms / 1e6);
    for (int pm = 0; pm < 2; ++pm) {
      const int* pp = pm ? perm : nullptr;
      int blocks = (int)((q / 32 + 7) / 8);
      cudaEventRecord(a); rd<<<blocks, 256>>>(h, pp, q, C, sink); cudaEventRecord(b); CK(cudaEventSynchronize(b));
      cudaEventElapsedTime(&ms, a, b); printf("zc read rows perm=%d %.2f ms %.1f GB/s\n", pm, ms, bytes / ms / 1e6);
      cudaEventRecord(a); wr<<<blocks, 256>>>(h, pp, q, C); cudaEventRecord(b); CK(cudaEventSynchronize(b));
      cudaEventElapsedTime(&ms, a, b); printf("zc write rows perm=%d %.2f ms %.1f GB/s\n", pm, ms, bytes / ms / 1e6);
      cudaEventRecord(a); wr_lane<<<(q + 255) / 256, 256>>>(h, pp, q, C); cudaEventRecord(b); CK(cudaEventSynchronize(b));
      cudaEventElapsedTime(&ms, a, b); printf("zc write lane-rows perm=%d %.2f ms %.1f GB/s\n", pm, ms, bytes / ms / 1e6);
      cudaEventRecord(a); wr_lane<<<(q + 255) / 256, 256>>>(d, pp, q, C); cudaEventRecord(b); CK(cudaEventSynchronize(b));
      cudaEventElapsedTime(&ms, a, b); printf("dev write lane-rows perm=%d %.2f ms %.1f GB/s\n", pm, ms, bytes / ms / 1e6);
      cudaEventRecord(a); wr<<<blocks, 256>>>(d, pp, q, C); cudaEventRecord(b); CK(cudaEventSynchronize(b));
      cudaEventElapsedTime(&ms, a, b); printf("dev write rows perm=%d %.2f ms %.1f GB/s\n", pm, ms, bytes / ms / 1e6);
    }
  }
  return 0;
}
