// tools/tcgen05_mn_major_probe.cu — probe of tcgen05.mma kind::tf32 operand layouts on B200
// (session 5; nvcc -O2 -gencode arch=compute_100a,code=sm_100a; run: ./probe MODE).
//
// Question: can the forward's radial product run as one long-K tcgen05 GEMM per
// query warp, D[channel][query] += rows^T[channel][entry] . w[entry][query]
// (M = 64, N = 32, K = 8 per MMA, accumulator resident in TMEM for the whole
// traversal)? Both operands arrive MN-major (a node's 48 moments are contiguous
// per entry, a warp's 32 weights are contiguous per entry), so it needs the
// instruction descriptor's a_major / b_major = MN.
//
// Result on B200 (driver 580.159, CUDA 12.9), D checked against fp64:
//   MODE 2  both operands K-major, SWIZZLE_128B (the layout tc_gemm.cu and
//           adjoint_tm.cu use): exact; confirms the M = 64 row -> TMEM lane map
//           32 (m / 16) + m % 16.
//   MODE 0, 1  MN-major, no swizzle (either LBO / SBO assignment): accumulator
//           all zero, no error.
//   MODE 3, 4  MN-major, SWIZZLE_128B atoms (8 k-rows x 128 B): all zero.
//   MODE 5  A K-major, only B MN-major SWIZZLE_128B: all zero.
//   MODE 7  MN-major, SWIZZLE_128B_BASE32B (layout type 1: atoms of 4 k-rows x
//           128 B, the 32-byte chunk c of row k stored at c ^ (k & 3); LBO = MN
//           atom stride, SBO = stride of the 4-row k groups): EXACT. This is the
//           layout forward_tm.cu uses. MODE 8 (LBO / SBO swapped) faults.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
#include <stdint.h>
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// no-swizzle descriptor: lbo / sbo in bytes
__device__ __forceinline__ uint64_t desc_ns(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  return d;  // layout type 0
}
__host__ __device__ constexpr uint32_t idesc(int m, int n, int amn, int bmn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)amn << 15) | ((uint32_t)bmn << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
constexpr int M = 64, N = 32, K = 8, KT = 3;  // KT k-steps accumulated
constexpr int CS = 144;                       // core stride (bytes)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
__global__ void kref(const float* A, const float* B, float* D, int mix = 0) {
  __shared__ __align__(1024) uint8_t sa[64 * 128], sb[32 * 128];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int i = tid; i < 64 * 32; i += blockDim.x) {
    int m = i / 32, kk = i % 32;
    float v = kk < KT * K ? A[kk * M + m] : 0.f;
    *reinterpret_cast<float*>(&sa[m * 128 + ((4 * kk) ^ ((m & 7) << 4))]) = v;
  }
  for (int i = tid; i < 32 * 32; i += blockDim.x) {
    int n = i / 32, kk = i % 32;
    float v = kk < KT * K ? B[kk * N + n] : 0.f;
    if (mix == 1)  // MN-major SW128: k-row kk (128 B = 32 n), atoms of 8 k-rows (1024 B)
      *reinterpret_cast<float*>(&sb[(kk / 8) * 1024 + (kk % 8) * 128 + (((n / 4) ^ (kk & 7)) << 4) + (n % 4) * 4]) = v;
    else
      *reinterpret_cast<float*>(&sb[n * 128 + ((4 * kk) ^ ((n & 7) << 4))]) = v;
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_addr(&slot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = slot;
  if (tid == 0) {
    for (int kt = 0; kt < KT; ++kt) {
      uint64_t da = sw128_desc(smem_addr(sa) + 32 * kt), db = sw128_desc(smem_addr(sb) + 32 * kt);
      if (mix == 1) db = sw128_desc(smem_addr(sb) + 1024 * kt);
      uint32_t acc = kt != 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem), "l"(da), "l"(db),
                   "r"(idesc(M, N, 0, mix == 1 ? 1 : 0)), "r"(acc) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_addr(&bar)) : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(done) : "r"(smem_addr(&bar)), "r"(0) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
        "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(tmem + ((uint32_t)(32 * w) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  for (int c = 0; c < 32; ++c) D[(32 * w + lane) * 32 + c] = __uint_as_float(r[c]);
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(32));
}
__device__ __forceinline__ uint64_t desc_mn128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
__global__ void kmn128(const float* A, const float* B, float* D, int variant) {
  __shared__ __align__(1024) uint8_t sa[KT][2048], sb[KT][1024];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int i = tid; i < KT * K * M; i += blockDim.x) {
    int kt = i / (K * M), kk = (i / M) % K, m = i % M;
    int atom = m / 32, c = (m % 32) / 4;
    *reinterpret_cast<float*>(&sa[kt][atom * 1024 + kk * 128 + ((c ^ (kk & 7)) << 4) + (m % 4) * 4]) = A[(kt * K + kk) * M + m];
  }
  for (int i = tid; i < KT * K * N; i += blockDim.x) {
    int kt = i / (K * N), kk = (i / N) % K, n = i % N;
    int c = n / 4;
    *reinterpret_cast<float*>(&sb[kt][kk * 128 + ((c ^ (kk & 7)) << 4) + (n % 4) * 4]) = B[(kt * K + kk) * N + n];
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_addr(&slot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = slot;
  if (tid == 0) {
    for (int kt = 0; kt < KT; ++kt) {
      uint32_t lbo = 1024, sbo = 2048;
      if (variant == 1) { lbo = 2048; sbo = 1024; }
      uint64_t da = desc_mn128(smem_addr(sa[kt]), lbo, sbo), db = desc_mn128(smem_addr(sb[kt]), lbo, sbo);
      uint32_t acc = kt != 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem), "l"(da), "l"(db),
                   "r"(idesc(M, N, 1, 1)), "r"(acc) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_addr(&bar)) : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(done) : "r"(smem_addr(&bar)), "r"(0) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
        "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(tmem + ((uint32_t)(32 * w) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  for (int c = 0; c < 32; ++c) D[(32 * w + lane) * 32 + c] = __uint_as_float(r[c]);
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(32));
}
__global__ void kmn32(const float* A, const float* B, float* D, int variant) {
  __shared__ __align__(1024) uint8_t sa[KT][2048], sb[KT][1024];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int i = tid; i < KT * K * M; i += blockDim.x) {
    int kt = i / (K * M), kk = (i / M) % K, m = i % M;
    int atom = m / 32, c = (m % 32) / 8;
    *reinterpret_cast<float*>(&sa[kt][atom * 1024 + (kk / 4) * 512 + (kk % 4) * 128 + ((c ^ (kk & 3)) << 5) + (m % 8) * 4]) = A[(kt * K + kk) * M + m];
  }
  for (int i = tid; i < KT * K * N; i += blockDim.x) {
    int kt = i / (K * N), kk = (i / N) % K, n = i % N;
    int c = n / 8;
    *reinterpret_cast<float*>(&sb[kt][(kk / 4) * 512 + (kk % 4) * 128 + ((c ^ (kk & 3)) << 5) + (n % 8) * 4]) = B[(kt * K + kk) * N + n];
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_addr(&slot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = slot;
  if (tid == 0) {
    for (int kt = 0; kt < KT; ++kt) {
      uint32_t lbo = 1024, sbo = 512;
      if (variant == 1) { lbo = 512; sbo = 1024; }
      uint64_t da = desc_mn128(smem_addr(sa[kt]), lbo, sbo), db = desc_mn128(smem_addr(sb[kt]), lbo, sbo);
      da = (da & ~((uint64_t)7 << 61)) | ((uint64_t)1 << 61);
      db = (db & ~((uint64_t)7 << 61)) | ((uint64_t)1 << 61);
      uint32_t acc = kt != 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem), "l"(da), "l"(db),
                   "r"(idesc(M, N, 1, 1)), "r"(acc) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_addr(&bar)) : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(done) : "r"(smem_addr(&bar)), "r"(0) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
        "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(tmem + ((uint32_t)(32 * w) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  for (int c = 0; c < 32; ++c) D[(32 * w + lane) * 32 + c] = __uint_as_float(r[c]);
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(32));
}
__global__ void k(const float* A, const float* B, float* D, int swap_lbo_sbo) {
  // A[kk][m] (MN-major: m contiguous), B[kk][n]
  __shared__ __align__(128) uint8_t sa[KT][16 * CS], sb[KT][8 * CS];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int i = tid; i < KT * K * M; i += blockDim.x) {
    int kt = i / (K * M), kk = (i / M) % K, m = i % M;
    *reinterpret_cast<float*>(&sa[kt][(m / 4) * CS + kk * 16 + (m % 4) * 4]) = A[(kt * K + kk) * M + m];
  }
  for (int i = tid; i < KT * K * N; i += blockDim.x) {
    int kt = i / (K * N), kk = (i / N) % K, n = i % N;
    *reinterpret_cast<float*>(&sb[kt][(n / 4) * CS + kk * 16 + (n % 4) * 4]) = B[(kt * K + kk) * N + n];
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_addr(&slot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = slot;
  if (tid == 0) {
    for (int kt = 0; kt < KT; ++kt) {
      uint32_t lbo = 16 * CS, sbo = CS;  // K-group stride (unused: one group), MN core stride
      if (swap_lbo_sbo) { uint32_t t = lbo; lbo = sbo; sbo = t; }
      uint64_t da = desc_ns(smem_addr(sa[kt]), lbo, sbo), db = desc_ns(smem_addr(sb[kt]), lbo, sbo);
      uint32_t acc = kt != 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem), "l"(da), "l"(db),
                   "r"(idesc(M, N, 1, 1)), "r"(acc) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_addr(&bar)) : "memory");
  }
  // wait
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(done) : "r"(smem_addr(&bar)), "r"(0) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  // warp w reads its lane quadrant: 32 lanes x 32 columns
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
        "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(tmem + ((uint32_t)(32 * w) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  for (int c = 0; c < 32; ++c) D[(32 * w + lane) * 32 + c] = __uint_as_float(r[c]);  // D[tmem lane][col]
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(32));
}
int main(int argc, char** argv) {
  int swap = argc > 1 ? atoi(argv[1]) : 0;
  float hA[KT * K * M], hB[KT * K * N], hD[128 * 32];
  srand(1);
  for (auto& v : hA) v = (float)(rand() % 17 - 8) / 4.f;  // tf32-exact values
  for (auto& v : hB) v = (float)(rand() % 13 - 6) / 2.f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, sizeof hD);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, sizeof hD);
  if (swap == 7 || swap == 8) kmn32<<<1, 128>>>(dA, dB, dD, swap - 7); else if (swap == 3 || swap == 4) kmn128<<<1, 128>>>(dA, dB, dD, swap - 3); else if (swap == 2 || swap == 5) kref<<<1, 128>>>(dA, dB, dD, swap == 5); else k<<<1, 128>>>(dA, dB, dD, swap);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
  // expected: D[m][n] = sum_k A[k][m] B[k][n]; M = 64 rows -> tmem lane 32 (m / 16) + m % 16
  int bad = 0; double maxerr = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int kk = 0; kk < KT * K; ++kk) s += (double)hA[kk * M + m] * hB[kk * N + n];
      int lane = 32 * (m / 16) + m % 16;
      double err = fabs(hD[lane * 32 + n] - s);
      if (err > 1e-3) ++bad;
      if (err > maxerr) maxerr = err;
    }
  printf("swap=%d mismatches %d of %d, max err %g; D[0][0..3] = %g %g %g %g\n", swap, bad, M * N, maxerr, hD[0], hD[1], hD[2], hD[3]);
  return 0;
}
