// tc_gemm.cu — tcgen05 / TMEM GEMM (see tc_gemm.cuh).
//
// One CTA of 4 warps computes a 128 x BN tile of D (BN <= 128; TMEM holds D
// and two A stages in 256 columns, so two CTAs share an SM). K is walked in
// chunks of 32 tf32, double-buffered, the next chunk's A loads in flight
// during the current chunk's MMAs:
//   * A (M = 128 rows): each thread owns one tile row (= one TMEM lane of its
//     warp's quadrant), loads its 32 values of the chunk, splits them into
//     tf32 hi / lo and writes both straight into TMEM (tcgen05.st) — the MMA
//     reads A from tensor memory, so A never occupies shared memory bandwidth;
//   * B (N = BN rows): either a pre-split, pre-swizzled image in global memory
//     (the MLP's weights, built once per head) fetched with one bulk async copy
//     (cp.async.bulk, mbarrier transaction count) per chunk, or staged by the
//     threads (split + swizzle, the weight-gradient GEMM's activations);
//   * one thread issues the chunk's 12 MMAs (M = 128, N = BN, K = 8,
//     kind::tf32; hi.hi + hi.lo + lo.hi per k-step) and commits them to the
//     stage's mbarrier, which frees the stage two chunks later.
// The fp32 accumulator (128 lanes x BN columns of TMEM) is read back by the
// warp owning each lane quadrant (tcgen05.ld 32x32b) for the fused epilogue.
#include <algorithm>
#include <cstdlib>
#include <atomic>

#include "dpl_internal.cuh"
#include "tc_gemm.cuh"

namespace dpl {

namespace {

constexpr int kTileM = 128;
constexpr int kChunkK = 32;            // tf32 elements per swizzle row (128 B)
constexpr int kRowBytes = kChunkK * 4;  // 128
constexpr uint32_t kTmemA = 128;  // A stages: columns 128 + 64 s (hi), + 32 (lo), after D (<= 128)

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// K-major SWIZZLE_128B shared-memory matrix descriptor (tcgen05): 8-row core
// groups of 8 x 128 B = 1024 B (SBO), the 16-byte chunks of row r permuted by
// XOR (r & 7); start address in 16-byte units; bit 46 = descriptor version 1
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;            // LBO (not used by swizzled K-major layouts)
  d |= (uint64_t)(1024u >> 4) << 32;  // SBO: next 8-row group
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;  // SWIZZLE_128B
  return d;
}

// instruction descriptor, kind::tf32: D fp32, A / B tf32, both K-major
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

// D[tmem] (+)= A[tmem] . B[smem]
__device__ __forceinline__ void mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   bar)
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %0;\n" ::"r"(bytes), "r"(bar)
               : "memory");
}

__device__ __forceinline__ void bulk_copy(uint32_t dst, const void* src, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]),
      "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]),
      "r"(r[30]), "r"(r[31])
      : "memory");
}

// swizzled byte offset of element (row, k) in a [rows][32] tf32 K-major tile
__host__ __device__ __forceinline__ uint32_t sw_off(int row, int k) {
  return (uint32_t)row * kRowBytes + ((uint32_t)(((k >> 2) ^ (row & 7)) << 4)) +
         ((uint32_t)(k & 3) << 2);
}

__device__ __forceinline__ uint32_t tf32_hi(float x) { return __float_as_uint(x) & 0xffffe000u; }

// threads stage rows [r0, r0 + ROWS) x k-chunk [k0, k0 + 32) of B (split + swizzle)
template <int ROWS, bool KCONTIG>
__device__ __forceinline__ void stage_b(const float* __restrict__ X, int64_t ld, int nrows, int r0,
                                        int kend, int k0, uint8_t* hi, uint8_t* lo, int tid) {
  constexpr int PER = ROWS * kChunkK / 128;
  if constexpr (!KCONTIG && ROWS % 32 == 0) {
    // B[k][n] (n contiguous, the weight-gradient GEMM's activations). A warp
    // covers 8 consecutive rows x 4 consecutive k per step: 32-byte row segments
    // of 4 k-lines from global memory, and 32 distinct banks in the swizzled
    // tile (row r's 16-byte chunk is XORed with r & 7, k & 3 picks the word; 32
    // consecutive rows at one k would hit every bank four times). Step i of
    // warp w: row octet w + 4 (i % (ROWS / 32)), k quad i / (ROWS / 32) — all
    // compile-time but the lane part, so a full tile needs one pointer, one
    // shared-memory base and immediate offsets.
    if (r0 + ROWS <= nrows && k0 + kChunkK <= kend) {
      constexpr int RO = ROWS / 32;  // row-octet steps per k quad
      const int w = tid >> 5, ln = tid & 31;
      const int rl = 8 * w + (ln & 7), kl = ln >> 3;
      const float* src = X + (int64_t)(k0 + kl) * ld + (r0 + rl);
      const uint32_t ob = (uint32_t)rl * kRowBytes + ((uint32_t)kl << 2);
      const uint32_t sw = (uint32_t)(ln & 7);
      float x[PER];
#pragma unroll
      for (int i = 0; i < PER; ++i) x[i] = __ldg(src + (int64_t)(4 * (i / RO)) * ld + 32 * (i % RO));
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const uint32_t o = ob + (uint32_t)(32 * (i % RO)) * kRowBytes + ((((uint32_t)(i / RO)) ^ sw) << 4);
        const uint32_t h = tf32_hi(x[i]);
        *reinterpret_cast<uint32_t*>(hi + o) = h;
        *reinterpret_cast<float*>(lo + o) = x[i] - __uint_as_float(h);
      }
      return;
    }
  }
#pragma unroll 8
  for (int i = 0; i < PER; ++i) {
    const int idx = tid + 128 * i;
    int r, k;
    if (KCONTIG) {
      r = idx >> 5, k = idx & 31;  // a warp reads 32 consecutive k of one row
    } else {
      const int blk = idx >> 5, ln = idx & 31;  // 8 rows x 4 k per warp step (see above)
      r = (blk % (ROWS / 8)) * 8 + (ln & 7);
      k = (blk / (ROWS / 8)) * 4 + (ln >> 3);
    }
    const int gr = r0 + r, gk = k0 + k;
    float x = 0.f;
    if (gr < nrows && gk < kend)
      x = KCONTIG ? __ldg(X + (int64_t)gr * ld + gk) : __ldg(X + (int64_t)gk * ld + gr);
    const uint32_t h = tf32_hi(x), o = sw_off(r, k);
    *reinterpret_cast<uint32_t*>(hi + o) = h;
    *reinterpret_cast<float*>(lo + o) = x - __uint_as_float(h);
  }
}

// this thread's A row (global row gr) for k-chunk [k0, k0 + 32), raw fp32
// (zero beyond M / K); issued a chunk ahead of its use so the load latency
// overlaps the previous chunk's MMAs
template <bool AK>
__device__ __forceinline__ void load_a(const TcGemm& g, int gr, int k0, int kend, bool vec,
                                       float (&x)[32]) {
  if (AK) {
    const float* src = g.A + (int64_t)gr * g.lda + k0;
    if (gr < g.M && vec && k0 + 32 <= kend) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(src) + j);
        x[4 * j] = v.x, x[4 * j + 1] = v.y, x[4 * j + 2] = v.z, x[4 * j + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] = (gr < g.M && k0 + j < kend) ? __ldg(src + j) : 0.f;
    }
  } else {  // A[k][m]: consecutive threads read consecutive m at each k (coalesced)
    const int64_t ld = g.lda;
    const float* src = g.A + (int64_t)k0 * ld + gr;
    if (gr < g.M && k0 + 32 <= kend) {  // full chunk: one pointer, strided loads
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] = __ldg(src + j * ld);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] = (gr < g.M && k0 + j < kend) ? __ldg(src + j * ld) : 0.f;
    }
  }
}

// split a chunk into tf32 hi / lo and write both into this thread's TMEM lane
__device__ __forceinline__ void store_a(uint32_t ta, const float (&x)[32]) {
  uint32_t hi[32], lo[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    hi[j] = tf32_hi(x[j]);
    lo[j] = __float_as_uint(x[j] - __uint_as_float(hi[j]));
  }
  tmem_st32(ta, hi);
  tmem_st32(ta + 32u, lo);
}

// BIMG: B comes from a pre-split image (bulk copies), else threads stage it
template <int BN, bool AK, bool BIMG, bool BK, int EPI>
__global__ void __launch_bounds__(128, 2) k_tc_gemm(TcGemm g) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  constexpr int BBYTES = BN * kRowBytes;  // one part (hi or lo) of a B chunk
  constexpr int STAGE = 2 * BBYTES;
  __shared__ __align__(8) uint64_t full[2], done[2];
  __shared__ uint32_t tmem_slot;
  // TMEM: D (BN <= 128 columns) + two A stages (2 x 64): 256 columns, so two
  // CTAs share an SM (one's prologue / epilogue overlaps the other's MMAs)
  constexpr uint32_t kTmemCols = 256;
  static_assert(BN <= 128, "D must fit below the A stages");

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // N tiles vary fastest: the CTAs sharing an A row block run together (A is
  // read from DRAM once)
  const int ntiles = (g.N + BN - 1) / BN;
  const int nt = (int)(blockIdx.x % ntiles), mt = (int)(blockIdx.x / ntiles);
  const int m0 = mt * kTileM, n0 = nt * BN;
  int kb = 0, ke = g.K;
  if (EPI == TC_ACC64) {
    const int per = (((g.K + gridDim.z - 1) / gridDim.z) + kChunkK - 1) / kChunkK * kChunkK;
    kb = blockIdx.z * per;
    ke = min(g.K, kb + per);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_addr(&tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) mbar_init(smem_addr(&full[i]), 1), mbar_init(smem_addr(&done[i]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  constexpr uint32_t IDESC = idesc_tf32(kTileM, BN);
  const int row = 32 * warp + lane, gr = m0 + row;
  const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
  const bool vec = AK && (g.lda & 3) == 0 && ((reinterpret_cast<uintptr_t>(g.A) & 15) == 0);
  const int nkc_total = (g.K + kChunkK - 1) / kChunkK;  // chunks per image column block
  const bool vec_d = EPI != TC_ACC64 && (g.ldd & 3) == 0 &&
                     ((reinterpret_cast<uintptr_t>(g.D) & 15) == 0) &&
                     (EPI != TC_GATE || ((g.ldaux & 3) == 0 && (reinterpret_cast<uintptr_t>(g.aux) & 15) == 0));

  const int nchunks = ke > kb ? (ke - kb + kChunkK - 1) / kChunkK : 0;
  float xa[32];  // the next chunk's A values, in flight during the current MMAs
  double bsum = 0.0;  // TC_ACC64 with bias_grad: this row's sum of A (delta) values
  // K-contiguous A with 16-byte rows: coalesced cp.async of the chunk into a
  // swizzled fp32 staging tile (a warp moves 4 rows x 128 B), then each thread
  // reads its own row back conflict-free (8 x LDS.128); otherwise direct loads
  uint8_t* astage = sm + 2 * STAGE;  // 2 x 16 KB
  auto issue_a = [&](int cidx) {
    const int k0c = kb + cidx * kChunkK;
    uint8_t* dst0 = astage + (cidx & 1) * (kTileM * kRowBytes);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int idx = tid + 128 * i, r = idx >> 3, j = idx & 7;
      const int grr = m0 + r, gk = k0c + 4 * j;
      const int bytes = grr < g.M ? max(0, min(16, (ke - gk) * 4)) : 0;
      const float* src = bytes ? g.A + (int64_t)grr * g.lda + gk : g.A;
      const uint32_t dst = smem_addr(dst0 + r * kRowBytes + ((j ^ (r & 7)) << 4));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  const bool smem_a = AK && vec;
  if (nchunks > 0) {
    if (smem_a)
      issue_a(0);
    else
      load_a<AK>(g, gr, kb, ke, vec, xa);
  }
  for (int c = 0; c < nchunks; ++c) {
    const int s = c & 1;
    uint8_t* bhi = sm + s * STAGE;
    uint8_t* blo = bhi + BBYTES;
    const int k0 = kb + c * kChunkK;
    if (c >= 2) mbar_wait(smem_addr(&done[s]), ((c - 2) >> 1) & 1);  // chunk c-2 freed stage s
    if (BIMG) {
      if (tid == 0) {
        const uint8_t* src = g.b_image + ((size_t)nt * nkc_total + k0 / kChunkK) * STAGE;
        mbar_expect_tx(smem_addr(&full[s]), STAGE);
        bulk_copy(smem_addr(bhi), src, STAGE, smem_addr(&full[s]));
      }
    } else {
      stage_b<BN, BK>(g.B, g.ldb, g.N, n0, ke, k0, bhi, blo, tid);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic -> async proxy
    }
    if (smem_a) {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      __syncthreads();  // chunk c's tile, copied by every thread, is complete
      if (c + 1 < nchunks) issue_a(c + 1);  // the other staging tile was read last chunk
      const uint8_t* src = astage + (c & 1) * (kTileM * kRowBytes) + row * kRowBytes;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 v = *reinterpret_cast<const float4*>(src + ((j ^ (row & 7)) << 4));
        xa[4 * j] = v.x, xa[4 * j + 1] = v.y, xa[4 * j + 2] = v.z, xa[4 * j + 3] = v.w;
      }
    }
    {
      if (EPI == TC_ACC64 && g.bias_grad) {
#pragma unroll
        for (int j = 0; j < 32; ++j) bsum += (double)xa[j];
      }
      store_a(tmem + lane_base + kTmemA + 64u * s, xa);
      if (!smem_a && c + 1 < nchunks) load_a<AK>(g, gr, k0 + kChunkK, ke, vec, xa);
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      if (BIMG) mbar_wait(smem_addr(&full[s]), (c >> 1) & 1);
      tc_fence_after();
      const uint32_t b_hi = smem_addr(bhi), b_lo = smem_addr(blo);
      const uint32_t a_hi = tmem + kTmemA + 64u * s, a_lo = a_hi + 32u;
#pragma unroll
      for (int ks = 0; ks < kChunkK / 8; ++ks) {  // k-step of 8 tf32: 8 TMEM columns, 32 B of B rows
        mma_ts(tmem, a_hi + 8u * ks, sw128_desc(b_hi + 32u * ks), IDESC, (c | ks) != 0);
        mma_ts(tmem, a_hi + 8u * ks, sw128_desc(b_lo + 32u * ks), IDESC, 1u);
        mma_ts(tmem, a_lo + 8u * ks, sw128_desc(b_hi + 32u * ks), IDESC, 1u);
      }
      mma_commit(smem_addr(&done[s]));
    }
  }
  if (nchunks > 0) {
    const int last = nchunks - 1;
    mbar_wait(smem_addr(&done[last & 1]), (last >> 1) & 1);  // every earlier MMA completed too
  }
  tc_fence_after();

  // epilogue: warp w owns TMEM lanes (= tile rows) 32w .. 32w + 31
  const bool row_ok = gr < g.M;
#pragma unroll 1
  for (int cb = 0; cb < BN; cb += 16) {
    float v[16];
    if (nchunks > 0) {
      tmem_ld16(tmem + lane_base + (uint32_t)cb, v);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = 0.f;
    }
    if (!row_ok) continue;
    const int nb = n0 + cb;
    if (EPI != TC_ACC64 && vec_d && nb + 16 <= g.N) {  // full 16-column group: 4 x 16-byte stores
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float x = v[j];
        if (EPI == TC_BIAS_RELU) x = fmaxf(x + __ldg(g.bias + nb + j), 0.f);
        if (EPI == TC_BIAS) x += __ldg(g.bias + nb + j);
        v[j] = x;
      }
      if (EPI == TC_GATE) {  // ReLU backward: the gate row as 4 x 16-byte loads
        const float4* ax = reinterpret_cast<const float4*>(g.aux + (int64_t)gr * g.ldaux + nb);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 a4 = __ldg(ax + j);
          v[4 * j] = a4.x > 0.f ? v[4 * j] : 0.f;
          v[4 * j + 1] = a4.y > 0.f ? v[4 * j + 1] : 0.f;
          v[4 * j + 2] = a4.z > 0.f ? v[4 * j + 2] : 0.f;
          v[4 * j + 3] = a4.w > 0.f ? v[4 * j + 3] : 0.f;
        }
      }
      float4* dst = reinterpret_cast<float4*>(g.D + (int64_t)gr * g.ldd + nb);
#pragma unroll
      for (int j = 0; j < 4; ++j) dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      continue;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int n = nb + j;
      if (n >= g.N) break;
      float x = v[j];
      if (EPI == TC_BIAS_RELU) x = fmaxf(x + __ldg(g.bias + n), 0.f);
      if (EPI == TC_BIAS) x += __ldg(g.bias + n);
      if (EPI == TC_GATE) x = __ldg(g.aux + (int64_t)gr * g.ldaux + n) > 0.f ? x : 0.f;
      if (EPI == TC_ACC64) {
        if (x != 0.f) atomicAdd(g.D64 + (int64_t)gr * g.ldd + n, (double)x);
      } else {
        g.D[(int64_t)gr * g.ldd + n] = x;
      }
    }
  }
  if (EPI == TC_ACC64 && g.bias_grad && nt == 0 && row_ok && bsum != 0.0)
    atomicAdd(g.bias_grad + gr, bsum);
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(kTmemCols)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}

// ---------------------------------------------------------------------------
// Persistent, warp-specialised variant for K-contiguous A and a pre-split B
// image (the MLP head's forward and input-gradient GEMMs). One CTA per SM
// walks the tiles round-robin:
//   warps 0-7  A producers in two sets of 4 warps taking alternate chunks:
//              cp.async of the chunk into the set's swizzled fp32 staging ring
//              (the set's next chunk in flight), split into tf32 hi / lo,
//              tcgen05.st into one of 4 TMEM A stages (warps w, w + 4 -> lanes
//              32w..); the set's thread 0 also issues the chunk's B bulk copy;
//   warp 12    MMA issuer (one thread): 12 tcgen05.mma per chunk into one of two
//              TMEM accumulators, commit -> stage free; after a tile's last
//              chunk, commit -> accumulator full;
//   warps 8-11 epilogue: tcgen05.ld of the finished accumulator (warp 8 + q ->
//              lane quadrant q), fused bias / ReLU / gate, stores, release.
// The epilogue of tile i and the producers of tile i + 1 run while the tensor
// core works, so per-tile fixed costs (TMEM allocation, barrier setup, the
// first loads, the drain) are paid once per SM instead of once per tile.
// TMEM: accumulators 2 x BN (<= 256) + A stages 4 x 64 = 512 columns.
constexpr int kWsStages = 4;
constexpr int kWsRing = 2;  // per producer set: A staging ring (prefetch distance 1)
constexpr int kWsThreads = 13 * 32;

template <int BN, int EPI>
__global__ void __launch_bounds__(kWsThreads, 1) k_tc_gemm_ws(TcGemm g) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  constexpr int BBYTES = BN * kRowBytes;
  constexpr int STAGEB = 2 * BBYTES;
  constexpr int ABYTES = kTileM * kRowBytes;
  uint8_t* bst = sm;                          // kWsStages x (hi | lo)
  uint8_t* ast = sm + kWsStages * STAGEB;     // 2 sets x kWsRing x raw fp32 A chunk
  __shared__ __align__(8) uint64_t afull[kWsStages], bfull[kWsStages], empty[kWsStages],
      dfull[2], dempty[2];
  __shared__ uint32_t tmem_slot;
  constexpr uint32_t TM_A = 256;  // A stages at columns 256 + 64 s (hi), + 32 (lo)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_addr(&tmem_slot)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  if (tid == 0) {
    for (int i = 0; i < kWsStages; ++i) {
      mbar_init(smem_addr(&afull[i]), 128);
      mbar_init(smem_addr(&bfull[i]), 1);
      mbar_init(smem_addr(&empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) mbar_init(smem_addr(&dfull[i]), 1), mbar_init(smem_addr(&dempty[i]), 128);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  const int mtiles = (g.M + kTileM - 1) / kTileM, ntiles = (g.N + BN - 1) / BN;
  const int ntotal = mtiles * ntiles;
  const int nkc = (g.K + kChunkK - 1) / kChunkK;  // chunks per tile (K > 0)

  if (warp < 8) {
    // ---------------- A producers (+ B bulk copies): two sets of 4 warps take
    // alternate chunks (set = warp / 4; warps w and w + 4 share lane quadrant w)
    const int set = warp >> 2, ptid = tid & 127;
    const int row = ptid;  // tile row = TMEM lane of quadrant warp % 4
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    uint8_t* ring = ast + set * kWsRing * ABYTES;
    // (tile, chunk) cursors over this set's chunks: every second chunk of the
    // CTA's sequence, starting at chunk `set`
    struct Cursor {
      int t, c;
    };
    auto step = [&](Cursor& k) {
      if (++k.c == nkc) k.c = 0, k.t += gridDim.x;
    };
    Cursor pf{(int)blockIdx.x, 0};
    if (set) step(pf);
    Cursor cs = pf;
    int pf_n = 0;  // chunks issued so far by this set
    auto issue = [&]() {
      if (pf.t < ntotal) {
        const int m0 = (pf.t / ntiles) * kTileM, k0 = pf.c * kChunkK;
        uint8_t* dst0 = ring + (pf_n % kWsRing) * ABYTES;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int idx = ptid + 128 * i, r = idx >> 3, j = idx & 7;
          const int grr = m0 + r, gk = k0 + 4 * j;
          const int bytes = grr < g.M ? max(0, min(16, (g.K - gk) * 4)) : 0;
          const float* src = bytes ? g.A + (int64_t)grr * g.lda + gk : g.A;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                           smem_addr(dst0 + r * kRowBytes + ((j ^ (r & 7)) << 4))),
                       "l"(src), "r"(bytes)
                       : "memory");
        }
        step(pf);
        step(pf);
      }
      ++pf_n;
      asm volatile("cp.async.commit_group;\n" ::: "memory");  // (possibly empty) group
    };
    issue();  // prefetch distance 1 within the set (2 chunks of the CTA's sequence)
    for (int n = 0; cs.t < ntotal; ++n) {
      const int gc = 2 * n + set;
      const int s = gc % kWsStages;
      const uint32_t ph = (uint32_t)(gc / kWsStages) & 1u;
      mbar_wait(smem_addr(&empty[s]), ph ^ 1u);  // the MMAs of chunk gc - 4 are done
      if (ptid == 0) {
        const uint8_t* src = g.b_image + ((size_t)(cs.t % ntiles) * nkc + cs.c) * STAGEB;
        mbar_expect_tx(smem_addr(&bfull[s]), STAGEB);
        bulk_copy(smem_addr(bst + s * STAGEB), src, STAGEB, smem_addr(&bfull[s]));
      }
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");  // this set's chunk n has landed
      asm volatile("bar.sync %0, 128;\n" ::"r"(1 + set) : "memory");  // ... everyone's; slot n-1 read
      issue();
      const uint8_t* src = ring + (n % kWsRing) * ABYTES + row * kRowBytes;
      float x[32];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 v = *reinterpret_cast<const float4*>(src + ((j ^ (row & 7)) << 4));
        x[4 * j] = v.x, x[4 * j + 1] = v.y, x[4 * j + 2] = v.z, x[4 * j + 3] = v.w;
      }
      store_a(tmem + lane_base + TM_A + 64u * s, x);
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      tc_fence_before();
      mbar_arrive(smem_addr(&afull[s]));
      step(cs);
      step(cs);
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  } else if (warp == 12) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC = idesc_tf32(kTileM, BN);
      int gc = 0, i = 0;
      for (int t = blockIdx.x; t < ntotal; t += gridDim.x, ++i) {
        const int b = i & 1;
        mbar_wait(smem_addr(&dempty[b]), ((uint32_t)(i >> 1) & 1u) ^ 1u);  // epilogue drained it
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(b * BN);
        for (int c = 0; c < nkc; ++c, ++gc) {
          const int s = gc % kWsStages;
          const uint32_t ph = (uint32_t)(gc / kWsStages) & 1u;
          mbar_wait(smem_addr(&afull[s]), ph);
          mbar_wait(smem_addr(&bfull[s]), ph);
          tc_fence_after();
          const uint32_t b_hi = smem_addr(bst + s * STAGEB), b_lo = b_hi + BBYTES;
          const uint32_t a_hi = tmem + TM_A + 64u * s, a_lo = a_hi + 32u;
#pragma unroll
          for (int ks = 0; ks < kChunkK / 8; ++ks) {
            mma_ts(d, a_hi + 8u * ks, sw128_desc(b_hi + 32u * ks), IDESC, (c | ks) != 0);
            mma_ts(d, a_hi + 8u * ks, sw128_desc(b_lo + 32u * ks), IDESC, 1u);
            mma_ts(d, a_lo + 8u * ks, sw128_desc(b_hi + 32u * ks), IDESC, 1u);
          }
          mma_commit(smem_addr(&empty[s]));
        }
        mma_commit(smem_addr(&dfull[b]));
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue (warps 8-11 -> lane quadrants 0-3)
    const int q = warp - 8;
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    const bool vec_d = (g.ldd & 3) == 0 && ((reinterpret_cast<uintptr_t>(g.D) & 15) == 0) &&
                       (EPI != TC_GATE || ((g.ldaux & 3) == 0 &&
                                           (reinterpret_cast<uintptr_t>(g.aux) & 15) == 0));
    int i = 0;
    for (int t = blockIdx.x; t < ntotal; t += gridDim.x, ++i) {
      const int b = i & 1;
      const int m0 = (t / ntiles) * kTileM, n0 = (t % ntiles) * BN;
      const int gr = m0 + 32 * q + lane;
      mbar_wait(smem_addr(&dfull[b]), (uint32_t)(i >> 1) & 1u);
      tc_fence_after();
#pragma unroll 1
      for (int cb = 0; cb < BN; cb += 16) {
        float v[16];
        tmem_ld16(tmem + lane_base + (uint32_t)(b * BN + cb), v);
        if (gr >= g.M) continue;
        const int nb = n0 + cb;
        if (vec_d && nb + 16 <= g.N) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float x = v[j];
            if (EPI == TC_BIAS_RELU) x = fmaxf(x + __ldg(g.bias + nb + j), 0.f);
            if (EPI == TC_BIAS) x += __ldg(g.bias + nb + j);
            v[j] = x;
          }
          if (EPI == TC_GATE) {
            const float4* ax = reinterpret_cast<const float4*>(g.aux + (int64_t)gr * g.ldaux + nb);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float4 a4 = __ldg(ax + j);
              v[4 * j] = a4.x > 0.f ? v[4 * j] : 0.f;
              v[4 * j + 1] = a4.y > 0.f ? v[4 * j + 1] : 0.f;
              v[4 * j + 2] = a4.z > 0.f ? v[4 * j + 2] : 0.f;
              v[4 * j + 3] = a4.w > 0.f ? v[4 * j + 3] : 0.f;
            }
          }
          float4* dst = reinterpret_cast<float4*>(g.D + (int64_t)gr * g.ldd + nb);
#pragma unroll
          for (int j = 0; j < 4; ++j) dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          continue;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int n = nb + j;
          if (n >= g.N) break;
          float x = v[j];
          if (EPI == TC_BIAS_RELU) x = fmaxf(x + __ldg(g.bias + n), 0.f);
          if (EPI == TC_BIAS) x += __ldg(g.bias + n);
          if (EPI == TC_GATE) x = __ldg(g.aux + (int64_t)gr * g.ldaux + n) > 0.f ? x : 0.f;
          g.D[(int64_t)gr * g.ldd + n] = x;
        }
      }
      tc_fence_before();
      mbar_arrive(smem_addr(&dempty[b]));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512u)
                 : "memory");
}

// B image: [n-tile][k-chunk] blocks of (BN x 128 B hi | BN x 128 B lo), swizzled
__global__ void k_b_image(const float* __restrict__ B, int64_t ldb, int kcontig, int N, int K,
                          int BN, int ntiles, int nkc, uint8_t* __restrict__ img) {
  const int64_t total = (int64_t)ntiles * nkc * BN * kChunkK;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % kChunkK);
    int64_t t = i / kChunkK;
    const int r = (int)(t % BN);
    t /= BN;
    const int kc = (int)(t % nkc);
    const int nt = (int)(t / nkc);
    const int gn = nt * BN + r, gk = kc * kChunkK + k;
    float x = 0.f;
    if (gn < N && gk < K) x = kcontig ? B[(int64_t)gn * ldb + gk] : B[(int64_t)gk * ldb + gn];
    uint8_t* blk = img + ((size_t)nt * nkc + kc) * (size_t)2 * BN * kRowBytes;
    const uint32_t h = x == x ? (__float_as_uint(x) & 0xffffe000u) : __float_as_uint(x);
    *reinterpret_cast<uint32_t*>(blk + sw_off(r, k)) = h;
    *reinterpret_cast<float*>(blk + (size_t)BN * kRowBytes + sw_off(r, k)) = x - __uint_as_float(h);
  }
}

inline int pick_bn(int n) { return n <= 16 ? 16 : n <= 32 ? 32 : n <= 64 ? 64 : 128; }

template <int BN, bool AK, bool BIMG, bool BK, int EPI>
void launch_bn(const TcGemm& g, int device, cudaStream_t s) {
  constexpr size_t smem = 1024 + 2 * 2 * (size_t)BN * kRowBytes + 2 * (size_t)kTileM * kRowBytes;
  static std::atomic<unsigned long long> attr{0};
  ensure_max_dyn_smem(k_tc_gemm<BN, AK, BIMG, BK, EPI>, device, smem, attr);
  dim3 grid((unsigned)(((g.M + kTileM - 1) / kTileM) * ((g.N + BN - 1) / BN)), 1u,
            (unsigned)(EPI == TC_ACC64 ? std::max(1, g.split_k) : 1));
  k_tc_gemm<BN, AK, BIMG, BK, EPI><<<grid, 128, smem, s>>>(g);
  count_launch();
}

template <bool AK, bool BIMG, bool BK, int EPI>
void launch_n(const TcGemm& g, int device, cudaStream_t s) {
  switch (pick_bn(g.N)) {
    case 16: return launch_bn<16, AK, BIMG, BK, EPI>(g, device, s);
    case 32: return launch_bn<32, AK, BIMG, BK, EPI>(g, device, s);
    case 64: return launch_bn<64, AK, BIMG, BK, EPI>(g, device, s);
    default: return launch_bn<128, AK, BIMG, BK, EPI>(g, device, s);
  }
}

template <int BN, int EPI>
void launch_ws(const TcGemm& g, int device, cudaStream_t s) {
  constexpr size_t smem = 1024 + (size_t)kWsStages * 2 * BN * kRowBytes +
                          2 * (size_t)kWsRing * kTileM * kRowBytes;
  static std::atomic<unsigned long long> attr{0};
  ensure_max_dyn_smem(k_tc_gemm_ws<BN, EPI>, device, smem, attr);
  int sms = 148;
  DPL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  const int64_t tiles = (int64_t)((g.M + kTileM - 1) / kTileM) * ((g.N + BN - 1) / BN);
  k_tc_gemm_ws<BN, EPI><<<(unsigned)std::min<int64_t>(tiles, sms), kWsThreads, smem, s>>>(g);
  count_launch();
}

bool ws_enabled() {
  static const bool off = getenv("DPL_TC_GEMM_SIMPLE") != nullptr;  // A/B switch for tests
  return !off;
}

template <int EPI>
void launch_epi(const TcGemm& g, int device, cudaStream_t s) {
  if constexpr (EPI != TC_ACC64) {
    const bool vec = g.a_kcontig && (g.lda & 3) == 0 && ((reinterpret_cast<uintptr_t>(g.A) & 15) == 0);
    if (g.b_image && vec && g.K > 0 && ws_enabled()) {  // persistent warp-specialised path
      switch (pick_bn(g.N)) {
        case 16: return launch_ws<16, EPI>(g, device, s);
        case 32: return launch_ws<32, EPI>(g, device, s);
        case 64: return launch_ws<64, EPI>(g, device, s);
        default: return launch_ws<128, EPI>(g, device, s);
      }
    }
  }
  if (g.b_image) {  // the layout of the image does not depend on B's order any more
    if (g.a_kcontig) return launch_n<true, true, true, EPI>(g, device, s);
    return launch_n<false, true, true, EPI>(g, device, s);
  }
  if (g.a_kcontig && g.b_kcontig) return launch_n<true, false, true, EPI>(g, device, s);
  if (g.a_kcontig && !g.b_kcontig) return launch_n<true, false, false, EPI>(g, device, s);
  if (!g.a_kcontig && !g.b_kcontig) return launch_n<false, false, false, EPI>(g, device, s);
  return launch_n<false, false, true, EPI>(g, device, s);
}

}  // namespace

size_t tc_b_image_bytes(int N, int K) {
  const int BN = pick_bn(N);
  const size_t ntiles = (size_t)((N + BN - 1) / BN), nkc = (size_t)((K + kChunkK - 1) / kChunkK);
  return ntiles * nkc * 2 * (size_t)BN * kRowBytes;
}

void tc_b_image(const float* B, int64_t ldb, bool kcontig, int N, int K, uint8_t* img,
                cudaStream_t s) {
  const int BN = pick_bn(N);
  const int ntiles = (N + BN - 1) / BN, nkc = (K + kChunkK - 1) / kChunkK;
  const int64_t total = (int64_t)ntiles * nkc * BN * kChunkK;
  const unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
  k_b_image<<<blocks, 256, 0, s>>>(B, ldb, kcontig ? 1 : 0, N, K, BN, ntiles, nkc, img);
  count_launch();
  DPL_CUDA(cudaGetLastError());
}

void tc_gemm(const TcGemm& g, int device, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0) return;
  switch (g.epi) {
    case TC_STORE: launch_epi<TC_STORE>(g, device, s); break;
    case TC_BIAS_RELU: launch_epi<TC_BIAS_RELU>(g, device, s); break;
    case TC_BIAS: launch_epi<TC_BIAS>(g, device, s); break;
    case TC_GATE: launch_epi<TC_GATE>(g, device, s); break;
    case TC_ACC64: launch_epi<TC_ACC64>(g, device, s); break;
    default: throw Error(1, "tc_gemm: bad epilogue");
  }
  DPL_CUDA(cudaGetLastError());
}

}  // namespace dpl
