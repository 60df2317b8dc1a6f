// forward_tm.cu — two-phase forward (K5) with the radial-channel accumulator in
// tensor memory (tcgen05.mma, kind::tf32; opt-in with DPL_FORWARD_TMEM=1).
//
// Same traversal, decisions and phase A as k_forward_tc (forward_tc.cu;
// DipoleTree::primal, proj/src/bhtree.cpp:188-234). Per query warp the radial
// part of the sum is one long-K matrix product over all of the warp's sources,
//     D[channel][query] = sum_e rows[e][channel] . w[e][query]       (48 x 32)
// so the accumulator can stay in 32 TMEM columns for the whole traversal instead
// of 48 registers per lane, and phase B shrinks from fragment loads, operand
// splits and 36 mma.sync per 8 sources to three tcgen05.mma (M = 64, N = 32,
// K = 8) issued by one lane: hi.hi + hi.lo + lo.hi of the tf32 split (fp32-class
// products, as forward_tc).
//
// Both operands arrive MN-major (a source's 48 moments and a warp's 32 weights
// are contiguous per source). For 32-bit elements that needs the
// SWIZZLE_128B_BASE32B shared-memory layout (probed in
// tools/tcgen05_mn_major_probe.cu: every other MN-major layout leaves the
// accumulator zero on B200): atoms of 4 k-rows x 128 B (32 MN elements), the
// 32-byte chunk c of row k stored at c ^ (k & 3); LBO = stride of MN atoms,
// SBO = stride of the 4-row k groups. A source's row is 12 cp.async chunks of
// 16 B (the split rows [hi | lo] are precomputed with the moments), its
// weights one conflict-free STS per lane.
#include <algorithm>

#include "forward.cuh"
#include "tc05.cuh"
#include "traverse.cuh"

namespace dpl {

namespace {
__device__ __forceinline__ void cp_async16(uint32_t smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(smem), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

__device__ __forceinline__ float4 fwd_w(float fx, float fy, float fz, float r2, float A,
                                        const KParams& kp) {
  const float inv_r = rsqrt_pos(r2);
  float W, R;
  if (kp.mode == KM_SINGULAR || (kp.mode == KM_REGULARIZED && r2 >= kp.near2)) {
    R = inv_r * inv_r;
    W = R * inv_r;
  } else {
    Co c = coeffs<0>(r2, kp);
    W = c.W;
    R = c.R;
  }
  const float aW = A * W;
  return make_float4(aW * fx, aW * fy, aW * fz, A * R);
}
__device__ __forceinline__ float4 fwd_w_far(float fx, float fy, float fz, float r2, float A) {
  const float inv_r = rsqrt_pos(r2);
  const float R = inv_r * inv_r;
  const float W = R * inv_r;
  const float aW = A * W;
  return make_float4(aW * fx, aW * fy, aW * fz, A * R);
}
__device__ __forceinline__ float4 fwd_w_far_m(float fx, float fy, float fz, float r2, float Am,
                                              float near2) {
  const float inv_r = rsqrt_far(r2, near2);
  const float R = inv_r * inv_r;
  const float aW = Am * (R * inv_r);
  return make_float4(aW * fx, aW * fy, aW * fz, Am * R);
}

constexpr int FT_WARPS = 4;
constexpr int FT_F4 = 13;  // row float4s: dipole + 48 radial
// per warp (bytes); tiles on 1024-byte boundaries. FT_NS stages of operand tiles:
// with 2 a batch is written while the previous batch's MMAs still read theirs,
// but only 3 CTAs fit an SM; measured on config 2 (forward incl. K9): 1 stage
// 13.9 ms, 2 stages 16.6 ms (k_forward_tc: 11.0 ms)
constexpr int FT_NS = 1;
constexpr uint32_t FT_A_HI = 0;      // [2 MN atoms][2 k groups][4 rows][128 B]
constexpr uint32_t FT_A_LO = 2048;
constexpr uint32_t FT_B_HI = 4096;   // [2 k groups][4 rows][128 B]
constexpr uint32_t FT_B_LO = 5120;
constexpr uint32_t FT_STAGE = 6144;
constexpr uint32_t FT_STK = FT_NS * FT_STAGE;  // traversal stack / node-record window
constexpr uint32_t FT_VB = FT_STK + DPL_STACK_PER_WARP * 8;  // [32] window dipole moments
constexpr uint32_t FT_WARP = FT_NS * FT_STAGE + 3072;
static_assert(FT_VB + 32 * 16 <= FT_WARP && FT_VB % 16 == 0, "per-warp layout");
static_assert(32 * 48 <= DPL_STACK_PER_WARP * 8, "record window fits the stack region");

// MN-major SWIZZLE_128B_BASE32B shared-memory descriptor (layout type 1)
__device__ __forceinline__ uint64_t mn32_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)1u << 61;
  return d;
}
// kind::tf32, D fp32, A and B MN-major
constexpr uint32_t ft_idesc(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}
}  // namespace

// LIST: replay the interaction lists; warps whose list is incomplete walk the
// tree (same arithmetic in the same entry order). REG: regularized kernel with
// (6.5 eps)^2 >= REG_MIN_NEAR2 (the mode tests fold away).
template <bool LIST, bool REG>
__global__ void __launch_bounds__(FT_WARPS * 32, FT_NS == 1 ? 4 : 3)
    k_forward_tm(TreeView tv, KParams kp_in, const double* __restrict__ xs,
                 const int32_t* __restrict__ perm, int64_t q, int nr,
                 const int* __restrict__ chmap, float* __restrict__ out, int out_stride,
                 int only_ch, IListView lv, int* overflow) {
  using namespace tc05;
  KParams kp = kp_in;
  if (REG) kp.mode = KM_REGULARIZED;
  constexpr int F4 = FT_F4;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bars[FT_WARPS][2];
  __shared__ uint32_t tmem_slot;
  __shared__ long long qidx[FT_WARPS][32];  // query of (warp, lane); -1: none
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint8_t* wb = sm + (size_t)w * FT_WARP;

  if (w == 0) tmem_alloc<32 * FT_WARPS>(&tmem_slot);
  if (threadIdx.x == 0) {
    for (int i = 0; i < FT_WARPS; ++i) mbar_init(smem_addr(&bars[i][0]), 1), mbar_init(smem_addr(&bars[i][1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  const int64_t sidx = ((int64_t)blockIdx.x * FT_WARPS + w) * 32 + lane;
  const bool valid = sidx < q;
  const int64_t qi = valid ? (perm ? (int64_t)perm[sidx] : sidx) : 0;
  qidx[w][lane] = valid ? qi : -1;
  // operand tiles start finite: a row slot that was never written (channels
  // 48..63, the tail of the last batch) only ever meets zero weights
  {
    float4* z = reinterpret_cast<float4*>(wb);
    for (int i = lane; i < (int)(FT_STK / 16); i += 32) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_slot + 32u * (uint32_t)w;  // this warp's 32 accumulator columns
  const uint32_t bar0 = smem_addr(&bars[w][0]);
  const unsigned active = __ballot_sync(FULL_MASK, valid);

  float accd = 0.f;
  if (active) {
    QueryPos x;
    if (valid) {
      x.x = xs[3 * qi], x.y = xs[3 * qi + 1], x.z = xs[3 * qi + 2];
    } else {
      x.x = x.y = x.z = 0.0;
    }
    const QueryDF qx = make_qdf(x, tv.cmax);
    const bool singular = kp.mode == KM_SINGULAR;
    const float4* __restrict__ node_row = tv.node_row;
    const float4* __restrict__ pt_row = tv.pt_row;
    // split rows [row][hi | lo]: row r starts at float4 index 2 F4 r
    const float4* __restrict__ node_split = tv.node_row_split;
    const float4* __restrict__ pt_split = tv.pt_row_split;
    int2* stk = reinterpret_cast<int2*>(wb + FT_STK);
    float4* vb = reinterpret_cast<float4*>(wb + FT_VB);
    const uint32_t s_a = smem_addr(wb + FT_A_HI), s_b = smem_addr(wb + FT_B_HI);
    // Tile offsets. Row k of a tile starts at (k >> 2) 512 + (k & 3) 128 and its
    // 32-byte chunks are permuted by XOR with (k & 3): every field sits in its own
    // bits, so an element's offset is (lane constant) ^ U(k) with the warp-uniform
    // U(k) = (k >> 2) 512 + (k & 3) (128 + 32). Weights: lane n is element n of the
    // row; source rows: lane L in 1..12 copies 16-byte chunk j = L - 1 (radial
    // channels 4 j .. 4 j + 3; MN atom j >> 3).
    const uint32_t b0 = (((uint32_t)lane >> 3) << 5) + ((uint32_t)lane & 7u) * 4u;
    const uint32_t j = (uint32_t)(lane - 1) & 15u;
    const uint32_t a0 = (j >> 3) * 1024u + (((j & 7u) >> 1) << 5) + (j & 1u) * 16u;
    const bool a_lane = lane >= 1 && lane < F4;
    constexpr uint32_t IDESC = ft_idesc(64, 32);
    int nent = 0;
    bool first = true;
    uint32_t st = 0;          // stage being filled
    uint32_t issued = 0;      // bit s: stage s has MMAs in flight (or not yet waited for)
    uint32_t phase = 0;       // bit s: parity the next wait on stage s uses
    uint8_t* tb = wb;         // tiles of the stage being filled

    // wait until the MMAs that last read stage s have completed
    auto stage_free = [&](uint32_t s_) {
      if ((issued >> s_) & 1u) {
        mbar_wait(bar0 + 8u * s_, (phase >> s_) & 1u);
        phase ^= 1u << s_;
        issued &= ~(1u << s_);
      }
    };
    // the batch's 8 sources -> three MMAs into the warp's accumulator
    auto evaluate = [&]() {
      for (int k = nent; k < 8; ++k) {  // rows without a source: zero weights
        const uint32_t off = b0 ^ ((uint32_t)(k >> 2) * 512u + (uint32_t)(k & 3) * 160u);
        *reinterpret_cast<float*>(tb + FT_B_HI + off) = 0.f;
        *reinterpret_cast<float*>(tb + FT_B_LO + off) = 0.f;
      }
      cp_async_wait_all();
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        fence_after();
        const uint32_t sa = s_a + st * FT_STAGE, sb = s_b + st * FT_STAGE;
        const uint64_t ah = mn32_desc(sa, 1024u, 512u), al = mn32_desc(sa + 2048u, 1024u, 512u);
        const uint64_t bh = mn32_desc(sb, 1024u, 512u), bl = mn32_desc(sb + 1024u, 1024u, 512u);
        mma_ss(tmem, ah, bh, IDESC, first ? 0u : 1u);
        mma_ss(tmem, ah, bl, IDESC, 1u);
        mma_ss(tmem, al, bh, IDESC, 1u);
        mma_commit(bar0 + 8u * st);
      }
      __syncwarp();
      issued |= 1u << st;
      first = false;
      nent = 0;
      st = (st + 1u) % (uint32_t)FT_NS;
      tb = wb + st * FT_STAGE;
    };
    // v: the source's dipole moment; split: the source's [hi | lo] row
    auto store_entry = [&](float4 wv, const float4* split, float4 v) {  // nent < 8
      if (nent == 0) stage_free(st);  // the MMAs that last read these tiles are done
      accd = fmaf(wv.x, v.x, fmaf(wv.y, v.y, fmaf(wv.z, v.z, accd)));
      const uint32_t u = (uint32_t)(nent >> 2) * 512u + (uint32_t)(nent & 3) * 160u;
      const uint32_t offb = b0 ^ u;
      const float wh = __uint_as_float(__float_as_uint(wv.w) & 0xffffe000u);
      *reinterpret_cast<float*>(tb + FT_B_HI + offb) = wh;
      *reinterpret_cast<float*>(tb + FT_B_LO + offb) = wv.w - wh;
      if (a_lane) {
        const uint32_t offa = st * FT_STAGE + (a0 ^ u);
        const float4* src = split + lane;
        cp_async16(s_a + offa, src);
        cp_async16(s_a + 2048u + offa, src + F4);
      }
      ++nent;
    };
    auto append = [&](float4 wv, const float4* rowsrc, const float4* split) {
      const float4 v = __ldg(rowsrc);
      if (nent == 8) evaluate();
      store_entry(wv, split, v);
    };

    const int64_t wg = (int64_t)blockIdx.x * FT_WARPS + w;
    const int total = LIST ? __ldg(lv.count + wg) : -1;
    if (LIST && total >= 0) {
      // 32 entries at a time; their node records are prefetched into the
      // (unused) stack region with cp.async, read back as broadcast LDS.128
      NodeRec* rb = reinterpret_cast<NodeRec*>(stk);
      const uint32_t s_rb = smem_addr(stk) + 48u * lane;
      const uint32_t s_vb = smem_addr(vb) + 16u * lane;
      const double* xq = xs + 3 * qi;
      int chunk = (int)wg;
      for (int base = 0; base < total; base += 32) {
        if (base > 0 && base % IL_CHUNK == 0) chunk = __ldg(lv.next + chunk);
        const uint2 my = il_load(lv, chunk, base, total, lane);
        const int n = min(32, total - base);
        __syncwarp();  // the previous window's records are consumed
        if (lane < n) {
          const NodeRec* r = tv.node_rec + (my.x & IL_NODE);
          cp_async16(s_rb, &r->hi);
          cp_async16(s_rb + 16u, &r->lo);
          cp_async16(s_rb + 32u, &r->topo);
          if (!(my.x & IL_LEAF)) cp_async16(s_vb, node_row + (size_t)(my.x & IL_NODE) * F4);
        }
        cp_async_wait_all();
        if (lane < n) *reinterpret_cast<uint2*>(&rb[lane].topo) = my;
        __syncwarp();
        for (int i = 0; i < n; ++i) {
          const int4 tpi = rb[i].topo;
          const uint32_t src = (uint32_t)tpi.x;
          if (nent == 8) evaluate();
          // two consecutive far entries without near lanes that fit the batch
          if (nent + 2 <= 8 && i + 1 < n &&
              !((src | (uint32_t)rb[i + 1].topo.x) & (IL_LEAF | IL_NEAR))) {
            const int4 tb = rb[i + 1].topo;
            const float4 ha = rb[i].hi, la = rb[i].lo, hb = rb[i + 1].hi, lb = rb[i + 1].lo;
            float ax, ay, az, bx, by, bz;
            const float sa = dist2_df(ha, la, qx, ax, ay, az);
            const float sb = dist2_df(hb, lb, qx, bx, by, bz);
            const bool fa = ((unsigned)tpi.y >> lane) & 1u, fb = ((unsigned)tb.y >> lane) & 1u;
            if (REG) {
              store_entry(fwd_w_far_m(ax, ay, az, sa, sel0(fa, la.w), kp.near2),
                          node_split + (size_t)(src & IL_NODE) * (2 * F4), vb[i]);
              store_entry(fwd_w_far_m(bx, by, bz, sb, sel0(fb, lb.w), kp.near2),
                          node_split + (size_t)((uint32_t)tb.x & IL_NODE) * (2 * F4), vb[i + 1]);
            } else {
              const float4 wa = fwd_w_far(ax, ay, az, sa, la.w), wbv = fwd_w_far(bx, by, bz, sb, lb.w);
              store_entry(make_float4(fa ? wa.x : 0.f, fa ? wa.y : 0.f, fa ? wa.z : 0.f, fa ? wa.w : 0.f),
                          node_split + (size_t)(src & IL_NODE) * (2 * F4), vb[i]);
              store_entry(make_float4(fb ? wbv.x : 0.f, fb ? wbv.y : 0.f, fb ? wbv.z : 0.f,
                                      fb ? wbv.w : 0.f),
                          node_split + (size_t)((uint32_t)tb.x & IL_NODE) * (2 * F4), vb[i + 1]);
            }
            ++i;
            continue;
          }
          const unsigned m = (unsigned)tpi.y;
          const int node = (int)(src & IL_NODE);
          const bool mine = (m >> lane) & 1u;
          if (!(src & IL_LEAF)) {
            const float4 hi = rb[i].hi, lo = rb[i].lo;
            float dx, dy, dz;
            const float s = dist2_df(hi, lo, qx, dx, dy, dz);
            float4 wv;
            if (src & IL_NEAR) {
              wv = mine ? fwd_w(dx, dy, dz, s, lo.w, kp) : make_float4(0.f, 0.f, 0.f, 0.f);
            } else if (REG) {
              wv = fwd_w_far_m(dx, dy, dz, s, sel0(mine, lo.w), kp.near2);
            } else {
              const float4 f = fwd_w_far(dx, dy, dz, s, lo.w);
              wv.x = mine ? f.x : 0.f, wv.y = mine ? f.y : 0.f;
              wv.z = mine ? f.z : 0.f, wv.w = mine ? f.w : 0.f;
            }
            if (nent == 8) evaluate();
            store_entry(wv, node_split + (size_t)node * (2 * F4), vb[i]);
          } else {
            for (int jp = tpi.z; jp < tpi.w; ++jp) {
              float4 wv = make_float4(0.f, 0.f, 0.f, 0.f);
              if (mine) {
                const PtRec* pr = tv.pt_rec + jp;
                const float4 ph = __ldg(&pr->hi);
                float dx, dy, dz;
                const float r2 = dist2_df(ph, __ldg(&pr->lo), qx, dx, dy, dz);
                if (!(singular && r2 == 0.f && coincident_exact(tv.pt_pos64 + 3 * (size_t)jp, xq)))
                  wv = fwd_w(dx, dy, dz, r2, ph.w, kp);
              }
              append(wv, pt_row + (size_t)jp * F4, pt_split + (size_t)jp * (2 * F4));
            }
          }
        }
      }
    }
    int sp = (LIST && total >= 0) ? 0 : 1;
    if (sp && lane == 0) stk[0] = make_int2(0, (int)active);
    __syncwarp();
    while (sp > 0) {
      --sp;
      const int2 e = stk[sp];
      __syncwarp();
      const int node = e.x;
      const unsigned mask = (unsigned)e.y;
      const bool mine = (mask >> lane) & 1u;
      const NodeRec* rec = tv.node_rec + node;
      const float4 hi = __ldg(&rec->hi);
      const float4 lo = __ldg(&rec->lo);
      const int4 tp = __ldg(&rec->topo);
      const float A = lo.w;
      float dx, dy, dz;
      const float s = dist2_df(hi, lo, qx, dx, dy, dz);
      const bool far = mine && far_test(s, hi, qx, x, tv.node_dec + node);
      const unsigned farm = __ballot_sync(FULL_MASK, far);
      if (farm && A > 0.f) {  // area > 0 (bhtree.cpp:205)
        const float4 wv = far ? fwd_w(dx, dy, dz, s, A, kp) : make_float4(0.f, 0.f, 0.f, 0.f);
        append(wv, node_row + (size_t)node * F4, node_split + (size_t)node * (2 * F4));
      }
      const unsigned openm = mask & ~farm;
      if (openm) {
        if (tp.y == 0) {
          const bool me_open = (openm >> lane) & 1u;
          for (int jp = tp.z; jp < tp.w; ++jp) {
            float4 wv = make_float4(0.f, 0.f, 0.f, 0.f);
            if (me_open) {
              const PtRec* pr = tv.pt_rec + jp;
              const float4 ph = __ldg(&pr->hi);
              const float r2 = dist2_df(ph, __ldg(&pr->lo), qx, dx, dy, dz);
              if (!(singular && r2 == 0.f && coincident_exact(tv.pt_pos64 + 3 * (size_t)jp, x)))
                wv = fwd_w(dx, dy, dz, r2, ph.w, kp);
            }
            append(wv, pt_row + (size_t)jp * F4, pt_split + (size_t)jp * (2 * F4));
          }
        } else {
          if (sp + tp.y > DPL_STACK_PER_WARP) {
            if (lane == 0) atomicExch(overflow, 1);
            break;
          }
          if (lane < tp.y) stk[sp + lane] = make_int2(tp.x + lane, (int)openm);
          sp += tp.y;
          __syncwarp();
        }
      }
    }
    // the last batch; a warp without any source still defines its accumulator
    // (all weights zero)
    if (nent || first) {
      if (nent == 0) stage_free(st);
      evaluate();
    }
    for (uint32_t s_ = 0; s_ < (uint32_t)FT_NS; ++s_) stage_free(s_);  // the accumulator is complete
    // the dipole value is lane-local
    if (only_ch >= 0) {
      if (valid && __ldg(chmap) == only_ch) out[qi] = accd;
    } else if (valid) {
      out[qi * out_stride + __ldg(chmap)] = accd;
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  // Radial outputs. A 64-row accumulator puts channel c in TMEM lane
  // 32 (c / 16) + c % 16, and a warp reads only its own lane quadrant: warp g
  // stores channels 16 g .. 16 g + 15 of all four accumulators of the CTA.
  if (w < 3 && 16 * w < nr) {
    const int c = 16 * w + lane;
    const bool okc = lane < 16 && c < nr;
    const int ch = okc ? __ldg(chmap + 1 + c) : 0;
    for (int a = 0; a < FT_WARPS; ++a) {
      if (qidx[a][0] < 0) continue;  // lane 0 of a warp is valid whenever any lane is
      uint32_t r[32];
      tmem_ld32(tmem_slot + ((uint32_t)(32 * w) << 16) + 32u * (uint32_t)a, r);
      if (okc) {
#pragma unroll
        for (int col = 0; col < 32; ++col) {
          const long long qq = qidx[a][col];
          if (qq >= 0) {
            if (only_ch < 0)
              out[qq * out_stride + ch] = __uint_as_float(r[col]);
            else if (ch == only_ch)
              out[qq] = __uint_as_float(r[col]);
          }
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<32 * FT_WARPS>(tmem_slot);
}

template <bool LIST, bool REG>
static void launch_ftm(const Tree& t, const KParams& kp, const FwdArgs& a, int nr, IListView lv) {
  // 128 TMEM columns per CTA: at most 4 CTAs of an SM can hold their accumulators.
  // The request is padded so that no fifth CTA becomes resident: it would spin in
  // tcgen05.alloc (9 % of the issued instructions in the first ncu capture) with
  // its other warps parked at the barrier behind it.
  const size_t smem = std::max<size_t>((size_t)FT_WARPS * FT_WARP + 1024, 47 * 1024);
  static std::atomic<unsigned long long> attr{0};
  ensure_max_dyn_smem(k_forward_tm<LIST, REG>, t.device, smem, attr);
  const unsigned blocks = (unsigned)((a.q + FT_WARPS * 32 - 1) / (FT_WARPS * 32));
  k_forward_tm<LIST, REG><<<blocks, FT_WARPS * 32, smem, t.stream>>>(
      t.view(), kp, a.xs, a.perm, a.q, nr, t.chmap.as<int>(), a.out, a.out_stride, a.only_ch, lv,
      a.overflow);
  count_launch();
}

// One Dipole + 48 Radial slots, values only; false when the call is outside its
// range (the caller falls back to forward_tc / forward2).
bool forward_tm_launch(const Tree& t, const KParams& kp, const FwdArgs& a) {
  if (a.grad_mode != 0 || a.counters || (a.single && a.only_ch < 0)) return false;
  if (t.Cd != 1 || t.PR != 48 || t.F4 != FT_F4 || !t.node_row_split.p) return false;
  if (a.only_ch >= 0 && t.kinds[a.only_ch] == 0) return false;  // dipole-only variant: forward_tc
  const int nr = a.nr_limit >= 0 ? std::min(a.nr_limit, t.Cr) : t.Cr;
  const bool reg = kp.mode == KM_REGULARIZED && kp.near2 >= REG_MIN_NEAR2;
  if (a.ilist && !no_ilist()) {
    ilist_build(t, *a.ilist, a.xs, a.perm, a.q, a.beta, ilist_near_thr(kp), a.overflow);
    if (reg)
      launch_ftm<true, true>(t, kp, a, nr, a.ilist->view());
    else
      launch_ftm<true, false>(t, kp, a, nr, a.ilist->view());
  } else if (reg) {
    launch_ftm<false, true>(t, kp, a, nr, IListView{});
  } else {
    launch_ftm<false, false>(t, kp, a, nr, IListView{});
  }
  return true;
}

}  // namespace dpl
