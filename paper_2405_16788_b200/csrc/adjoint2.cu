// adjoint2.cu — two-phase adjoint traversal (K7) for the SceneModel layout
// (one Dipole channel + Cr <= 64 Radial channels).
//
// Same semantics as k_adjoint (adjoint.cu; DipoleTree::adjoint,
// proj/src/bhtree.cpp:345-417), restructured like forward2.cu:
//   phase A (traverse, lanes = queries): exact fp64 opening tests; for every
//     source (far node / opened leaf point) each lane computes its
//     coefficients once and writes to the warp's shared batch
//       wR[l] = A R, wE[l] = A dR_de            (radial weights, eps weights)
//       vq[0..3][l] = node:  A W ds0 d  (- A (W dg + Wp_r (dg.d) d))   , 0
//                     point: dn (3), d mu_0                        (:394-406)
//     and adds its dipole epsilon terms to a per-lane fp64 accumulator. The
//     radial payload row is staged (cp.async) only when some lane is within
//     6.5 eps (the only case with radial epsilon terms).
//   phase B (evaluate, lanes = channels): the warp's d_out tile is held
//     TRANSPOSED in registers — lane L owns radial channel L for all 32
//     queries and channel 32 + (L & 15) for the 16 queries of its half-warp
//     (48 registers, every lane busy for Cr = 48) — so each entry's
//       node_s[t, c] (or point_mu[m, c]) += sum_l wR[l] ds[l, c]
//     is 8 broadcast LDS.128 + 48 FFMA per lane and one coalesced fp64 RED per
//     channel. The 4 per-lane vector quantities are reduced with one LDS.128,
//     3 FADD and 3 shuffles and land in node_v / point_n / point_mu_0 with at
//     most 4 REDs. Accumulators are fp64 (SURVEY §7 hard part 4).
//   tensor-core phase B (MT > 0, opt-in with DPL_ADJOINT_TC=1; measured slower
//     than the FFMA phase B on config 2, see adj2_plan): the radial product
//     D[channel][entry] = sum_l dsT[channel][l] wR[entry][l] (and its epsilon
//     twin with wE) runs on mma.sync: A = the warp's transposed d_out tile,
//     held as TF32 fragments in registers for the whole traversal (16 MT
//     registers, the same budget as the FFMA tile) with its low part as BF16
//     fragments in shared memory; B = the batch's weights. Three-term split
//     A_hi B_hi + A_hi B_lo (TF32) + A_lo B_hi (BF16): per-product error
//     ~2^-19 relative, fp32-class. The epilogue REDs 8 consecutive channels of
//     4 entries per instruction (8 sectors per 32 lanes, as the FFMA path).
#include <type_traits>

#include "adjoint.cuh"
#include "traverse.cuh"

namespace dpl {

namespace {
// cvt.rna.tf32.f32 for finite a (round to nearest, ties away: add half a tf32
// ulp to the magnitude bits, truncate): 2 integer ops instead of the 4 that the
// cvt lowers to on sm_100 (its inf / NaN guard is not needed here)
__device__ __forceinline__ uint32_t to_tf32(float a) {
  return (__float_as_uint(a) + 0x1000u) & 0xffffe000u;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo_col, float hi_col) {
  uint32_t r;  // lower 16 bits: the smaller k index
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;\n" : "=r"(r) : "f"(hi_col), "f"(lo_col));
  return r;
}
__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint4& a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}
// smallest stride >= n floats with stride = 8 or 24 (mod 32): conflict-free
// fragment gathers from a [32][stride] tile
// packed fp32 FMA (Blackwell FFMA2): acc.{x,y} += a.{x,y} * b.{x,y}, one issue slot
__device__ __forceinline__ void fma2(float2& acc, float2 a, float2 b) {
  unsigned long long A, B, C;
  asm("mov.b64 %0, {%1, %2};" : "=l"(A) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(B) : "f"(b.x), "f"(b.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(C) : "f"(acc.x), "f"(acc.y));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(C) : "l"(A), "l"(B));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(acc.x), "=f"(acc.y) : "l"(C));
}
constexpr int tile_stride(int n) {
  int r = n;
  while (r % 32 != 8 && r % 32 != 24) ++r;
  return r;
}
__device__ __forceinline__ void cp_async16(uint32_t smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(smem), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
}  // namespace

// Coefficients for the adjoint: beyond 6.5 eps (and for the singular kernel)
// tau = 1, tau' = tau'' = 0 (kernels.cpp:50-55), so only W, R (and Wp_r when
// query-gradient adjoints are present) are non-zero.
template <int GM>
__device__ __forceinline__ Co adj_coeffs(float r2, const KParams& kp) {
  if (kp.mode == KM_SINGULAR || (kp.mode == KM_REGULARIZED && r2 >= kp.near2)) {
    Co c;
    const float inv_r = rsqrtf(r2);
    c.R = inv_r * inv_r;
    c.W = c.R * inv_r;
    c.Wp_r = GM ? -3.0f * c.W * c.R : 0.f;
    c.Rp_r = 0.f;
    c.dW_de = c.dWp_r_de = c.dR_de = 0.f;
    c.near = false;
    return c;
  }
  return coeffs<2>(r2, kp);
}

struct Adj2Ptrs {
  double* node_v;  // nodes x Cd(=1) x 3
  double* node_s;  // nodes x Cr
  double* pt_mud;  // N x 1
  double* pt_mur;  // N x Cr
  double* pt_n;    // N x 3
  double* d_eps;
};

// Per-warp shared-memory layout. The d_out tile staged by the tensor-core
// prologue aliases the batch arrays (it is consumed before the first entry).
// VR: radial channels reduced with the vector quantities (NB = 3, nr <= 4):
// 8 per-lane slots per entry, no weight rows and no staged payload rows.
template <int MT, int ENT, int RR, bool VR = false>
struct AdjLayout {
  static constexpr int WS = MT ? 36 : 32;  // weight row stride: conflict-free B gathers
  static constexpr int F4 = VR ? 0 : 1 + RR;  // smem row capacity (float4)
  static constexpr int VQ = VR ? 8 : 4;       // per-lane slots per entry
  static constexpr int S = tile_stride(16 * (MT ? MT : 1));
  static constexpr int BATCH = (VR ? 0 : ENT * WS * 2) + ENT * 32 * VQ + ENT * F4 * 4;
  static constexpr int TILE = MT ? 32 * S : 0;
  static constexpr int UNION = BATCH > TILE ? BATCH : TILE;
  static constexpr int ALO = MT * 2 * 32 * 4;  // BF16 A_lo fragments (uint32 words)
  static constexpr int PTR = 2 * ENT;  // per-entry radial destination row (double*)
  static constexpr int WARP_FLOATS =
      (UNION + ALO + PTR + ENT + (ENT & 1) + 2 * DPL_STACK_PER_WARP + 3) & ~3;
};

// NB: 0 -> Cr <= 32; 1 -> 32 < Cr <= 48 (split); 2 -> Cr <= 64 (FFMA phase B);
//     3 -> Cr <= 4 (render path: each lane forms A R ds_c for its own query and
//     the radial sums ride along the vector-quantity reduction, no d_out tile).
// MT: > 0 selects the tensor-core phase B with MT m-tiles (Cr <= 16 MT); NB unused.
// GM: 0 no d_grad; 1 d_grad q x dstride x 3; 2 d_grad q x 3 (channel 0).
// MAXR: register cap (occupancy vs. spills; chosen by measurement)
// LIST: replay the batch's interaction lists (ilist.cuh); warps whose list is
// incomplete walk the tree as the fused kernel does (same entry order).
// REG: compiled for the regularized kernel (the mode tests fold away)
template <int NB, int GM, int WARPS, int ENT, int RR, int MAXR = 128, int MT = 0, bool LIST = false,
          bool REG = false>
__global__ void __launch_bounds__(WARPS * 32) __maxnreg__(MAXR)
    k_adjoint2(TreeView tv, KParams kp_in, const double* __restrict__ xs,
               const int32_t* __restrict__ perm, int64_t q, const float* __restrict__ d_out,
               int dstride, const float* __restrict__ d_grad, int nr,
               const int* __restrict__ chmap, Adj2Ptrs acc, IListView lv, int* overflow) {
  KParams kp = kp_in;
  if (REG) kp.mode = KM_REGULARIZED;
  constexpr bool VR = NB == 3;
  static_assert(!VR || MT == 0, "VR is an FFMA-path layout");
  using L = AdjLayout<MT, ENT, RR, VR>;
  constexpr int VQ = L::VQ;
  constexpr int F4 = L::F4;
  constexpr int WS = L::WS;
  static_assert(MT == 0 || ENT == 8, "tensor-core phase B uses one n-tile of 8 entries");
  static_assert((ENT & (ENT - 1)) == 0 && ENT <= 32, "ENT: a power of two <= 32");
  extern __shared__ float4 smem_f4[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;  // mma fragment coordinates
  float* base = reinterpret_cast<float*>(smem_f4) + (size_t)w * L::WARP_FLOATS;
  float* wR = base;
  float* wE = wR + ENT * WS;
  float* vq = VR ? base : wE + ENT * WS;
  float4* rows = reinterpret_cast<float4*>(vq + ENT * 32 * VQ);
  const uint4* alo = reinterpret_cast<const uint4*>(base + L::UNION);
  // per entry: the radial destination row, resolved once by lane 0 in phase A
  double** dptr = reinterpret_cast<double**>(base + L::UNION + L::ALO);
  int* meta = reinterpret_cast<int*>(base + L::UNION + L::ALO + L::PTR);
  int2* stk = reinterpret_cast<int2*>(meta + ENT + (ENT & 1));
  const uint32_t s_rows = smem_u32(rows) + 16u * lane;
  const int F4g = tv.F4;               // global row stride
  const int F4c = F4g < F4 ? F4g : F4;  // float4 staged per row (dipole + radial slots used)

  const int64_t sidx = ((int64_t)blockIdx.x * WARPS + w) * 32 + lane;
  const bool valid = sidx < q;
  const int64_t qi = valid ? (perm ? (int64_t)perm[sidx] : sidx) : 0;
  QueryPos x;
  if (valid) {
    x.x = xs[3 * qi], x.y = xs[3 * qi + 1], x.z = xs[3 * qi + 2];
  } else {
    x.x = x.y = x.z = 0.0;
  }
  const unsigned active = __ballot_sync(FULL_MASK, valid);
  if (!active) return;
  const int Cr = tv.Cr;
  const QueryDF qx = make_qdf(x, tv.cmax);
  // fp64 position for the exact fallbacks, re-read there (invalid lanes never test)
  const double* xq = xs + 3 * qi;

  // own-query dipole upstream gradients (channel slot 0)
  const int ch0 = __ldg(chmap);
  const float ds0 = valid ? __ldg(d_out + qi * dstride + ch0) : 0.f;
  float dg0 = 0.f, dg1 = 0.f, dg2 = 0.f;
  if (GM && valid) {
    const float* g = GM == 1 ? d_grad + (qi * dstride + ch0) * 3 : d_grad + qi * 3;
    dg0 = g[0], dg1 = g[1], dg2 = g[2];
  }
  // FFMA phase B: transposed radial tile in registers. Lane (h, g) = (lane >> 4,
  // lane & 15) owns channels g, 16 + g, .. (NG groups of 16) for the 16 queries
  // of half-warp h: each entry's weights are then 4 LDS.128 with a
  // half-warp-uniform address (8 shared-memory wavefronts) instead of 12
  // warp-uniform ones (24) — shared-memory wavefronts, not issue slots, bound
  // this kernel (profiles/r02_smem_wavefronts.md) — and the two halves' partial
  // sums meet through one shuffle per channel-group pair.
  constexpr bool FF = MT == 0;
  constexpr int NG = NB == 0 ? 2 : (NB == 1 ? 3 : (NB == 2 ? 4 : 1));
  const int hw = lane >> 4, g16 = lane & 15;
  float col[FF && !VR ? NG : 1][16];
  bool okg[NG];
#pragma unroll
  for (int k = 0; k < NG; ++k) okg[k] = FF && !VR && 16 * k + g16 < nr;
  // VR: this lane's own radial upstream gradients (slots >= nr read as 0)
  float dsr[4] = {0.f, 0.f, 0.f, 0.f};
  if constexpr (VR) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (valid && c < nr) dsr[c] = __ldg(d_out + qi * dstride + __ldg(chmap + 1 + c));
  }
  // tensor-core phase B: A = d_out tile^T [channel][query] as TF32 fragments
  uint32_t ahi[MT ? MT : 1][4][4];
  if constexpr (FF && !VR) {
    int chg[NG];
#pragma unroll
    for (int k = 0; k < NG; ++k) chg[k] = okg[k] ? __ldg(chmap + 1 + 16 * k + g16) : 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int srcl = 16 * hw + i;
      const int64_t ql = __shfl_sync(FULL_MASK, qi, srcl);
      const bool vl = (active >> srcl) & 1u;
#pragma unroll
      for (int k = 0; k < NG; ++k)
        col[k][i] = (okg[k] && vl) ? __ldg(d_out + ql * dstride + chg[k]) : 0.f;
    }
  } else {
    // coalesced staging of the tile T[query l][slot c] (c < 16 MT), then
    // fragment gathers (stride S = 8 or 24 mod 32: conflict-free)
    constexpr int S = L::S;
    float* T = base;
    const int c1 = lane + 32;
    const int chm0 = lane < nr ? __ldg(chmap + 1 + lane) : 0;
    const int chm1 = (16 * MT > 32 && c1 < nr) ? __ldg(chmap + 1 + c1) : 0;
    for (int l = 0; l < 32; ++l) {
      const int64_t ql = __shfl_sync(FULL_MASK, qi, l);
      const bool vl = (active >> l) & 1u;
      if (lane < 16 * MT)
        T[l * S + lane] = (vl && lane < nr) ? __ldg(d_out + ql * dstride + chm0) : 0.f;
      if (16 * MT > 32 && c1 < 16 * MT)
        T[l * S + c1] = (vl && c1 < nr) ? __ldg(d_out + ql * dstride + chm1) : 0.f;
    }
    __syncwarp();
#pragma unroll
    for (int mt = 0; mt < (MT ? MT : 1); ++mt)
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const float* t0 = T + (8 * ks + tq) * S + 16 * mt + g;  // A[g][tq] = T[q][ch]
        ahi[mt][ks][0] = to_tf32(t0[0]);
        ahi[mt][ks][1] = to_tf32(t0[8]);
        ahi[mt][ks][2] = to_tf32(t0[4 * S]);
        ahi[mt][ks][3] = to_tf32(t0[4 * S + 8]);
      }
    auto lo = [](float v) { return v - __uint_as_float(to_tf32(v)); };
    uint4* alo_w = reinterpret_cast<uint4*>(base + L::UNION);
#pragma unroll
    for (int mt = 0; mt < (MT ? MT : 1); ++mt)
#pragma unroll
      for (int ks2 = 0; ks2 < 2; ++ks2) {
        const float* u0 = T + (16 * ks2 + 2 * tq) * S + 16 * mt + g;
        uint4 a;
        a.x = pack_bf16(lo(u0[0]), lo(u0[S]));               // (g,   2tq | 2tq+1)
        a.y = pack_bf16(lo(u0[8]), lo(u0[S + 8]));           // (g+8, 2tq | 2tq+1)
        a.z = pack_bf16(lo(u0[8 * S]), lo(u0[9 * S]));       // (g,   2tq+8 | +9)
        a.w = pack_bf16(lo(u0[8 * S + 8]), lo(u0[9 * S + 8]));
        alo_w[(mt * 2 + ks2) * 32 + lane] = a;
      }
    __syncwarp();  // the tile region becomes the batch arrays
  }
  double eps_acc = 0.0;
  int nent = 0;

  // D[slot][entry] += A . W^T over the 32 queries for a batch of <= 8 entries
  // (columns >= nent hold stale weights; they only reach columns never read)
  auto tc_product = [&](const float* wbase, float (&d)[MT ? MT : 1][4]) {
#pragma unroll
    for (int mt = 0; mt < (MT ? MT : 1); ++mt) d[mt][0] = d[mt][1] = d[mt][2] = d[mt][3] = 0.f;
    const float* wrow = wbase + g * WS;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const float b0 = wrow[8 * ks + tq], b1 = wrow[8 * ks + tq + 4];
      // truncating split, the residual read by the tensor core at tf32 precision
      const uint32_t h0 = __float_as_uint(b0) & 0xffffe000u, h1 = __float_as_uint(b1) & 0xffffe000u;
      const uint32_t l0 = __float_as_uint(b0 - __uint_as_float(h0));
      const uint32_t l1 = __float_as_uint(b1 - __uint_as_float(h1));
#pragma unroll
      for (int mt = 0; mt < (MT ? MT : 1); ++mt) {
        mma_tf32(d[mt], ahi[mt][ks], h0, h1);
        mma_tf32(d[mt], ahi[mt][ks], l0, l1);
      }
    }
#pragma unroll
    for (int ks2 = 0; ks2 < 2; ++ks2) {
      const float2 p0 = *reinterpret_cast<const float2*>(wrow + 16 * ks2 + 2 * tq);
      const float2 p1 = *reinterpret_cast<const float2*>(wrow + 16 * ks2 + 2 * tq + 8);
      const uint32_t b0 = pack_bf16(p0.x, p0.y), b1 = pack_bf16(p1.x, p1.y);
#pragma unroll
      for (int mt = 0; mt < (MT ? MT : 1); ++mt) mma_bf16(d[mt], alo[(mt * 2 + ks2) * 32 + lane], b0, b1);
    }
  };

  auto evaluate = [&]() {
    cp_async_wait_all();
    __syncwarp();
    if constexpr (!FF) {
      float d[MT ? MT : 1][4];
      tc_product(wR, d);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int e = 2 * tq + j;
        double* dst = dptr[e];  // stale beyond nent: those REDs are predicated off
#pragma unroll
        for (int mt = 0; mt < (MT ? MT : 1); ++mt) {
          const int c = 16 * mt + g;
          red_add_f32_if(dst + c, d[mt][j], e < nent && c < nr);
          red_add_f32_if(dst + c + 8, d[mt][2 + j], e < nent && c + 8 < nr);
        }
      }
      // radial epsilon terms (:379, :409) for entries with a lane within 6.5 eps
      const unsigned nb = __ballot_sync(FULL_MASK, lane < nent && ((meta[lane & 7] >> 29) & 1));
      if (nb) {
        tc_product(wE, d);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int e = 2 * tq + j;
          if ((nb >> e) & 1u) {
            const float* rad = reinterpret_cast<const float*>(rows + e * F4 + 1);
#pragma unroll
            for (int mt = 0; mt < (MT ? MT : 1); ++mt) {
              const int c = 16 * mt + g;
              if (c < nr) eps_acc += (double)(d[mt][j] * rad[c]);
              if (c + 8 < nr) eps_acc += (double)(d[mt][2 + j] * rad[c + 8]);
            }
          }
        }
      }
    }
    // NG == 3: channel group 2 (16 channels) of two consecutive entries shares one
    // exchange and one full-warp RED: half 0 completes the even entry, half 1 the odd
    float sg2_prev = 0.f;
    double* dst_prev = nullptr;
#pragma unroll 2
    for (int e = 0; e < nent; ++e) {
      const int m = meta[e];
      if constexpr (FF && !VR) {
        const float4* wr4 = reinterpret_cast<const float4*>(wR + e * WS + 16 * hw);
        // even / odd query partial sums on the packed FMA pipe (FFMA2)
        float2 p[NG];
#pragma unroll
        for (int k = 0; k < NG; ++k) p[k] = make_float2(0.f, 0.f);
#pragma unroll
        for (int i4 = 0; i4 < 4; ++i4) {
          const float4 ww = wr4[i4];
#pragma unroll
          for (int k = 0; k < NG; ++k) {
            fma2(p[k], make_float2(ww.x, ww.y), make_float2(col[k][4 * i4], col[k][4 * i4 + 1]));
            fma2(p[k], make_float2(ww.z, ww.w), make_float2(col[k][4 * i4 + 2], col[k][4 * i4 + 3]));
          }
        }
        float sg[NG];
#pragma unroll
        for (int k = 0; k < NG; ++k) sg[k] = p[k].x + p[k].y;
        // half 0 completes groups 0 (and 2), half 1 groups 1 (and 3): each lane
        // sends the partial its partner completes, so group pair (0, 1) ends as
        // channel `lane` in lane `lane`
        const float t01 = (hw ? sg[1] : sg[0]) + __shfl_xor_sync(FULL_MASK, hw ? sg[0] : sg[1], 16);
        double* dst_s = dptr[e];
        if (NB > 0)  // nr > 32: every lane owns a channel; no predicate, no branch
          red_add_f32(dst_s + lane, t01);
        else
          red_add_f32_if(dst_s + lane, t01, lane < nr && t01 != 0.f);
        if constexpr (NG == 3) {
          if (e & 1) {  // own partial + the partner's, as the one-entry form: the same sums
            const float mine = hw ? sg[2] : sg2_prev;
            const float t2 = mine + __shfl_xor_sync(FULL_MASK, hw ? sg2_prev : sg[2], 16);
            red_add_f32_if((hw ? dst_s : dst_prev) + 32 + g16, t2, okg[2] && t2 != 0.f);
          } else {
            sg2_prev = sg[2];
            dst_prev = dst_s;
          }
        }
        if constexpr (NG == 4) {
          const float t23 = (hw ? sg[NG - 1] : sg[2]) +
                            __shfl_xor_sync(FULL_MASK, hw ? sg[2] : sg[NG - 1], 16);
          red_add_f32_if(dst_s + 32 + lane, t23, 32 + lane < nr && t23 != 0.f);
        }
      }
    }
    if constexpr (FF && !VR && NG == 3) {
      if (nent & 1) {  // the last entry of an odd batch has no partner
        const float t2 = sg2_prev + __shfl_xor_sync(FULL_MASK, sg2_prev, 16);
        red_add_f32_if(dst_prev + 32 + g16, t2, hw == 0 && okg[2] && t2 != 0.f);
      }
    }
    if constexpr (FF && !VR) {
      // radial epsilon terms (:379, :409) of the batch's near entries, out of
      // the main loop so it carries no per-entry branch
      unsigned nm = __ballot_sync(FULL_MASK, lane < nent && ((meta[lane & (ENT - 1)] >> 29) & 1));
      while (nm) {
        const int e = __ffs(nm) - 1;
        nm &= nm - 1;
        const float4* we4 = reinterpret_cast<const float4*>(wE + e * WS + 16 * hw);
        float ev[NG];
#pragma unroll
        for (int k = 0; k < NG; ++k) ev[k] = 0.f;
#pragma unroll
        for (int i4 = 0; i4 < 4; ++i4) {
          const float4 ww = we4[i4];
          const float wv[4] = {ww.x, ww.y, ww.z, ww.w};
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int k = 0; k < NG; ++k) ev[k] = fmaf(wv[u], col[k][4 * i4 + u], ev[k]);
        }
        // each half's partial sum times the channel's moment: no cross-half step
        // (eps_acc is reduced over the warp at the end)
        const float* rad = reinterpret_cast<const float*>(rows + e * F4 + 1);
#pragma unroll
        for (int k = 0; k < NG; ++k)
          if (okg[k]) eps_acc += (double)(ev[k] * rad[16 * k + g16]);
      }
    }
    // vector quantities of the whole batch: lane L sums pair (e, k) = (L / VQ, L % VQ)
    // of vq[e][k][0..31] (8 LDS.128, rotated by L so the 8 lanes of each phase
    // hit distinct bank groups) and issues at most one RED
    for (int p0 = 0; p0 < VQ * nent; p0 += 32) {
      const int pr = p0 + lane;
      if (pr < VQ * nent) {
        const float4* row = reinterpret_cast<const float4*>(vq + pr * 32);
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 v4 = row[(j + lane) & 7];
          s += (v4.x + v4.y) + (v4.z + v4.w);
        }
        const int e = pr / VQ, k = pr % VQ;  // 0..2 vector, 3 = d mu_0, 4.. radial (VR)
        const int m = meta[e];
        const bool is_point = m & (1 << 30);
        const int64_t src = m & ((1 << 29) - 1);
        double* dst = is_point ? (k < 3 ? acc.pt_n + 3 * src + k : acc.pt_mud + src)
                               : acc.node_v + 3 * src + k;
        bool use = is_point || k < 3;
        if (VR && k >= 4) {
          dst = (is_point ? acc.pt_mur : acc.node_s) + src * Cr + (k - 4);
          use = k - 4 < nr;
        }
        red_add_if(dst, (double)s, s != 0.f && use);
      }
    }
    __syncwarp();
    nent = 0;
  };

  // VR: the radial epsilon terms (:379, :409) of a lane within 6.5 eps, from the
  // source's first radial float4 (called inside the near-field branches only)
  auto vr_eps = [&](float e_, const float4* row) {
    const float4 rad = __ldg(row + 1);
    eps_acc += (double)(e_ * fmaf(dsr[0], rad.x, fmaf(dsr[1], rad.y,
                                                        fmaf(dsr[2], rad.z, dsr[3] * rad.w))));
  };
  // VR: this lane's slots of the current entry — vector terms, d mu_0 (points),
  // and the radial products A R ds_c
  auto vr_store = [&](float r_, float v0, float v1, float v2, float v3, bool point) {
    float* vqe = vq + nent * 32 * VQ;
    vqe[lane] = v0, vqe[32 + lane] = v1, vqe[64 + lane] = v2;
    if (point) vqe[96 + lane] = v3;  // slot 3 is never read for nodes
    vqe[128 + lane] = r_ * dsr[0], vqe[160 + lane] = r_ * dsr[1];
    vqe[192 + lane] = r_ * dsr[2];
    if (nr > 3) vqe[224 + lane] = r_ * dsr[3];  // slot 7 is read only when nr == 4
  };

  auto begin_entry = [&]() {
    if (nent == ENT) evaluate();
  };

  // far-field lane values beyond 6.5 eps (tau = 1: W = R / r, Wp_r = -3 W R, no
  // epsilon terms; kernels.cpp:50-55), branch-free: every lane evaluates,
  // non-far lanes select 0 (bhtree.cpp:361-376)
  // REG: one select on the area instead of one per value (rsqrt_far keeps the
  // non-member lanes finite, kept lanes are bit-identical)
  auto far_fast = [&](float A, float s, float fx, float fy, float fz, bool far, float& r_,
                      float& u0, float& u1, float& u2) {
    if (REG) {
      const float Am = sel0(far, A);
      const float inv_r = rsqrt_far(s, kp.near2);
      const float R = inv_r * inv_r;
      r_ = Am * R;
      if (GM == 0) {
        const float aWds = Am * (R * inv_r) * ds0;
        u0 = aWds * fx, u1 = aWds * fy, u2 = aWds * fz;
      } else {  // with the query-gradient adjoint d_grad (:372-376)
        const float W = R * inv_r;
        const float Wp_r = -3.0f * W * R;
        const float aWds = Am * W * ds0;
        const float gd = fmaf(dg0, fx, fmaf(dg1, fy, dg2 * fz));
        const float t = Wp_r * gd;
        u0 = aWds * fx - Am * fmaf(W, dg0, t * fx);
        u1 = aWds * fy - Am * fmaf(W, dg1, t * fy);
        u2 = aWds * fz - Am * fmaf(W, dg2, t * fz);
      }
      return;
    }
    const float inv_r = rsqrt_pos(s);
    const float R = inv_r * inv_r;
    r_ = sel0(far, A * R);
    if (GM == 0) {
      const float aWds = A * (R * inv_r) * ds0;
      u0 = sel0(far, aWds * fx), u1 = sel0(far, aWds * fy), u2 = sel0(far, aWds * fz);
    } else {  // with the query-gradient adjoint d_grad (:372-376)
      const float W = R * inv_r;
      const float Wp_r = -3.0f * W * R;
      const float aWds = A * W * ds0;
      const float gd = fmaf(dg0, fx, fmaf(dg1, fy, dg2 * fz));
      const float t = Wp_r * gd;
      u0 = sel0(far, aWds * fx - A * fmaf(W, dg0, t * fx));
      u1 = sel0(far, aWds * fy - A * fmaf(W, dg1, t * fy));
      u2 = sel0(far, aWds * fz - A * fmaf(W, dg2, t * fz));
    }
  };

  // one far source (node) for the lanes in `far` (bhtree.cpp:361-381).
  // hint: the list's NEAR flag (0: no far lane needs the series, 1: some may),
  // -1 on the tree walk (decided by a vote)
  auto far_entry = [&](int node, float A, float s, float fx, float fy, float fz, bool far,
                       int hint) {
    begin_entry();
    float r_ = 0.f, e_ = 0.f, u0 = 0.f, u1 = 0.f, u2 = 0.f;
    bool nr_ = false;
    if (GM == 0) {
      // far lanes beyond 6.5 eps (or singular): tau = 1, no epsilon terms
      // (kernels.cpp:50-55); the coefficient series only under a warp-uniform
      // branch, so a batch without near lanes never issues it
      const bool slow = far && !(kp.mode == KM_SINGULAR ||
                                 (kp.mode == KM_REGULARIZED && s >= kp.near2));
      far_fast(A, s, fx, fy, fz, far, r_, u0, u1, u2);
      if (hint != 0 && (hint > 0 || __any_sync(FULL_MASK, slow))) {
        if (slow) {
          const Co c = coeffs<2>(s, kp);
          nr_ = c.near;
          r_ = A * c.R;
          e_ = A * c.dR_de;
          if (VR && e_ != 0.f) vr_eps(e_, tv.node_row + (size_t)node * F4g);
          const float aWds = A * c.W * ds0;
          u0 = aWds * fx, u1 = aWds * fy, u2 = aWds * fz;
          if (c.near) {
            const float4 v = __ldg(tv.node_row + (size_t)node * F4g);
            const float vd = fmaf(v.x, fx, fmaf(v.y, fy, v.z * fz));
            eps_acc += (double)(ds0 * A * c.dW_de * vd);  // :370
          }
        }
      }
    } else {
      // d_grad present (render path). Far lanes beyond 6.5 eps: tau = 1, so
      // W = R / r, Wp_r = -3 W R and every epsilon term vanishes (the moment row
      // is not even read); the series and the epsilon terms run under a
      // warp-uniform branch for the near lanes only
      const bool slow = far && !(kp.mode == KM_SINGULAR ||
                                 (kp.mode == KM_REGULARIZED && s >= kp.near2));
      far_fast(A, s, fx, fy, fz, far, r_, u0, u1, u2);
      if (hint != 0 && (hint > 0 || __any_sync(FULL_MASK, slow))) {
        if (slow) {
          const Co c = adj_coeffs<GM>(s, kp);
          nr_ = c.near;
          r_ = A * c.R;
          e_ = A * c.dR_de;
          if (VR && e_ != 0.f) vr_eps(e_, tv.node_row + (size_t)node * F4g);
          const float aWds = A * c.W * ds0;
          u0 = aWds * fx, u1 = aWds * fy, u2 = aWds * fz;
          const float4 v = __ldg(tv.node_row + (size_t)node * F4g);
          const float vd = fmaf(v.x, fx, fmaf(v.y, fy, v.z * fz));
          float e = ds0 * A * c.dW_de * vd;  // :370
          const float gd = fmaf(dg0, fx, fmaf(dg1, fy, dg2 * fz));  // :372-374
          const float t = c.Wp_r * gd;
          u0 -= A * fmaf(c.W, dg0, t * fx);
          u1 -= A * fmaf(c.W, dg1, t * fy);
          u2 -= A * fmaf(c.W, dg2, t * fz);
          const float k2 = c.dWp_r_de * vd;
          e -= A * fmaf(dg0, fmaf(c.dW_de, v.x, k2 * fx),
                        fmaf(dg1, fmaf(c.dW_de, v.y, k2 * fy), dg2 * fmaf(c.dW_de, v.z, k2 * fz)));
          eps_acc += (double)e;
        }
      }
    }
    if constexpr (VR) {
      vr_store(r_, u0, u1, u2, 0.f, false);
      meta[nent] = node;  // every lane stores the same word: no branch
      ++nent;
      return;
    }
    wR[nent * WS + lane] = r_;
    float* vqe = vq + nent * 128;
    vqe[lane] = u0, vqe[32 + lane] = u1, vqe[64 + lane] = u2;  // slot 3 (d mu_0) is never read for nodes
    const bool any_near = hint != 0 && __any_sync(FULL_MASK, nr_);
    if (any_near) {  // warp-uniform; rare beyond the first tree levels
      wE[nent * WS + lane] = e_;  // read by phase B for near entries only
      if (lane < F4c) cp_async16(s_rows + 16u * F4 * nent, tv.node_row + (size_t)node * F4g + lane);
    }
    // every lane stores the same words: no branch
    meta[nent] = node | (any_near ? (1 << 29) : 0);
    dptr[nent] = acc.node_s + (size_t)node * Cr;
    ++nent;
  };
  // K consecutive list entries r[0..K): far nodes whose far lanes are all beyond
  // 6.5 eps — far_entry's fast path for each, interleaved
  auto far_group = [&](const NodeRec* r, auto kc) {
    constexpr int K = decltype(kc)::value;
    float s[K], fx[K], fy[K], fz[K], A[K];
    bool f[K];
    int nd[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int4 t = r[k].topo;
      const float4 h = r[k].hi, l = r[k].lo;
      s[k] = dist2_df(h, l, qx, fx[k], fy[k], fz[k]);
      f[k] = ((unsigned)t.y >> lane) & 1u;
      nd[k] = t.x & IL_NODE;
      A[k] = l.w;
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      float r_, u0, u1, u2;
      far_fast(A[k], s[k], fx[k], fy[k], fz[k], f[k], r_, u0, u1, u2);
      if constexpr (VR) {
        vr_store(r_, u0, u1, u2, 0.f, false);
        meta[nent] = nd[k];
      } else {
        wR[nent * WS + lane] = r_;
        float* v = vq + nent * 128;
        v[lane] = u0, v[32 + lane] = u1, v[64 + lane] = u2;
        meta[nent] = nd[k];
        dptr[nent] = acc.node_s + (size_t)nd[k] * Cr;
      }
      ++nent;
    }
    if (nent == ENT) evaluate();  // keeps the nent + K <= ENT checks cheap
  };
  // the points of an opened leaf for the lanes in `me_open` (:382-412)
  auto leaf_points = [&](const int4 tp, bool me_open) {
    for (int j = tp.z; j < tp.w; ++j) {
      begin_entry();
      float r_ = 0.f, e_ = 0.f, n0 = 0.f, n1 = 0.f, n2 = 0.f, dmu = 0.f;
      bool nr_ = false;
      if (me_open) {
        const PtRec* pr = tv.pt_rec + j;
        const float4 ph = __ldg(&pr->hi);
        float fx, fy, fz;
        const float r2 = dist2_df(ph, __ldg(&pr->lo), qx, fx, fy, fz);
        // :387 skips exact coincidence (fp64); fp32 r2 == 0 triggers the exact check
        if (!(r2 == 0.f && coincident_exact(tv.pt_pos64 + 3 * (size_t)j, xq))) {
          const Co c = adj_coeffs<GM>(r2, kp);
          const float Am = ph.w;
          nr_ = c.near;
          r_ = Am * c.R;
          e_ = Am * c.dR_de;
          if (VR && e_ != 0.f) vr_eps(e_, tv.pt_row + (size_t)j * F4g);
          const float mu = __ldg(tv.pt_mu + j);
          const float nx = __ldg(tv.pt_nrm + 3 * (size_t)j), ny = __ldg(tv.pt_nrm + 3 * (size_t)j + 1),
                      nz = __ldg(tv.pt_nrm + 3 * (size_t)j + 2);
          const float nu = fmaf(nx, fx, fmaf(ny, fy, nz * fz));
          const float aW = Am * c.W;
          dmu = ds0 * aW * nu;
          const float sc = ds0 * aW * mu;
          n0 = sc * fx, n1 = sc * fy, n2 = sc * fz;
          float e = ds0 * Am * mu * c.dW_de * nu;
          if (GM) {
            const float gd = fmaf(dg0, fx, fmaf(dg1, fy, dg2 * fz));
            const float gn = fmaf(dg0, nx, fmaf(dg1, ny, dg2 * nz));
            dmu -= Am * fmaf(c.W, gn, c.Wp_r * nu * gd);
            const float am = Am * mu, t = c.Wp_r * gd;
            n0 -= am * fmaf(c.W, dg0, t * fx);
            n1 -= am * fmaf(c.W, dg1, t * fy);
            n2 -= am * fmaf(c.W, dg2, t * fz);
            e -= am * fmaf(c.dW_de, gn, c.dWp_r_de * nu * gd);
          }
          eps_acc += (double)e;
        }
      }
      if constexpr (VR) {
        vr_store(r_, n0, n1, n2, dmu, true);
        meta[nent] = j | (1 << 30);
        ++nent;
        continue;
      }
      wR[nent * WS + lane] = r_;
      float* vqe = vq + nent * 128;
      vqe[lane] = n0, vqe[32 + lane] = n1, vqe[64 + lane] = n2, vqe[96 + lane] = dmu;
      const bool any_near = __any_sync(FULL_MASK, nr_);
      if (any_near) {
        wE[nent * WS + lane] = e_;
        if (lane < F4c) cp_async16(s_rows + 16u * F4 * nent, tv.pt_row + (size_t)j * F4g + lane);
      }
      meta[nent] = j | (1 << 30) | (any_near ? (1 << 29) : 0);
      dptr[nent] = acc.pt_mur + (size_t)j * Cr;
      ++nent;
    }
  };
  const int64_t wg = (int64_t)blockIdx.x * WARPS + w;
  const int total = LIST ? __ldg(lv.count + wg) : -1;
  if (LIST && total >= 0) {
    // replay the interaction list (ilist.cuh): 32 entries at a time, their node
    // records prefetched into the (unused) stack region with cp.async
    NodeRec* rb = reinterpret_cast<NodeRec*>(stk);
    const uint32_t s_rb = smem_u32(stk) + 48u * lane;
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
      }
      cp_async_wait_all();
      // the entry itself goes into its record's unused child fields (topo.x/y;
      // the replay reads only the point range z/w): one broadcast LDS.128 per
      // entry instead of two shuffles
      if (lane < n) *reinterpret_cast<uint2*>(&rb[lane].topo) = my;
      __syncwarp();
      for (int i = 0; i < n;) {
        const int4 tpi = rb[i].topo;
        const uint32_t src = (uint32_t)tpi.x;
        if constexpr (true) {  // FFMA and tensor-core phase B alike
          // two consecutive far entries without near lanes that fit the batch:
          // one interleaved pass (independent dependency chains for the
          // scheduler; groups of 4 measured no faster); batches fill exactly as
          // on the tree walk, so results stay bitwise those of the walk
          if (nent + 2 <= ENT && i + 1 < n &&
              !((src | (uint32_t)rb[i + 1].topo.x) & (IL_LEAF | IL_NEAR))) {
            far_group(rb + i, std::integral_constant<int, 2>{});
            i += 2;
            continue;
          }
        }
        const unsigned m = (unsigned)tpi.y;
        const bool mine = (m >> lane) & 1u;
        if (!(src & IL_LEAF)) {
          const float4 hi = rb[i].hi, lo = rb[i].lo;
          float fx, fy, fz;
          const float s = dist2_df(hi, lo, qx, fx, fy, fz);
          far_entry((int)(src & IL_NODE), lo.w, s, fx, fy, fz, mine, (src & IL_NEAR) ? 1 : 0);
        } else {
          leaf_points(tpi, mine);
        }
        ++i;
      }
    }
  }
  int sp = (LIST && total >= 0) ? 0 : 1;
  if (sp && lane == 0) stk[0] = make_int2(0, (int)active);
  __syncwarp();
  while (sp > 0) {
    --sp;
    const int2 en = stk[sp];
    __syncwarp();
    const int node = en.x;
    const unsigned mask = (unsigned)en.y;
    const bool mine = (mask >> lane) & 1u;
    const NodeRec* rec = tv.node_rec + node;
    const float4 hi = __ldg(&rec->hi);
    const float4 lo = __ldg(&rec->lo);
    const int4 tp = __ldg(&rec->topo);
    const float A = lo.w;
    float fx, fy, fz;
    const float s = dist2_df(hi, lo, qx, fx, fy, fz);
    const bool far = mine && far_test(s, hi, qx, xq, tv.node_dec + node);
    const unsigned farm = __ballot_sync(FULL_MASK, far);
    if (farm && A > 0.f) {
      far_entry(node, A, s, fx, fy, fz, far, -1);
    }
    const unsigned openm = mask & ~farm;
    if (openm) {
      if (tp.y == 0) {
        leaf_points(tp, (openm >> lane) & 1u);
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
  if (nent) evaluate();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) eps_acc += __shfl_xor_sync(FULL_MASK, eps_acc, o);
  if (lane == 0 && eps_acc != 0.0) atomicAdd(acc.d_eps, eps_acc);
}

template <int NB, int GM, int RR, int WARPS, int ENT, int MAXR, int MT, bool LIST, bool REG>
static void launch_adj2c(const Tree& t, const KParams& kp, const AdjArgs& a, GradBuf& b, int nr,
                         IListView lv) {
  const size_t smem = (size_t)WARPS * AdjLayout<MT, ENT, RR, NB == 3>::WARP_FLOATS * 4;
  static std::atomic<unsigned long long> attr{0};
  ensure_max_dyn_smem(k_adjoint2<NB, GM, WARPS, ENT, RR, MAXR, MT, LIST, REG>, t.device, smem, attr);
  Adj2Ptrs p{b.node_v, b.node_s, b.pt_mud, b.pt_mur, b.pt_n, b.d_eps};
  unsigned blocks = (unsigned)((a.q + WARPS * 32 - 1) / (WARPS * 32));
  k_adjoint2<NB, GM, WARPS, ENT, RR, MAXR, MT, LIST, REG><<<blocks, WARPS * 32, smem, t.stream>>>(
      t.view(), kp, a.xs, a.perm, a.q, a.d_out, a.dstride, a.d_grad, nr, t.chmap.as<int>(), p, lv,
      a.overflow);
  count_launch();
}

// builds (or reuses) the interaction lists when the caller provides the workspace
// SPEC: also instantiate the regularized-mode kernels (production configurations)
template <int NB, int GM, int RR, int WARPS = 4, int ENT = 8, int MAXR = 128, int MT = 0,
          bool SPEC = false>
static void launch_adj2(const Tree& t, const KParams& kp, const AdjArgs& a, GradBuf& b, int nr) {
  const bool reg = SPEC && kp.mode == KM_REGULARIZED && kp.near2 >= REG_MIN_NEAR2;
  if (a.ilist && !no_ilist()) {
    ilist_build(t, *a.ilist, a.xs, a.perm, a.q, a.beta, ilist_near_thr(kp), a.overflow);
    if (reg)
      launch_adj2c<NB, GM, RR, WARPS, ENT, MAXR, MT, true, SPEC>(t, kp, a, b, nr, a.ilist->view());
    else
      launch_adj2c<NB, GM, RR, WARPS, ENT, MAXR, MT, true, false>(t, kp, a, b, nr, a.ilist->view());
  } else if (reg) {
    launch_adj2c<NB, GM, RR, WARPS, ENT, MAXR, MT, false, SPEC>(t, kp, a, b, nr, IListView{});
  } else {
    launch_adj2c<NB, GM, RR, WARPS, ENT, MAXR, MT, false, false>(t, kp, a, b, nr, IListView{});
  }
}

template <int GM>
static bool adj2_plan(const Tree& t, const KParams& kp, const AdjArgs& a, GradBuf& b) {
  const int nr = a.nr_limit >= 0 ? std::min(a.nr_limit, t.Cr) : t.Cr;
  // Tensor-core phase B: correct (parity-tested) but measured SLOWER on config 2
  // (34.9-36.6 ms vs 29.2 ms FFMA: the 48 A_hi registers push the traversal
  // into spills or lower occupancy) -> opt-in experiment.
  static const bool tc = getenv("DPL_ADJOINT_TC") != nullptr;
  if (tc) {  // rows staged up to the slots used
    if (nr <= 16) return launch_adj2<0, GM, 4, 4, 8, 128, 1, true>(t, kp, a, b, nr), true;
    if (nr <= 32) return launch_adj2<0, GM, 8, 4, 8, 128, 2, true>(t, kp, a, b, nr), true;
    // best measured (warps, register cap) for the 48-channel tile: 2 warps at 160
    // (2 at 144 / 136 and 4 at 128 spill and run slower)
    if (nr <= 48) return launch_adj2<0, GM, 12, 2, 8, 160, 3, true>(t, kp, a, b, nr), true;
  }
  if (t.F4 - 1 > 16) return false;
  if (nr <= 4) return launch_adj2<3, GM, 1, 4, 8, 96, 0, true>(t, kp, a, b, nr), true;
  if (nr <= 32) return launch_adj2<0, GM, 16, 4, 8, 128, 0, true>(t, kp, a, b, nr), true;
  if (nr <= 48) return launch_adj2<1, GM, 16, 4, 8, 128, 0, true>(t, kp, a, b, nr), true;
  if (nr <= 64) return launch_adj2<2, GM, 16>(t, kp, a, b, nr), true;
  return false;
}

bool adjoint2_launch(const Tree& t, const KParams& kp, const AdjArgs& a, GradBuf& b) {
  if (t.Cd != 1 || t.Cr > 64) return false;
  if (a.grad_mode == 0) return adj2_plan<0>(t, kp, a, b);
  if (a.grad_mode == 1) return adj2_plan<1>(t, kp, a, b);
  return adj2_plan<2>(t, kp, a, b);
}

}  // namespace dpl
