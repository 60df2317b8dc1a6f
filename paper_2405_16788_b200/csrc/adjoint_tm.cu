// adjoint_tm.cu — adjoint traversal (K7) with the radial channel product on the
// 5th-generation tensor cores (tcgen05.mma, accumulators in tensor memory).
//
// Same semantics as k_adjoint2 (adjoint2.cu; DipoleTree::adjoint,
// proj/src/bhtree.cpp:345-417) for the SceneModel layout with 4 < Cr <= 48
// radial channels. Per far source / leaf point t and radial channel c the
// adjoint adds (bhtree.cpp:377-381, :407-411)
//     node_s[t, c] (or point_mu[m, c]) += sum_l  w[l] ds[l, c]
// over the 32 queries l of a warp, w[l] = A R(|x_l - c_t|) for member lanes and
// 0 otherwise. That is, per warp, the matrix product
//     D[c][t] = sum_l  dsT[c][l] . w[t][l]          (48 x T) = (48 x 32) (32 x T)
// whose left operand (the warp's transposed upstream-gradient tile) is constant
// for the whole traversal. k_adjoint2 keeps that tile in 48 registers and
// spends 24 FFMA2 + 12 LDS.128 per source on the product; here
//   * the tile lives in shared memory as a K-major SWIZZLE_128B tcgen05 operand
//     (tf32 hi / lo parts, 2 x 6 KB per warp), written once;
//   * the 4 PRODUCER warps of a CTA run phase A only (lanes = queries: opening
//     decisions from the interaction list, coefficients, the dipole vector
//     terms) and write each source's weights as one row of a B tile (16 rows =
//     16 sources, tf32 hi / lo, double-buffered);
//   * a full tile is multiplied by ONE lane with 12 tcgen05.mma (M = 64, N = 16,
//     K = 8, kind::tf32; hi.hi + hi.lo + lo.hi per k-step: fp32-class products)
//     into a 16-column TMEM accumulator, committed to an mbarrier;
//   * 3 EPILOGUE warps (TMEM lane quadrants 0..2 = channels 16 q .. 16 q + 15)
//     read the accumulator with tcgen05.ld and issue the fp64 REDs (one
//     128-byte RED per source and quadrant), then hand the buffer back.
// The radial epsilon terms (:379, :409) of sources with a lane inside 6.5 eps
// ride along as one more tile row (weights A dR_de), whose accumulator column
// the epilogue dots with the source's moment row instead of adding it.
// Producers never wait for the tensor core or the REDs unless both of their
// buffers are in flight. Accumulators are fp64 (SURVEY §7 hard part 4).
#include <type_traits>

#include "adjoint.cuh"
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

template <int GM>
__device__ __forceinline__ Co adj_coeffs_tm(float r2, const KParams& kp) {
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

constexpr int TM_PROD = 4;    // producer warps per CTA
constexpr int TM_EPI = 3;     // epilogue warps (quadrants 0..2: channels 0..47)
constexpr int TM_N = 16;      // sources per B tile = accumulator columns
constexpr int TM_VQ = 8;      // sources per vector-quantity batch
constexpr int TM_ROWS = 48;   // radial channel rows of the A tile
constexpr uint32_t TM_COLS = TM_PROD * 2 * TM_N;  // TMEM columns per CTA (128)

// per producer warp (bytes); every tile starts on a 1024-byte boundary. The
// M = 64 MMA reads 16 rows past each 48-row A tile: A_lo after A_hi, the first
// B tile after A_lo — finite or not, those rows only reach TMEM lanes that are
// never read (accumulator rows are independent).
constexpr uint32_t TM_A_HI = 0;
constexpr uint32_t TM_A_LO = TM_ROWS * 128;                 // 6144
constexpr uint32_t TM_B = 2 * TM_ROWS * 128;                // 12288: [buf][hi | lo] x 2 KB
constexpr uint32_t TM_VQO = TM_B + 2 * 2 * TM_N * 128;      // 20480: vq[8][4][32] floats
constexpr uint32_t TM_RB = TM_VQO + TM_VQ * 4 * 32 * 4;     // 24576: node records / stack
constexpr uint32_t TM_RBSZ = DPL_STACK_PER_WARP * 8 > 32 * 48 ? DPL_STACK_PER_WARP * 8 : 32 * 48;
constexpr uint32_t TM_DP = TM_RB + TM_RBSZ;                 // dptr[2][16]
constexpr uint32_t TM_META = TM_DP + 2 * TM_N * 8;          // meta[8], ncols[2]
constexpr uint32_t TM_WARP = 27648;                         // 27 KB
static_assert(TM_META + (TM_VQ + 2) * 4 <= TM_WARP, "per-warp layout");
static_assert(TM_DP % 16 == 0, "destination rows are read as 16-byte pairs");
static_assert(TM_WARP % 1024 == 0 && TM_B % 1024 == 0, "tile alignment");
}  // namespace

struct AdjTmPtrs {
  double* node_v;
  double* node_s;
  double* pt_mud;
  double* pt_mur;
  double* pt_n;
  double* d_eps;
};

// GM: 0 no d_grad; 1 d_grad q x dstride x 3; 2 d_grad q x 3 (channel 0).
// LIST: replay the interaction lists (warps with an incomplete list walk the tree).
// REG: compiled for the regularized kernel with (6.5 eps)^2 >= REG_MIN_NEAR2.
template <int GM, bool LIST, bool REG>
__global__ void __launch_bounds__((TM_PROD + TM_EPI) * 32, 2)
    k_adjoint_tm(TreeView tv, KParams kp_in, const double* __restrict__ xs,
                 const int32_t* __restrict__ perm, int64_t q, const float* __restrict__ d_out,
                 int dstride, const float* __restrict__ d_grad, int nr,
                 const int* __restrict__ chmap, AdjTmPtrs acc, IListView lv, int* overflow) {
  using namespace tc05;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full_bar[TM_PROD][2], empty_bar[TM_PROD][2];
  __shared__ uint32_t tmem_slot;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;

  if (w == TM_PROD) tmem_alloc<TM_COLS>(&tmem_slot);
  if (threadIdx.x == 0) {
    for (int i = 0; i < TM_PROD; ++i)
      for (int b = 0; b < 2; ++b) {
        mbar_init(smem_addr(&full_bar[i][b]), 2);  // tcgen05.commit + the producer's release
        mbar_init(smem_addr(&empty_bar[i][b]), TM_EPI);
      }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_slot;

  if (w >= TM_PROD) {
    // ------------------------------------------------------------- epilogue
    const int qd = w - TM_PROD;  // TMEM lane quadrant (w % 4) = channel group
    const int c = 16 * qd + lane;
    const bool ok = lane < 16 && c < nr;
    double eps_acc = 0.0;
    unsigned alive = (1u << TM_PROD) - 1;
    int round[TM_PROD];
#pragma unroll
    for (int i = 0; i < TM_PROD; ++i) round[i] = 0;
    while (alive) {
#pragma unroll
      for (int i = 0; i < TM_PROD; ++i) {
        if (!((alive >> i) & 1u)) continue;
        const int r = round[i], b = r & 1;
        mbar_wait(smem_addr(&full_bar[i][b]), (r >> 1) & 1);
        fence_after();
        const uint8_t* wb = sm + (size_t)i * TM_WARP;
        const int word = reinterpret_cast<const int*>(wb + TM_META)[TM_VQ + b];
        const int n = word & 0xff;
        const unsigned emask = (unsigned)word >> 16;  // columns holding epsilon weights
        if (n > 0 && 16 * qd < nr) {
          float v[16];
          tmem_ld16(tmem + ((uint32_t)(32 * qd) << 16) + (uint32_t)((2 * i + b) * TM_N), v);
          // the 16 destination rows with 8 broadcast LDS.128, then 16 predicated
          // REDs back to back (no per-column branch)
          const ulonglong2* dp2 = reinterpret_cast<const ulonglong2*>(wb + TM_DP) + b * (TM_N / 2);
          unsigned long long d[TM_N];
#pragma unroll
          for (int j = 0; j < TM_N / 2; ++j) {
            const ulonglong2 t2 = dp2[j];
            d[2 * j] = t2.x, d[2 * j + 1] = t2.y;
          }
          const unsigned live = ok ? (((1u << n) - 1u) & ~emask) : 0u;
#pragma unroll
          for (int j = 0; j < TM_N; ++j)
            red_add_f32_if(reinterpret_cast<double*>(d[j]) + c, v[j], (live >> j) & 1u);
          if (emask) {  // radial epsilon terms: dot with the source's moment row (rare)
#pragma unroll
            for (int j = 0; j < TM_N; ++j)
              if (((emask >> j) & 1u) && ok)
                eps_acc += (double)(v[j] * __ldg(reinterpret_cast<const float*>(d[j]) + c));
          }
        }
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_addr(&empty_bar[i][b]));
        round[i] = r + 1;
        if (word & 0x100) alive &= ~(1u << i);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) eps_acc += __shfl_xor_sync(FULL_MASK, eps_acc, o);
    if (lane == 0 && eps_acc != 0.0) atomicAdd(acc.d_eps, eps_acc);
  } else {
    // ------------------------------------------------------------- producer
    KParams kp = kp_in;
    if (REG) kp.mode = KM_REGULARIZED;
    uint8_t* wb = sm + (size_t)w * TM_WARP;
    float* vq = reinterpret_cast<float*>(wb + TM_VQO);
    int2* stk = reinterpret_cast<int2*>(wb + TM_RB);
    unsigned long long* dptr = reinterpret_cast<unsigned long long*>(wb + TM_DP);
    int* meta = reinterpret_cast<int*>(wb + TM_META);
    const int F4g = tv.F4;
    const int Cr = tv.Cr;

    const int64_t sidx = ((int64_t)blockIdx.x * TM_PROD + w) * 32 + lane;
    const bool valid = sidx < q;
    const int64_t qi = valid ? (perm ? (int64_t)perm[sidx] : sidx) : 0;
    QueryPos x;
    if (valid) {
      x.x = xs[3 * qi], x.y = xs[3 * qi + 1], x.z = xs[3 * qi + 2];
    } else {
      x.x = x.y = x.z = 0.0;
    }
    const unsigned active = __ballot_sync(FULL_MASK, valid);
    const QueryDF qx = make_qdf(x, tv.cmax);
    const double* xq = xs + 3 * qi;

    const int ch0 = __ldg(chmap);
    const float ds0 = valid ? __ldg(d_out + qi * dstride + ch0) : 0.f;
    float dg0 = 0.f, dg1 = 0.f, dg2 = 0.f;
    if (GM && valid) {
      const float* g = GM == 1 ? d_grad + (qi * dstride + ch0) * 3 : d_grad + qi * 3;
      dg0 = g[0], dg1 = g[1], dg2 = g[2];
    }
    // the warp's transposed upstream-gradient tile A[channel][query] (tf32 hi / lo):
    // coalesced reads (lanes = channels of one query), rows >= nr zero
    {
      const bool okA = lane < nr, okB = lane < 16 && 32 + lane < nr;
      const int chA = okA ? __ldg(chmap + 1 + lane) : 0;
      const int chB = okB ? __ldg(chmap + 33 + lane) : 0;
#pragma unroll 4
      for (int l = 0; l < 32; ++l) {
        const int64_t ql = __shfl_sync(FULL_MASK, qi, l);
        const bool vl = (active >> l) & 1u;
        const float a = (okA && vl) ? __ldg(d_out + ql * dstride + chA) : 0.f;
        const uint32_t h = tf32_hi(a), o = sw_off((uint32_t)lane, (uint32_t)l);
        *reinterpret_cast<uint32_t*>(wb + TM_A_HI + o) = h;
        *reinterpret_cast<float*>(wb + TM_A_LO + o) = a - __uint_as_float(h);
        if (lane < 16) {
          const float b2 = (okB && vl) ? __ldg(d_out + ql * dstride + chB) : 0.f;
          const uint32_t h2 = tf32_hi(b2), o2 = sw_off((uint32_t)(32 + lane), (uint32_t)l);
          *reinterpret_cast<uint32_t*>(wb + TM_A_HI + o2) = h2;
          *reinterpret_cast<float*>(wb + TM_A_LO + o2) = b2 - __uint_as_float(h2);
        }
      }
    }
    const uint32_t s_a_hi = smem_addr(wb + TM_A_HI), s_a_lo = smem_addr(wb + TM_A_LO);
    const uint32_t s_b0 = smem_addr(wb + TM_B);
    const uint32_t lane4 = 4u * (uint32_t)lane;
    constexpr uint32_t IDESC = idesc_tf32(64, TM_N);

    double eps_acc = 0.0;
    int ncol = 0, nvq = 0, kb = 0;
    unsigned emask = 0;  // tile rows holding epsilon weights (A dR_de)
    uint8_t* bt = wb + TM_B;  // current B tile pair: hi at +0, lo at +2048

    // hand the current tile to the tensor core and the epilogue warps
    auto flush = [&](bool last) {
      fence_async_smem();
      __syncwarp();
      const int b = kb & 1;
      if (lane == 0) {
        meta[TM_VQ + b] = ncol | (last ? 0x100 : 0) | (int)(emask << 16);
        const uint32_t fb = smem_addr(&full_bar[w][b]);
        if (ncol > 0) {
          fence_after();
          const uint32_t d = tmem + (uint32_t)((2 * w + b) * TM_N);
          const uint32_t s_hi = s_b0 + (uint32_t)b * 4096u, s_lo = s_hi + 2048u;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t ah = sw128_desc(s_a_hi + 32u * ks), al = sw128_desc(s_a_lo + 32u * ks);
            const uint64_t bh = sw128_desc(s_hi + 32u * ks), bl = sw128_desc(s_lo + 32u * ks);
            mma_ss(d, ah, bh, IDESC, ks != 0);
            mma_ss(d, ah, bl, IDESC, 1u);
            mma_ss(d, al, bh, IDESC, 1u);
          }
          mma_commit(fb);  // arrives when the 12 MMAs have completed
        } else {
          mbar_arrive(fb);
        }
        mbar_arrive(fb);  // release: the column count and the destination rows
      }
      __syncwarp();
      ++kb;
      ncol = 0;
      emask = 0;
      bt = wb + TM_B + (size_t)(kb & 1) * 4096;
      // the next buffer: its MMAs and REDs of two tiles ago are complete
      if (!last && kb >= 2) mbar_wait(smem_addr(&empty_bar[w][kb & 1]), ((kb >> 1) + 1) & 1);
    };
    // one tile row: the 32 lane weights of a source and where its column goes
    auto put_col = [&](float v, unsigned long long dst) {
      const uint32_t off = (uint32_t)ncol * 128u + (lane4 ^ (((uint32_t)ncol & 7u) << 4));
      const uint32_t h = tf32_hi(v);
      *reinterpret_cast<uint32_t*>(bt + off) = h;
      *reinterpret_cast<float*>(bt + 2048 + off) = v - __uint_as_float(h);
      dptr[(kb & 1) * TM_N + ncol] = dst;  // every lane stores the same word
      ++ncol;
    };
    // vector quantities of the batch: lane L sums pair (e, k) = (L / 4, L % 4) of
    // vq[e][k][0..31] and issues at most one RED (as k_adjoint2)
    auto eval_vq = [&]() {
      __syncwarp();
      if (lane < 4 * nvq) {
        const float4* row = reinterpret_cast<const float4*>(vq + lane * 32);
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 v4 = row[(j + lane) & 7];
          s += (v4.x + v4.y) + (v4.z + v4.w);
        }
        const int e = lane >> 2, k = lane & 3;  // 0..2 vector, 3 = d mu_0
        const int m = meta[e];
        const bool is_point = m & (1 << 30);
        const int64_t src = m & ((1 << 29) - 1);
        double* dst = is_point ? (k < 3 ? acc.pt_n + 3 * src + k : acc.pt_mud + src)
                               : acc.node_v + 3 * src + k;
        red_add_if(dst, (double)s, s != 0.f && (is_point || k < 3));
      }
      __syncwarp();
      nvq = 0;
    };

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
        } else {
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
      } else {
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

    // one far source (node) for the lanes in `far` (bhtree.cpp:361-381). hint:
    // the list's NEAR flag (0 / 1), -1 on the tree walk (decided by a vote)
    auto far_entry = [&](int node, float A, float s, float fx, float fy, float fz, bool far,
                         int hint) {
      float r_ = 0.f, e_ = 0.f, u0 = 0.f, u1 = 0.f, u2 = 0.f;
      bool nr_ = false;
      const bool slow = far && !(kp.mode == KM_SINGULAR ||
                                 (kp.mode == KM_REGULARIZED && s >= kp.near2));
      far_fast(A, s, fx, fy, fz, far, r_, u0, u1, u2);
      if (hint != 0 && (hint > 0 || __any_sync(FULL_MASK, slow))) {
        if (slow) {
          const Co c = adj_coeffs_tm<GM>(s, kp);
          nr_ = c.near;
          r_ = A * c.R;
          e_ = A * c.dR_de;
          const float aWds = A * c.W * ds0;
          u0 = aWds * fx, u1 = aWds * fy, u2 = aWds * fz;
          if (GM == 0) {
            if (c.near) {
              const float4 v = __ldg(tv.node_row + (size_t)node * F4g);
              const float vd = fmaf(v.x, fx, fmaf(v.y, fy, v.z * fz));
              eps_acc += (double)(ds0 * A * c.dW_de * vd);  // :370
            }
          } else {
            const float4 v = __ldg(tv.node_row + (size_t)node * F4g);
            const float vd = fmaf(v.x, fx, fmaf(v.y, fy, v.z * fz));
            float e = ds0 * A * c.dW_de * vd;                          // :370
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
      const bool any_near = hint != 0 && __any_sync(FULL_MASK, nr_);
      if (ncol + (any_near ? 2 : 1) > TM_N) flush(false);
      put_col(r_, reinterpret_cast<unsigned long long>(acc.node_s + (size_t)node * Cr));
      if (any_near) {  // warp-uniform; rare beyond the first tree levels
        emask |= 1u << ncol;
        put_col(e_, reinterpret_cast<unsigned long long>(tv.node_row + (size_t)node * F4g + 1));
      }
      if (nvq == TM_VQ) eval_vq();
      float* vqe = vq + nvq * 128;
      vqe[lane] = u0, vqe[32 + lane] = u1, vqe[64 + lane] = u2;  // slot 3 is never read for nodes
      meta[nvq] = node;
      ++nvq;
    };
    // K consecutive list entries: far nodes whose far lanes are all beyond 6.5 eps
    // (the caller checked that the tile and the vector batch have room)
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
        put_col(r_, reinterpret_cast<unsigned long long>(acc.node_s + (size_t)nd[k] * Cr));
        float* v = vq + nvq * 128;
        v[lane] = u0, v[32 + lane] = u1, v[64 + lane] = u2;
        meta[nvq] = nd[k];
        ++nvq;
      }
    };
    // the points of an opened leaf for the lanes in `me_open` (:382-412)
    auto leaf_points = [&](const int4 tp, bool me_open) {
      for (int j = tp.z; j < tp.w; ++j) {
        float r_ = 0.f, e_ = 0.f, n0 = 0.f, n1 = 0.f, n2 = 0.f, dmu = 0.f;
        bool nr_ = false;
        if (me_open) {
          const PtRec* pr = tv.pt_rec + j;
          const float4 ph = __ldg(&pr->hi);
          float fx, fy, fz;
          const float r2 = dist2_df(ph, __ldg(&pr->lo), qx, fx, fy, fz);
          if (!(r2 == 0.f && coincident_exact(tv.pt_pos64 + 3 * (size_t)j, xq))) {
            const Co c = adj_coeffs_tm<GM>(r2, kp);
            const float Am = ph.w;
            nr_ = c.near;
            r_ = Am * c.R;
            e_ = Am * c.dR_de;
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
        const bool any_near = __any_sync(FULL_MASK, nr_);
        if (ncol + (any_near ? 2 : 1) > TM_N) flush(false);
        put_col(r_, reinterpret_cast<unsigned long long>(acc.pt_mur + (size_t)j * Cr));
        if (any_near) {
          emask |= 1u << ncol;
          put_col(e_, reinterpret_cast<unsigned long long>(tv.pt_row + (size_t)j * F4g + 1));
        }
        if (nvq == TM_VQ) eval_vq();
        float* vqe = vq + nvq * 128;
        vqe[lane] = n0, vqe[32 + lane] = n1, vqe[64 + lane] = n2, vqe[96 + lane] = dmu;
        meta[nvq] = j | (1 << 30);
        ++nvq;
      }
    };

    if (active) {
      const int64_t wg = (int64_t)blockIdx.x * TM_PROD + w;
      const int total = LIST ? __ldg(lv.count + wg) : -1;
      if (LIST && total >= 0) {
        // replay the interaction list: 32 entries at a time, their node records
        // prefetched into the (unused) stack region with cp.async
        NodeRec* rb = reinterpret_cast<NodeRec*>(stk);
        const uint32_t s_rb = smem_addr(stk) + 48u * lane;
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
          if (lane < n) *reinterpret_cast<uint2*>(&rb[lane].topo) = my;
          __syncwarp();
          for (int i = 0; i < n;) {
            const int4 tpi = rb[i].topo;
            const uint32_t src = (uint32_t)tpi.x;
            if (i + 1 < n && !((src | (uint32_t)rb[i + 1].topo.x) & (IL_LEAF | IL_NEAR))) {
              // two consecutive far entries without near lanes: one interleaved pass
              if (ncol + 2 > TM_N) flush(false);
              if (nvq + 2 > TM_VQ) eval_vq();
              far_group(rb + i, std::integral_constant<int, 2>{});
              i += 2;
              continue;
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
        if (farm && A > 0.f) far_entry(node, A, s, fx, fy, fz, far, -1);
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
      if (nvq) eval_vq();
    }
    flush(true);  // the last tile (possibly empty): tells the epilogue this warp is done
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) eps_acc += __shfl_xor_sync(FULL_MASK, eps_acc, o);
    if (lane == 0 && eps_acc != 0.0) atomicAdd(acc.d_eps, eps_acc);
  }
  fence_before();
  __syncthreads();
  if (w == TM_PROD) tmem_dealloc<TM_COLS>(tmem);
}

template <int GM, bool LIST, bool REG>
static void launch_tm(const Tree& t, const KParams& kp, const AdjArgs& a, GradBuf& b, int nr,
                      IListView lv) {
  const size_t smem = (size_t)TM_PROD * TM_WARP + 1024;
  static std::atomic<unsigned long long> attr{0};
  ensure_max_dyn_smem(k_adjoint_tm<GM, LIST, REG>, t.device, smem, attr);
  AdjTmPtrs p{b.node_v, b.node_s, b.pt_mud, b.pt_mur, b.pt_n, b.d_eps};
  const unsigned blocks = (unsigned)((a.q + TM_PROD * 32 - 1) / (TM_PROD * 32));
  k_adjoint_tm<GM, LIST, REG><<<blocks, (TM_PROD + TM_EPI) * 32, smem, t.stream>>>(
      t.view(), kp, a.xs, a.perm, a.q, a.d_out, a.dstride, a.d_grad, nr, t.chmap.as<int>(), p, lv,
      a.overflow);
  count_launch();
}

template <int GM>
static void plan_tm(const Tree& t, const KParams& kp, const AdjArgs& a, GradBuf& b, int nr) {
  const bool reg = kp.mode == KM_REGULARIZED && kp.near2 >= REG_MIN_NEAR2;
  if (a.ilist && !no_ilist()) {
    ilist_build(t, *a.ilist, a.xs, a.perm, a.q, a.beta, ilist_near_thr(kp), a.overflow);
    if (reg)
      launch_tm<GM, true, true>(t, kp, a, b, nr, a.ilist->view());
    else
      launch_tm<GM, true, false>(t, kp, a, b, nr, a.ilist->view());
  } else if (reg) {
    launch_tm<GM, false, true>(t, kp, a, b, nr, IListView{});
  } else {
    launch_tm<GM, false, false>(t, kp, a, b, nr, IListView{});
  }
}

// The tensor-memory adjoint for one Dipole + (4, 48] Radial channels; false when
// the layout is outside its range (the caller falls back to k_adjoint2).
bool adjoint_tm_launch(const Tree& t, const KParams& kp, const AdjArgs& a, GradBuf& b) {
  if (t.Cd != 1) return false;
  const int nr = a.nr_limit >= 0 ? std::min(a.nr_limit, t.Cr) : t.Cr;
  if (nr <= 4 || nr > TM_ROWS) return false;
  if (a.grad_mode == 0)
    plan_tm<0>(t, kp, a, b, nr);
  else if (a.grad_mode == 1)
    plan_tm<1>(t, kp, a, b, nr);
  else
    plan_tm<2>(t, kp, a, b, nr);
  return true;
}

}  // namespace dpl
