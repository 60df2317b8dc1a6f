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
#include "adjoint.cuh"
#include "traverse.cuh"

namespace dpl {

namespace {
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

// NB: 0 -> Cr <= 32; 1 -> 32 < Cr <= 48 (split); 2 -> Cr <= 64.
// GM: 0 no d_grad; 1 d_grad q x dstride x 3; 2 d_grad q x 3 (channel 0).
// MAXR: register cap (occupancy vs. spills; chosen by measurement)
template <int NB, int GM, int WARPS, int ENT, int RR, int MAXR = 128>
__global__ void __launch_bounds__(WARPS * 32) __maxnreg__(MAXR)
    k_adjoint2(TreeView tv, KParams kp, const double* __restrict__ xs,
               const int32_t* __restrict__ perm, int64_t q, const float* __restrict__ d_out,
               int dstride, const float* __restrict__ d_grad, int nr,
               const int* __restrict__ chmap, Adj2Ptrs acc, int* overflow) {
  constexpr int F4 = 1 + RR;  // smem row capacity: [dipole float4 | up to RR radial float4]
  // per-warp shared layout (floats): wR[ENT][32] wE[ENT][32] vq[ENT][4][32]
  //                                  rows[ENT][F4*4] meta[ENT] stack[2*STACK]
  constexpr int WARP_FLOATS = ENT * 32 * 6 + ENT * F4 * 4 + ENT + 2 * DPL_STACK_PER_WARP;
  extern __shared__ float4 smem_f4[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* base = reinterpret_cast<float*>(smem_f4) + (size_t)w * ((WARP_FLOATS + 3) & ~3);
  float* wR = base;
  float* wE = wR + ENT * 32;
  float* vq = wE + ENT * 32;
  float4* rows = reinterpret_cast<float4*>(vq + ENT * 128);
  int* meta = reinterpret_cast<int*>(rows + ENT * F4);
  int2* stk = reinterpret_cast<int2*>(meta + ENT + (ENT & 1));
  const uint32_t s_rows = smem_u32(rows) + 16u * lane;
  const int F4g = tv.F4;  // global row stride (<= F4)

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
  const QueryDF qx = make_qdf(x);

  // own-query dipole upstream gradients (channel slot 0)
  const int ch0 = __ldg(chmap);
  const float ds0 = valid ? __ldg(d_out + qi * dstride + ch0) : 0.f;
  float dg0 = 0.f, dg1 = 0.f, dg2 = 0.f;
  if (GM && valid) {
    const float* g = GM == 1 ? d_grad + (qi * dstride + ch0) * 3 : d_grad + qi * 3;
    dg0 = g[0], dg1 = g[1], dg2 = g[2];
  }
  // transposed radial tile
  float colA[32];
  float colB[NB == 2 ? 32 : (NB == 1 ? 16 : 1)];
  const bool okA = lane < nr;
  const int chA = okA ? __ldg(chmap + 1 + lane) : 0;
  const int slotB = NB == 1 ? 32 + (lane & 15) : 32 + lane;
  const bool okB = NB > 0 && slotB < nr;
  const int chB = okB ? __ldg(chmap + 1 + slotB) : 0;
#pragma unroll
  for (int l = 0; l < 32; ++l) {
    const int64_t ql = __shfl_sync(FULL_MASK, qi, l);
    const bool vl = (active >> l) & 1u;
    colA[l] = (okA && vl) ? __ldg(d_out + ql * dstride + chA) : 0.f;
    if (NB == 2) colB[l] = (okB && vl) ? __ldg(d_out + ql * dstride + chB) : 0.f;
  }
  if (NB == 1) {
    const int h = lane >> 4;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int l = 16 * h + i;
      const int64_t ql = __shfl_sync(FULL_MASK, qi, l);  // all lanes participate
      const bool vl = (active >> l) & 1u;
      colB[i] = (okB && vl) ? __ldg(d_out + ql * dstride + chB) : 0.f;
    }
  }
  double eps_acc = 0.0;
  int nent = 0;

  auto evaluate = [&]() {
    cp_async_wait_all();
    __syncwarp();
    for (int e = 0; e < nent; ++e) {
      const int m = meta[e];
      const bool is_point = m & (1 << 30);
      const bool near = m & (1 << 29);
      const int64_t src = m & ((1 << 29) - 1);
      const float4* wr4 = reinterpret_cast<const float4*>(wR + e * 32);
      float sA = 0.f, sB = 0.f;
#pragma unroll
      for (int l4 = 0; l4 < 8; ++l4) {
        const float4 ww = wr4[l4];
        const float wv[4] = {ww.x, ww.y, ww.z, ww.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int l = 4 * l4 + u;
          sA = fmaf(wv[u], colA[l], sA);
          if (NB == 2) sB = fmaf(wv[u], colB[l], sB);
        }
      }
      if (NB == 1) {
        // half-warp split: lanes 0-15 cover queries 0-15, lanes 16-31 queries 16-31
        const float* wh = wR + e * 32 + 16 * (lane >> 4);
#pragma unroll
        for (int i4 = 0; i4 < 4; ++i4) {
          const float4 ww = reinterpret_cast<const float4*>(wh)[i4];
          sB = fmaf(ww.x, colB[4 * i4 + 0], sB);
          sB = fmaf(ww.y, colB[4 * i4 + 1], sB);
          sB = fmaf(ww.z, colB[4 * i4 + 2], sB);
          sB = fmaf(ww.w, colB[4 * i4 + 3], sB);
        }
        sB += __shfl_xor_sync(FULL_MASK, sB, 16);
      }
      double* dst_s = is_point ? acc.pt_mur + src * Cr : acc.node_s + src * Cr;
      if (okA && sA != 0.f) atomicAdd(dst_s + lane, (double)sA);
      const bool ownB = NB == 2 ? okB : (NB == 1 ? (okB && lane < 16) : false);
      if (ownB && sB != 0.f) atomicAdd(dst_s + slotB, (double)sB);
      if (near) {  // radial epsilon terms (:379, :409)
        const float4* we4 = reinterpret_cast<const float4*>(wE + e * 32);
        float eA = 0.f, eB = 0.f;
#pragma unroll
        for (int l4 = 0; l4 < 8; ++l4) {
          const float4 ww = we4[l4];
          const float wv[4] = {ww.x, ww.y, ww.z, ww.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            eA = fmaf(wv[u], colA[4 * l4 + u], eA);
            if (NB == 2) eB = fmaf(wv[u], colB[4 * l4 + u], eB);
          }
        }
        if (NB == 1) {
          const float* wh = wE + e * 32 + 16 * (lane >> 4);
#pragma unroll
          for (int i = 0; i < 16; ++i) eB = fmaf(wh[i], colB[i], eB);
          eB += __shfl_xor_sync(FULL_MASK, eB, 16);
        }
        const float* rad = reinterpret_cast<const float*>(rows + e * F4 + 1);
        if (okA) eps_acc += (double)(eA * rad[lane]);
        if (ownB) eps_acc += (double)(eB * rad[slotB]);
      }
      // vector quantities: transposed sum of vq[e][k][l] over l
      const float4 v4 = reinterpret_cast<const float4*>(vq + e * 128)[lane];
      float s = (v4.x + v4.y) + (v4.z + v4.w);
      s += __shfl_xor_sync(FULL_MASK, s, 1);
      s += __shfl_xor_sync(FULL_MASK, s, 2);
      s += __shfl_xor_sync(FULL_MASK, s, 4);
      if ((lane & 7) == 0 && s != 0.f) {
        const int k = lane >> 3;  // 0..2 vector, 3 = d mu_0
        double* dst = is_point ? (k < 3 ? acc.pt_n + 3 * src + k : acc.pt_mud + src)
                               : acc.node_v + 3 * src + k;
        if (is_point || k < 3) atomicAdd(dst, (double)s);
      }
    }
    __syncwarp();
    nent = 0;
  };

  auto begin_entry = [&]() {
    if (nent == ENT) evaluate();
  };

  int sp = 1;
  if (lane == 0) stk[0] = make_int2(0, (int)active);
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
    const bool far = mine && far_test(s, hi, qx, x, tv.node_dec + node);
    const unsigned farm = __ballot_sync(FULL_MASK, far);
    if (farm && A > 0.f) {
      begin_entry();
      float r_ = 0.f, e_ = 0.f, u0 = 0.f, u1 = 0.f, u2 = 0.f;
      bool nr_ = false;
      if (far) {
        const Co c = adj_coeffs<GM>(s, kp);
        nr_ = c.near;
        r_ = A * c.R;
        e_ = A * c.dR_de;
        const float aWds = A * c.W * ds0;
        u0 = aWds * fx, u1 = aWds * fy, u2 = aWds * fz;
        if (c.near || GM) {
          const float4 v = __ldg(tv.node_row + (size_t)node * F4g);
          const float vd = fmaf(v.x, fx, fmaf(v.y, fy, v.z * fz));
          float e = ds0 * A * c.dW_de * vd;  // :370
          if (GM) {                          // :372-374
            const float gd = fmaf(dg0, fx, fmaf(dg1, fy, dg2 * fz));
            const float t = c.Wp_r * gd;
            u0 -= A * fmaf(c.W, dg0, t * fx);
            u1 -= A * fmaf(c.W, dg1, t * fy);
            u2 -= A * fmaf(c.W, dg2, t * fz);
            const float k2 = c.dWp_r_de * vd;
            e -= A * fmaf(dg0, fmaf(c.dW_de, v.x, k2 * fx),
                          fmaf(dg1, fmaf(c.dW_de, v.y, k2 * fy), dg2 * fmaf(c.dW_de, v.z, k2 * fz)));
          }
          eps_acc += (double)e;
        }
      }
      wR[nent * 32 + lane] = r_;
      wE[nent * 32 + lane] = e_;
      float* vqe = vq + nent * 128;
      vqe[lane] = u0, vqe[32 + lane] = u1, vqe[64 + lane] = u2, vqe[96 + lane] = 0.f;
      const bool any_near = __any_sync(FULL_MASK, nr_);
      if (any_near && lane < F4g)
        cp_async16(s_rows + 16u * F4 * nent, tv.node_row + (size_t)node * F4g + lane);
      if (lane == 0) meta[nent] = node | (any_near ? (1 << 29) : 0);
      ++nent;
    }
    const unsigned openm = mask & ~farm;
    if (openm) {
      if (tp.y == 0) {
        const bool me_open = (openm >> lane) & 1u;
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
            if (!(r2 == 0.f && coincident_exact(tv.pt_pos64 + 3 * (size_t)j, x))) {
              const Co c = adj_coeffs<GM>(r2, kp);
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
          wR[nent * 32 + lane] = r_;
          wE[nent * 32 + lane] = e_;
          float* vqe = vq + nent * 128;
          vqe[lane] = n0, vqe[32 + lane] = n1, vqe[64 + lane] = n2, vqe[96 + lane] = dmu;
          const bool any_near = __any_sync(FULL_MASK, nr_);
          if (any_near && lane < F4g)
            cp_async16(s_rows + 16u * F4 * nent, tv.pt_row + (size_t)j * F4g + lane);
          if (lane == 0) meta[nent] = j | (1 << 30) | (any_near ? (1 << 29) : 0);
          ++nent;
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
  if (nent) evaluate();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) eps_acc += __shfl_xor_sync(FULL_MASK, eps_acc, o);
  if (lane == 0 && eps_acc != 0.0) atomicAdd(acc.d_eps, eps_acc);
}

template <int NB, int GM, int RR, int WARPS = 4, int ENT = 8, int MINB = 128>
static void launch_adj2(const Tree& t, const KParams& kp, const AdjArgs& a, GradBuf& b, int nr) {
  constexpr int F4 = 1 + RR;
  constexpr int WARP_FLOATS = ENT * 32 * 6 + ENT * F4 * 4 + ENT + 2 * DPL_STACK_PER_WARP;
  const size_t smem = (size_t)WARPS * ((WARP_FLOATS + 3) & ~3) * 4;
  static bool attr = false;
  if (!attr) {
    DPL_CUDA(cudaFuncSetAttribute(k_adjoint2<NB, GM, WARPS, ENT, RR, MINB>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  Adj2Ptrs p{b.node_v, b.node_s, b.pt_mud, b.pt_mur, b.pt_n, b.d_eps};
  unsigned blocks = (unsigned)((a.q + WARPS * 32 - 1) / (WARPS * 32));
  k_adjoint2<NB, GM, WARPS, ENT, RR, MINB><<<blocks, WARPS * 32, smem, t.stream>>>(
      t.view(), kp, a.xs, a.perm, a.q, a.d_out, a.dstride, a.d_grad, nr, t.chmap.as<int>(), p,
      a.overflow);
  count_launch();
}

template <int GM>
static bool adj2_plan(const Tree& t, const KParams& kp, const AdjArgs& a, GradBuf& b) {
  const int nr = a.nr_limit >= 0 ? std::min(a.nr_limit, t.Cr) : t.Cr;
  if (t.F4 - 1 > 16) return false;
  if (nr <= 32) return launch_adj2<0, GM, 16>(t, kp, a, b, nr), true;
  if (nr <= 48 && GM == 0) {
    const char* v = getenv("DPL_TUNE_ADJ");
    switch (v ? atoi(v) : 0) {  // occupancy / batch experiments
      case 1: return launch_adj2<1, GM, 16, 4, 8, 112>(t, kp, a, b, nr), true;
      case 2: return launch_adj2<1, GM, 16, 4, 8, 104>(t, kp, a, b, nr), true;
      case 3: return launch_adj2<1, GM, 16, 4, 4, 112>(t, kp, a, b, nr), true;
      case 4: return launch_adj2<1, GM, 16, 4, 4, 96>(t, kp, a, b, nr), true;
      case 5: return launch_adj2<1, GM, 16, 4, 6, 112>(t, kp, a, b, nr), true;
      default: break;
    }
  }
  if (nr <= 48) return launch_adj2<1, GM, 16>(t, kp, a, b, nr), true;
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
