// adjoint.cu — K7 adjoint traversal and K8 top-down gradient push-down.
//
// Restates DipoleTree::adjoint (proj/src/bhtree.cpp:345-417) and
// flush_gradients (:419-463) for a batch of queries.
//
// K7 walks the tree exactly like the forward kernel (same fp64 decisions) and
// scatters per-interaction gradients into fp64 accumulators, aggregated per
// warp so that one atomic per (warp, node, channel) replaces 32:
//   * radial slots: the warp contribution to node_s[t, c] is
//       sum_l  w_l * ds[l, c],   w_l = A R(|d_l|) for the lanes that accepted t,
//     a (1 x 32) . (32 x TR) product. The warp's d_out tile is held TRANSPOSED
//     in registers (lane L owns channel column L of all 32 queries), the 32
//     weights are broadcast through shared memory, and lane L finishes channel
//     L with 32 FMAs — every lane busy, one coalesced fp64 RED per channel.
//     The epsilon terms use the same product with weights A dR_de.
//   * dipole slots: per-lane vector contributions (bhtree.cpp:367-376) reduced
//     with warp shuffles, one RED per component.
//   * leaf points: the same two paths into point accumulators (:382-412).
// K8 replaces the reference's per-point ancestor walk (:441-457) with the
// equivalent push-down G_t = G_parent + node_v[t] / area_t (level by level,
// fp64), then one pass over points: d mu = point_mu + a_m (n . G_leaf) etc.
#include <cub/cub.cuh>

#include "adjoint.cuh"
#include "traverse.cuh"

namespace dpl {

constexpr int ADJ_WARPS = 4;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
  return v;
}

// Reduce 4 floats across the warp with 6 shuffles (reduce-scatter, then a
// butterfly on one value); returns the full sums in every lane.
__device__ __forceinline__ void warp_sum4(float& a, float& b, float& c, float& d, int lane) {
  // step 1: pairs (a,b) vs (c,d) over xor 16
  {
    bool hi = lane & 16;
    float s0 = hi ? a : c, s1 = hi ? b : d;
    float r0 = __shfl_xor_sync(FULL_MASK, s0, 16), r1 = __shfl_xor_sync(FULL_MASK, s1, 16);
    if (hi) { c += r0; d += r1; } else { a += r0; b += r1; }
  }
  // lanes < 16 hold (a,b), lanes >= 16 hold (c,d)
  float x0 = (lane & 16) ? c : a, x1 = (lane & 16) ? d : b;
  {
    bool hi = lane & 8;
    float s = hi ? x0 : x1;
    float r = __shfl_xor_sync(FULL_MASK, s, 8);
    if (hi) x1 += r; else x0 += r;
  }
  float y = (lane & 8) ? x1 : x0;
  y += __shfl_xor_sync(FULL_MASK, y, 4);
  y += __shfl_xor_sync(FULL_MASK, y, 2);
  y += __shfl_xor_sync(FULL_MASK, y, 1);
  // lane groups: [0,8) a, [8,16) b, [16,24) c, [24,32) d
  a = __shfl_sync(FULL_MASK, y, 0);
  b = __shfl_sync(FULL_MASK, y, 8);
  c = __shfl_sync(FULL_MASK, y, 16);
  d = __shfl_sync(FULL_MASK, y, 24);
}

struct AdjPtrs {
  double* node_v;   // nodes x Cd x 3
  double* node_s;   // nodes x Cr
  double* pt_mud;   // N x Cd   (sorted order)
  double* pt_mur;   // N x Cr   (sorted order)
  double* pt_n;     // N x 3    (sorted order)
  double* d_eps;    // 1
};

// per-interaction dipole-slot work for far nodes (lane-local part)
template <int TD>
struct DipLane {
  float ds[TD > 0 ? TD : 1];
  float dg[TD > 0 ? TD : 1][3];
};

// NCOL: radial column groups of 32 channels handled by this tile (0..2).
// GM: d_grad mode 0 none, 1 per channel (q x dstride x 3), 2 channel-0 only (q x 3).
template <int TD, int NCOL, int GM>
__global__ void __launch_bounds__(ADJ_WARPS * 32)
    k_adjoint(TreeView tv, KParams kp, const float4* __restrict__ node_payd,
              const float* __restrict__ node_payr, const float4* __restrict__ pt_payd,
              const float* __restrict__ pt_payr, const double* __restrict__ xs,
              const int32_t* __restrict__ perm, int64_t q, const float* __restrict__ d_out,
              int dstride, const float* __restrict__ d_grad, int d0, int nd, int r0, int nr,
              const int* __restrict__ chmap, AdjPtrs acc, int* overflow) {
  __shared__ int2 stk[ADJ_WARPS][DPL_STACK_PER_WARP];
  __shared__ float4 wsh[ADJ_WARPS][32];  // per lane: (w_R, w_eps, -, -)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t sidx = ((int64_t)blockIdx.x * ADJ_WARPS + w) * 32 + lane;
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
  const int Cd = tv.Cd, Cr = tv.Cr, F4 = tv.F4;

  // own-query dipole upstream gradients
  DipLane<TD> dl;
#pragma unroll
  for (int k = 0; k < (TD > 0 ? TD : 1); ++k) {
    dl.ds[k] = 0.f;
    dl.dg[k][0] = dl.dg[k][1] = dl.dg[k][2] = 0.f;
    if (k < nd && valid) {
      int ch = __ldg(chmap + d0 + k);
      dl.ds[k] = d_out[qi * dstride + ch];
      if (GM == 1) {
        const float* g = d_grad + (qi * dstride + ch) * 3;
        dl.dg[k][0] = g[0], dl.dg[k][1] = g[1], dl.dg[k][2] = g[2];
      } else if (GM == 2 && ch == 0) {
        const float* g = d_grad + qi * 3;
        dl.dg[k][0] = g[0], dl.dg[k][1] = g[1], dl.dg[k][2] = g[2];
      }
    }
  }
  // transposed radial tile: col[m][l] = d_out[query of lane l, radial slot r0 + 32 m + lane]
  float col[NCOL > 0 ? NCOL : 1][32];
  bool colok[NCOL > 0 ? NCOL : 1];
#pragma unroll
  for (int m = 0; m < NCOL; ++m) {
    const int slot = 32 * m + lane;
    colok[m] = slot < nr;
    const int ch = colok[m] ? __ldg(chmap + Cd + r0 + slot) : 0;
#pragma unroll
    for (int l = 0; l < 32; ++l) {
      int64_t ql = __shfl_sync(FULL_MASK, qi, l);
      bool vl = (active >> l) & 1u;
      col[m][l] = (colok[m] && vl) ? __ldg(d_out + ql * dstride + ch) : 0.f;
    }
  }
  double eps_acc = 0.0;
  const bool skip_coincident = true;  // adjoint always skips r = 0 (:387)

  int sp = 1;
  if (lane == 0) stk[w][0] = make_int2(0, (int)active);
  __syncwarp();

  // one source (far node or leaf point) for the lanes in `me`
  auto source = [&](bool me, double dx, double dy, double dz, double dist2, float A,
                    const float4* pd, const float* pr, int64_t src, bool is_point) {
    const float fx = (float)dx, fy = (float)dy, fz = (float)dz;
    Co c{};
    if (me) c = coeffs<2>((float)dist2, kp);
    // ---- radial slots: warp mat-vec
    if (NCOL > 0) {
      float wR = me ? A * c.R : 0.f;
      float wE = me ? A * c.dR_de : 0.f;
      wsh[w][lane] = make_float4(wR, wE, 0.f, 0.f);
      const bool any_eps = __any_sync(FULL_MASK, me && c.near);
      __syncwarp();
#pragma unroll
      for (int m = 0; m < NCOL; ++m) {
        float s = 0.f, se = 0.f;
#pragma unroll
        for (int l = 0; l < 32; ++l) {
          float4 ww = wsh[w][l];
          s = fmaf(ww.x, col[m][l], s);
          if (any_eps) se = fmaf(ww.y, col[m][l], se);
        }
        if (colok[m]) {
          const int slot = r0 + 32 * m + lane;
          if (s != 0.f) {
            double* dst = is_point ? acc.pt_mur + src * Cr + slot : acc.node_s + src * Cr + slot;
            atomicAdd(dst, (double)s);
          }
          if (any_eps && se != 0.f) {
            // reference: d_eps += ds A dR_de s_node (:379) / ds A mu dR_de (:409)
            float sv = __ldg(pr - r0 + slot);
            eps_acc += (double)(se * sv);
          }
        }
      }
      __syncwarp();
    }
    // ---- dipole slots
#pragma unroll
    for (int k = 0; k < TD; ++k) {
      if (k >= nd) continue;
      float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f;  // reduced quantities
      if (me) {
        const float ds = dl.ds[k];
        if (!is_point) {
          // far node (:367-376): node_v += A W ds d - A (W dg + Wp_r (dg.d) d)
          float4 v = __ldg(pd + k);
          float vd = fmaf(v.x, fx, fmaf(v.y, fy, v.z * fz));
          float aWds = A * c.W * ds;
          v0 = aWds * fx, v1 = aWds * fy, v2 = aWds * fz;
          float e = ds * A * c.dW_de * vd;
          if (GM) {
            const float* g = dl.dg[k];
            float gd = fmaf(g[0], fx, fmaf(g[1], fy, g[2] * fz));
            float t = c.Wp_r * gd;
            v0 -= A * fmaf(c.W, g[0], t * fx);
            v1 -= A * fmaf(c.W, g[1], t * fy);
            v2 -= A * fmaf(c.W, g[2], t * fz);
            float u0 = fmaf(c.dW_de, v.x, c.dWp_r_de * vd * fx);
            float u1 = fmaf(c.dW_de, v.y, c.dWp_r_de * vd * fy);
            float u2 = fmaf(c.dW_de, v.z, c.dWp_r_de * vd * fz);
            e -= A * fmaf(g[0], u0, fmaf(g[1], u1, g[2] * u2));
          }
          eps_acc += (double)e;
        } else {
          // leaf point (:394-406): d mu, d n, d eps
          const float mu = __ldg(tv.pt_mu + src * Cd + d0 + k);
          const float nx = __ldg(tv.pt_nrm + 3 * src), ny = __ldg(tv.pt_nrm + 3 * src + 1),
                      nz = __ldg(tv.pt_nrm + 3 * src + 2);
          float nu = fmaf(nx, fx, fmaf(ny, fy, nz * fz));
          float aW = A * c.W;
          float dmu = ds * aW * nu;
          float s = ds * aW * mu;
          float n0 = s * fx, n1 = s * fy, n2 = s * fz;
          float e = ds * A * mu * c.dW_de * nu;
          if (GM) {
            const float* g = dl.dg[k];
            float gd = fmaf(g[0], fx, fmaf(g[1], fy, g[2] * fz));
            float gn = fmaf(g[0], nx, fmaf(g[1], ny, g[2] * nz));
            dmu -= A * fmaf(c.W, gn, c.Wp_r * nu * gd);
            float am = A * mu, t = c.Wp_r * gd;
            n0 -= am * fmaf(c.W, g[0], t * fx);
            n1 -= am * fmaf(c.W, g[1], t * fy);
            n2 -= am * fmaf(c.W, g[2], t * fz);
            e -= am * fmaf(c.dW_de, gn, c.dWp_r_de * nu * gd);
          }
          eps_acc += (double)e;
          v0 = n0, v1 = n1, v2 = n2, v3 = dmu;
        }
      }
      warp_sum4(v0, v1, v2, v3, lane);
      if (!is_point) {
        if (lane < 3) {
          float val = lane == 0 ? v0 : (lane == 1 ? v1 : v2);
          if (val != 0.f) atomicAdd(acc.node_v + (src * Cd + d0 + k) * 3 + lane, (double)val);
        }
      } else {
        if (lane < 4) {
          float val = lane == 0 ? v0 : (lane == 1 ? v1 : (lane == 2 ? v2 : v3));
          if (val != 0.f) {
            double* dst = lane < 3 ? acc.pt_n + 3 * src + lane : acc.pt_mud + src * Cd + d0 + k;
            atomicAdd(dst, (double)val);
          }
        }
      }
    }
  };

  while (sp > 0) {
    --sp;
    const int2 e = stk[w][sp];
    __syncwarp();
    const int node = e.x;
    const unsigned mask = (unsigned)e.y;
    const bool mine = (mask >> lane) & 1u;
    const double4 dec = ld_dec(tv.node_dec + node);
    const int4 tp = __ldg(tv.node_topo + node);
    double dx, dy, dz;
    const double dist2 = dist2_rn(dec.x, dec.y, dec.z, x, dx, dy, dz);
    const bool far = mine && (dist2 > dec.w);
    const unsigned farm = __ballot_sync(FULL_MASK, far);
    if (farm && (__ldg(tv.node_flag + node) & 1)) {
      source(far, dx, dy, dz, dist2, __ldg(tv.node_geo + node).w,
             node_payd + (int64_t)node * F4 + d0,
             reinterpret_cast<const float*>(node_payd + (int64_t)node * F4 + Cd) + r0, node,
             false);
    }
    const unsigned openm = mask & ~farm;
    if (openm) {
      if (tp.y == 0) {
        const bool me_open = (openm >> lane) & 1u;
        for (int j = tp.z; j < tp.w; ++j) {
          double px = __ldg(tv.pt_pos64 + 3 * (int64_t)j);
          double py = __ldg(tv.pt_pos64 + 3 * (int64_t)j + 1);
          double pz = __ldg(tv.pt_pos64 + 3 * (int64_t)j + 2);
          const double r2 = dist2_rn(px, py, pz, x, dx, dy, dz);
          const bool me = me_open && !(r2 == 0.0 && skip_coincident);
          if (__any_sync(FULL_MASK, me))
            source(me, dx, dy, dz, r2, __ldg(tv.pt_geo + j).w, pt_payd + (int64_t)j * F4 + d0,
                   reinterpret_cast<const float*>(pt_payd + (int64_t)j * F4 + Cd) + r0, j, true);
        }
      } else {
        if (sp + tp.y > DPL_STACK_PER_WARP) {
          if (lane == 0) atomicExch(overflow, 1);
          break;
        }
        if (lane < tp.y) stk[w][sp + lane] = make_int2(tp.x + lane, (int)openm);
        sp += tp.y;
        __syncwarp();
      }
    }
  }
  double e = warp_sum_d(eps_acc);
  if (lane == 0 && e != 0.0) atomicAdd(acc.d_eps, e);
}

// ---------------------------------------------------------------- K8

// G_t = G_parent + node_acc[t] / area_t  (area_t > 0), in place, one level.
__global__ void k_pushdown_level(int64_t off, int64_t cnt, int W, const int32_t* __restrict__ parent,
                                 const double* __restrict__ narea, double* gv, int Wv, double* gs,
                                 int Ws) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= cnt * W) return;
  int64_t node = off + g / W;
  int comp = (int)(g % W);
  double a = narea[node];
  int32_t p = parent[node];
  double* arr = comp < Wv ? gv : gs;
  int cw = comp < Wv ? Wv : Ws;
  int cc = comp < Wv ? comp : comp - Wv;
  double v = arr[node * cw + cc];
  double own = a > 0 ? v / a : 0.0;
  double up = p >= 0 ? arr[(int64_t)p * cw + cc] : 0.0;
  arr[node * cw + cc] = up + own;
}

// per sorted point j (original m = order[j]):
//   d mu_c = pt_mu[j, c] + a_m (n_m . G_leaf,c)  (dipole)  |  + a_m S_leaf,c (radial)
//   d n_m  = pt_n[j] + a_m sum_c mu_{m,c} G_leaf,c
__global__ void k_flush_points(int64_t n, int C, int Cd, int Cr, const int* __restrict__ chmap,
                               const int32_t* __restrict__ order,
                               const int32_t* __restrict__ pt_leaf,
                               const double* __restrict__ area, const double* __restrict__ nrm,
                               const double* __restrict__ mu, const double* __restrict__ gv,
                               const double* __restrict__ gs, const double* __restrict__ pmud,
                               const double* __restrict__ pmur, const double* __restrict__ pn,
                               float* moments, float* normals) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  int64_t m = order[j];
  int64_t leaf = pt_leaf[j];
  double a = area[m];
  double nx = nrm[3 * m], ny = nrm[3 * m + 1], nz = nrm[3 * m + 2];
  double dn0 = pn[3 * j], dn1 = pn[3 * j + 1], dn2 = pn[3 * j + 2];
  for (int k = 0; k < Cd; ++k) {
    int ch = chmap[k];
    const double* g = gv + (leaf * Cd + k) * 3;
    double v = pmud[j * Cd + k] + a * (nx * g[0] + ny * g[1] + nz * g[2]);
    if (moments) moments[m * C + ch] = (float)v;
    double am = a * mu[m * C + ch];
    dn0 += am * g[0], dn1 += am * g[1], dn2 += am * g[2];
  }
  if (normals) {
    normals[3 * m] = (float)dn0, normals[3 * m + 1] = (float)dn1, normals[3 * m + 2] = (float)dn2;
  }
}

// radial moments: one warp per point, lanes over its radial slots (coalesced;
// same arithmetic as the per-point loop it replaces)
__global__ void k_flush_radial(int64_t n, int C, int Cd, int Cr, const int* __restrict__ chmap,
                               const int32_t* __restrict__ order,
                               const int32_t* __restrict__ pt_leaf,
                               const double* __restrict__ area, const double* __restrict__ gs,
                               const double* __restrict__ pmur, float* moments) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < n; j += nw) {
    const int64_t m = order[j];
    const int64_t leaf = pt_leaf[j];
    const double a = area[m];
    for (int k = lane; k < Cr; k += 32)
      moments[m * C + chmap[Cd + k]] = (float)(pmur[j * Cr + k] + a * gs[leaf * Cr + k]);
  }
}

// one warp per sorted point j in [lo, hi): row (j - lo) = [d mu (C) | d n (3)],
// the arithmetic of k_flush_points (lane 0, dipole slots + normal) and
// k_flush_radial (lanes over radial slots), so rows hold the same values
__global__ void k_flush_rows(int64_t lo, int64_t hi, int C, int Cd, int Cr,
                             const int* __restrict__ chmap, const int32_t* __restrict__ order,
                             const int32_t* __restrict__ pt_leaf, const double* __restrict__ area,
                             const double* __restrict__ nrm, const double* __restrict__ mu,
                             const double* __restrict__ gv, const double* __restrict__ gs,
                             const double* __restrict__ pmud, const double* __restrict__ pmur,
                             const double* __restrict__ pn, float* __restrict__ rows) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int W = C + 3;
  for (int64_t j = lo + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); j < hi; j += nw) {
    const int64_t m = order[j];
    const int64_t leaf = pt_leaf[j];
    const double a = area[m];
    float* row = rows + (j - lo) * W;
    for (int k = lane; k < Cr; k += 32)
      row[chmap[Cd + k]] = (float)(pmur[j * Cr + k] + a * gs[leaf * Cr + k]);
    if (lane == 0) {
      double nx = nrm[3 * m], ny = nrm[3 * m + 1], nz = nrm[3 * m + 2];
      double dn0 = pn[3 * j], dn1 = pn[3 * j + 1], dn2 = pn[3 * j + 2];
      for (int k = 0; k < Cd; ++k) {
        int ch = chmap[k];
        const double* g = gv + (leaf * Cd + k) * 3;
        double v = pmud[j * Cd + k] + a * (nx * g[0] + ny * g[1] + nz * g[2]);
        row[ch] = (float)v;
        double am = a * mu[m * C + ch];
        dn0 += am * g[0], dn1 += am * g[1], dn2 += am * g[2];
      }
      row[C] = (float)dn0, row[C + 1] = (float)dn1, row[C + 2] = (float)dn2;
    }
  }
}

// rows (tree order, C + 3 wide) -> moments N x C / normals N x 3 (original order)
__global__ void k_unpermute_rows(int64_t n, int C, const int32_t* __restrict__ order,
                                 const float* __restrict__ rows, float* moments, float* normals) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int W = C + 3;
  for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < n; j += nw) {
    const int64_t m = order[j];
    const float* row = rows + j * W;
    for (int k = lane; k < W; k += 32) {
      const float v = row[k];
      if (k < C) {
        if (moments) moments[m * C + k] = v;
      } else if (normals) {
        normals[3 * m + (k - C)] = v;
      }
    }
  }
}

__global__ void k_axpy_d(double* __restrict__ dst, const double* __restrict__ src, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] += src[i];
}

// ---------------------------------------------------------------- host

void gradbuf_alloc(GradBuf& b, const Tree& t) {
  b.nodes = t.nodes;
  b.n = t.n;
  b.Cd = t.Cd;
  b.Cr = t.Cr;
  size_t nv = (size_t)t.nodes * t.Cd * 3, ns = (size_t)t.nodes * t.Cr;
  size_t pd = (size_t)t.n * t.Cd, pr = (size_t)t.n * t.Cr, pn = (size_t)t.n * 3;
  b.total = nv + ns + pd + pr + pn + 1;
  b.mem.reserve(b.total * sizeof(double));
  double* base = b.mem.as<double>();
  b.node_v = base;
  b.node_s = b.node_v + nv;
  b.pt_mud = b.node_s + ns;
  b.pt_mur = b.pt_mud + pd;
  b.pt_n = b.pt_mur + pr;
  b.d_eps = b.pt_n + pn;
}

void gradbuf_zero(GradBuf& b, cudaStream_t s) {
  DPL_CUDA(cudaMemsetAsync(b.mem.p, 0, b.total * sizeof(double), s));
}

template <int TD, int NCOL, int GM>
static void adj_launch(const Tree& t, const KParams& kp, const AdjArgs& a, GradBuf& b, int d0,
                       int nd, int r0, int nr) {
  TreeView tv = t.view();
  AdjPtrs p{b.node_v, b.node_s, b.pt_mud, b.pt_mur, b.pt_n, b.d_eps};
  unsigned blocks = (unsigned)((a.q + ADJ_WARPS * 32 - 1) / (ADJ_WARPS * 32));
  k_adjoint<TD, NCOL, GM><<<blocks, ADJ_WARPS * 32, 0, t.stream>>>(
      tv, kp, t.node_row.as<float4>(), nullptr, t.pt_row.as<float4>(), nullptr, a.xs, a.perm, a.q, a.d_out, a.dstride, a.d_grad, d0, nd, r0, nr,
      t.chmap.as<int>(), p, a.overflow);
  count_launch();
}

template <int GM>
static void adj_plan(const Tree& t, const KParams& kp, const AdjArgs& a, GradBuf& b) {
  const int Cd = t.Cd;
  const int Cr = std::min(t.Cr, a.nr_limit >= 0 ? a.nr_limit : t.Cr);
  if (Cd <= 1 && Cr == 0) return adj_launch<1, 0, GM>(t, kp, a, b, 0, Cd, 0, 0);
  if (Cd <= 1 && Cr <= 32) return adj_launch<1, 1, GM>(t, kp, a, b, 0, Cd, 0, Cr);
  if (Cd <= 1 && Cr <= 64) return adj_launch<1, 2, GM>(t, kp, a, b, 0, Cd, 0, Cr);
  // general: first tile carries up to 4 dipole slots and 64 radial slots
  int d = 0, r = 0;
  while (d < Cd || r < Cr) {
    int nd = std::min(4, Cd - d), nr = std::min(64, Cr - r);
    if (nd > 0)
      adj_launch<4, 2, GM>(t, kp, a, b, d, nd, r, std::max(nr, 0));
    else
      adj_launch<0, 2, GM>(t, kp, a, b, 0, 0, r, nr);
    d += std::max(nd, 0);
    r += std::max(nr, 0);
  }
}

void adjoint_launch(const Tree& t, const KParams& kp, const AdjArgs& a, GradBuf& b) {
  static const bool single_phase = getenv("DPL_ADJOINT_SINGLE_PHASE") != nullptr;
  // tensor-memory adjoint (adjoint_tm.cu: tcgen05.mma, accumulators in TMEM) for
  // 4 < Cr <= 48: parity-tested, measured SLOWER than the register-tile FFMA2
  // kernel on B200 (config 2: 23.7 ms vs 13.6 ms, profiles/r02_adjoint_tmem.md),
  // so it is opt-in with DPL_ADJOINT_TMEM=1
  static const bool tmem = getenv("DPL_ADJOINT_TMEM") != nullptr;
  if (!single_phase && tmem && adjoint_tm_launch(t, kp, a, b)) return;
  if (!single_phase && adjoint2_launch(t, kp, a, b)) return;
  if (a.grad_mode == 0) return adj_plan<0>(t, kp, a, b);
  if (a.grad_mode == 1) return adj_plan<1>(t, kp, a, b);
  return adj_plan<2>(t, kp, a, b);
}

void gradbuf_accumulate(GradBuf& dst, const GradBuf& src, cudaStream_t s) {
  k_axpy_d<<<(unsigned)((dst.total + 255) / 256), 256, 0, s>>>(dst.mem.as<double>(),
                                                               src.mem.as<double>(), dst.total);
  count_launch();
}

void flush_pushdown(Tree& t, GradBuf& b) {
  const int B = 256;
  int Wv = 3 * t.Cd, Ws = t.Cr, W = Wv + Ws;
  int levels = (int)t.level_off.size() - 1;
  for (int d = 0; d < levels && W > 0; ++d) {
    int64_t off = t.level_off[d], cnt = t.level_off[d + 1] - off;
    if (!cnt) continue;
    k_pushdown_level<<<(unsigned)((cnt * W + B - 1) / B), B, 0, t.stream>>>(
        off, cnt, W, t.node_parent.as<int32_t>(), t.node_area64.as<double>(), b.node_v, Wv,
        b.node_s, Ws);
    count_launch();
  }
  DPL_CUDA(cudaGetLastError());
}

void flush_rows(Tree& t, const GradBuf& b, int64_t lo, int64_t hi, float* rows) {
  if (hi <= lo) return;
  const int64_t warps = hi - lo;
  const unsigned blocks = (unsigned)std::min<int64_t>((warps + 7) / 8, 148 * 16);
  k_flush_rows<<<blocks, 256, 0, t.stream>>>(
      lo, hi, t.C, t.Cd, t.Cr, t.chmap.as<int>(), t.order.as<int32_t>(), t.pt_leaf.as<int32_t>(),
      t.area64.as<double>(), t.nrm64.as<double>(), t.mu64.as<double>(), b.node_v, b.node_s,
      b.pt_mud, b.pt_mur, b.pt_n, rows);
  count_launch();
  DPL_CUDA(cudaGetLastError());
}

void flush_unpermute(Tree& t, const float* rows, float* moments, float* normals) {
  k_unpermute_rows<<<148 * 16, 256, 0, t.stream>>>(t.n, t.C, t.order.as<int32_t>(), rows, moments,
                                                  normals);
  count_launch();
  DPL_CUDA(cudaGetLastError());
}

void flush_launch(Tree& t, GradBuf& b, float* moments, float* normals) {
  const int B = 256;
  int Wv = 3 * t.Cd, Ws = t.Cr, W = Wv + Ws;
  int levels = (int)t.level_off.size() - 1;
  for (int d = 0; d < levels && W > 0; ++d) {
    int64_t off = t.level_off[d], cnt = t.level_off[d + 1] - off;
    if (!cnt) continue;
    k_pushdown_level<<<(unsigned)((cnt * W + B - 1) / B), B, 0, t.stream>>>(
        off, cnt, W, t.node_parent.as<int32_t>(), t.node_area64.as<double>(), b.node_v, Wv,
        b.node_s, Ws);
    count_launch();
  }
  k_flush_points<<<(unsigned)((t.n + B - 1) / B), B, 0, t.stream>>>(
      t.n, t.C, t.Cd, t.Cr, t.chmap.as<int>(), t.order.as<int32_t>(), t.pt_leaf.as<int32_t>(),
      t.area64.as<double>(), t.nrm64.as<double>(), t.mu64.as<double>(), b.node_v, b.node_s,
      b.pt_mud, b.pt_mur, b.pt_n, moments, normals);
  count_launch();
  if (moments && t.Cr > 0) {
    k_flush_radial<<<148 * 16, B, 0, t.stream>>>(t.n, t.C, t.Cd, t.Cr, t.chmap.as<int>(),
                                                t.order.as<int32_t>(), t.pt_leaf.as<int32_t>(),
                                                t.area64.as<double>(), b.node_s, b.pt_mur, moments);
    count_launch();
  }
  DPL_CUDA(cudaGetLastError());
}

}  // namespace dpl
