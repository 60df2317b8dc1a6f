// forward.cu — K5/K6 forward traversals and K10 query Morton sort.
//
// Restates DipoleTree::primal / primal_channel / primal_with_gradient
// (proj/src/bhtree.cpp:188-334) for a batch of queries. Channels are processed
// in tiles of TD dipole and TR radial slots (template parameters) so that all
// accumulators live in registers; the common layouts (C = 2, 4, 49 with channel
// 0 Dipole) run in one pass.
//
// Interaction (far node or leaf point), with d = source - x, A = area/(4 pi):
//   dipole slot:  out += A W (v . d);      grad -= A (W v + Wp_r (v . d) d)
//   radial slot:  out += A R s;            grad -= A Rp_r s d
// where (v, s) are the node moments (bhtree.cpp:205-213, :295-310) or, for a
// leaf point, (mu_c n_m, mu_c) (bhtree.cpp:214-229, :311-329) — one formula.
#include <cub/cub.cuh>

#include "forward.cuh"
#include "traverse.cuh"

namespace dpl {

constexpr int FWD_WARPS = 4;

template <int TD, int TR, int GRAD>
struct FAcc {
  float vd[TD > 0 ? TD : 1];
  float vr[TR > 0 ? TR : 1];
  float gd[(GRAD && TD > 0) ? TD : 1][3];
  float gr[(GRAD == 1 && TR > 0) ? TR : 1][3];
};

// coeffs()'s tau = 1 branch (kernels.cpp:50-55, and the singular kernel), for
// list entries whose far lanes are all beyond 6.5 eps (IL_NEAR clear)
template <int ORDER>
__device__ __forceinline__ Co far_coeffs(float r2) {
  Co c;
  const float inv_r = rsqrt_pos(r2);
  const float inv_r2 = inv_r * inv_r;
  c.R = inv_r2;
  c.W = inv_r2 * inv_r;
  c.Wp_r = ORDER >= 1 ? -3.0f * c.W * inv_r2 : 0.f;
  c.Rp_r = ORDER >= 1 ? -2.0f * inv_r2 * inv_r2 : 0.f;
  c.dW_de = c.dWp_r_de = c.dR_de = 0.f;
  c.near = false;
  return c;
}

template <int TD, int TR, int GRAD>
__device__ __forceinline__ void f_interact(FAcc<TD, TR, GRAD>& a, float fx, float fy, float fz,
                                           float r2, float A, const float4* __restrict__ pd,
                                           const float* __restrict__ pr, int nd, int nr,
                                           const KParams& kp, bool& near, bool tau1 = false) {
  Co c = tau1 ? far_coeffs<GRAD ? 1 : 0>(r2) : coeffs<GRAD ? 1 : 0>(r2, kp);
  near = c.near;
  const float aW = A * c.W, aR = A * c.R;
#pragma unroll
  for (int k = 0; k < TD; ++k) {
    if (k < nd) {
      float4 v = __ldg(pd + k);
      float vdot = fmaf(v.x, fx, fmaf(v.y, fy, v.z * fz));
      a.vd[k] = fmaf(aW, vdot, a.vd[k]);
      if (GRAD == 1 || (GRAD == 2 && k == 0)) {
        float t = A * c.Wp_r * vdot;
        a.gd[k][0] -= fmaf(aW, v.x, t * fx);
        a.gd[k][1] -= fmaf(aW, v.y, t * fy);
        a.gd[k][2] -= fmaf(aW, v.z, t * fz);
      }
    }
  }
  if (TR % 4 == 0) {
#pragma unroll
    for (int k4 = 0; k4 < TR / 4; ++k4) {
      if (4 * k4 < nr) {
        float4 s = __ldg(reinterpret_cast<const float4*>(pr) + k4);
        float sv[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = 4 * k4 + u;
          a.vr[k] = fmaf(aR, sv[u], a.vr[k]);
          if (GRAD == 1) {
            float t = A * c.Rp_r * sv[u];
            a.gr[k][0] = fmaf(-t, fx, a.gr[k][0]);
            a.gr[k][1] = fmaf(-t, fy, a.gr[k][1]);
            a.gr[k][2] = fmaf(-t, fz, a.gr[k][2]);
          }
        }
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < TR; ++k) {
      if (k < nr) {
        float s = __ldg(pr + k);
        a.vr[k] = fmaf(aR, s, a.vr[k]);
        if (GRAD == 1) {
          float t = A * c.Rp_r * s;
          a.gr[k][0] = fmaf(-t, fx, a.gr[k][0]);
          a.gr[k][1] = fmaf(-t, fy, a.gr[k][1]);
          a.gr[k][2] = fmaf(-t, fz, a.gr[k][2]);
        }
      }
    }
  }
}

namespace {
__device__ __forceinline__ void cp_async16(uint32_t smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(smem), "l"(gmem));
}
}  // namespace

// GRAD: 0 values only; 1 gradients of every channel in the tile; 2 gradient of
// dipole slot 0 only (render step). single: write column 0 of a q x 1 output.
// LIST: replay the batch's interaction lists (ilist.cuh; same entries in the
// same order as the walk, so identical results); incomplete warps walk.
// SPEC: regularized kernel and a full tile (nd == TD, every radial slot of the
// tile evaluated — rows are padded — and only the first nr stored), so the
// mode and slot tests fold away
template <int TD, int TR, int GRAD, bool COUNT, bool LIST = false, bool SPEC = false>
__global__ void __launch_bounds__(FWD_WARPS * 32)
    k_forward(TreeView tv, KParams kp_in, const float4* __restrict__ payd_n,
              const float* __restrict__ payr_n, const float4* __restrict__ payd_p,
              const float* __restrict__ payr_p, const double* __restrict__ xs,
              const int32_t* __restrict__ perm, int64_t q, int d0, int nd, int r0, int nr,
              const int* __restrict__ chmap, float* __restrict__ out, int out_stride, int single,
              float* __restrict__ grad, long long* __restrict__ counters, IListView lv,
              int* overflow) {
  __shared__ __align__(16) int2 stk[FWD_WARPS][DPL_STACK_PER_WARP];
  KParams kp = kp_in;
  if (SPEC) kp.mode = KM_REGULARIZED;
  const int ndi = SPEC ? TD : nd, nri = SPEC ? TR : nr;  // slots evaluated
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t sidx = ((int64_t)blockIdx.x * FWD_WARPS + w) * 32 + lane;
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
  // double-float query + the fp64 position re-read only on the exact paths
  const QueryDF qx = make_qdf(x, tv.cmax);
  const double* xq = xs + 3 * qi;
  FAcc<TD, TR, GRAD> a;
#pragma unroll
  for (int k = 0; k < (TD > 0 ? TD : 1); ++k) a.vd[k] = 0.f;
#pragma unroll
  for (int k = 0; k < ((GRAD && TD > 0) ? TD : 1); ++k) a.gd[k][0] = a.gd[k][1] = a.gd[k][2] = 0.f;
#pragma unroll
  for (int k = 0; k < (TR > 0 ? TR : 1); ++k) a.vr[k] = 0.f;
#pragma unroll
  for (int k = 0; k < ((GRAD == 1 && TR > 0) ? TR : 1); ++k) a.gr[k][0] = a.gr[k][1] = a.gr[k][2] = 0.f;
  long long c_vis = 0, c_fn = 0, c_ff = 0, c_pn = 0, c_pf = 0;
  // payload rows: [dipole float4 x Cd | radial floats]; row stride F4 float4
  const float4* pdn = payd_n + d0;
  const float* prn = reinterpret_cast<const float*>(payd_n + tv.Cd) + r0;
  const float4* pdp = payd_p + d0;
  const float* prp = reinterpret_cast<const float*>(payd_p + tv.Cd) + r0;
  const bool skip_coincident = GRAD != 0 || kp.mode == KM_SINGULAR;  // :219 vs :316

  // the points of an opened leaf for this lane (bhtree.cpp:214-229, :311-329)
  auto leaf = [&](const int4 tp) {
    for (int j = tp.z; j < tp.w; ++j) {
      const PtRec* pr = tv.pt_rec + j;
      const float4 ph = __ldg(&pr->hi);
      float dx, dy, dz;
      const float r2 = dist2_df(ph, __ldg(&pr->lo), qx, dx, dy, dz);
      // exact coincidence (fp64) is only possible when the fp32 r2 is 0
      if (skip_coincident && r2 == 0.f && coincident_exact(tv.pt_pos64 + 3 * (size_t)j, xq))
        continue;
      bool near;
      f_interact<TD, TR, GRAD>(a, dx, dy, dz, r2, ph.w, pdp + (int64_t)j * tv.F4,
                               prp + (int64_t)j * 4 * tv.F4, ndi, nri, kp, near);
      if (COUNT) near ? ++c_pn : ++c_pf;
    }
  };

  const int64_t wg = (int64_t)blockIdx.x * FWD_WARPS + w;
  const int total = LIST ? __ldg(lv.count + wg) : -1;
  if (LIST && total >= 0) {
    // 32 entries at a time, their node records prefetched into the (unused)
    // stack region with cp.async and read back as broadcast loads
    NodeRec* rb = reinterpret_cast<NodeRec*>(stk[w]);
    const uint32_t s_rb = (uint32_t)__cvta_generic_to_shared(stk[w]) + 48u * lane;
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
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      // the entry itself goes into its record's unused child fields (topo.x/y;
      // the replay reads only the point range z/w): one broadcast LDS.128 per
      // entry instead of two shuffles
      if (lane < n) *reinterpret_cast<uint2*>(&rb[lane].topo) = my;
      __syncwarp();
      for (int i = 0; i < n; ++i) {
        const int4 tpi = rb[i].topo;
        const uint32_t src = (uint32_t)tpi.x;
        const unsigned m = (unsigned)tpi.y;
        if (i + 1 < n && !((src | (uint32_t)rb[i + 1].topo.x) & (IL_LEAF | IL_NEAR))) {
          // two far entries without near lanes, interleaved and branch-free:
          // a lane outside an entry's mask adds exact zeros (area 0, finite r)
          const int4 tpj = rb[i + 1].topo;
          const bool ma = (m >> lane) & 1u, mb = ((unsigned)tpj.y >> lane) & 1u;
          const float4 ha = rb[i].hi, la = rb[i].lo, hb = rb[i + 1].hi, lb = rb[i + 1].lo;
          float ax, ay, az, bx, by, bz;
          const float sa = dist2_df(ha, la, qx, ax, ay, az);
          const float sb = dist2_df(hb, lb, qx, bx, by, bz);
          const int na = (int)(src & IL_NODE), nb = (int)((uint32_t)tpj.x & IL_NODE);
          bool near;
          f_interact<TD, TR, GRAD>(a, ax, ay, az, ma ? sa : 1.f, ma ? la.w : 0.f,
                                   pdn + (int64_t)na * tv.F4, prn + (int64_t)na * 4 * tv.F4, ndi,
                                   nri, kp, near, true);
          f_interact<TD, TR, GRAD>(a, bx, by, bz, mb ? sb : 1.f, mb ? lb.w : 0.f,
                                   pdn + (int64_t)nb * tv.F4, prn + (int64_t)nb * 4 * tv.F4, ndi,
                                   nri, kp, near, true);
          ++i;
          continue;
        }
        if (!((m >> lane) & 1u)) continue;
        const int node = (int)(src & IL_NODE);
        if (!(src & IL_LEAF)) {
          const float4 hi = rb[i].hi, lo = rb[i].lo;
          float dx, dy, dz;
          const float s = dist2_df(hi, lo, qx, dx, dy, dz);
          bool near;
          f_interact<TD, TR, GRAD>(a, dx, dy, dz, s, lo.w, pdn + (int64_t)node * tv.F4,
                                   prn + (int64_t)node * 4 * tv.F4, ndi, nri, kp, near,
                                   !(src & IL_NEAR));
        } else {
          leaf(tpi);
        }
      }
    }
  }

  int sp = (LIST && total >= 0) ? 0 : 1;
  if (sp && lane == 0) stk[w][0] = make_int2(0, (int)active);
  __syncwarp();
  while (sp > 0) {
    --sp;
    const int2 e = stk[w][sp];
    __syncwarp();
    const int node = e.x;
    const unsigned mask = (unsigned)e.y;
    const bool mine = (mask >> lane) & 1u;
    // the reference's opening test (bhtree.cpp:202-204) decided in fp32 on the
    // double-float record, exactly in fp64 inside the error band (traverse.cuh)
    const NodeRec* rec = tv.node_rec + node;
    const float4 hi = __ldg(&rec->hi);
    const float4 lo = __ldg(&rec->lo);
    const int4 tp = __ldg(&rec->topo);
    float dx, dy, dz;
    const float s = dist2_df(hi, lo, qx, dx, dy, dz);
    const bool far = mine && far_test(s, hi, qx, xq, tv.node_dec + node);
    const unsigned farm = __ballot_sync(FULL_MASK, far);
    if (COUNT && mine) ++c_vis;
    if (far && (__ldg(tv.node_flag + node) & 1)) {
      bool near;
      f_interact<TD, TR, GRAD>(a, dx, dy, dz, s, lo.w,
                               pdn + (int64_t)node * tv.F4, prn + (int64_t)node * 4 * tv.F4,
                               ndi, nri,
                               kp, near);
      if (COUNT) near ? ++c_fn : ++c_ff;
    }
    const unsigned openm = mask & ~farm;
    if (openm) {
      if (tp.y == 0) {
        if ((openm >> lane) & 1u) leaf(tp);
        __syncwarp();
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
  if (!valid) return;
  if (single) {
    out[qi] = TD > 0 && nd > 0 ? a.vd[0] : a.vr[0];
  } else {
#pragma unroll
    for (int k = 0; k < TD; ++k)
      if (k < nd) {
        int ch = __ldg(chmap + d0 + k);
        out[qi * out_stride + ch] = a.vd[k];
        if (GRAD == 1) {
          float* g = grad + (qi * out_stride + ch) * 3;
          g[0] = a.gd[k][0], g[1] = a.gd[k][1], g[2] = a.gd[k][2];
        }
      }
    if (GRAD == 2 && TD > 0 && nd > 0 && d0 == 0) {
      float* g = grad + qi * 3;
      g[0] = a.gd[0][0], g[1] = a.gd[0][1], g[2] = a.gd[0][2];
    }
    const int cd = tv.Cd;
#pragma unroll
    for (int k = 0; k < TR; ++k)
      if (k < nr) {
        int ch = __ldg(chmap + cd + r0 + k);
        out[qi * out_stride + ch] = a.vr[k];
        if (GRAD == 1) {
          float* g = grad + (qi * out_stride + ch) * 3;
          g[0] = a.gr[k][0], g[1] = a.gr[k][1], g[2] = a.gr[k][2];
        }
      }
  }
  if (COUNT) {
    long long* cq = counters + 5 * qi;
    cq[0] = c_vis, cq[1] = c_fn, cq[2] = c_ff, cq[3] = c_pn, cq[4] = c_pf;
  }
}

// ---------------------------------------------------------------- K10
__device__ __forceinline__ uint32_t spread10(uint32_t v) {
  v &= 0x3ff;
  v = (v | (v << 16)) & 0x030000FF;
  v = (v | (v << 8)) & 0x0300F00F;
  v = (v | (v << 4)) & 0x030C30C3;
  v = (v | (v << 2)) & 0x09249249;
  return v;
}

// 3-D Hilbert index of 10-bit coordinates (Skilling's transpose form): no
// long jumps between consecutive cells, so the 32 queries of a warp are more
// compact than along the Morton curve
__device__ __forceinline__ uint32_t hilbert3(uint32_t x, uint32_t y, uint32_t z) {
  uint32_t X[3] = {x, y, z};
  for (uint32_t Q = 1u << 9; Q > 1; Q >>= 1) {
    const uint32_t P = Q - 1;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      if (X[i] & Q) {
        X[0] ^= P;
      } else {
        const uint32_t t = (X[0] ^ X[i]) & P;
        X[0] ^= t;
        X[i] ^= t;
      }
    }
  }
  X[1] ^= X[0];
  X[2] ^= X[1];
  uint32_t t = 0;
  for (uint32_t Q = 1u << 9; Q > 1; Q >>= 1)
    if (X[2] & Q) t ^= Q - 1;
  X[0] ^= t, X[1] ^= t, X[2] ^= t;
  uint32_t key = 0;
  for (int bit = 9; bit >= 0; --bit)
    key = (key << 3) | (((X[0] >> bit) & 1) << 2) | (((X[1] >> bit) & 1) << 1) | ((X[2] >> bit) & 1);
  return key;
}

__global__ void k_morton(const double* __restrict__ xs, int64_t q, double lx, double ly,
                         double lz, double inv, int hilbert, uint32_t* keys, int32_t* idx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= q) return;
  auto qz = [&](double v, double lo) {
    double f = (v - lo) * inv;
    f = f < 0 ? 0 : (f > 1023 ? 1023 : f);
    return (uint32_t)f;
  };
  uint32_t a = qz(xs[3 * i], lx), b = qz(xs[3 * i + 1], ly), c = qz(xs[3 * i + 2], lz);
  keys[i] = hilbert ? hilbert3(a, b, c) : (spread10(a) | (spread10(b) << 1) | (spread10(c) << 2));
  idx[i] = (int32_t)i;
}

void morton_order(Tree& t, const double* xs_dev, int64_t q, int32_t* perm_out, DevBuf& ws) {
  if (q <= 0) return;
  double ext = 0;
  for (int a = 0; a < 3; ++a) ext = std::max(ext, t.root_hi[a] - t.root_lo[a]);
  double pad = 0.5 * ext + 1e-12;
  double lo[3];
  for (int a = 0; a < 3; ++a) lo[a] = 0.5 * (t.root_lo[a] + t.root_hi[a]) - 2 * pad;
  double inv = 1024.0 / (4 * pad);  // frame: 2x the root cell around its centre
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (int32_t*)nullptr, (int32_t*)nullptr, (int)q, 0, 30, t.stream);
  size_t need = q * 4 * 3 + tb + 256;
  ws.reserve(need);
  char* base = ws.as<char>();
  uint32_t* keys = (uint32_t*)base;
  uint32_t* keys_s = keys + q;
  int32_t* idx = (int32_t*)(keys_s + q);
  void* tmp = (void*)(((uintptr_t)(idx + q) + 255) & ~(uintptr_t)255);
  // Hilbert order by default (config 2: step 38.3 -> 36.0 ms vs Morton);
  // DPL_ORDER_MORTON=1 restores the Morton curve
  static const bool hilbert = getenv("DPL_ORDER_MORTON") == nullptr;
  k_morton<<<(unsigned)((q + 255) / 256), 256, 0, t.stream>>>(xs_dev, q, lo[0], lo[1], lo[2], inv,
                                                               hilbert ? 1 : 0, keys, idx);
  count_launch();
  DPL_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys_s, idx, perm_out, (int)q, 0, 30,
                                           t.stream));
  count_launch(3);
}

// ---------------------------------------------------------------- dispatch
// LISTS: also instantiate the list-replay kernel (used when a.ilist is set)
template <int TD, int TR, int GRAD, bool LISTS = false>
static void launch_one(const Tree& t, const KParams& kp, FwdArgs& a, int d0, int nd, int r0,
                       int nr) {
  TreeView tv = t.view();
  unsigned blocks = (unsigned)((a.q + FWD_WARPS * 32 - 1) / (FWD_WARPS * 32));
  IListView lv{};
  auto run = [&](auto kern) {
    kern<<<blocks, FWD_WARPS * 32, 0, t.stream>>>(
        tv, kp, t.node_row.as<float4>(), nullptr, t.pt_row.as<float4>(), nullptr, a.xs, a.perm,
        a.q, d0, nd, r0, nr, t.chmap.as<int>(), a.out, a.out_stride, a.single, a.grad, a.counters,
        lv, a.overflow);
  };
  if (a.counters) {
    run(k_forward<TD, TR, GRAD, true>);
  } else if (LISTS && a.ilist && !no_ilist()) {
    ilist_build(t, *a.ilist, a.xs, a.perm, a.q, a.beta, ilist_near_thr(kp), a.overflow);
    lv = a.ilist->view();
    if (kp.mode == KM_REGULARIZED && nd == TD && nr >= 1)
      run(k_forward<TD, TR, GRAD, false, true, true>);
    else
      run(k_forward<TD, TR, GRAD, false, true>);
  } else if (LISTS && kp.mode == KM_REGULARIZED && nd == TD && nr >= 1) {
    run(k_forward<TD, TR, GRAD, false, false, true>);
  } else {
    run(k_forward<TD, TR, GRAD, false>);
  }
  a.counters = nullptr;  // later tiles re-walk the same decisions: count once
  count_launch();
}

// Channel-tile plan: (TD, TR) instantiations tried in order; the first that
// covers the tile in one pass wins, otherwise tiles of the largest are used.
void forward_launch(const Tree& t, const KParams& kp, FwdArgs a) {
  static const bool single_phase = getenv("DPL_FORWARD_SINGLE_PHASE") != nullptr;
  static const bool no_tc = getenv("DPL_FORWARD_NO_TC") != nullptr;
  // accumulator in tensor memory (forward_tm.cu), opt-in with DPL_FORWARD_TMEM=1
  if (!single_phase && !no_tc && forward_tmem_enabled() && forward_tm_launch(t, kp, a)) return;
  if (!single_phase && !no_tc && forward_tc_launch(t, kp, a)) return;
  if (!single_phase && forward2_launch(t, kp, a)) return;
  const int Cd = a.only_dip >= 0 ? 1 : (a.only_rad >= 0 ? 0 : t.Cd);
  const int Cr = a.only_rad >= 0 ? 1
                 : (a.only_dip >= 0 ? 0 : (a.nr_limit >= 0 ? std::min(a.nr_limit, t.Cr) : t.Cr));
  const int dbase = a.only_dip >= 0 ? a.only_dip : 0;
  const int rbase = a.only_rad >= 0 ? a.only_rad : 0;
  if (a.grad_mode == 0) {
    if (Cd <= 1 && Cr == 0) return launch_one<1, 0, 0>(t, kp, a, dbase, Cd, 0, 0);
    if (Cd == 0 && Cr == 1) return launch_one<0, 1, 0>(t, kp, a, 0, 0, rbase, 1);
    if (Cd <= 1 && Cr <= 1) return launch_one<1, 1, 0>(t, kp, a, 0, Cd, 0, Cr);
    if (Cd <= 1 && Cr <= 4) return launch_one<1, 4, 0>(t, kp, a, 0, Cd, 0, Cr);
    if (Cd <= 1 && Cr <= 16) return launch_one<1, 16, 0>(t, kp, a, 0, Cd, 0, Cr);
    if (Cd <= 1 && Cr <= 48) return launch_one<1, 48, 0>(t, kp, a, 0, Cd, 0, Cr);
    // general: dipole tiles of 4, radial tiles of 48
    for (int d = 0; d < Cd; d += 4) launch_one<4, 0, 0>(t, kp, a, d, std::min(4, Cd - d), 0, 0);
    for (int r = 0; r < Cr; r += 48) launch_one<0, 48, 0>(t, kp, a, 0, 0, r, std::min(48, Cr - r));
    return;
  }
  if (a.grad_mode == 2) {  // values of all channels + gradient of dipole slot 0
    if (Cd < 1) throw Error(1, "grad0 requires a dipole channel 0");
    if (Cd == 1 && Cr <= 4) return launch_one<1, 4, 2, true>(t, kp, a, 0, 1, 0, Cr);
    if (Cd == 1 && Cr <= 16) return launch_one<1, 16, 2>(t, kp, a, 0, 1, 0, Cr);
    if (Cd == 1 && Cr <= 48) return launch_one<1, 48, 2>(t, kp, a, 0, 1, 0, Cr);
    launch_one<1, 0, 2>(t, kp, a, 0, 1, 0, 0);
    for (int d = 1; d < Cd; d += 4) launch_one<4, 0, 0>(t, kp, a, d, std::min(4, Cd - d), 0, 0);
    for (int r = 0; r < Cr; r += 48) launch_one<0, 48, 0>(t, kp, a, 0, 0, r, std::min(48, Cr - r));
    return;
  }
  // full gradients
  if (Cd <= 1 && Cr == 0) return launch_one<1, 0, 1>(t, kp, a, dbase, Cd, 0, 0);
  if (Cd == 0 && Cr == 1) return launch_one<0, 1, 1>(t, kp, a, 0, 0, rbase, 1);
  if (Cd <= 1 && Cr <= 1) return launch_one<1, 1, 1>(t, kp, a, 0, Cd, 0, Cr);
  if (Cd <= 1 && Cr <= 4) return launch_one<1, 4, 1>(t, kp, a, 0, Cd, 0, Cr);
  for (int d = 0; d < Cd; d += 4) launch_one<4, 0, 1>(t, kp, a, d, std::min(4, Cd - d), 0, 0);
  for (int r = 0; r < Cr; r += 16) launch_one<0, 16, 1>(t, kp, a, 0, 0, r, std::min(16, Cr - r));
}

}  // namespace dpl
