// forward2.cu — two-phase (traverse / evaluate) forward traversal, values only.
//
// Same semantics as k_forward<TD, TR, 0> (forward.cu; DipoleTree::primal,
// proj/src/bhtree.cpp:188-234), restructured for the B200 issue model. Each
// warp owns 32 Morton-adjacent queries and alternates two phases over a
// shared-memory batch of ENT interaction entries:
//   phase A (traverse): pop a node, read its packed 64-byte record, evaluate
//     every lane's exact fp64 opening test; for each source the warp interacts
//     with (a far node, or a point of an opened leaf) append one entry — the
//     lane's weights (A W d, A R), zero for lanes that do not take the source,
//     go to shared memory (one STS.128 per lane) and the source's payload row
//     is copied global -> shared with cp.async (one LDGSTS.128 per lane), so
//     the row fetch overlaps the rest of the traversal;
//   phase B (evaluate): a branch-free loop over the batch: one LDS.128 of the
//     lane's weights, broadcast LDS.128 of the row, 3*TD + TR FFMAs.
// The row shape is compile-time (TD dipole float4 + TR/4 radial float4), so
// all address arithmetic is 32-bit and constant-strided.
#include "forward.cuh"
#include "traverse.cuh"

namespace dpl {

__device__ __forceinline__ void cp_async16(uint32_t smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(smem), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// lane weights of one source: (A W dx, A W dy, A W dz, A R)
__device__ __forceinline__ float4 fwd_weights(float fx, float fy, float fz, float r2, float A,
                                              const KParams& kp) {
  const float inv_r = rsqrt_pos(r2);
  float W, R;
  if (kp.mode == KM_SINGULAR || (kp.mode == KM_REGULARIZED && r2 >= kp.near2)) {
    R = inv_r * inv_r;  // tau = 1 beyond t = 6.5 (kernels.cpp:50-55)
    W = R * inv_r;
  } else {
    Co c = coeffs<0>(r2, kp);
    W = c.W;
    R = c.R;
  }
  const float aW = A * W;
  return make_float4(aW * fx, aW * fy, aW * fz, A * R);
}

// MAXR: register cap (occupancy vs. spills; chosen by measurement)
template <int TD, int TR, int WARPS, int ENT, int MAXR = 128, bool COUNT = false>
__global__ void __launch_bounds__(WARPS * 32) __maxnreg__(MAXR)
    k_forward2(TreeView tv, KParams kp, const double* __restrict__ xs,
               const int32_t* __restrict__ perm, int64_t q, int nd, int nr,
               const int* __restrict__ chmap, float* __restrict__ out, int out_stride,
               int only_ch, long long* __restrict__ counters, int* overflow) {
  constexpr int RR = TR / 4;          // radial float4 per row
  constexpr int F4 = TD + RR;         // float4 per row (== tree F4)
  constexpr int WARP_F4 = ENT * 32 + ENT * F4 + DPL_STACK_PER_WARP / 2;
  extern __shared__ float4 smem_f4[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float4* wts = smem_f4 + (size_t)w * WARP_F4;
  float4* rows = wts + ENT * 32;
  int2* stk = reinterpret_cast<int2*>(rows + ENT * F4);
  const uint32_t s_wts = smem_u32(wts) + 16u * lane;  // this lane's weight slot, entry 0
  const uint32_t s_rows = smem_u32(rows) + 16u * lane;

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
  const QueryDF qx = make_qdf(x, tv.cmax);

  float accd[TD > 0 ? TD : 1], accr[TR > 0 ? TR : 1];
#pragma unroll
  for (int k = 0; k < (TD > 0 ? TD : 1); ++k) accd[k] = 0.f;
#pragma unroll
  for (int k = 0; k < (TR > 0 ? TR : 1); ++k) accr[k] = 0.f;

  const bool singular = kp.mode == KM_SINGULAR;
  const float4* __restrict__ node_row = tv.node_row;
  const float4* __restrict__ pt_row = tv.pt_row;
  int nent = 0;

  auto evaluate = [&]() {
    cp_async_wait_all();
    __syncwarp();
    for (int e = 0; e < nent; ++e) {
      const float4 wv = wts[e * 32 + lane];
      const float4* row = rows + e * F4;
#pragma unroll
      for (int k = 0; k < TD; ++k) {
        const float4 v = row[k];
        accd[k] = fmaf(wv.x, v.x, fmaf(wv.y, v.y, fmaf(wv.z, v.z, accd[k])));
      }
#pragma unroll
      for (int k4 = 0; k4 < RR; ++k4) {
        const float4 s = row[TD + k4];
        accr[4 * k4 + 0] = fmaf(wv.w, s.x, accr[4 * k4 + 0]);
        accr[4 * k4 + 1] = fmaf(wv.w, s.y, accr[4 * k4 + 1]);
        accr[4 * k4 + 2] = fmaf(wv.w, s.z, accr[4 * k4 + 2]);
        accr[4 * k4 + 3] = fmaf(wv.w, s.w, accr[4 * k4 + 3]);
      }
    }
    __syncwarp();
    nent = 0;
  };

  auto append = [&](float4 wv, const float4* rowsrc) {
    if (nent == ENT) evaluate();
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(s_wts + 512u * nent),
                 "f"(wv.x), "f"(wv.y), "f"(wv.z), "f"(wv.w));
    if (lane < F4) cp_async16(s_rows + 16u * F4 * nent, rowsrc + lane);
    ++nent;
  };

  // COUNT: per-query replay counters (visited, far near/far, point near/far);
  // same kernel as the values-only launch so primal(visited) == primal()
  long long c_vis = 0, c_fn = 0, c_ff = 0, c_pn = 0, c_pf = 0;
  const bool reg = kp.mode == KM_REGULARIZED;

  int sp = 1;
  if (lane == 0) stk[0] = make_int2(0, (int)active);
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
    if (COUNT && mine) ++c_vis;
    if (COUNT && far) (reg && s < kp.near2) ? ++c_fn : ++c_ff;
    const unsigned farm = __ballot_sync(FULL_MASK, far);
    if (farm && A > 0.f) {  // area > 0 (bhtree.cpp:205)
      const float4 wv = far ? fwd_weights(dx, dy, dz, s, A, kp) : make_float4(0.f, 0.f, 0.f, 0.f);
      append(wv, node_row + (size_t)node * F4);
    }
    const unsigned openm = mask & ~farm;
    if (openm) {
      if (tp.y == 0) {
        const bool me_open = (openm >> lane) & 1u;
        for (int j = tp.z; j < tp.w; ++j) {
          float4 wv = make_float4(0.f, 0.f, 0.f, 0.f);
          if (me_open) {
            const PtRec* pr = tv.pt_rec + j;
            const float4 ph = __ldg(&pr->hi);
            const float r2 = dist2_df(ph, __ldg(&pr->lo), qx, dx, dy, dz);
            // exact coincidence only matters for the singular kernel (bhtree.cpp:219);
            // the regularized kernel's r = 0 contribution is identically zero
            if (!(singular && r2 == 0.f && coincident_exact(tv.pt_pos64 + 3 * (size_t)j, x))) {
              wv = fwd_weights(dx, dy, dz, r2, ph.w, kp);
              if (COUNT) (reg && r2 < kp.near2) ? ++c_pn : ++c_pf;
            }
          }
          append(wv, pt_row + (size_t)j * F4);
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
  if (!valid) return;
  if (COUNT) {
    long long* cq = counters + 5 * qi;
    cq[0] = c_vis, cq[1] = c_fn, cq[2] = c_ff, cq[3] = c_pn, cq[4] = c_pf;
  }
  if (only_ch >= 0) {  // primal_channel: same arithmetic, one column stored
#pragma unroll
    for (int k = 0; k < TD; ++k)
      if (k < nd && __ldg(chmap + k) == only_ch) out[qi] = accd[k];
#pragma unroll
    for (int k = 0; k < TR; ++k)
      if (k < nr && __ldg(chmap + TD + k) == only_ch) out[qi] = accr[k];
    return;
  }
  float* o = out + qi * out_stride;
#pragma unroll
  for (int k = 0; k < TD; ++k)
    if (k < nd) o[__ldg(chmap + k)] = accd[k];
#pragma unroll
  for (int k = 0; k < TR; ++k)
    if (k < nr) o[__ldg(chmap + TD + k)] = accr[k];
}

template <int TD, int TR, int WARPS, int ENT, int MAXR, bool COUNT>
static void launch2c(const Tree& t, const KParams& kp, const FwdArgs& a, int nd, int nr) {
  constexpr int F4 = TD + TR / 4;
  const size_t smem = (size_t)WARPS * (ENT * 32 + ENT * F4 + DPL_STACK_PER_WARP / 2) * 16;
  static std::atomic<unsigned long long> attr{0};
  ensure_max_dyn_smem(k_forward2<TD, TR, WARPS, ENT, MAXR, COUNT>, t.device, smem, attr);
  unsigned blocks = (unsigned)((a.q + WARPS * 32 - 1) / (WARPS * 32));
  k_forward2<TD, TR, WARPS, ENT, MAXR, COUNT><<<blocks, WARPS * 32, smem, t.stream>>>(
      t.view(), kp, a.xs, a.perm, a.q, nd, nr, t.chmap.as<int>(), a.out, a.out_stride, a.only_ch,
      a.counters, a.overflow);
  count_launch();
}

template <int TD, int TR, int WARPS, int ENT, int MAXR = 128>
static void launch2(const Tree& t, const KParams& kp, const FwdArgs& a, int nd, int nr) {
  if (a.counters)
    launch2c<TD, TR, WARPS, ENT, MAXR, true>(t, kp, a, nd, nr);
  else
    launch2c<TD, TR, WARPS, ENT, MAXR, false>(t, kp, a, nd, nr);
}

static int tune_choice(const char* env) {
  const char* v = getenv(env);
  return v ? atoi(v) : 0;
}

// Values-only plan for the two-phase kernel: the compile-time row shape must
// equal the tree's (one dipole slot + PR radial floats). Returns false when
// not covered (the caller falls back to the single-phase kernels).
bool forward2_launch(const Tree& t, const KParams& kp, const FwdArgs& a) {
  if (a.grad_mode != 0 || (a.single && a.only_ch < 0)) return false;
  if (t.Cd != 1) return false;
  const int nr = a.nr_limit >= 0 ? std::min(a.nr_limit, t.Cr) : t.Cr;
  constexpr int W = 4, E = 16;
  switch (t.PR) {
    case 4: return launch2<1, 4, W, E>(t, kp, a, 1, nr), true;
    case 16: return launch2<1, 16, W, E>(t, kp, a, 1, nr), true;
    case 48:
      switch (tune_choice("DPL_TUNE_FWD")) {  // (batch, register cap) experiments
        case 1: return launch2<1, 48, W, 8, 128>(t, kp, a, 1, nr), true;
        case 2: return launch2<1, 48, W, 8, 112>(t, kp, a, 1, nr), true;
        case 3: return launch2<1, 48, W, 8, 104>(t, kp, a, 1, nr), true;
        case 4: return launch2<1, 48, W, 8, 96>(t, kp, a, 1, nr), true;
        case 5: return launch2<1, 48, W, 12, 112>(t, kp, a, 1, nr), true;
        case 6: return launch2<1, 48, W, 16, 128>(t, kp, a, 1, nr), true;
        default: return launch2<1, 48, W, 8, 128>(t, kp, a, 1, nr), true;  // measured best
      }
    default: return false;
  }
}

}  // namespace dpl
