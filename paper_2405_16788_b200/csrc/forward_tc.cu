// forward_tc.cu — two-phase forward with the radial-channel contraction on
// tensor cores (mma.sync m16n8k8 TF32, 3xTF32 split for fp32 accuracy).
//
// Phase A is forward2.cu's (exact opening decisions, per-lane weights into
// shared memory, cp.async-staged payload rows). Phase B is a dense product
// per batch of ENT entries:
//     out[32 queries x TR radial] += Wr[32 x ENT] . Rows[ENT x TR]
// with Wr[l][e] = A R of lane l for entry e (0 when lane l does not take e).
// Each operand is split a = hi + lo (hi = a truncated to tf32, lo = a - hi
// exact, read by the tensor core at tf32 precision) and hi.hi + hi.lo + lo.hi
// is accumulated in fp32 (error <~ 2^-19 relative per product; the dropped
// lo.lo term is < 2^-20). The dipole slot (3 FMA per entry) stays on the FP32
// pipe.
// Shared-memory strides are padded so every fragment load is bank-conflict
// free: weights Wr[ENT][40], rows [ENT][RSF] with RSF = 8 or 24 mod 32 floats.
#include "forward.cuh"
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
// a = hi + lo with hi = a truncated to tf32 (exact residual lo, |lo| < 2^-10 |a|);
// lo goes to the MMA as raw fp32 bits — the tensor core reads its top 19 bits,
// an error <= 2^-10 |lo| <= 2^-20 |a|. 2 instructions instead of 2 roundings.
__device__ __forceinline__ void split_tf32(float a, uint32_t& hi, uint32_t& lo) {
  hi = __float_as_uint(a) & 0xffffe000u;
  lo = __float_as_uint(a - __uint_as_float(hi));
}
__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
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

// fwd_w's far-field branch for every lane (tau = 1; the list says no far lane
// of this entry is within 6.5 eps, or the kernel is singular)
__device__ __forceinline__ float4 fwd_w_far(float fx, float fy, float fz, float r2, float A) {
  const float inv_r = rsqrt_pos(r2);
  const float R = inv_r * inv_r;
  const float W = R * inv_r;
  const float aW = A * W;
  return make_float4(aW * fx, aW * fy, aW * fz, A * R);
}

// fwd_w_far with the non-member lanes' area already zeroed (regularized
// kernels: members have r2 >= near2, see rsqrt_far)
__device__ __forceinline__ float4 fwd_w_far_m(float fx, float fy, float fz, float r2, float Am,
                                              float near2) {
  const float inv_r = rsqrt_far(r2, near2);
  const float R = inv_r * inv_r;
  const float aW = Am * (R * inv_r);
  return make_float4(aW * fx, aW * fy, aW * fz, Am * R);
}

constexpr int row_stride_floats(int f4) {
  int r = 4 * f4;
  while (r % 32 != 8 && r % 32 != 24) r += 4;
  return r;
}
}  // namespace

// NT: radial n-tiles of 8 channels (TR = 8 NT); one dipole slot.
// LIST: replay the batch's interaction lists (ilist.cuh) instead of walking the
// tree; warps whose list is incomplete walk it as in the fused kernel. Both
// paths run the same arithmetic in the same entry order -> identical results.
// REG: compiled for the regularized kernel (the mode tests fold away)
template <int NT, int WARPS, int ENT, int MAXR, bool COUNT, bool LIST, bool REG = false>
__global__ void __launch_bounds__(WARPS * 32) __maxnreg__(MAXR)
    k_forward_tc(TreeView tv, KParams kp_in, const double* __restrict__ xs,
                 const int32_t* __restrict__ perm, int64_t q, int nr,
                 const int* __restrict__ chmap, float* __restrict__ out, int out_stride,
                 int only_ch, long long* __restrict__ counters, IListView lv, int* overflow) {
  static_assert(ENT % 8 == 0, "ENT must be a multiple of the mma K (8)");
  KParams kp = kp_in;
  if (REG) kp.mode = KM_REGULARIZED;
  constexpr int TR = 8 * NT;
  constexpr int F4 = 1 + TR / 4;               // global row float4 (dipole + radial)
  constexpr int RSF = row_stride_floats(F4);   // padded smem row stride (floats)
  constexpr int WSTR = 40;                     // padded Wr row stride (floats)
  // the dipole slot is accumulated in phase A (its moment float4 arrives with the
  // node-record window, vb), so no per-lane dipole weights go through shared memory
  constexpr int WARP_FLOATS = ENT * WSTR + ENT * RSF + 2 * DPL_STACK_PER_WARP + 32 * 4;
  extern __shared__ float4 smem_f4[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;  // mma fragment coordinates
  float* base = reinterpret_cast<float*>(smem_f4) + (size_t)w * WARP_FLOATS;
  float* wr = base;                 // [ENT][WSTR]  A R
  float* rows = wr + ENT * WSTR;    // [ENT][RSF] (the dipole float4 of each row is not staged)
  int2* stk = reinterpret_cast<int2*>(rows + ENT * RSF);
  float4* vb = reinterpret_cast<float4*>(stk + DPL_STACK_PER_WARP);  // [32] window dipole moments
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

  float accd = 0.f;
  float acc[2][NT ? NT : 1][4];  // NT = 0: dipole-only variant (primal_channel of the dipole)
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = acc[mt][nt][2] = acc[mt][nt][3] = 0.f;

  const bool singular = kp.mode == KM_SINGULAR;
  const float4* __restrict__ node_row = tv.node_row;
  const float4* __restrict__ pt_row = tv.pt_row;
  const int F4g = NT > 0 ? F4 : tv.F4;  // row stride in HBM (== F4, compile-time, unless NT = 0)
  int nent = 0;

  auto evaluate = [&]() {
    // zero-fill the batch tail so the K=8 steps read zeros
    for (int e = nent; e < ((nent + 7) & ~7); ++e) wr[e * WSTR + lane] = 0.f;
    cp_async_wait_all();
    __syncwarp();
    // radial channels on the tensor cores
    const int ksteps = NT > 0 ? (nent + 7) >> 3 : 0;
    for (int ks = 0; ks < ksteps; ++ks) {
      const int e0 = 8 * ks;
      uint32_t ah[2][4], al[2][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const float* wcol = wr + 16 * mt + g;
        split_tf32(wcol[(e0 + tq) * WSTR], ah[mt][0], al[mt][0]);
        split_tf32(wcol[(e0 + tq) * WSTR + 8], ah[mt][1], al[mt][1]);
        split_tf32(wcol[(e0 + tq + 4) * WSTR], ah[mt][2], al[mt][2]);
        split_tf32(wcol[(e0 + tq + 4) * WSTR + 8], ah[mt][3], al[mt][3]);
      }
      // rows of this k-step: entry e0 + tq (b0) and e0 + tq + 4 (b1), radial col 8 nt + g
      const float* r0 = rows + (e0 + tq) * RSF + 4 + g;
      const float* r1 = rows + (e0 + tq + 4) * RSF + 4 + g;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        uint32_t bh0, bl0, bh1, bl1;
        const float v0 = (e0 + tq < nent) ? r0[8 * nt] : 0.f;
        const float v1 = (e0 + tq + 4 < nent) ? r1[8 * nt] : 0.f;
        split_tf32(v0, bh0, bl0);
        split_tf32(v1, bh1, bl1);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          mma_tf32(acc[mt][nt], ah[mt], bh0, bh1);
          mma_tf32(acc[mt][nt], ah[mt], bl0, bl1);
          mma_tf32(acc[mt][nt], al[mt], bh0, bh1);
        }
      }
    }
    __syncwarp();
    nent = 0;
  };

  // v: the source's dipole moment (first float4 of its row); the dipole slot is
  // three FMAs on the FP32 pipe, in entry order (bitwise the batch loop it replaces)
  auto store_entry = [&](float4 wv, const float4* rowsrc, float4 v) {  // nent < ENT
    accd = fmaf(wv.x, v.x, fmaf(wv.y, v.y, fmaf(wv.z, v.z, accd)));
    wr[nent * WSTR + lane] = wv.w;
    if (lane >= 1 && lane < F4) cp_async16(s_rows + 4u * RSF * nent, rowsrc + lane);
    ++nent;
  };
  auto append = [&](float4 wv, const float4* rowsrc) {
    const float4 v = __ldg(rowsrc);
    if (nent == ENT) evaluate();
    store_entry(wv, rowsrc, v);
  };

  // COUNT: per-query replay counters (visited, far near/far, point near/far)
  long long c_vis = 0, c_fn = 0, c_ff = 0, c_pn = 0, c_pf = 0;
  const bool reg = kp.mode == KM_REGULARIZED;

  const int64_t wg = (int64_t)blockIdx.x * WARPS + w;
  const int total = LIST ? __ldg(lv.count + wg) : -1;
  if (LIST && total >= 0) {
    // 32 entries at a time; their node records are prefetched into the
    // (unused) stack region with cp.async, read back as broadcast LDS.128
    NodeRec* rb = reinterpret_cast<NodeRec*>(stk);
    const uint32_t s_rb = smem_u32(stk) + 48u * lane;
    const uint32_t s_vb = smem_u32(vb) + 16u * lane;
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
        if (!(my.x & IL_LEAF)) cp_async16(s_vb, node_row + (size_t)(my.x & IL_NODE) * F4g);
      }
      cp_async_wait_all();
      // the entry itself goes into its record's unused child fields (topo.x/y;
      // the replay reads only the point range z/w): one broadcast LDS.128 per
      // entry instead of two shuffles
      if (lane < n) *reinterpret_cast<uint2*>(&rb[lane].topo) = my;
      __syncwarp();
      for (int i = 0; i < n; ++i) {
        const int4 tpi = rb[i].topo;
        const uint32_t src = (uint32_t)tpi.x;
        if (nent == ENT) evaluate();  // as append() would, before deciding on a pair
        // two consecutive far entries without near lanes that fit the batch:
        // one interleaved pass; batches fill exactly as on the tree walk
        if (nent + 2 <= ENT && i + 1 < n &&
            !((src | (uint32_t)rb[i + 1].topo.x) & (IL_LEAF | IL_NEAR))) {
          const int4 tb = rb[i + 1].topo;
          const float4 ha = rb[i].hi, la = rb[i].lo, hb = rb[i + 1].hi, lb = rb[i + 1].lo;
          float ax, ay, az, bx, by, bz;
          const float sa = dist2_df(ha, la, qx, ax, ay, az);
          const float sb = dist2_df(hb, lb, qx, bx, by, bz);
          const bool fa = ((unsigned)tpi.y >> lane) & 1u, fb = ((unsigned)tb.y >> lane) & 1u;
          if (REG) {  // one select on the area per entry (see rsqrt_far)
            store_entry(fwd_w_far_m(ax, ay, az, sa, sel0(fa, la.w), kp.near2),
                        node_row + (size_t)(src & IL_NODE) * F4g, vb[i]);
            store_entry(fwd_w_far_m(bx, by, bz, sb, sel0(fb, lb.w), kp.near2),
                        node_row + (size_t)((uint32_t)tb.x & IL_NODE) * F4g, vb[i + 1]);
          } else {
            const float4 wa = fwd_w_far(ax, ay, az, sa, la.w), wb = fwd_w_far(bx, by, bz, sb, lb.w);
            store_entry(make_float4(fa ? wa.x : 0.f, fa ? wa.y : 0.f, fa ? wa.z : 0.f, fa ? wa.w : 0.f),
                        node_row + (size_t)(src & IL_NODE) * F4g, vb[i]);
            store_entry(make_float4(fb ? wb.x : 0.f, fb ? wb.y : 0.f, fb ? wb.z : 0.f, fb ? wb.w : 0.f),
                        node_row + (size_t)((uint32_t)tb.x & IL_NODE) * F4g, vb[i + 1]);
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
          } else if (REG) {  // branch-free, one select on the area
            wv = fwd_w_far_m(dx, dy, dz, s, sel0(mine, lo.w), kp.near2);
          } else {  // branch-free: every lane evaluates, non-members select 0
            const float4 f = fwd_w_far(dx, dy, dz, s, lo.w);
            wv.x = mine ? f.x : 0.f, wv.y = mine ? f.y : 0.f;
            wv.z = mine ? f.z : 0.f, wv.w = mine ? f.w : 0.f;
          }
          if (nent == ENT) evaluate();
          store_entry(wv, node_row + (size_t)node * F4g, vb[i]);
        } else {
          const int4 tp = tpi;
          for (int j = tp.z; j < tp.w; ++j) {
            float4 wv = make_float4(0.f, 0.f, 0.f, 0.f);
            if (mine) {
              const PtRec* pr = tv.pt_rec + j;
              const float4 ph = __ldg(&pr->hi);
              float dx, dy, dz;
              const float r2 = dist2_df(ph, __ldg(&pr->lo), qx, dx, dy, dz);
              if (!(singular && r2 == 0.f && coincident_exact(tv.pt_pos64 + 3 * (size_t)j, xq)))
                wv = fwd_w(dx, dy, dz, r2, ph.w, kp);
            }
            append(wv, pt_row + (size_t)j * F4g);
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
    if (COUNT && mine) ++c_vis;
    if (farm && A > 0.f) {  // area > 0 (bhtree.cpp:205)
      const float4 wv = far ? fwd_w(dx, dy, dz, s, A, kp) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (COUNT && far) (reg && s < kp.near2) ? ++c_fn : ++c_ff;
      append(wv, node_row + (size_t)node * F4g);
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
            if (!(singular && r2 == 0.f && coincident_exact(tv.pt_pos64 + 3 * (size_t)j, x))) {
              wv = fwd_w(dx, dy, dz, r2, ph.w, kp);
              if (COUNT) (reg && r2 < kp.near2) ? ++c_pn : ++c_pf;
            }
          }
          append(wv, pt_row + (size_t)j * F4g);
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
  if (COUNT && valid) {
    long long* cq = counters + 5 * qi;
    cq[0] = c_vis, cq[1] = c_fn, cq[2] = c_ff, cq[3] = c_pn, cq[4] = c_pf;
  }
  if (nent) evaluate();
  // outputs: the dipole value is lane-local; radial values live in mma C fragments
  if (only_ch >= 0) {  // primal_channel: same kernel as primal, one column stored
    if (valid && __ldg(chmap) == only_ch) out[qi] = accd;
  } else if (valid) {
    out[qi * out_stride + __ldg(chmap)] = accd;
  }
#pragma unroll
  for (int mt = 0; mt < (NT > 0 ? 2 : 0); ++mt)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int row = 16 * mt + 8 * h + g;  // lane whose query this row is
      const int64_t qr = __shfl_sync(FULL_MASK, qi, row);
      const bool vr = (active >> row) & 1u;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int col = 8 * nt + 2 * tq + u;
          if (vr && col < nr) {
            const int ch = __ldg(chmap + 1 + col);
            if (only_ch < 0)
              out[qr * out_stride + ch] = acc[mt][nt][2 * h + u];
            else if (ch == only_ch)
              out[qr] = acc[mt][nt][2 * h + u];
          }
        }
    }
}

template <int NT, int WARPS, int ENT, int MAXR, bool COUNT, bool LIST, bool REG = false>
static void launch_tc1(const Tree& t, const KParams& kp, const FwdArgs& a, int nr,
                       IListView lv = {}) {
  constexpr int F4 = 1 + 2 * NT;
  constexpr int RSF = row_stride_floats(F4);
  constexpr int WARP_FLOATS = ENT * 40 + ENT * RSF + 2 * DPL_STACK_PER_WARP + 32 * 4;
  const size_t smem = (size_t)WARPS * WARP_FLOATS * 4;
  static std::atomic<unsigned long long> attr{0};
  ensure_max_dyn_smem(k_forward_tc<NT, WARPS, ENT, MAXR, COUNT, LIST, REG>, t.device, smem, attr);
  unsigned blocks = (unsigned)((a.q + WARPS * 32 - 1) / (WARPS * 32));
  k_forward_tc<NT, WARPS, ENT, MAXR, COUNT, LIST, REG><<<blocks, WARPS * 32, smem, t.stream>>>(
      t.view(), kp, a.xs, a.perm, a.q, nr, t.chmap.as<int>(), a.out, a.out_stride, a.only_ch,
      a.counters, lv, a.overflow);
  count_launch();
}

// SPEC: also instantiate the regularized-mode kernels (production configurations)
template <int NT, int WARPS, int ENT, int MAXR, bool SPEC = false>
static void launch_tc(const Tree& t, const KParams& kp, const FwdArgs& a, int nr) {
  const bool reg = SPEC && kp.mode == KM_REGULARIZED && kp.near2 >= REG_MIN_NEAR2;
  if (a.counters) {
    launch_tc1<NT, WARPS, ENT, MAXR, true, false>(t, kp, a, nr);
  } else if (a.ilist && !no_ilist()) {
    ilist_build(t, *a.ilist, a.xs, a.perm, a.q, a.beta, ilist_near_thr(kp), a.overflow);
    if (reg)
      launch_tc1<NT, WARPS, ENT, MAXR, false, true, SPEC>(t, kp, a, nr, a.ilist->view());
    else
      launch_tc1<NT, WARPS, ENT, MAXR, false, true>(t, kp, a, nr, a.ilist->view());
  } else if (reg) {
    launch_tc1<NT, WARPS, ENT, MAXR, false, false, SPEC>(t, kp, a, nr);
  } else {
    launch_tc1<NT, WARPS, ENT, MAXR, false, false>(t, kp, a, nr);
  }
}

// Tensor-core plan: one dipole slot and PR a multiple of 8 (8..64 radial).
bool forward_tc_launch(const Tree& t, const KParams& kp, const FwdArgs& a) {
  if (a.grad_mode != 0 || (a.single && a.only_ch < 0)) return false;
  // primal_channel of the dipole channel: the dipole-only variant runs the same
  // entry sequence and the same dipole arithmetic as every values kernel
  // (forward_tc / forward2), so it is bitwise primal()[c] at a fraction of the work
  const bool two_phase_values = t.PR == 0 || t.PR == 4 || t.PR == 16 || t.PR == 48 || t.PR == 64;
  if (a.only_ch >= 0 && t.Cd == 1 && t.kinds[a.only_ch] == 0 && two_phase_values)
    return launch_tc<0, 4, 8, 128, true>(t, kp, a, 0), true;
  if (t.Cd != 1 || t.PR % 8 != 0) return false;
  const int nr = a.nr_limit >= 0 ? std::min(a.nr_limit, t.Cr) : t.Cr;
  const char* v = getenv("DPL_TUNE_TC");
  const int choice = v ? atoi(v) : 0;
  switch (t.PR) {
    case 0: return launch_tc<0, 4, 8, 128>(t, kp, a, 0), true;  // dipole only (C = 1)
    case 16: return launch_tc<2, 4, 8, 128>(t, kp, a, nr), true;
    case 48:
      switch (choice) {
        case 1: return launch_tc<6, 4, 16, 128>(t, kp, a, nr), true;
        case 2: return launch_tc<6, 4, 8, 112>(t, kp, a, nr), true;
        case 3: return launch_tc<6, 8, 8, 128>(t, kp, a, nr), true;
        default: return launch_tc<6, 4, 8, 128, true>(t, kp, a, nr), true;  // measured best
      }
    case 64: return launch_tc<8, 4, 8, 128>(t, kp, a, nr), true;
    default: return false;
  }
}

}  // namespace dpl
