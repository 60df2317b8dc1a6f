// traverse.cuh — warp-cooperative Barnes-Hut traversal shared by the forward
// (K5/K6) and adjoint (K7) kernels.
//
// One warp owns 32 Morton-adjacent queries and walks the tree with ONE shared
// stack of (node, lane-mask) entries in shared memory. Every lane keeps its
// own opening decisions (SURVEY §7 hard part 2): at a popped node each lane in
// the mask evaluates the reference's fp64 test
//     d = centroid - x;  (dx*dx + dy*dy) + dz*dz  >  (beta^2 * r) * r
// (bhtree.cpp:202-204; __dmul_rn/__dadd_rn, no FMA), the far lanes accumulate
// the far field, and only the lanes that opened the node descend (children
// pushed with the opening lanes' mask; a leaf's points are visited once for
// all its opening lanes). Node and point records are warp-uniform loads
// (one broadcast transaction each). `__ballot_sync` gives the far / open
// masks, so a node every lane accepts costs one pass and no divergence.
#pragma once

#include "coeffs.cuh"
#include "dpl_internal.cuh"

namespace dpl {

#define FULL_MASK 0xffffffffu

struct QueryPos {
  double x, y, z;
};

// exact fp64 opening test; returns dist2 and d (fp64)
__device__ __forceinline__ double dist2_rn(double cx, double cy, double cz, const QueryPos& q,
                                           double& dx, double& dy, double& dz) {
  dx = __dsub_rn(cx, q.x);
  dy = __dsub_rn(cy, q.y);
  dz = __dsub_rn(cz, q.z);
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// Query in double-float form (x = hi + lo to ~2^-48) plus its fp64 original.
struct QueryDF {
  float hx, hy, hz, lx, ly, lz;
  float m;  // absolute part of the opening-test error band, 1e-13 (cmax + max|x|)^2
};

// the empty asm makes each value opaque, so the compiler keeps the 7 floats
// instead of re-deriving them from a live fp64 position inside the loops
__device__ __forceinline__ float opaque(float v) {
  asm volatile("" : "+f"(v));
  return v;
}

// cmax >= max |centroid coordinate| over the tree (TreeView::cmax)
__device__ __forceinline__ QueryDF make_qdf(const QueryPos& x, float cmax) {
  QueryDF q;
  q.hx = (float)x.x, q.hy = (float)x.y, q.hz = (float)x.z;
  q.lx = opaque((float)(x.x - (double)q.hx)), q.ly = opaque((float)(x.y - (double)q.hy)),
  q.lz = opaque((float)(x.z - (double)q.hz));
  const float M = cmax + fmaxf(fmaxf(fabsf(q.hx), fabsf(q.hy)), fabsf(q.hz));
  q.m = opaque(1e-13f * M * M);
  q.hx = opaque(q.hx), q.hy = opaque(q.hy), q.hz = opaque(q.hz);
  return q;
}

// d = source - x from double-float operands: |d - d_exact| <= 2^-23 |d| + 2^-46 (|c| + |x|).
__device__ __forceinline__ float dist2_df(const float4& hi, const float4& lo, const QueryDF& q,
                                          float& dx, float& dy, float& dz) {
  dx = (hi.x - q.hx) + (lo.x - q.lx);
  dy = (hi.y - q.hy) + (lo.y - q.ly);
  dz = (hi.z - q.hz) + (lo.z - q.lz);
  return fmaf(dz, dz, fmaf(dy, dy, dx * dx));
}

// The reference's opening test dist2 > (beta^2 r) r (bhtree.cpp:204), decided
// in fp32 when the margin exceeds a rigorous error bound (dist2 error
// <= 2^-21 s + 2^-46 M^2 with M = |c| + |x| <= cmax + max|x|, threshold
// rounding 2^-24 thr; the band below is 2x that, its absolute part precomputed
// per query in QueryDF::m), else re-evaluated exactly in fp64 with the
// reference's operation order. NaN / inf thresholds (beta = inf) always take
// the exact path.
__device__ __forceinline__ bool far_test(float s, const float4& hi, const QueryDF& q,
                                         const QueryPos& x, const double4* __restrict__ dec) {
  const float thr = hi.w;
  const float band = 2e-6f * (s + thr) + q.m;
  const float diff = s - thr;
  if (diff > band) return true;
  if (-diff > band) return false;
  const double2 a = __ldg(reinterpret_cast<const double2*>(dec));
  const double2 b = __ldg(reinterpret_cast<const double2*>(dec) + 1);
  double ex, ey, ez;
  return dist2_rn(a.x, a.y, b.x, x, ex, ey, ez) > b.y;
}

// Same test with the fp64 query re-read from memory on the (rare) exact path:
// keeps the 6 registers of the fp64 position out of the traversal loop.
__device__ __forceinline__ bool far_test(float s, const float4& hi, const QueryDF& q,
                                         const double* __restrict__ xq,
                                         const double4* __restrict__ dec) {
  const float thr = hi.w;
  const float band = 2e-6f * (s + thr) + q.m;
  const float diff = s - thr;
  if (diff > band) return true;
  if (-diff > band) return false;
  const double2 a = __ldg(reinterpret_cast<const double2*>(dec));
  const double2 b = __ldg(reinterpret_cast<const double2*>(dec) + 1);
  const QueryPos x{xq[0], xq[1], xq[2]};
  double ex, ey, ez;
  return dist2_rn(a.x, a.y, b.x, x, ex, ey, ez) > b.y;
}

// exact fp64 opening test out of line: the call is one (predicated) instruction
// on the common path, where an inlined body would be if-converted into ~17
// predicated-off instructions issued on every pop
static __device__ __noinline__ bool far_exact(const double* __restrict__ xq,
                                              const double4* __restrict__ dec) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(dec));
  const double2 b = __ldg(reinterpret_cast<const double2*>(dec) + 1);
  const QueryPos x{xq[0], xq[1], xq[2]};
  double ex, ey, ez;
  return dist2_rn(a.x, a.y, b.x, x, ex, ey, ez) > b.y;
}

// The same decision with the lane mask folded in: every lane forms the fp32
// verdict without a branch (|diff| > band decides by the sign of diff, as the
// two one-sided tests above), and only member lanes inside the band (or with a
// NaN / inf threshold) take the exact fp64 path. Bitwise the same decisions as
// `mine && far_test(...)`, fewer instructions on the common path.
__device__ __forceinline__ bool far_test_masked(float s, const float4& hi, const QueryDF& q,
                                                const double* __restrict__ xq,
                                                const double4* __restrict__ dec, bool mine) {
  const float thr = hi.w;
  const float band = 2e-6f * (s + thr) + q.m;
  const float diff = s - thr;
  bool far = mine && diff > 0.f;
  if (mine && !(fabsf(diff) > band)) far = far_exact(xq, dec);
  return far;
}

// exact fp64 coincidence check for a leaf point (bhtree.cpp:219,316,387)
__device__ __forceinline__ bool coincident_exact(const double* __restrict__ p,
                                                 const double* __restrict__ xq) {
  const QueryPos x{xq[0], xq[1], xq[2]};
  double ex, ey, ez;
  return dist2_rn(__ldg(p), __ldg(p + 1), __ldg(p + 2), x, ex, ey, ez) == 0.0;
}

// exact fp64 coincidence check for a leaf point (bhtree.cpp:219,316,387)
__device__ __forceinline__ bool coincident_exact(const double* __restrict__ p, const QueryPos& x) {
  double ex, ey, ez;
  return dist2_rn(__ldg(p), __ldg(p + 1), __ldg(p + 2), x, ex, ey, ez) == 0.0;
}

__device__ __forceinline__ double4 ld_dec(const double4* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  double2 a = __ldg(q), b = __ldg(q + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

}  // namespace dpl
