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

__device__ __forceinline__ double4 ld_dec(const double4* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  double2 a = __ldg(q), b = __ldg(q + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

}  // namespace dpl
