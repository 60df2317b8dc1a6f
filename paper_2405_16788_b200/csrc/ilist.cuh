// ilist.cuh — interaction lists: the Barnes-Hut opening decisions of a query
// batch, recorded once and replayed by the evaluation kernels.
//
// K9 (k_build_list, ilist.cu) walks the tree exactly like the fused kernels —
// warp = 32 Morton-adjacent queries, one shared (node, lane-mask) stack, the
// reference's fp64 opening test (bhtree.cpp:202-204) — but does no arithmetic
// beyond the decision, so it runs with few registers at high occupancy. For
// each warp it records, in traversal order, one 8-byte entry per
//   far source   {node,          far-lane mask}   (area > 0, bhtree.cpp:205)
//   opened leaf  {node | LEAF,   open-lane mask}  (points visited, :214-229)
// The forward, gradient and adjoint kernels then stream these entries (their
// node records prefetched into shared memory 32 at a time) instead of
// re-deriving them, and one list serves a primal and the adjoint that follows
// on the same queries. A warp whose list did not fit the pool is marked
// incomplete (count -1) and the evaluation kernels traverse for it themselves,
// so the pool size affects speed only, never results.
#pragma once

#include <cstdlib>

#include "tree.cuh"

namespace dpl {

constexpr int IL_CHUNK = 128;             // entries per pool chunk (1 KB)
constexpr uint32_t IL_LEAF = 1u << 30;    // entry.x flag: opened leaf
constexpr uint32_t IL_NODE = IL_LEAF - 1;  // entry.x node-index mask
// entry.x flag on far sources: some far lane has dist^2 < near_thr (the
// lanes that need the near-field coefficient series); a far entry without
// it is evaluated with tau = 1 by every lane, no per-lane branch or vote
constexpr uint32_t IL_NEAR = 1u << 31;

// near_thr for the NEAR flag: regularized kernel (6.5 eps)^2 (kernels.cpp:50-55),
// singular never near, desingularized always (its coefficients have no far form)
inline float ilist_near_thr(const KParams& kp) {
  if (kp.mode == KM_REGULARIZED) return kp.near2;
  return kp.mode == KM_SINGULAR ? -1.0f : __builtin_huge_valf();
}

struct IListView {
  const uint2* pool = nullptr;  // [chunks][IL_CHUNK] entries {src, lane mask}
  const int* next = nullptr;    // next chunk of a chunk (warp w starts at chunk w)
  const int* count = nullptr;   // per warp: entries, or -1 when incomplete
};

struct IList {
  DevBuf pool, next, count, ctr;
  int64_t chunks = 0, nwarps = 0;
  unsigned long long* used_host = nullptr;  // pinned: chunks used by the last build
  double per_warp = 6.0;                    // chunk budget per warp (grows on use)
  // validity for reuse by a later call on the same batch
  bool valid = false;
  int64_t q = 0;
  double beta = 0;
  float near_thr = 0;
  uint64_t tree_version = 0;
  DevBuf xs_copy;  // the queries the list was built for (exact reuse check)
  DevBuf same;     // device int: 1 when this batch equals xs_copy (set per call)
  IListView view() const {
    return {pool.as<uint2>(), next.as<int>(), count.as<int>()};
  }
  ~IList();
};

// DPL_NO_ILIST set: every kernel walks the tree itself (fused kernels)
inline bool no_ilist() {
  static const bool v = getenv("DPL_NO_ILIST") != nullptr;
  return v;
}
// DPL_ILIST_ALWAYS set: every primal / adjoint builds or reuses lists,
// whatever the call pattern (tests of the replay kernels)
inline bool ilist_always() {
  static const bool v = getenv("DPL_ILIST_ALWAYS") != nullptr && !no_ilist();
  return v;
}

// Lists for q queries (device xs, Morton permutation perm) at opening
// parameter beta. When the previous lists were built for the same tree
// version, beta, q and bit-identical query positions (checked on the device,
// no host sync) the build kernels exit at once and the lists are reused:
// the decisions depend only on (tree geometry, beta, xs).
void ilist_build(const Tree& t, IList& il, const double* xs, const int32_t* perm, int64_t q,
                 double beta, float near_thr, int* overflow);

// Device-side iteration of warp wg's list: entries [base, base + 32) of the
// list live at pool[chunk * IL_CHUNK + base % IL_CHUNK + lane].
__device__ __forceinline__ uint2 il_load(const IListView& lv, int chunk, int base, int total,
                                         int lane) {
  return lane < total - base ? __ldg(lv.pool + (size_t)chunk * IL_CHUNK + (base % IL_CHUNK) + lane)
                             : make_uint2(0u, 0u);
}

}  // namespace dpl
