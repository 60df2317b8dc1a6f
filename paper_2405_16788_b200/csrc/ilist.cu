// ilist.cu — K9: record the Barnes-Hut opening decisions of a query batch
// (see ilist.cuh). Same traversal and decisions as DipoleTree::primal /
// adjoint (proj/src/bhtree.cpp:188-234, 345-417): pop order, the fp64 test
// (:202-204), far sources with area > 0 (:205), far test before the leaf test.
#include <algorithm>
#include <cstdlib>

#include "ilist.cuh"
#include "traverse.cuh"

namespace dpl {

IList::~IList() {
  if (used_host) cudaFreeHost(used_host);
}

namespace {
__global__ void k_set_u64(unsigned long long* p, unsigned long long v, const int* skip) {
  if (skip && *skip) return;
  *p = v;
}
__global__ void k_set_int(int* p, int v) { *p = v; }
// chunk usage to mapped pinned memory: a kernel store, not a D2H copy that
// would wait behind a host-async download on the copy engine
__global__ void k_publish_u64(volatile unsigned long long* host, const unsigned long long* v) {
  *host = *v;
}
// SM copy (not cudaMemcpy: a D2D copy-engine transfer would queue behind a
// host-async D2H in flight on the same engine); skipped when the batch is unchanged
__global__ void k_copy_u64(unsigned long long* __restrict__ dst,
                           const unsigned long long* __restrict__ src, int64_t n,
                           const int* skip) {
  if (skip && *skip) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __ldg(src + i);
}
// same = 0 if any coordinate differs bitwise (NaN payloads included)
__global__ void k_compare(const unsigned long long* __restrict__ a,
                          const unsigned long long* __restrict__ b, int64_t n, int* same) {
  bool diff = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    diff |= __ldg(a + i) != __ldg(b + i);
  if (__syncthreads_or(diff) && threadIdx.x == 0) *same = 0;
}
}  // namespace

// WARPS warps per block, MINB blocks per SM: few registers, high occupancy
// (the walk is latency-bound on the node-record loads).
template <int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB)
    k_build_list(TreeView tv, const double* __restrict__ xs, const int32_t* __restrict__ perm,
                 int64_t q, uint2* __restrict__ pool, int* __restrict__ next,
                 int* __restrict__ count, unsigned long long* ctr, int64_t chunks,
                 float near_thr, const int* skip, int* overflow) {
  if (skip && *skip) return;  // lists of this exact batch are already in place
  __shared__ int2 stk_all[WARPS][DPL_STACK_PER_WARP];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int2* stk = stk_all[w];
  const int64_t wg = (int64_t)blockIdx.x * WARPS + w;
  const int64_t sidx = wg * 32 + lane;
  const bool valid = sidx < q;
  const int64_t qi = valid ? (perm ? (int64_t)perm[sidx] : sidx) : 0;
  QueryPos x;
  if (valid) {
    x.x = xs[3 * qi], x.y = xs[3 * qi + 1], x.z = xs[3 * qi + 2];
  } else {
    x.x = x.y = x.z = 0.0;
  }
  const unsigned active = __ballot_sync(FULL_MASK, valid);
  if (!active) return;  // evaluation kernels return for such warps too
  const QueryDF qx = make_qdf(x, tv.cmax);
  const double* xq = xs + 3 * qi;
  const unsigned lanebit = 1u << lane;

  int cur = (int)wg;  // chunk being filled (warp w owns chunk w)
  int total = 0;      // entries written to the pool
  // entries are collected in registers — lane k holds entry k of the current
  // block of 32 — and written as one coalesced 256-byte store per block (a
  // chunk holds 4 blocks, so a block never straddles two chunks). Returns false
  // when the pool is exhausted: the warp then leaves its list incomplete (count
  // -1) and the evaluation kernels walk the tree for it.
  uint2 pend = make_uint2(0u, 0u);
  int npend = 0;
  auto flush = [&]() -> bool {
    const int b = total >> 5;  // block index: total is a multiple of 32 here
    if (b > 0 && (b & 3) == 0) {  // chunk full: link a fresh one
      unsigned long long c = 0;
      if (lane == 0) c = atomicAdd(ctr, 1ull);
      c = __shfl_sync(FULL_MASK, c, 0);
      if (c >= (unsigned long long)chunks) return false;
      if (lane == 0) next[cur] = (int)c;
      cur = (int)c;
    }
    if (lane < npend) pool[(size_t)cur * IL_CHUNK + (b & 3) * 32 + lane] = pend;
    total += npend;
    npend = 0;
    return true;
  };

  int sp = 1;
  if (lane == 0) stk[0] = make_int2(0, (int)active);
  __syncwarp();
  // the exhaustion exits are gotos, so the loop carries no status flag
  while (sp > 0) {
    --sp;
    // no __syncwarp after the pop: every lane has consumed e (the record
    // address) before the ballot below, the warp's next convergence point,
    // and pushes happen only after it
    const int2 e = stk[sp];
    const int node = e.x;
    const unsigned mask = (unsigned)e.y;
    const bool mine = (mask & lanebit) != 0u;
    const NodeRec* rec = tv.node_rec + node;
    const float4 hi = __ldg(&rec->hi);
    const float4 lo = __ldg(&rec->lo);
    const int4 tp = __ldg(&rec->topo);
    float dx, dy, dz;
    const float s = dist2_df(hi, lo, qx, dx, dy, dz);
    const bool far = far_test_masked(s, hi, qx, xq, tv.node_dec + node, mine);
    const unsigned farm = __ballot_sync(FULL_MASK, far);
    if (farm && lo.w > 0.f) {
      const bool nr = __any_sync(FULL_MASK, far && s < near_thr);
      if (lane == npend) pend = make_uint2((uint32_t)node | (nr ? IL_NEAR : 0u), farm);
      if (++npend == 32 && !flush()) goto exhausted;
    }
    const unsigned openm = mask & ~farm;
    if (openm) {
      if (tp.y == 0) {
        if (lane == npend) pend = make_uint2((uint32_t)node | IL_LEAF, openm);
        if (++npend == 32 && !flush()) goto exhausted;
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
  if (npend && !flush()) goto exhausted;
  if (lane == 0) count[wg] = total;
  return;
exhausted:
  if (lane == 0) count[wg] = -1;
}

void ilist_build(const Tree& t, IList& il, const double* xs, const int32_t* perm, int64_t q,
                 double beta, float near_thr, int* overflow) {
  constexpr int WARPS = 4, MINB = 12;
  const int64_t nwarps = (q + 31) / 32;
  static const char* pool_env = getenv("DPL_ILIST_POOL");  // chunks per warp (tests: 1 forces
  if (pool_env && il.nwarps == 0) il.per_warp = atof(pool_env);  // incomplete lists)
  // pool budget: warps' own chunks + overflow chunks, sized from the last use
  if (il.used_host && il.nwarps > 0 && *il.used_host > 0) {
    const double used = (double)*il.used_host / (double)il.nwarps;
    if (used > 0.8 * il.per_warp && !pool_env) il.per_warp = std::min(64.0, used * 1.5);
  }
  if (!il.used_host) {
    DPL_CUDA(cudaHostAlloc(&il.used_host, sizeof(unsigned long long), cudaHostAllocMapped));
    *il.used_host = 0;
  }
  il.same.reserve(sizeof(int));
  const int* skip = nullptr;
  if (il.valid && il.q == q && il.beta == beta && il.near_thr == near_thr &&
      il.tree_version == t.version) {
    k_set_int<<<1, 1, 0, t.stream>>>(il.same.as<int>(), 1);
    k_compare<<<4 * 148, 256, 0, t.stream>>>(reinterpret_cast<const unsigned long long*>(xs),
                                              il.xs_copy.as<unsigned long long>(), 3 * q,
                                              il.same.as<int>());
    count_launch(2);
    skip = il.same.as<int>();
  } else {
    // pool sizing happens only on a real rebuild (a reused pool must stay put)
    il.valid = false;
  }
  const int64_t chunks = skip ? il.chunks
                              : std::max<int64_t>(nwarps + 1, (int64_t)(il.per_warp * (double)nwarps));
  il.pool.reserve((size_t)chunks * IL_CHUNK * sizeof(uint2));
  il.next.reserve((size_t)chunks * sizeof(int));
  il.count.reserve((size_t)std::max<int64_t>(1, nwarps) * sizeof(int));
  il.ctr.reserve(sizeof(unsigned long long));
  il.chunks = chunks;
  il.nwarps = nwarps;
  k_set_u64<<<1, 1, 0, t.stream>>>(il.ctr.as<unsigned long long>(), (unsigned long long)nwarps,
                                   skip);
  count_launch();
  const unsigned blocks = (unsigned)((nwarps + WARPS - 1) / WARPS);
  k_build_list<WARPS, MINB><<<blocks, WARPS * 32, 0, t.stream>>>(
      t.view(), xs, perm, q, il.pool.as<uint2>(), il.next.as<int>(), il.count.as<int>(),
      il.ctr.as<unsigned long long>(), chunks, near_thr, skip, overflow);
  count_launch();
  // chunks actually used, read back without a sync (sizes the next build)
  unsigned long long* used_dev = nullptr;
  DPL_CUDA(cudaHostGetDevicePointer((void**)&used_dev, il.used_host, 0));
  k_publish_u64<<<1, 1, 0, t.stream>>>(used_dev, il.ctr.as<unsigned long long>());
  count_launch();
  // remember the batch the lists now describe (whether rebuilt or reused; the
  // host cannot tell without a sync, and the copy is ~0.03 ms per 4M queries)
  il.xs_copy.reserve((size_t)q * 24);
  k_copy_u64<<<8 * 148, 256, 0, t.stream>>>(il.xs_copy.as<unsigned long long>(),
                                             reinterpret_cast<const unsigned long long*>(xs),
                                             3 * q, skip);
  count_launch();
  il.valid = true;
  il.q = q;
  il.beta = beta;
  il.near_thr = near_thr;
  il.tree_version = t.version;
}

}  // namespace dpl
