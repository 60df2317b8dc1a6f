// tree.cu — GPU octree build (K1-K4) reproducing DipoleTree::build bit-exactly.
//
// Reference: proj/src/bhtree.cpp:20-176. The reference builds breadth-first
// with a FIFO queue and stable 8-way bucket partitions (:36-105). Because the
// FIFO processes whole levels in order and appends children in octant order
// (skipping empty octants), the BFS id of a node equals its level offset plus
// the rank of its point range within that level, and within a level nodes
// are ordered by range start. We therefore:
//   K1  compute, per point, the octant digit at every depth with the same fp64
//       centre recursion (c <- c + (0.5 h)(+-1), h <- 0.5 h; :77-78, :93-95) and
//       pack them into a 3*max_depth-bit key;
//   K2  stable radix-sort (key, index), then walk the levels: a node at depth d
//       is a maximal run of points sharing the top-d digits whose parent was
//       internal; it is internal iff size > max_leaf and d < max_depth (:69);
//       a second stable sort restores original index order inside every leaf
//       (the reference's stable partitions keep it), giving point_order;
//   K3  geometry per node, sequentially over its range in point_order with the
//       reference's fp64 operation order and no FMA (:107-134) -> bit-exact;
//   K4  moments bottom-up in fp64 (level by level, children summed), then
//       normalised by area and stored fp32 for the traversals (:136-156).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <string>

#include "tree.cuh"

namespace dpl {

// ---- guard mode (DPL_GUARD=1): every engine allocation gets 4 KB guard zones
// before and after it, filled with a byte pattern; dpl_guard_check() (and the
// release of a buffer) verifies them. compute-sanitizer is not available on the
// GPU pool, so this is the engine's own out-of-bounds-write detector.
namespace {
constexpr size_t kGuard = 4096;
constexpr unsigned char kGuardByte = 0xA5;
bool guard_mode() {
  static const bool on = getenv("DPL_GUARD") != nullptr;
  return on;
}
std::mutex& guard_mu() {
  static std::mutex m;
  return m;
}
std::set<DevBuf*>& guard_live() {
  static std::set<DevBuf*> s;
  return s;
}
std::string& guard_report() {
  static std::string r;
  return r;
}
bool guard_intact(const DevBuf& b) {
  std::vector<unsigned char> h(2 * kGuard);
  const char* base = static_cast<const char*>(b.p) - kGuard;
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(h.data(), base, kGuard, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess)
    e = cudaMemcpy(h.data() + kGuard, static_cast<const char*>(b.p) + b.bytes, kGuard,
                   cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    cudaGetLastError();  // reported here, not left pending for the next engine call
    guard_report() += std::string("guard zones of a ") + std::to_string(b.bytes) +
                      "-byte buffer unreadable (" + cudaGetErrorString(e) + "); ";
    return true;
  }
  for (unsigned char c : h)
    if (c != kGuardByte) return false;
  return true;
}
}  // namespace

void DevBuf::reserve(size_t b) {
  if (b <= bytes && p) return;
  release();
  size_t a = b ? b : 16;
  a = (a + 255) & ~(size_t)255;
  const bool g = guard_mode();
  if (g) {
    cudaError_t pe = cudaPeekAtLastError();
    if (pe != cudaSuccess)
      throw Error(4, std::string("guard mode: CUDA error pending before an allocation: ") +
                         cudaGetErrorString(pe));
  }
  void* raw = nullptr;
  cudaError_t e = cudaMalloc(&raw, a + (g ? 2 * kGuard : 0));
  if (e != cudaSuccess) {
    p = nullptr;
    bytes = 0;
    throw Error(4, std::string("cudaMalloc(") + std::to_string(a) + "): " + cudaGetErrorString(e));
  }
  if (g) {
    DPL_CUDA(cudaMemset(raw, kGuardByte, kGuard));
    DPL_CUDA(cudaMemset(static_cast<char*>(raw) + kGuard + a, kGuardByte, kGuard));
    DPL_CUDA(cudaDeviceSynchronize());
    p = static_cast<char*>(raw) + kGuard;
    guarded = true;
    std::lock_guard<std::mutex> lk(guard_mu());
    guard_live().insert(this);
  } else {
    p = raw;
  }
  bytes = a;
}

void DevBuf::release() {
  if (p) {
    if (guarded) {
      std::lock_guard<std::mutex> lk(guard_mu());
      guard_live().erase(this);
      if (!guard_intact(*this))
        guard_report() += "guard zone of a released " + std::to_string(bytes) + "-byte buffer overwritten; ";
      cudaFree(static_cast<char*>(p) - kGuard);
    } else {
      cudaFree(p);
    }
  }
  p = nullptr;
  bytes = 0;
  guarded = false;
}

void DevBuf::swap(DevBuf& o) {
  if (guarded || o.guarded) {
    std::lock_guard<std::mutex> lk(guard_mu());
    guard_live().erase(this);
    guard_live().erase(&o);
    std::swap(p, o.p);
    std::swap(bytes, o.bytes);
    std::swap(guarded, o.guarded);
    if (guarded) guard_live().insert(this);
    if (o.guarded) guard_live().insert(&o);
    return;
  }
  std::swap(p, o.p);
  std::swap(bytes, o.bytes);
}

// number of live guarded buffers whose guard zones were overwritten (plus
// earlier findings at release time); msg receives a description
int guard_check_all(std::string& msg) {
  std::lock_guard<std::mutex> lk(guard_mu());
  int bad = 0;
  for (DevBuf* b : guard_live())
    if (!guard_intact(*b)) {
      ++bad;
      msg += "guard zone of a live " + std::to_string(b->bytes) + "-byte buffer overwritten; ";
    }
  if (!guard_report().empty()) {
    ++bad;
    msg += guard_report();
    guard_report().clear();
  }
  return bad;
}

int guard_live_count() {
  std::lock_guard<std::mutex> lk(guard_mu());
  return (int)guard_live().size();
}

cudaEvent_t Tree::take_event() {
  if (!ev_pool.empty()) {
    cudaEvent_t e = ev_pool.back();
    ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  DPL_CUDA(cudaEventCreate(&e));
  return e;
}

PhaseTimer::PhaseTimer(Tree& tr, int ph) : t(tr), phase(ph) {
  if (!t.prof) return;
  a = t.take_event();
  cudaEventRecord(a, t.stream);
}

PhaseTimer::~PhaseTimer() {
  if (!a) return;
  cudaEvent_t b = t.take_event();
  cudaEventRecord(b, t.stream);
  t.recs.push_back({phase, a, b});
}

static constexpr double kInvFourPi = 0.07957747154594766788444188168625718101;

static inline unsigned grid_for(int64_t n, int block) {
  return (unsigned)std::max<int64_t>(1, (n + block - 1) / block);
}

KParams make_kparams(double eps, int desing, double delta) {
  KParams k{};
  if (desing) {
    k.mode = KM_DESING;
    k.delta2 = (float)(delta * delta);
  } else if (eps <= 0.0) {
    k.mode = KM_SINGULAR;
  } else {
    k.mode = KM_REGULARIZED;
    k.eps = (float)eps;
    k.inv_eps = (float)(1.0 / eps);
    k.inv_eps3 = (float)(1.0 / (eps * eps * eps));
    k.inv_eps4 = (float)(1.0 / (eps * eps * eps * eps));
    k.inv_eps5 = (float)(1.0 / (eps * eps * eps * eps * eps));
    k.inv_eps6 = (float)(1.0 / (eps * eps * eps * eps * eps * eps));
    k.near2 = (float)((6.5 * eps) * (6.5 * eps));
  }
  return k;
}

TreeView Tree::view() const {
  TreeView v;
  v.node_dec = node_dec.as<double4>();
  v.node_topo = node_topo.as<int4>();
  v.node_geo = node_geo.as<float4>();
  v.node_flag = node_flag.as<uint8_t>();
  v.node_rec = node_rec.as<NodeRec>();
  v.node_row = node_row.as<float4>();
  v.pt_pos64 = pt_pos64.as<double>();
  v.pt_geo = pt_geo.as<float4>();
  v.pt_row = pt_row.as<float4>();
  v.pt_rec = pt_rec.as<PtRec>();
  v.node_row_split = node_row_split.as<float4>();
  v.pt_row_split = pt_row_split.as<float4>();
  v.pt_nrm = pt_nrm.as<float>();
  v.pt_mu = pt_mud.as<float>();
  v.P = PR;
  v.F4 = F4;
  v.Cd = Cd;
  v.Cr = Cr;
  v.C = C;
  v.nodes = nodes;
  v.n = n;
  v.max_depth = max_depth;
  double cm = 0.0;  // centroids lie in the root bounding box
  for (int a = 0; a < 3; ++a) cm = std::max(cm, std::max(std::fabs(root_lo[a]), std::fabs(root_hi[a])));
  v.cmax = (float)(cm * 1.001) + 1e-30f;
  return v;
}

void Tree::set_layout() {
  dip_ch.clear();
  rad_ch.clear();
  slot_of.assign(C, 0);
  for (int c = 0; c < C; ++c) {
    if (kinds[c] == 0) {
      slot_of[c] = (int)dip_ch.size();
      dip_ch.push_back(c);
    } else {
      slot_of[c] = (int)rad_ch.size();
      rad_ch.push_back(c);
    }
  }
  Cd = (int)dip_ch.size();
  Cr = (int)rad_ch.size();
  PR = round_up4(std::max(Cr, 1));
  F4 = Cd + PR / 4;
  std::vector<int> m(dip_ch);
  m.insert(m.end(), rad_ch.begin(), rad_ch.end());
  chmap.reserve(sizeof(int) * std::max(1, C));
  DPL_CUDA(cudaMemcpyAsync(chmap.p, m.data(), sizeof(int) * C, cudaMemcpyHostToDevice, stream));
}

// ---------------------------------------------------------------- kernels

__global__ void k_bbox_partial(const double* __restrict__ pos, int64_t n, double* part) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int a = 0; a < 3; ++a) {
      double v = pos[3 * i + a];
      lo[a] = fmin(lo[a], v);
      hi[a] = fmax(hi[a], v);
    }
  __shared__ double s[6][256];
  for (int a = 0; a < 3; ++a) s[a][threadIdx.x] = lo[a], s[3 + a][threadIdx.x] = hi[a];
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w)
      for (int a = 0; a < 3; ++a) {
        s[a][threadIdx.x] = fmin(s[a][threadIdx.x], s[a][threadIdx.x + w]);
        s[3 + a][threadIdx.x] = fmax(s[3 + a][threadIdx.x], s[3 + a][threadIdx.x + w]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int a = 0; a < 6; ++a) part[6 * blockIdx.x + a] = s[a][0];
}

// K1: octant digits along the point's own descent (bhtree.cpp:77-78, 93-95).
// Up to 21 digits fit one 64-bit key; deeper trees (max_depth <= 42) put the
// digits of levels 22.. into a second key word (keys_lo, else nullptr).
__global__ void k_keys(const double* __restrict__ pos, int64_t n, double cx, double cy, double cz,
                       double half, int depth, uint64_t* keys, uint64_t* keys_lo, int32_t* idx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double px = pos[3 * i], py = pos[3 * i + 1], pz = pos[3 * i + 2];
  double c0 = cx, c1 = cy, c2 = cz, h = half;
  uint64_t key = 0, key_lo = 0;
  for (int d = 0; d < depth; ++d) {
    int o = (px >= c0 ? 1 : 0) | (py >= c1 ? 2 : 0) | (pz >= c2 ? 4 : 0);
    if (d < 21)
      key = (key << 3) | (uint64_t)o;
    else
      key_lo = (key_lo << 3) | (uint64_t)o;
    double hh = __dmul_rn(0.5, h);
    c0 = __dadd_rn(c0, (o & 1) ? hh : -hh);
    c1 = __dadd_rn(c1, (o & 2) ? hh : -hh);
    c2 = __dadd_rn(c2, (o & 4) ? hh : -hh);
    h = __dmul_rn(0.5, h);
  }
  keys[i] = key;
  if (keys_lo) keys_lo[i] = key_lo;
  idx[i] = (int32_t)i;
}

__global__ void k_iota(int32_t* p, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) p[i] = (int32_t)i;
}
__global__ void k_gather_u64(const uint64_t* __restrict__ src, const int32_t* __restrict__ at,
                             int64_t n, uint64_t* dst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[at[i]];
}
__global__ void k_gather_i32(const int32_t* __restrict__ src, const int32_t* __restrict__ at,
                             int64_t n, int32_t* dst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[at[i]];
}

// per sorted point: active at level d iff its level-(d-1) node is internal;
// marks heads of level-d runs and records leaves reached at level d-1.
__global__ void k_level_heads(const uint64_t* __restrict__ keys, const int32_t* __restrict__ cur,
                              const uint8_t* __restrict__ internal, int64_t n, int shift,
                              int32_t* head, int32_t* pt_leaf) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  int32_t c = cur[j];
  bool act = c >= 0 && internal[c];
  if (c >= 0 && !internal[c]) pt_leaf[j] = c;
  int h = 0;
  if (act) {
    if (j == 0) {
      h = 1;
    } else {
      int32_t cp = cur[j - 1];
      bool actp = cp >= 0 && internal[cp];
      h = (!actp || cp != c || (keys[j] >> shift) != (keys[j - 1] >> shift)) ? 1 : 0;
    }
  }
  head[j] = h;
}

__global__ void k_level_assign(const uint64_t* __restrict__ keys, const int32_t* __restrict__ cur,
                               const uint8_t* __restrict__ internal,
                               const int32_t* __restrict__ incl, const int32_t* __restrict__ head,
                               int64_t n, int shift, int64_t off, int32_t* next, int32_t* nbeg,
                               int32_t* nend, int32_t* nparent, int32_t* cbeg, int32_t* ccnt,
                               const int32_t* __restrict__ pbeg) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  int32_t c = cur[j];
  bool act = c >= 0 && internal[c];
  if (!act) {
    next[j] = -1;
    return;
  }
  int32_t id = (int32_t)(off + incl[j] - 1);
  next[j] = id;
  if (head[j]) {
    nbeg[id] = (int32_t)j;
    nparent[id] = c;
    if (pbeg[c] == (int32_t)j) cbeg[c] = id;
    atomicAdd(&ccnt[c], 1);
  }
  bool tail = (j + 1 == n);
  if (!tail) {
    int32_t cn = cur[j + 1];
    bool actn = cn >= 0 && internal[cn];
    tail = !actn || cn != c || (keys[j + 1] >> shift) != (keys[j] >> shift);
  }
  if (tail) nend[id] = (int32_t)(j + 1);
}

__global__ void k_level_internal(const int32_t* __restrict__ beg, const int32_t* __restrict__ end,
                                 int64_t off, int64_t cnt, int max_leaf, bool at_max_depth,
                                 uint8_t* internal, int32_t* nint) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= cnt) return;
  int64_t id = off + i;
  bool in = (end[id] - beg[id] > max_leaf) && !at_max_depth;
  internal[id] = in ? 1 : 0;
  if (in) atomicAdd(nint, 1);
}

__global__ void k_leaf_order_keys(const int32_t* __restrict__ pt_leaf,
                                  const int32_t* __restrict__ beg, const int32_t* __restrict__ idx,
                                  int64_t n, uint64_t* key2) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  key2[j] = ((uint64_t)(uint32_t)beg[pt_leaf[j]] << 32) | (uint64_t)(uint32_t)idx[j];
}

__global__ void k_finish_points(const uint64_t* __restrict__ key2, int64_t n, int32_t* order,
                                const int32_t* __restrict__ pt_leaf, int32_t* leaf_of) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  int32_t m = (int32_t)(key2[j] & 0xffffffffu);
  order[j] = m;
  leaf_of[m] = pt_leaf[j];
}

// sorted fp64 / fp32 point copies
__global__ void k_gather_points(const int32_t* __restrict__ order, const double* __restrict__ pos,
                                const double* __restrict__ area, int64_t n, double* pt_pos64,
                                float4* pt_geo, PtRec* pt_rec) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  int64_t m = order[j];
  double x = pos[3 * m], y = pos[3 * m + 1], z = pos[3 * m + 2];
  pt_pos64[3 * j] = x, pt_pos64[3 * j + 1] = y, pt_pos64[3 * j + 2] = z;
  float A = (float)(area[m] * kInvFourPi);
  float hx = (float)x, hy = (float)y, hz = (float)z;
  pt_geo[j] = make_float4(hx, hy, hz, A);
  PtRec r;
  r.hi = make_float4(hx, hy, hz, A);
  r.lo = make_float4((float)(x - (double)hx), (float)(y - (double)hy), (float)(z - (double)hz), 0.f);
  pt_rec[j] = r;
}

// K3: geometry, sequential in point_order (bit-exact). Nodes of up to
// GEO_BIG points: one thread per node. Larger nodes: k_geometry_warp.
constexpr int GEO_BIG = 64;

__global__ void k_geometry(const int32_t* __restrict__ beg, const int32_t* __restrict__ end,
                           int64_t nodes, const double* __restrict__ pt_pos64,
                           const int32_t* __restrict__ order, const double* __restrict__ area,
                           double* ctr, double* narea, double* nrad, uint8_t* flag,
                           float4* geo) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nodes) return;
  int32_t b = beg[i], e = end[i];
  if (e - b > GEO_BIG) return;
  double cx, cy, cz, asum, rad;
  if (e - b == 1) {  // bitwise copies for single-point nodes (:109-116)
    asum = area[order[b]];
    cx = pt_pos64[3 * b], cy = pt_pos64[3 * b + 1], cz = pt_pos64[3 * b + 2];
    rad = 0.0;
  } else {
    asum = 0;
    double px = 0, py = 0, pz = 0, mx = 0, my = 0, mz = 0;
    for (int32_t j = b; j < e; ++j) {
      double a = area[order[j]];
      double x = pt_pos64[3 * j], y = pt_pos64[3 * j + 1], z = pt_pos64[3 * j + 2];
      asum = __dadd_rn(asum, a);
      px = __dadd_rn(px, __dmul_rn(a, x));
      py = __dadd_rn(py, __dmul_rn(a, y));
      pz = __dadd_rn(pz, __dmul_rn(a, z));
      mx = __dadd_rn(mx, x);
      my = __dadd_rn(my, y);
      mz = __dadd_rn(mz, z);
    }
    if (asum > 0) {
      cx = __ddiv_rn(px, asum), cy = __ddiv_rn(py, asum), cz = __ddiv_rn(pz, asum);
    } else {
      double cnt = (double)(e - b);
      cx = __ddiv_rn(mx, cnt), cy = __ddiv_rn(my, cnt), cz = __ddiv_rn(mz, cnt);
    }
    double r2max = 0;
    for (int32_t j = b; j < e; ++j) {
      double dx = __dsub_rn(pt_pos64[3 * j], cx);
      double dy = __dsub_rn(pt_pos64[3 * j + 1], cy);
      double dz = __dsub_rn(pt_pos64[3 * j + 2], cz);
      double s = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      r2max = r2max < s ? s : r2max;
    }
    rad = __dsqrt_rn(r2max);
  }
  ctr[3 * i] = cx, ctr[3 * i + 1] = cy, ctr[3 * i + 2] = cz;
  narea[i] = asum;
  nrad[i] = rad;
  flag[i] = asum > 0 ? 1 : 0;
  geo[i] = make_float4((float)cx, (float)cy, (float)cz, (float)(asum * kInvFourPi));
}

// Large nodes, one warp each. The sums stay sequential in point_order (the
// reference's rounding, bhtree.cpp:117-124): the warp stages 32 points in
// shared memory with coalesced loads and lane 0 runs the fp64 chains, so the
// load latency is off the dependency chain. The radius is a max (order-free:
// the same `r < s ? s : r` comparator in a lane-parallel reduction).
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_geometry_warp(const int32_t* __restrict__ beg, const int32_t* __restrict__ end,
                    int64_t nodes, const double* __restrict__ pt_pos64,
                    const int32_t* __restrict__ order, const double* __restrict__ area,
                    double* ctr, double* narea, double* nrad, uint8_t* flag, float4* geo) {
  // batches of 128 points (4 per lane): while lane 0 runs the chains of one
  // batch (~10 cycles per point, bound by the fp64 add latency), the loads of
  // the next batch — including the area gather through point_order — are in
  // flight in every lane's registers
  constexpr int PER = 4;
  __shared__ double4 stage[WARPS][32 * PER];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * WARPS + w;
  if (i >= nodes) return;
  const int32_t b = beg[i], e = end[i];
  if (e - b <= GEO_BIG) return;
  double asum = 0, px = 0, py = 0, pz = 0, mx = 0, my = 0, mz = 0;
  auto fetch = [&](int32_t base, double4 (&v)[PER]) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int32_t j = base + 32 * u + lane;
      if (j < e)
        v[u] = make_double4(area[order[j]], pt_pos64[3 * (size_t)j], pt_pos64[3 * (size_t)j + 1],
                            pt_pos64[3 * (size_t)j + 2]);
    }
  };
  double4 nxt[PER];
  fetch(b, nxt);
  for (int32_t base = b; base < e; base += 32 * PER) {
#pragma unroll
    for (int u = 0; u < PER; ++u) stage[w][32 * u + lane] = nxt[u];
    __syncwarp();
    if (base + 32 * PER < e) fetch(base + 32 * PER, nxt);
    if (lane == 0) {
      const int n = min(32 * PER, e - base);
      for (int k = 0; k < n; ++k) {
        const double4 v = stage[w][k];
        asum = __dadd_rn(asum, v.x);
        px = __dadd_rn(px, __dmul_rn(v.x, v.y));
        py = __dadd_rn(py, __dmul_rn(v.x, v.z));
        pz = __dadd_rn(pz, __dmul_rn(v.x, v.w));
        mx = __dadd_rn(mx, v.y);
        my = __dadd_rn(my, v.z);
        mz = __dadd_rn(mz, v.w);
      }
    }
    __syncwarp();
  }
  double cx = 0, cy = 0, cz = 0;
  if (lane == 0) {
    if (asum > 0) {
      cx = __ddiv_rn(px, asum), cy = __ddiv_rn(py, asum), cz = __ddiv_rn(pz, asum);
    } else {
      const double cnt = (double)(e - b);
      cx = __ddiv_rn(mx, cnt), cy = __ddiv_rn(my, cnt), cz = __ddiv_rn(mz, cnt);
    }
  }
  cx = __shfl_sync(0xffffffffu, cx, 0);
  cy = __shfl_sync(0xffffffffu, cy, 0);
  cz = __shfl_sync(0xffffffffu, cz, 0);
  double r2max = 0;
  for (int32_t j = b + lane; j < e; j += 32) {
    const double dx = __dsub_rn(pt_pos64[3 * (size_t)j], cx);
    const double dy = __dsub_rn(pt_pos64[3 * (size_t)j + 1], cy);
    const double dz = __dsub_rn(pt_pos64[3 * (size_t)j + 2], cz);
    const double s = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    r2max = r2max < s ? s : r2max;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double other = __shfl_xor_sync(0xffffffffu, r2max, o);
    r2max = r2max < other ? other : r2max;
  }
  if (lane == 0) {
    ctr[3 * i] = cx, ctr[3 * i + 1] = cy, ctr[3 * i + 2] = cz;
    narea[i] = asum;
    nrad[i] = __dsqrt_rn(r2max);
    flag[i] = asum > 0 ? 1 : 0;
    geo[i] = make_float4((float)cx, (float)cy, (float)cz, (float)(asum * kInvFourPi));
  }
}

__global__ void k_topo(const int32_t* __restrict__ beg, const int32_t* __restrict__ end,
                       const int32_t* __restrict__ cbeg, const int32_t* __restrict__ ccnt,
                       const uint8_t* __restrict__ internal, int64_t nodes, int4* topo) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nodes) return;
  topo[i] = internal[i] ? make_int4(cbeg[i], ccnt[i], beg[i], end[i])
                        : make_int4(0, 0, beg[i], end[i]);
}

// opening thresholds thr = (beta^2 * r) * r (bhtree.cpp:193,204); IEEE keeps
// inf * 0 = NaN so radius-0 nodes never pass at beta = inf. Also writes the
// packed 64-byte node records the two-phase kernels read.
__global__ void k_thresholds(const double* __restrict__ ctr, const double* __restrict__ rad,
                             const int4* __restrict__ topo, const float4* __restrict__ geo,
                             int64_t nodes, double beta2, double4* dec, NodeRec* rec) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nodes) return;
  double r = rad[i];
  double thr = __dmul_rn(__dmul_rn(beta2, r), r);
  dec[i] = make_double4(ctr[3 * i], ctr[3 * i + 1], ctr[3 * i + 2], thr);
  NodeRec nr;
  float hx = (float)ctr[3 * i], hy = (float)ctr[3 * i + 1], hz = (float)ctr[3 * i + 2];
  nr.hi = make_float4(hx, hy, hz, (float)thr);
  nr.lo = make_float4((float)(ctr[3 * i] - (double)hx), (float)(ctr[3 * i + 1] - (double)hy),
                      (float)(ctr[3 * i + 2] - (double)hz), geo[i].w);
  nr.topo = topo[i];
  rec[i] = nr;
}

// K4a: per sorted point payload row [mu_c * n (dipole slots, float4 each) |
// mu_c (radial slots) | pad] and fp32 normal / dipole-mu copies for the
// adjoint's leaf terms.
__global__ void k_point_payload(const int32_t* __restrict__ order, const double* __restrict__ nrm,
                                const double* __restrict__ mu, int64_t n, int C, int Cd, int Cr,
                                int F4, const int* __restrict__ chmap, float4* rows, float* pnrm,
                                float* pmud) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  int64_t m = order[j];
  double nx = nrm[3 * m], ny = nrm[3 * m + 1], nz = nrm[3 * m + 2];
  pnrm[3 * j] = (float)nx, pnrm[3 * j + 1] = (float)ny, pnrm[3 * j + 2] = (float)nz;
  float4* row = rows + j * F4;
  for (int k = 0; k < Cd; ++k) {
    double u = mu[m * C + chmap[k]];
    row[k] = make_float4((float)(u * nx), (float)(u * ny), (float)(u * nz), 0.f);
    pmud[j * Cd + k] = (float)u;
  }
  float* r = reinterpret_cast<float*>(row + Cd);
  for (int k = 0; k < 4 * (F4 - Cd); ++k) r[k] = k < Cr ? (float)mu[m * C + chmap[Cd + k]] : 0.f;
}

// K4b: fp64 unnormalised sums, one thread per (node, component) of a level.
// Leaves sum their points (a_m mu_c n_m / a_m mu_c); internal nodes sum children.
__global__ void k_moments_level(int64_t off, int64_t cnt, int W, int C, int Cd,
                                const int4* __restrict__ topo, const int32_t* __restrict__ order,
                                const double* __restrict__ nrm, const double* __restrict__ area,
                                const double* __restrict__ mu, const int* __restrict__ chmap,
                                double* sumv, double* sums, int Cr) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= cnt * W) return;
  int64_t node = off + g / W;
  int comp = (int)(g % W);
  int4 tp = topo[node];
  double acc = 0;
  if (comp < 3 * Cd) {
    int k = comp / 3, a = comp % 3;
    if (tp.y == 0) {
      int ch = chmap[k];
      for (int32_t j = tp.z; j < tp.w; ++j) {
        int64_t m = order[j];
        acc += (area[m] * mu[m * C + ch]) * nrm[3 * m + a];
      }
    } else {
      for (int c = 0; c < tp.y; ++c) acc += sumv[((int64_t)(tp.x + c) * Cd + k) * 3 + a];
    }
    sumv[(node * Cd + k) * 3 + a] = acc;
  } else {
    int k = comp - 3 * Cd;
    if (tp.y == 0) {
      int ch = chmap[Cd + k];
      for (int32_t j = tp.z; j < tp.w; ++j) {
        int64_t m = order[j];
        acc += area[m] * mu[m * C + ch];
      }
    } else {
      for (int c = 0; c < tp.y; ++c) acc += sums[(int64_t)(tp.x + c) * Cr + k];
    }
    sums[node * Cr + k] = acc;
  }
}

__global__ void k_moments_normalise(int64_t nodes, int Cd, int Cr, int F4,
                                    const double* __restrict__ narea,
                                    const double* __restrict__ sumv,
                                    const double* __restrict__ sums, float4* rows) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nodes) return;
  double a = narea[i];
  bool ok = a > 0;  // nodes with area <= 0 keep zero moments (:142)
  float4* row = rows + i * F4;
  for (int k = 0; k < Cd; ++k) {
    const double* s = sumv + (i * Cd + k) * 3;
    row[k] = ok ? make_float4((float)(s[0] / a), (float)(s[1] / a), (float)(s[2] / a), 0.f)
                : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float* r = reinterpret_cast<float*>(row + Cd);
  for (int k = 0; k < 4 * (F4 - Cd); ++k)
    r[k] = (ok && k < Cr) ? (float)(sums[i * Cr + k] / a) : 0.f;
}

// ---------------------------------------------------------------- host

bool forward_tmem_enabled() {
  static const bool v = getenv("DPL_FORWARD_TMEM") != nullptr;
  return v;
}

// out[row] = [hi | lo] with hi = v truncated to tf32 (10 mantissa bits), lo = v - hi
// (exact); W floats per row
__global__ void k_rows_split(const float* __restrict__ rows, float* __restrict__ out, int64_t n,
                             int W) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = rows[i];
    const float h = __uint_as_float(__float_as_uint(v) & 0xffffe000u);
    const int64_t r = i / W, c = i - r * W;
    out[2 * r * W + c] = h;
    out[(2 * r + 1) * W + c] = v - h;
  }
}

template <typename T>
static T* sbuf(Tree& t, int slot, size_t count) {
  t.scratch[slot].reserve(count * sizeof(T));
  return t.scratch[slot].as<T>();
}

void tree_update_points(Tree& t, const double* pos, const double* nrm, const double* area,
                        const double* mu) {
  ++t.version;
  size_t n = (size_t)t.n;
  DPL_CUDA(cudaMemcpyAsync(t.pos64.p, pos, n * 3 * 8, cudaMemcpyDefault, t.stream));
  DPL_CUDA(cudaMemcpyAsync(t.nrm64.p, nrm, n * 3 * 8, cudaMemcpyDefault, t.stream));
  DPL_CUDA(cudaMemcpyAsync(t.area64.p, area, n * 8, cudaMemcpyDefault, t.stream));
  DPL_CUDA(cudaMemcpyAsync(t.mu64.p, mu, n * (size_t)t.C * 8, cudaMemcpyDefault, t.stream));
}

void tree_compute_moments(Tree& t) {
  PhaseTimer ptimer(t, PH_MOMENTS);
  const int B = 256;
  int W = 3 * t.Cd + t.Cr;
  t.node_sumv.reserve(sizeof(double) * std::max<int64_t>(1, t.nodes * t.Cd * 3));
  t.node_sums.reserve(sizeof(double) * std::max<int64_t>(1, t.nodes * t.Cr));
  t.node_row.reserve(sizeof(float4) * (t.nodes + 1) * t.F4);
  t.pt_row.reserve(sizeof(float4) * (t.n + 1) * t.F4);
  t.pt_nrm.reserve(sizeof(float) * t.n * 3);
  t.pt_mud.reserve(sizeof(float) * std::max<int64_t>(1, t.n * t.Cd));
  k_point_payload<<<grid_for(t.n, B), B, 0, t.stream>>>(
      t.order.as<int32_t>(), t.nrm64.as<double>(), t.mu64.as<double>(), t.n, t.C, t.Cd, t.Cr,
      t.F4, t.chmap.as<int>(), t.pt_row.as<float4>(), t.pt_nrm.as<float>(), t.pt_mud.as<float>());
  count_launch();
  int levels = (int)t.level_off.size() - 1;
  for (int d = levels - 1; d >= 0; --d) {
    int64_t off = t.level_off[d], cnt = t.level_off[d + 1] - off;
    if (cnt == 0 || W == 0) continue;
    k_moments_level<<<grid_for(cnt * W, B), B, 0, t.stream>>>(
        off, cnt, W, t.C, t.Cd, t.node_topo.as<int4>(), t.order.as<int32_t>(),
        t.nrm64.as<double>(), t.area64.as<double>(), t.mu64.as<double>(), t.chmap.as<int>(),
        t.node_sumv.as<double>(), t.node_sums.as<double>(), t.Cr);
    count_launch();
  }
  k_moments_normalise<<<grid_for(t.nodes, B), B, 0, t.stream>>>(
      t.nodes, t.Cd, t.Cr, t.F4, t.node_area64.as<double>(), t.node_sumv.as<double>(),
      t.node_sums.as<double>(), t.node_row.as<float4>());
  count_launch();
  if (forward_tmem_enabled()) {
    const int Wf = 4 * t.F4;
    t.node_row_split.reserve(sizeof(float) * 2 * (size_t)(t.nodes + 1) * Wf);
    t.pt_row_split.reserve(sizeof(float) * 2 * (size_t)(t.n + 1) * Wf);
    k_rows_split<<<8 * 148, 256, 0, t.stream>>>(t.node_row.as<float>(), t.node_row_split.as<float>(),
                                                 (int64_t)t.nodes * Wf, Wf);
    k_rows_split<<<8 * 148, 256, 0, t.stream>>>(t.pt_row.as<float>(), t.pt_row_split.as<float>(),
                                                 (int64_t)t.n * Wf, Wf);
    count_launch(2);
  }
  DPL_CUDA(cudaGetLastError());
}

void tree_set_kinds(Tree& t, const uint8_t* kinds) {
  t.kinds.assign(kinds, kinds + t.C);
  t.set_layout();
  tree_compute_moments(t);
}

void tree_ensure_thresholds(Tree& t, double beta) {
  if (t.thr_valid && (t.thr_beta == beta)) return;
  double beta2 = beta * beta;
  t.node_rec.reserve(sizeof(NodeRec) * std::max<int64_t>(1, t.nodes));
  k_thresholds<<<grid_for(t.nodes, 256), 256, 0, t.stream>>>(
      t.node_ctr64.as<double>(), t.node_rad64.as<double>(), t.node_topo.as<int4>(),
      t.node_geo.as<float4>(), t.nodes, beta2, t.node_dec.as<double4>(), t.node_rec.as<NodeRec>());
  count_launch();
  DPL_CUDA(cudaGetLastError());
  t.thr_beta = beta;
  t.thr_valid = !std::isnan(beta);
}

// bounding box of the current point positions (OrientedPointCloud::bounding_box,
// pointcloud.cpp:22-29); synchronous
void tree_point_bbox(Tree& t, double lo[3], double hi[3]) {
  const int B = 256;
  const int64_t n = t.n;
  int nb = (int)std::max<int64_t>(1, std::min<int64_t>(1024, (n + B - 1) / B));
  double* part = sbuf<double>(t, 0, 6 * nb);
  k_bbox_partial<<<nb, B, 0, t.stream>>>(t.pos64.as<double>(), n, part);
  count_launch();
  std::vector<double> hp(6 * nb);
  DPL_CUDA(cudaMemcpyAsync(hp.data(), part, 6 * nb * 8, cudaMemcpyDeviceToHost, t.stream));
  DPL_CUDA(cudaStreamSynchronize(t.stream));
  for (int a = 0; a < 3; ++a) {
    lo[a] = hp[a];
    hi[a] = hp[3 + a];
    for (int b = 1; b < nb; ++b) {
      lo[a] = std::min(lo[a], hp[6 * b + a]);
      hi[a] = std::max(hi[a], hp[6 * b + 3 + a]);
    }
  }
}

void tree_build(Tree& t, const double* pos, const double* nrm, const double* area,
                const double* mu, int64_t n, int C, int max_leaf, int max_depth) {
  if (n <= 0) throw Error(2, "DipoleTree::build: empty cloud");
  ++t.version;
  if (n >= (int64_t)INT32_MAX) throw Error(1, "dpl_tree_build: more than 2^31-1 points");
  if (C < 1 || C > DPL_MAX_CHANNELS) throw Error(1, "dpl_tree_build: channel count out of range");
  max_leaf = std::max(1, max_leaf);   // :162
  max_depth = std::max(0, max_depth); // :163
  if (max_depth > DPL_MAX_DEPTH)
    throw Error(1, "dpl_tree_build: max_depth > 42 not supported on GPU (two 63-bit key words)");
  t.n = n;
  t.C = C;
  t.max_leaf = max_leaf;
  t.max_depth = max_depth;
  t.thr_valid = false;
  t.kinds.assign(C, 0);  // channel_kernels_ all Dipole (:164)
  const int B = 256;
  cudaStream_t s = t.stream;
  t.pos64.reserve(n * 24);
  t.nrm64.reserve(n * 24);
  t.area64.reserve(n * 8);
  t.mu64.reserve(n * (size_t)C * 8);
  tree_update_points(t, pos, nrm, area, mu);

  // root cell (:43-50)
  double lo[3], hi[3];
  tree_point_bbox(t, lo, hi);
  double ctr[3], ext[3];
  for (int a = 0; a < 3; ++a) {
    ctr[a] = 0.5 * (lo[a] + hi[a]);
    ext[a] = hi[a] - lo[a];
    t.root_lo[a] = lo[a];
    t.root_hi[a] = hi[a];
  }
  double mx = ext[0];
  if (mx < ext[1]) mx = ext[1];
  if (mx < ext[2]) mx = ext[2];
  double half = 0.5 * mx;
  volatile double one_plus = 1.0 + 1e-7;
  half = half > 0 ? half * one_plus : 1.0;

  // K1 + K2: keys, stable sort
  uint64_t* keys = sbuf<uint64_t>(t, 1, n);
  int32_t* idx = sbuf<int32_t>(t, 2, n);
  uint64_t* keys_s = sbuf<uint64_t>(t, 3, n);
  int32_t* idx_s = sbuf<int32_t>(t, 4, n);
  const bool deep = max_depth > 21;  // second key word for levels 22..max_depth
  DevBuf klo, klo_s;                 // its unsorted / sorted copies (deep trees only)
  if (deep) klo.reserve(n * 8), klo_s.reserve(n * 8);
  k_keys<<<grid_for(n, B), B, 0, s>>>(t.pos64.as<double>(), n, ctr[0], ctr[1], ctr[2], half,
                                       max_depth, keys, deep ? klo.as<uint64_t>() : nullptr, idx);
  count_launch();
  size_t tmp_bytes = 0;
  if (!deep) {
    int end_bit = std::max(1, 3 * max_depth);
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys_s, idx, idx_s, (int)n, 0, end_bit, s);
    void* tmp = sbuf<char>(t, 5, tmp_bytes + 16);
    DPL_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys_s, idx, idx_s, (int)n, 0,
                                             end_bit, s));
    count_launch(4);
  } else {
    // stable LSD over the two words: by the low word, then by the high word
    DevBuf lo1, idx1, hi1, pos0, pos1;
    lo1.reserve(n * 8), idx1.reserve(n * 4), hi1.reserve(n * 8), pos0.reserve(n * 4),
        pos1.reserve(n * 4);
    const int lo_bits = 3 * (max_depth - 21);
    size_t b1 = 0, b2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b1, klo.as<uint64_t>(), lo1.as<uint64_t>(), idx,
                                    idx1.as<int32_t>(), (int)n, 0, lo_bits, s);
    cub::DeviceRadixSort::SortPairs(nullptr, b2, hi1.as<uint64_t>(), keys_s, pos0.as<int32_t>(),
                                    pos1.as<int32_t>(), (int)n, 0, 63, s);
    tmp_bytes = std::max(b1, b2);
    void* tmp = sbuf<char>(t, 5, tmp_bytes + 16);
    DPL_CUDA(cub::DeviceRadixSort::SortPairs(tmp, b1, klo.as<uint64_t>(), lo1.as<uint64_t>(), idx,
                                             idx1.as<int32_t>(), (int)n, 0, lo_bits, s));
    k_gather_u64<<<grid_for(n, B), B, 0, s>>>(keys, idx1.as<int32_t>(), n, hi1.as<uint64_t>());
    k_iota<<<grid_for(n, B), B, 0, s>>>(pos0.as<int32_t>(), n);
    DPL_CUDA(cub::DeviceRadixSort::SortPairs(tmp, b2, hi1.as<uint64_t>(), keys_s,
                                             pos0.as<int32_t>(), pos1.as<int32_t>(), (int)n, 0, 63,
                                             s));
    k_gather_u64<<<grid_for(n, B), B, 0, s>>>(lo1.as<uint64_t>(), pos1.as<int32_t>(), n,
                                              klo_s.as<uint64_t>());
    k_gather_i32<<<grid_for(n, B), B, 0, s>>>(idx1.as<int32_t>(), pos1.as<int32_t>(), n, idx_s);
    count_launch(12);
    DPL_CUDA(cudaStreamSynchronize(s));  // the temporaries are released here
  }

  // level walk. Node arrays grow level by level.
  std::vector<int64_t> off{0, 1};
  int64_t cap = std::max<int64_t>(1024, n / 2);
  DevBuf beg, end, par, cb, cc, internal;
  auto alloc_nodes = [&](int64_t c) {
    DevBuf nb_[6];
    size_t szs[6] = {4, 4, 4, 4, 4, 1};
    DevBuf* olds[6] = {&beg, &end, &par, &cb, &cc, &internal};
    int64_t have = off.back();
    for (int k = 0; k < 6; ++k) {
      nb_[k].reserve(c * szs[k]);
      DPL_CUDA(cudaMemsetAsync(nb_[k].p, 0, c * szs[k], s));
      if (olds[k]->p && have)
        DPL_CUDA(cudaMemcpyAsync(nb_[k].p, olds[k]->p, have * szs[k], cudaMemcpyDeviceToDevice, s));
    }
    for (int k = 0; k < 6; ++k) olds[k]->swap(nb_[k]);
    DPL_CUDA(cudaStreamSynchronize(s));  // old buffers freed by nb_ destructors
    cap = c;
  };
  alloc_nodes(cap);
  int32_t root_vals[4] = {0, (int32_t)n, -1, 0};
  DPL_CUDA(cudaMemcpyAsync(beg.p, &root_vals[0], 4, cudaMemcpyHostToDevice, s));
  DPL_CUDA(cudaMemcpyAsync(end.p, &root_vals[1], 4, cudaMemcpyHostToDevice, s));
  DPL_CUDA(cudaMemcpyAsync(par.p, &root_vals[2], 4, cudaMemcpyHostToDevice, s));
  int32_t* nint = sbuf<int32_t>(t, 6, 1);
  DPL_CUDA(cudaMemsetAsync(nint, 0, 4, s));
  k_level_internal<<<1, 32, 0, s>>>(beg.as<int32_t>(), end.as<int32_t>(), 0, 1, max_leaf,
                                    max_depth == 0, internal.as<uint8_t>(), nint);
  count_launch();
  int32_t* cur = idx;  // reuse: node id per sorted point at current level
  int32_t* nxt = sbuf<int32_t>(t, 7, n);
  DPL_CUDA(cudaMemsetAsync(cur, 0, n * 4, s));
  t.pt_leaf.reserve(n * 4);
  int32_t* head = reinterpret_cast<int32_t*>(keys);           // keys buffer reused (8n bytes)
  int32_t* incl = reinterpret_cast<int32_t*>(keys) + n;
  int32_t h_nint = 0;
  DPL_CUDA(cudaMemcpyAsync(&h_nint, nint, 4, cudaMemcpyDeviceToHost, s));
  DPL_CUDA(cudaStreamSynchronize(s));
  for (int d = 1; d <= max_depth && h_nint > 0; ++d) {
    // the key word holding digit d (points of one parent share every higher digit)
    const uint64_t* kw = (deep && d > 21) ? klo_s.as<uint64_t>() : keys_s;
    const int shift = !deep ? 3 * (max_depth - d) : (d <= 21 ? 3 * (21 - d) : 3 * (max_depth - d));
    k_level_heads<<<grid_for(n, B), B, 0, s>>>(kw, cur, internal.as<uint8_t>(), n, shift, head,
                                               t.pt_leaf.as<int32_t>());
    count_launch();
    size_t sb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, sb, head, incl, (int)n, s);
    void* stmp = sbuf<char>(t, 5, std::max(sb, tmp_bytes) + 16);
    DPL_CUDA(cub::DeviceScan::InclusiveSum(stmp, sb, head, incl, (int)n, s));
    count_launch();
    int32_t cnt = 0;
    DPL_CUDA(cudaMemcpyAsync(&cnt, incl + n - 1, 4, cudaMemcpyDeviceToHost, s));
    DPL_CUDA(cudaStreamSynchronize(s));
    int64_t o = off.back();
    if (o + cnt > cap) alloc_nodes(std::max<int64_t>(2 * cap, o + cnt));
    k_level_assign<<<grid_for(n, B), B, 0, s>>>(
        kw, cur, internal.as<uint8_t>(), incl, head, n, shift, o, nxt, beg.as<int32_t>(),
        end.as<int32_t>(), par.as<int32_t>(), cb.as<int32_t>(), cc.as<int32_t>(),
        beg.as<int32_t>());
    count_launch();
    off.push_back(o + cnt);
    DPL_CUDA(cudaMemsetAsync(nint, 0, 4, s));
    k_level_internal<<<grid_for(cnt, B), B, 0, s>>>(beg.as<int32_t>(), end.as<int32_t>(), o, cnt,
                                                   max_leaf, d >= max_depth,
                                                   internal.as<uint8_t>(), nint);
    count_launch();
    DPL_CUDA(cudaMemcpyAsync(&h_nint, nint, 4, cudaMemcpyDeviceToHost, s));
    DPL_CUDA(cudaStreamSynchronize(s));
    std::swap(cur, nxt);
  }
  // leaves of the last level
  k_level_heads<<<grid_for(n, B), B, 0, s>>>(keys_s, cur, internal.as<uint8_t>(), n, 0, head,
                                             t.pt_leaf.as<int32_t>());
  count_launch();
  int64_t nodes = off.back();
  t.nodes = nodes;
  t.level_off = off;

  // restore index order within leaves: stable sort by (leaf begin, index)
  uint64_t* key2 = sbuf<uint64_t>(t, 1, n);  // keys buffer (head/incl no longer needed)
  uint64_t* key2_s = keys_s;                 // reuse
  k_leaf_order_keys<<<grid_for(n, B), B, 0, s>>>(t.pt_leaf.as<int32_t>(), beg.as<int32_t>(), idx_s,
                                                 n, key2);
  count_launch();
  size_t tb2 = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tb2, key2, key2_s, (int)n, 0, 64, s);
  void* tmp2 = sbuf<char>(t, 5, std::max(tb2, tmp_bytes) + 16);
  DPL_CUDA(cub::DeviceRadixSort::SortKeys(tmp2, tb2, key2, key2_s, (int)n, 0, 64, s));
  count_launch(4);
  t.order.reserve(n * 4);
  t.leaf_of.reserve(n * 4);
  k_finish_points<<<grid_for(n, B), B, 0, s>>>(key2_s, n, t.order.as<int32_t>(),
                                               t.pt_leaf.as<int32_t>(), t.leaf_of.as<int32_t>());
  count_launch();

  // node arrays in final form
  t.node_parent.reserve(nodes * 4);
  DPL_CUDA(cudaMemcpyAsync(t.node_parent.p, par.p, nodes * 4, cudaMemcpyDeviceToDevice, s));
  t.node_topo.reserve(nodes * sizeof(int4));
  k_topo<<<grid_for(nodes, B), B, 0, s>>>(beg.as<int32_t>(), end.as<int32_t>(), cb.as<int32_t>(),
                                          cc.as<int32_t>(), internal.as<uint8_t>(), nodes,
                                          t.node_topo.as<int4>());
  count_launch();
  t.pt_pos64.reserve(n * 24);
  t.pt_geo.reserve((n + 1) * sizeof(float4));
  t.pt_rec.reserve((n + 1) * sizeof(PtRec));
  k_gather_points<<<grid_for(n, B), B, 0, s>>>(t.order.as<int32_t>(), t.pos64.as<double>(),
                                                t.area64.as<double>(), n, t.pt_pos64.as<double>(),
                                                t.pt_geo.as<float4>(), t.pt_rec.as<PtRec>());
  count_launch();
  t.node_ctr64.reserve(nodes * 24);
  t.node_area64.reserve(nodes * 8);
  t.node_rad64.reserve(nodes * 8);
  t.node_flag.reserve(nodes);
  t.node_geo.reserve((nodes + 1) * sizeof(float4));
  t.node_dec.reserve(nodes * sizeof(double4));
  k_geometry<<<grid_for(nodes, 64), 64, 0, s>>>(
      beg.as<int32_t>(), end.as<int32_t>(), nodes, t.pt_pos64.as<double>(), t.order.as<int32_t>(),
      t.area64.as<double>(), t.node_ctr64.as<double>(), t.node_area64.as<double>(),
      t.node_rad64.as<double>(), t.node_flag.as<uint8_t>(), t.node_geo.as<float4>());
  k_geometry_warp<4><<<(unsigned)((nodes + 3) / 4), 128, 0, s>>>(
      beg.as<int32_t>(), end.as<int32_t>(), nodes, t.pt_pos64.as<double>(), t.order.as<int32_t>(),
      t.area64.as<double>(), t.node_ctr64.as<double>(), t.node_area64.as<double>(),
      t.node_rad64.as<double>(), t.node_flag.as<uint8_t>(), t.node_geo.as<float4>());
  count_launch(2);
  DPL_CUDA(cudaGetLastError());
  t.set_layout();
  tree_compute_moments(t);
  DPL_CUDA(cudaStreamSynchronize(s));
}

void tree_refresh_sorted_positions(Tree& t) {
  k_gather_points<<<grid_for(t.n, 256), 256, 0, t.stream>>>(
      t.order.as<int32_t>(), t.pos64.as<double>(), t.area64.as<double>(), t.n,
      t.pt_pos64.as<double>(), t.pt_geo.as<float4>(), t.pt_rec.as<PtRec>());
  count_launch();
  DPL_CUDA(cudaGetLastError());
}

// export: node records + point permutation
void tree_export(Tree& t, double* geo, int32_t* topo, int32_t* order, int32_t* leaf_of) {
  cudaStream_t s = t.stream;
  int64_t nn = t.nodes;
  if (geo) {
    std::vector<double> c(nn * 3), a(nn), r(nn);
    DPL_CUDA(cudaMemcpyAsync(c.data(), t.node_ctr64.p, nn * 24, cudaMemcpyDeviceToHost, s));
    DPL_CUDA(cudaMemcpyAsync(a.data(), t.node_area64.p, nn * 8, cudaMemcpyDeviceToHost, s));
    DPL_CUDA(cudaMemcpyAsync(r.data(), t.node_rad64.p, nn * 8, cudaMemcpyDeviceToHost, s));
    DPL_CUDA(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < nn; ++i) {
      geo[5 * i] = c[3 * i], geo[5 * i + 1] = c[3 * i + 1], geo[5 * i + 2] = c[3 * i + 2];
      geo[5 * i + 3] = a[i], geo[5 * i + 4] = r[i];
    }
  }
  if (topo) {
    std::vector<int4> tp(nn);
    std::vector<int32_t> par(nn);
    DPL_CUDA(cudaMemcpyAsync(tp.data(), t.node_topo.p, nn * 16, cudaMemcpyDeviceToHost, s));
    DPL_CUDA(cudaMemcpyAsync(par.data(), t.node_parent.p, nn * 4, cudaMemcpyDeviceToHost, s));
    DPL_CUDA(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < nn; ++i) {
      int32_t* o = topo + 6 * i;
      o[0] = tp[i].z, o[1] = tp[i].w, o[2] = tp[i].x, o[3] = tp[i].y, o[4] = par[i];
      o[5] = tp[i].y == 0 ? 1 : 0;
    }
  }
  if (order) DPL_CUDA(cudaMemcpyAsync(order, t.order.p, t.n * 4, cudaMemcpyDeviceToHost, s));
  if (leaf_of) DPL_CUDA(cudaMemcpyAsync(leaf_of, t.leaf_of.p, t.n * 4, cudaMemcpyDeviceToHost, s));
  DPL_CUDA(cudaStreamSynchronize(s));
}

// fp64 moments for every channel in both forms, straight from the definition
// (used by dump; the reference stores both for all channels, bhtree.cpp:136-156).
__global__ void k_full_moments(int64_t nodes, int C, const int4* __restrict__ topo,
                               const int32_t* __restrict__ order, const double* __restrict__ nrm,
                               const double* __restrict__ area, const double* __restrict__ mu,
                               const double* __restrict__ narea, double* mv, double* ms) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= nodes * C) return;
  int64_t i = g / C;
  int c = (int)(g % C);
  int4 tp = topo[i];
  double v0 = 0, v1 = 0, v2 = 0, s = 0;
  double a = narea[i];
  if (a > 0) {
    for (int32_t j = tp.z; j < tp.w; ++j) {
      int64_t m = order[j];
      // the reference rounds am * normal before the add (bhtree.cpp:146-147):
      // explicit _rn intrinsics keep nvcc from contracting them into an FMA
      double am = __dmul_rn(area[m], mu[m * C + c]);
      v0 = __dadd_rn(v0, __dmul_rn(am, nrm[3 * m]));
      v1 = __dadd_rn(v1, __dmul_rn(am, nrm[3 * m + 1]));
      v2 = __dadd_rn(v2, __dmul_rn(am, nrm[3 * m + 2]));
      s = __dadd_rn(s, am);
    }
    v0 /= a, v1 /= a, v2 /= a, s /= a;
  }
  mv[3 * g] = v0, mv[3 * g + 1] = v1, mv[3 * g + 2] = v2;
  ms[g] = s;
}

void tree_full_moments(Tree& t, std::vector<double>& mv, std::vector<double>& ms) {
  int64_t tot = t.nodes * t.C;
  DevBuf dmv, dms;
  dmv.reserve(tot * 24);
  dms.reserve(tot * 8);
  k_full_moments<<<grid_for(tot, 128), 128, 0, t.stream>>>(
      t.nodes, t.C, t.node_topo.as<int4>(), t.order.as<int32_t>(), t.nrm64.as<double>(),
      t.area64.as<double>(), t.mu64.as<double>(), t.node_area64.as<double>(), dmv.as<double>(),
      dms.as<double>());
  count_launch();
  mv.resize(tot * 3);
  ms.resize(tot);
  DPL_CUDA(cudaMemcpyAsync(mv.data(), dmv.p, tot * 24, cudaMemcpyDeviceToHost, t.stream));
  DPL_CUDA(cudaMemcpyAsync(ms.data(), dms.p, tot * 8, cudaMemcpyDeviceToHost, t.stream));
  DPL_CUDA(cudaStreamSynchronize(t.stream));
}

}  // namespace dpl
