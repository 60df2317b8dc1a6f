// dpl_internal.cuh — shared device/host definitions of the B200 dipole engine.
//
// HBM layout of one tree (all device-resident, built by build.cu):
//   node_dec   double4 [nodes]   {cx, cy, cz, thr}   fp64 centroid + opening threshold
//                                thr = (beta^2 * radius) * radius for the current beta
//   node_topo  int4    [nodes]   {child_begin, child_count, begin, end}; leaf <=> count == 0
//   node_geo   float4  [nodes]   {cx, cy, cz, A = area/(4 pi)} fp32 copies for arithmetic
//   node_flag  uint8   [nodes]   bit0: area > 0 (far field allowed, bhtree.cpp:205)
//   node_pay   float   [nodes x P]  payload row: [3 x Cd dipole moments | Cr radial moments | pad]
//   pt_pos64   double  [N x 3]   sorted (tree) order, fp64 positions (leaf distances)
//   pt_geo     float4  [N]       {px, py, pz, A_m = a_m/(4 pi)} sorted order
//   pt_pay     float   [N x P]   payload row: [mu_c * n (3 x Cd) | mu_c (Cr) | pad]
//   pt_nrm/pt_mu fp32 sorted copies for the adjoint's leaf terms
// Channel layout: dipole channels first (dip_ch[k] = reference channel id),
// radial channels after (rad_ch[k]); P = round_up(3*Cd + Cr, 4).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <stdexcept>
#include <string>

#define DPL_WARP 32
#define DPL_MAX_CHANNELS 1024
// Deepest tree the GPU build supports: 3 key bits per level in two 64-bit key
// words (tree.cu rejects max_depth > 42 at build time with a usage error; the
// reference's default is 20, bhtree.hpp:54).
#define DPL_MAX_DEPTH 42
// Traversal stack per warp. A popped internal node pushes its child_count
// children, so along any root-to-leaf path the stack holds at most
// 1 + sum (child_count - 1) <= 1 + 7 * depth entries (the reference sizes its
// stack the same way, bhtree.cpp:185); 304 covers every supported depth.
#define DPL_STACK_PER_WARP 304
static_assert(DPL_STACK_PER_WARP >= 7 * DPL_MAX_DEPTH + 8, "traversal stack below 7 * depth + 8");

namespace dpl {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define DPL_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw ::dpl::Error(4, std::string(#call) + ": " + cudaGetErrorString(e_));        \
  } while (0)

void count_launch(int n = 1);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is a per-device property of
// a kernel: `done` keeps one bit per device (benign race: two threads may both
// set the same attribute value).
template <typename K>
inline void ensure_max_dyn_smem(K* kernel, int device, size_t smem,
                                std::atomic<unsigned long long>& done) {
  const unsigned long long bit = 1ull << (device & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  DPL_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  done.fetch_or(bit, std::memory_order_acq_rel);
}

// kernel radial-profile mode
enum KMode : int { KM_REGULARIZED = 0, KM_SINGULAR = 1, KM_DESING = 2 };

// Launch-constant kernel parameters (fp32 powers of 1/eps precomputed in fp64).
struct KParams {
  int mode;
  float eps, inv_eps, inv_eps3, inv_eps4, inv_eps5, inv_eps6;
  float delta2;
  float near2;  // (6.5 eps)^2: beyond it tau = 1 (kernels.cpp:50-55)
};

// Packed 48-byte node record for the two-phase kernels. The fp64 centroid c
// is stored as a double-float pair (hi = fl32(c), lo = fl32(c - hi)), so
// d = (c_hi - x_hi) + (c_lo - x_lo) carries ~2^-23 relative error and the
// opening test can run in fp32 with a rigorous ambiguity band; only inside
// the band is the reference's exact fp64 test re-evaluated (node_dec).
struct alignas(16) NodeRec {
  float4 hi;     // c_hi.xyz, thr32 = fl32((beta^2 r) r)
  float4 lo;     // c_lo.xyz, A = area / (4 pi)
  int4 topo;     // child_begin, child_count (0 = leaf), begin, end
};

// Double-float point record (tree order): p_hi.xyz + A, p_lo.xyz.
struct alignas(16) PtRec {
  float4 hi;
  float4 lo;
};

// Per-launch view of a tree for the traversal kernels.
struct TreeView {
  const double4* node_dec;
  const int4* node_topo;
  const float4* node_geo;
  const uint8_t* node_flag;
  const NodeRec* node_rec;
  const PtRec* pt_rec;
  const float4* node_row;   // nodes x F4: [dipole float4 x Cd | radial floats | pad]
  const double* pt_pos64;
  const float4* pt_geo;
  const float4* pt_row;     // N x F4 (sorted order)
  // tf32 split of the payload rows, [row][hi F4 float4 | lo F4 float4] (hi = row
  // truncated to tf32, lo = row - hi), only when the TMEM forward is enabled
  // (forward_tm.cu); null otherwise
  const float4* node_row_split;
  const float4* pt_row_split;
  const float* pt_nrm;  // N x 3 sorted
  const float* pt_mu;   // N x C sorted (reference channel order)
  int P;                // radial pad (floats, multiple of 4)
  int F4;               // payload row stride (float4)
  int Cd, Cr, C;
  int64_t nodes, n;
  int max_depth;
  float cmax;  // >= max |centroid coordinate| (root bounding box, with margin)
};

// Fast host->device constant table of channel mapping for kernels.
struct ChanMap {
  int dip_ch[64];   // dipole slot -> channel id (tiles only use the first TD)
  int rad_ch[1024];
};

inline int round_up4(int x) { return (x + 3) & ~3; }

// smallest (6.5 eps)^2 for which the regularized-mode kernels zero a far
// entry's non-member lanes through their area: R <= 1e12, W <= 1e18 and the
// query-gradient term W R <= 1e30 stay finite (eps >= 1.6e-7; smaller eps runs
// the generic kernels)
constexpr float REG_MIN_NEAR2 = 1e-12f;

#ifdef __CUDACC__
// 1/sqrt(x): the MUFU.RSQ that rsqrtf issues for normal inputs (bit-identical
// there), without rsqrtf's denormal rescaling — x is clamped to FLT_MIN instead.
// Callers either have x >= FLT_MIN (far field: x > the opening threshold) or
// discard the result (r2 == 0 at coincidence takes the near-field series)
__device__ __forceinline__ float rsqrt_pos(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(fmaxf(x, 1.17549435e-38f)));
  return r;
}

// 1/sqrt(max(x, m)) for the regularized far field beyond 6.5 eps: every lane
// whose value is kept has x >= m = (6.5 eps)^2, so the clamp changes nothing
// for it; the other lanes get a finite W <= m^-1.5 (hosts only pick these
// kernels when m >= REG_MIN_NEAR2), which their zeroed area turns into exact 0s
__device__ __forceinline__ float rsqrt_far(float x, float m) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(fmaxf(x, m)));
  return r;
}

// p ? a : 0 as one SEL the compiler cannot turn back into a branch around the
// computation of a (keeps branch-free lane values branch-free)
__device__ __forceinline__ float sel0(bool p, float a) {
  float r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\tselp.f32 %0, %1, 0f00000000, q;\n\t}\n"
      : "=f"(r)
      : "f"(a), "r"((int)p));
  return r;
}

// fp64 RED under a PTX predicate (no C++ branch; the address needs no guard)
__device__ __forceinline__ void red_add_if(double* p, double v, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q red.global.add.f64 [%0], %1;\n\t}\n" ::"l"(p),
      "d"(v), "r"((int)pred)
      : "memory");
}

// fp32 value added to an fp64 accumulator: conversion and RED in one predicated
// PTX block (keeps ptxas from branching around the pair)
__device__ __forceinline__ void red_add_f32_if(double* p, float v, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\t.reg .f64 d;\n\tsetp.ne.b32 q, %2, 0;\n\t"
      "cvt.f64.f32 d, %1;\n\t@q red.global.add.f64 [%0], d;\n\t}\n" ::"l"(p),
      "f"(v), "r"((int)pred)
      : "memory");
}
__device__ __forceinline__ void red_add_f32(double* p, float v) {
  asm volatile("{\n\t.reg .f64 d;\n\tcvt.f64.f32 d, %1;\n\tred.global.add.f64 [%0], d;\n\t}\n" ::"l"(p),
               "f"(v)
               : "memory");
}

#endif

}  // namespace dpl
