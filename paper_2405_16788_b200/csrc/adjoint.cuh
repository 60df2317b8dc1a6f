// adjoint.cuh — GradientBuffer on device and the adjoint / flush entry points.
#pragma once

#include "ilist.cuh"
#include "tree.cuh"

namespace dpl {

// GradientBuffer (bhtree.hpp:40-49) in fp64, one allocation. Point
// accumulators are kept in tree (sorted) order; flush maps them back.
struct GradBuf {
  int64_t nodes = 0, n = 0;
  int Cd = 0, Cr = 0;
  size_t total = 0;
  DevBuf mem;
  double *node_v = nullptr, *node_s = nullptr, *pt_mud = nullptr, *pt_mur = nullptr,
         *pt_n = nullptr, *d_eps = nullptr;
};

struct AdjArgs {
  const double* xs = nullptr;
  const int32_t* perm = nullptr;
  int64_t q = 0;
  const float* d_out = nullptr;  // q x dstride
  int dstride = 0;
  const float* d_grad = nullptr;
  int grad_mode = 0;   // 0 none, 1 q x dstride x 3, 2 q x 3 for channel 0
  int nr_limit = -1;   // only the first nr_limit radial slots carry non-zero d_out
  int* overflow = nullptr;
  double beta = 0;         // opening parameter (interaction-list reuse key)
  IList* ilist = nullptr;  // interaction lists (ilist.cuh); reused when the previous
                           // call built them for the same queries / beta / tree
};

void gradbuf_alloc(GradBuf& b, const Tree& t);
void gradbuf_zero(GradBuf& b, cudaStream_t s);
void gradbuf_accumulate(GradBuf& dst, const GradBuf& src, cudaStream_t s);
void adjoint_launch(const Tree& t, const KParams& kp, const AdjArgs& a, GradBuf& b);
// two-phase kernel for one Dipole + <= 64 Radial channels (adjoint2.cu)
bool adjoint2_launch(const Tree& t, const KParams& kp, const AdjArgs& a, GradBuf& b);
// tcgen05 / TMEM kernel for one Dipole + (4, 48] Radial channels (adjoint_tm.cu)
bool adjoint_tm_launch(const Tree& t, const KParams& kp, const AdjArgs& a, GradBuf& b);
// consumes b's node accumulators (push-down in place); caller zeroes afterwards
void flush_launch(Tree& t, GradBuf& b, float* moments, float* normals);
// flush_launch split for cross-rank reduction: the node
// push-down, then per-point gradient ROWS [moments (C) | normals (3)] in tree
// order for the sorted-point range [lo, hi) (identical on every rank: the tree
// is bit-identical), then the scatter of summed rows to the original order.
void flush_pushdown(Tree& t, GradBuf& b);
void flush_rows(Tree& t, const GradBuf& b, int64_t lo, int64_t hi, float* rows);
void flush_unpermute(Tree& t, const float* rows, float* moments, float* normals);

}  // namespace dpl
