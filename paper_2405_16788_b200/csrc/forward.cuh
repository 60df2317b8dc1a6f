// forward.cuh — host entry points of the forward traversals (forward.cu).
#pragma once

#include "ilist.cuh"
#include "tree.cuh"

namespace dpl {

struct FwdArgs {
  const double* xs = nullptr;     // device, q x 3 (original order)
  const int32_t* perm = nullptr;  // device, sorted position -> query index (or null)
  int64_t q = 0;
  float* out = nullptr;           // device, q x out_stride
  int out_stride = 1;
  int single = 0;                 // primal_channel: q x 1 output
  float* grad = nullptr;          // grad_mode 1: q x C x 3; grad_mode 2: q x 3
  int grad_mode = 0;              // 0 none, 1 all channels, 2 dipole slot 0 only
  long long* counters = nullptr;  // q x 5 (dpl_counters)
  int* overflow = nullptr;        // device flag
  int only_dip = -1, only_rad = -1;  // primal_channel: the single slot
  int only_ch = -1;  // primal_channel on the two-phase kernels: same kernel as
                     // primal, only channel only_ch stored (q x 1) -> bitwise
                     // primal_channel(c) == primal()[c] (test_bhtree.cpp:140)
  int nr_limit = -1;                 // only the first nr_limit radial slots (render step)
  double beta = 0;         // opening parameter (interaction-list reuse key)
  IList* ilist = nullptr;  // interaction-list workspace (ilist.cuh): built and replayed by the
                           // kernels that support it, unless DPL_NO_ILIST is set
};

void forward_launch(const Tree& t, const KParams& kp, FwdArgs a);
// two-phase values-only kernel (forward2.cu); false if the layout is not covered
bool forward2_launch(const Tree& t, const KParams& kp, const FwdArgs& a);
// tensor-core (3xTF32 mma.sync) values-only kernel (forward_tc.cu)
bool forward_tc_launch(const Tree& t, const KParams& kp, const FwdArgs& a);
// tcgen05 / TMEM values-only kernel for one Dipole + 48 Radial slots (forward_tm.cu)
bool forward_tm_launch(const Tree& t, const KParams& kp, const FwdArgs& a);
void morton_order(Tree& t, const double* xs_dev, int64_t q, int32_t* perm_out, DevBuf& ws);

}  // namespace dpl
