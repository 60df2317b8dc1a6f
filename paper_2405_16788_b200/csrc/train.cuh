// train.cuh — device-side point-parameter update of Trainer::step (train.cu).
#pragma once

#include "tree.cuh"

namespace dpl {

struct PointAdam {
  int64_t n = 0;
  int C = 0;
  int64_t t = 0;  // Adam::t (optimizer.hpp:54-59)
  DevBuf state;   // m_mu, v_mu (N x C), m_n, v_n (N x 3), fp64
};

void point_adam_alloc(PointAdam& o, const Tree& t);
// g_mu: N x C, g_n: N x 3 (device fp32, original point order)
void point_adam_step(Tree& t, PointAdam& o, const float* g_mu, const float* g_n, double lr,
                     double b1, double b2, double eps);

}  // namespace dpl
