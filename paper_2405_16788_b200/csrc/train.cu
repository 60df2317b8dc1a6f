// train.cu — the point-parameter half of Trainer::step on the device.
//
// Restates proj/src/optimizer.cpp:161-205 for the point groups: Adam
// (optimizer.cpp:65-81) on the geometry moments beta, the appearance moments
// alpha and the raw normals n, one step counter shared by the three groups
// (they are stepped together every iteration), then the write-back: moments
// copied, normals renormalised only when the update changed them (:196-200),
// and finally update_moments (bhtree.cpp:171-176) refreshes the tree's node
// moments and payload rows. fp64 with the reference's operation order and no
// FMA, so given identical gradients the parameters match the reference's bits.
#include <cmath>

#include "train.cuh"

namespace dpl {

__device__ __forceinline__ double adam1(double p, double g, double& m, double& v, double lr,
                                        double b1, double b2, double eps, double c1, double c2) {
  m = __dadd_rn(__dmul_rn(b1, m), __dmul_rn(__dsub_rn(1.0, b1), g));
  v = __dadd_rn(__dmul_rn(b2, v), __dmul_rn(__dmul_rn(__dsub_rn(1.0, b2), g), g));
  const double step = __ddiv_rn(__dmul_rn(lr, __ddiv_rn(m, c1)),
                                __dadd_rn(__dsqrt_rn(__ddiv_rn(v, c2)), eps));
  return __dsub_rn(p, step);
}

// appearance / geometry moments: one thread per (point, channel) element,
// coalesced (the groups are elementwise, optimizer.cpp:65-81)
__global__ void k_moment_adam(int64_t nm, double* __restrict__ mu, const float* __restrict__ g_mu,
                              double* __restrict__ m_mu, double* __restrict__ v_mu, double lr,
                              double b1, double b2, double eps, double c1, double c2) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nm;
       k += (int64_t)gridDim.x * blockDim.x) {
    double m = m_mu[k], v = v_mu[k];
    mu[k] = adam1(mu[k], (double)g_mu[k], m, v, lr, b1, b2, eps, c1, c2);
    m_mu[k] = m, v_mu[k] = v;
  }
}

// raw normals: one thread per point (original order), renormalised only when
// the update changed them (optimizer.cpp:196-200)
__global__ void k_normal_adam(int64_t n, double* __restrict__ nrm, const float* __restrict__ g_n,
                              double* __restrict__ m_n, double* __restrict__ v_n, double lr,
                              double b1, double b2, double eps, double c1, double c2) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double old[3], nw[3];
  for (int a = 0; a < 3; ++a) {
    const int64_t k = 3 * i + a;
    old[a] = nrm[k];
    double m = m_n[k], v = v_n[k];
    nw[a] = adam1(old[a], (double)g_n[k], m, v, lr, b1, b2, eps, c1, c2);
    m_n[k] = m, v_n[k] = v;
  }
  if (nw[0] != old[0] || nw[1] != old[1] || nw[2] != old[2]) {  // n != p.normal (:197)
    const double len = __dsqrt_rn(
        __dadd_rn(__dadd_rn(__dmul_rn(nw[0], nw[0]), __dmul_rn(nw[1], nw[1])), __dmul_rn(nw[2], nw[2])));
    if (len > 1e-12)
      for (int a = 0; a < 3; ++a) nrm[3 * i + a] = __ddiv_rn(nw[a], len);
  }
}

void point_adam_alloc(PointAdam& o, const Tree& t) {
  o.n = t.n;
  o.C = t.C;
  o.t = 0;
  size_t nm = (size_t)t.n * t.C, nn = (size_t)t.n * 3;
  o.state.reserve((2 * nm + 2 * nn) * sizeof(double));
  DPL_CUDA(cudaMemsetAsync(o.state.p, 0, (2 * nm + 2 * nn) * sizeof(double), t.stream));
}

void point_adam_step_range(Tree& t, PointAdam& o, const float* g_mu, const float* g_n,
                           int64_t lo, int64_t hi, double lr, double b1, double b2, double eps) {
  ++o.t;  // one step per call, as Adam::step (:73)
  if (hi <= lo) return;
  const double c1 = 1.0 - std::pow(b1, (double)o.t);
  const double c2 = 1.0 - std::pow(b2, (double)o.t);
  const size_t nm = (size_t)t.n * t.C, nn = (size_t)t.n * 3;
  const int64_t cnt = hi - lo;
  double* s = o.state.as<double>();
  const size_t om = (size_t)lo * t.C, on = (size_t)lo * 3;
  k_moment_adam<<<148 * 16, 256, 0, t.stream>>>(cnt * t.C, t.mu64.as<double>() + om, g_mu, s + om,
                                                 s + nm + om, lr, b1, b2, eps, c1, c2);
  k_normal_adam<<<(unsigned)((cnt + 255) / 256), 256, 0, t.stream>>>(
      cnt, t.nrm64.as<double>() + on, g_n, s + 2 * nm + on, s + 2 * nm + nn + on, lr, b1, b2, eps,
      c1, c2);
  count_launch(2);
  DPL_CUDA(cudaGetLastError());
}

void point_adam_step(Tree& t, PointAdam& o, const float* g_mu, const float* g_n, double lr,
                     double b1, double b2, double eps) {
  ++o.t;  // Adam::step increments before use (:73)
  const double c1 = 1.0 - std::pow(b1, (double)o.t);
  const double c2 = 1.0 - std::pow(b2, (double)o.t);
  size_t nm = (size_t)t.n * t.C, nn = (size_t)t.n * 3;
  double* s = o.state.as<double>();
  k_moment_adam<<<148 * 16, 256, 0, t.stream>>>((int64_t)nm, t.mu64.as<double>(), g_mu, s,
                                                 s + nm, lr, b1, b2, eps, c1, c2);
  k_normal_adam<<<(unsigned)((t.n + 255) / 256), 256, 0, t.stream>>>(
      t.n, t.nrm64.as<double>(), g_n, s + 2 * nm, s + 2 * nm + nn, lr, b1, b2, eps, c1, c2);
  count_launch(2);
  DPL_CUDA(cudaGetLastError());
  tree_compute_moments(t);  // update_moments (bhtree.cpp:171-176)
}

}  // namespace dpl
