// dipole_b200.hpp — C++ mirror of dipole::DipoleTree (proj/include/dipole/
// bhtree.hpp:51-130) over the C-ABI in dipole_b200.h.
//
// Same method names and argument meaning as the reference class; queries are
// batched (a query is 3 doubles, like Vec3) and outputs are fp32. Status codes
// come back as the reference's exception types (DataError / NumericalError,
// util.hpp:35-40). Header-only; link libdipole_b200.so.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "dipole_b200.h"

namespace dipole_b200 {

struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == DPL_OK) return;
  const std::string msg = dpl_last_error();
  if (rc == DPL_ERR_DATA) throw DataError(msg);
  if (rc == DPL_ERR_NUMERICAL) throw NumericalError(msg);
  if (rc == DPL_ERR_CUDA) throw CudaError(msg);
  throw std::invalid_argument(msg);
}

enum class ChannelKernel : uint8_t { Dipole = DPL_DIPOLE, Radial = DPL_RADIAL };

struct KernelParams {  // kernels.hpp:24-29
  double epsilon = 0.0;
  bool desingularized = false;
  double desing_delta = 0.0;
  double coincident_value = 0.0;
  dpl_kernel_params c() const {
    return {epsilon, desingularized ? 1 : 0, 0, desing_delta, coincident_value};
  }
};

// SoA cloud: moments[i * C + 0] is the geometry moment, 1..C-1 appearance.
struct PointCloud {
  std::vector<double> positions, normals, areas, moments;
  int channels = 1;
  int64_t size() const { return (int64_t)areas.size(); }
};

struct TreeNode {  // bhtree.hpp:15-24
  double centroid[3] = {0, 0, 0};
  double area = 0, radius = 0;
  int begin = 0, end = 0, child_begin = 0, child_count = 0, parent = -1;
  bool leaf = false;
};

struct PointGradients {  // bhtree.hpp:28-36
  int channels = 0;
  std::vector<float> moments;  // N x C
  std::vector<float> normals;  // N x 3
  double d_epsilon = 0.0;
  float moment(size_t point, int channel) const { return moments[point * channels + channel]; }
};

class DipoleTree;

class GradientBuffer {  // bhtree.hpp:40-49 (device, fp64)
 public:
  GradientBuffer(GradientBuffer&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  GradientBuffer& operator=(GradientBuffer&& o) noexcept {
    std::swap(h_, o.h_);
    return *this;
  }
  GradientBuffer(const GradientBuffer&) = delete;
  ~GradientBuffer() {
    if (h_) dpl_gradbuf_destroy(h_);
  }
  void reset() { check(dpl_gradbuf_zero(h_)); }
  dpl_gradbuf_t handle() const { return h_; }

 private:
  friend class DipoleTree;
  explicit GradientBuffer(dpl_gradbuf_t h) : h_(h) {}
  dpl_gradbuf_t h_ = nullptr;
};

class DipoleTree {
 public:
  static constexpr int kDefaultMaxLeafSize = 8;
  static constexpr int kDefaultMaxDepth = 20;

  explicit DipoleTree(int device = 0, void* stream = nullptr) {
    check(dpl_tree_create(device, stream, &h_));
  }
  ~DipoleTree() {
    if (h_) dpl_tree_destroy(h_);
  }
  DipoleTree(const DipoleTree&) = delete;
  DipoleTree& operator=(const DipoleTree&) = delete;

  void build(const PointCloud& c, int max_leaf_size = kDefaultMaxLeafSize,
             int max_depth = kDefaultMaxDepth) {
    check(dpl_tree_build(h_, c.positions.data(), c.normals.data(), c.areas.data(),
                         c.moments.data(), c.size(), c.channels, max_leaf_size, max_depth));
  }
  void update_moments(const PointCloud& c) {
    check(dpl_tree_update_moments(h_, c.positions.data(), c.normals.data(), c.areas.data(),
                                  c.moments.data(), c.size(), c.channels));
  }
  void set_channel_kernels(const std::vector<ChannelKernel>& k) {
    std::vector<uint8_t> v(k.size());
    for (size_t i = 0; i < k.size(); ++i) v[i] = (uint8_t)k[i];
    check(dpl_tree_set_channel_kernels(h_, v.data(), (int32_t)v.size()));
  }
  int channels() const {
    int32_t c = 0;
    check(dpl_tree_channels(h_, &c));
    return c;
  }
  size_t point_count() const {
    int64_t n = 0;
    check(dpl_tree_point_count(h_, &n));
    return (size_t)n;
  }
  std::vector<TreeNode> nodes() const {
    int64_t nn = 0;
    check(dpl_tree_node_count(h_, &nn));
    std::vector<double> geo(nn * 5);
    std::vector<int32_t> topo(nn * 6);
    check(dpl_tree_export(h_, geo.data(), topo.data(), nullptr, nullptr));
    std::vector<TreeNode> out(nn);
    for (int64_t i = 0; i < nn; ++i) {
      TreeNode& t = out[i];
      for (int a = 0; a < 3; ++a) t.centroid[a] = geo[5 * i + a];
      t.area = geo[5 * i + 3], t.radius = geo[5 * i + 4];
      t.begin = topo[6 * i], t.end = topo[6 * i + 1], t.child_begin = topo[6 * i + 2];
      t.child_count = topo[6 * i + 3], t.parent = topo[6 * i + 4], t.leaf = topo[6 * i + 5] != 0;
    }
    return out;
  }
  std::vector<int> point_order() const {
    std::vector<int> o(point_count());
    check(dpl_tree_export(h_, nullptr, nullptr, o.data(), nullptr));
    return o;
  }

  // primal (bhtree.cpp:188-234) for q queries xs[3 q]: out[q * C]; visited optional
  void primal(const double* xs, int64_t q, const KernelParams& p, double beta_bh, float* out,
              dpl_counters* counters = nullptr) const {
    dpl_kernel_params kp = p.c();
    check(dpl_primal(h_, &kp, beta_bh, xs, q, out, nullptr, counters));
  }
  // primal_channel (bhtree.cpp:236-274): out[q]
  void primal_channel(const double* xs, int64_t q, const KernelParams& p, double beta_bh,
                      int channel, float* out) const {
    dpl_kernel_params kp = p.c();
    check(dpl_primal_channel(h_, &kp, beta_bh, xs, q, channel, out));
  }
  // primal_with_gradient (bhtree.cpp:276-334): out[q * C], grad[q * C * 3]
  void primal_with_gradient(const double* xs, int64_t q, const KernelParams& p, double beta_bh,
                            float* out, float* grad) const {
    dpl_kernel_params kp = p.c();
    check(dpl_primal(h_, &kp, beta_bh, xs, q, out, grad, nullptr));
  }

  // sample_grid (meshing.cpp:33-59): values[(k * r1 + j) * r0 + i] = 0.5 - D0(node)
  std::vector<float> sample_grid(const KernelParams& p, double beta_bh, const int32_t res[3],
                                 const double lo[3], const double hi[3], double lo_out[3] = nullptr,
                                 double hi_out[3] = nullptr) const {
    dpl_kernel_params kp = p.c();
    std::vector<float> v((size_t)res[0] * res[1] * res[2]);
    check(dpl_sample_grid(h_, &kp, beta_bh, res, lo, hi, v.data(), lo_out, hi_out));
    return v;
  }
  // sample_ray (renderer.cpp:46-86) for R rays (origin, dir): t / delta R x max_samples
  void sample_rays(const KernelParams& p, double beta_bh, const double* rays, int64_t R,
                   const dpl_ray_sampler& cfg, int32_t max_samples, double* t, double* delta,
                   int32_t* count, uint8_t* bracketed) const {
    dpl_kernel_params kp = p.c();
    check(dpl_sample_rays(h_, &kp, beta_bh, rays, R, &cfg, max_samples, t, delta, count,
                          bracketed));
  }

  GradientBuffer make_buffer() const {
    dpl_gradbuf_t b = nullptr;
    check(dpl_gradbuf_create(h_, &b));
    return GradientBuffer(b);
  }
  // adjoint (bhtree.cpp:345-417): d_out[q * C], d_grad nullptr or [q * C * 3]
  void adjoint(const double* xs, int64_t q, const KernelParams& p, double beta_bh,
               const float* d_out, const float* d_grad, GradientBuffer& buf) const {
    dpl_kernel_params kp = p.c();
    check(dpl_adjoint(h_, &kp, beta_bh, xs, q, d_out, d_grad, buf.handle()));
  }
  // flush_gradients (bhtree.cpp:419-463): zeroes the buffers
  PointGradients flush_gradients(std::vector<GradientBuffer*> bufs) const {
    std::vector<dpl_gradbuf_t> hs;
    for (GradientBuffer* b : bufs) hs.push_back(b->handle());
    PointGradients g;
    g.channels = channels();
    g.moments.resize(point_count() * g.channels);
    g.normals.resize(point_count() * 3);
    check(dpl_flush(h_, hs.data(), (int32_t)hs.size(), g.moments.data(), g.normals.data(),
                    &g.d_epsilon));
    return g;
  }
  PointGradients flush_gradients(GradientBuffer& b) const { return flush_gradients({&b}); }

  void dump(const std::string& path) const { check(dpl_tree_dump(h_, path.c_str())); }
  // host-async mode: see dpl_tree_set_host_async
  void set_host_async(bool on) { check(dpl_tree_set_host_async(h_, on ? 1 : 0)); }
  void synchronize() const { check(dpl_tree_sync(h_)); }
  dpl_tree_t handle() const { return h_; }

 private:
  dpl_tree_t h_ = nullptr;
};

}  // namespace dipole_b200
