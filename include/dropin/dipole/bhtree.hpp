// Drop-in replacement for the reference's dipole/bhtree.hpp (the public
// surface of proj/include/dipole/bhtree.hpp:13-105, signatures unchanged),
// implemented on the B200 engine through the C-ABI of include/dipole_b200.h
// (paper_2405_16788_b200/dropin/bhtree_b200.cpp). A project switches by putting
// include/dropin ahead of its own include directory, compiling
// bhtree_b200.cpp instead of src/bhtree.cpp and linking libdipole_b200.so;
// callers (fields.cpp, renderer.cpp, optimizer.cpp, verify.cpp, oracles.cpp)
// compile unchanged. INTEGRATION.md describes the deviations:
//  * per-query calls are correct but launch-bound; the batched overloads at the
//    end of the class are the fast path;
//  * query arithmetic is fp32 (fp64 opening decisions and accumulators);
//  * GradientBuffer's accumulators live on the device; its reference fields
//    are read-only views that materialise on access, and per-query adjoint()
//    calls are queued and evaluated in batches.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "dipole/kernels.hpp"
#include "dipole/pointcloud.hpp"

namespace dipole {

enum class ChannelKernel { Dipole, Radial };  // bhtree.hpp:13

struct TreeNode {  // bhtree.hpp:15-24 (same fields, same defaults)
  Vec3 centroid = Vec3::Zero();
  double area = 0.0;
  double radius = 0.0;
  int begin = 0, end = 0;
  int child_begin = 0;
  int child_count = 0;
  int parent = -1;
  bool leaf = false;
};

struct PointGradients {  // bhtree.hpp:28-36
  int channels = 0;
  std::vector<double> moments;  // M x channels
  std::vector<Vec3> normals;    // M
  double d_epsilon = 0.0;

  double& moment(std::size_t point, int channel) { return moments[point * channels + channel]; }
  double moment(std::size_t point, int channel) const { return moments[point * channels + channel]; }
};

struct GradientBuffer;

namespace b200 {
struct BufferState;  // device accumulators + queued per-query adjoints
struct TreeState;    // the engine handle + host mirrors of the tree

// One of GradientBuffer's reference fields, read through the device buffer:
// any read first evaluates the queued adjoint queries and downloads the
// accumulators (only when they changed since the last download).
template <typename T>
class DeviceMirror {
 public:
  using value_type = T;
  using const_iterator = const T*;
  explicit DeviceMirror(int field) : field_(field) {}
  std::size_t size() const { return view().size(); }
  bool empty() const { return view().empty(); }
  const T& operator[](std::size_t i) const { return view()[i]; }
  const T& at(std::size_t i) const { return view().at(i); }
  const T* data() const { return view().data(); }
  const T* begin() const { return view().data(); }
  const T* end() const { return view().data() + view().size(); }
  const T& front() const { return view().front(); }
  const T& back() const { return view().back(); }
  operator const std::vector<T>&() const { return view(); }

 private:
  friend struct ::dipole::GradientBuffer;
  const std::vector<T>& view() const;
  int field_;
  BufferState* owner_ = nullptr;
};
}  // namespace b200

// Per-worker adjoint accumulator (bhtree.hpp:38-49). Move-only: it owns a
// device buffer. Fields read as in the reference (views of the device data).
struct GradientBuffer {
  b200::DeviceMirror<Vec3> node_v{0};     // nodes x channels
  b200::DeviceMirror<double> node_s{1};   // nodes x channels
  b200::DeviceMirror<double> point_mu{2}; // M x channels
  b200::DeviceMirror<Vec3> point_n{3};    // M
  double d_epsilon = 0.0;                 // host copy, refreshed with the views
  bool dirty = false;

  void reset();

  GradientBuffer();
  ~GradientBuffer();
  GradientBuffer(GradientBuffer&&) noexcept;
  GradientBuffer& operator=(GradientBuffer&&) noexcept;
  GradientBuffer(const GradientBuffer&) = delete;
  GradientBuffer& operator=(const GradientBuffer&) = delete;

 private:
  friend class DipoleTree;
  template <typename T>
  friend class b200::DeviceMirror;
  void bind();
  std::unique_ptr<b200::BufferState> state_;
};

class DipoleTree {
 public:
  static constexpr int kDefaultMaxLeafSize = 8;
  static constexpr int kDefaultMaxDepth = 20;

  DipoleTree();
  ~DipoleTree();
  DipoleTree(const DipoleTree& other);  // rebuilds the copy on the device
  DipoleTree& operator=(const DipoleTree& other);
  DipoleTree(DipoleTree&&) noexcept;
  DipoleTree& operator=(DipoleTree&&) noexcept;

  // ---- the reference's API (bhtree.hpp:51-105), unchanged ------------------
  void build(const OrientedPointCloud& cloud, int max_leaf_size = kDefaultMaxLeafSize,
             int max_depth = kDefaultMaxDepth);
  void update_moments(const OrientedPointCloud& cloud);

  void set_channel_kernels(std::vector<ChannelKernel> kernels);
  const std::vector<ChannelKernel>& channel_kernels() const;

  int channels() const;
  std::size_t point_count() const;
  const std::vector<TreeNode>& nodes() const;
  const std::vector<int>& point_order() const;

  void primal(const Vec3& x, const KernelParams& params, double beta_bh, std::span<double> out,
              long* visited = nullptr) const;
  double primal_channel(const Vec3& x, const KernelParams& params, double beta_bh, int channel,
                        long* visited = nullptr) const;
  void primal_with_gradient(const Vec3& x, const KernelParams& params, double beta_bh,
                            std::span<double> out, std::span<Vec3> grad_out,
                            long* visited = nullptr) const;
  void adjoint(const Vec3& x, const KernelParams& params, double beta_bh,
               std::span<const double> d_out, std::span<const Vec3> d_grad,
               GradientBuffer& buf) const;

  GradientBuffer make_buffer() const;
  PointGradients flush_gradients(std::span<GradientBuffer> buffers) const;
  PointGradients flush_gradients(GradientBuffer& buffer) const;

  void dump(const std::string& path) const;

  // ---- batched overloads (the fast path): xs Q points, out Q x C ------------
  void primal(std::span<const Vec3> xs, const KernelParams& params, double beta_bh,
              std::span<double> out, std::span<long> visited = {}) const;
  void primal_channel(std::span<const Vec3> xs, const KernelParams& params, double beta_bh,
                      int channel, std::span<double> out) const;
  void primal_with_gradient(std::span<const Vec3> xs, const KernelParams& params, double beta_bh,
                            std::span<double> out, std::span<Vec3> grad_out) const;
  // d_out Q x C; d_grad empty or Q x C
  void adjoint(std::span<const Vec3> xs, const KernelParams& params, double beta_bh,
               std::span<const double> d_out, std::span<const Vec3> d_grad,
               GradientBuffer& buf) const;

  // engine device for trees built after the call (default: DPL_DEVICE or 0)
  static void set_device(int device);

 private:
  std::shared_ptr<b200::TreeState> s_;
};

}  // namespace dipole
