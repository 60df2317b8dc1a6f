// bhtree_b200.cpp — dipole::DipoleTree (include/dropin/dipole/bhtree.hpp, the
// reference's proj/include/dipole/bhtree.hpp:51-105 signatures) on the B200
// engine. Every method is a call through the C-ABI (include/dipole_b200.h);
// nothing here computes a dipole sum on the CPU.
//
// Mapping (reference method -> engine entry point, reference lines):
//   build            -> dpl_tree_build + dpl_tree_export        bhtree.cpp:158-169
//   update_moments   -> dpl_tree_update_moments                  :171-176
//   set_channel_kernels -> dpl_tree_set_channel_kernels          :178-182
//   primal / primal_channel / primal_with_gradient (one query)
//                    -> dpl_primal with gradients, one query      :188-334
//   adjoint (one query) -> queued, dpl_adjoint per batch          :345-417
//   make_buffer      -> dpl_gradbuf_create                       :336-343
//   flush_gradients  -> dpl_flush                                 :419-463
//   dump             -> dpl_tree_dump                             :465-494
// Per-query forward calls all run the engine's gradient kernel, so primal,
// primal_channel and primal_with_gradient values are bitwise equal to each
// other as the reference's tests require (test_bhtree.cpp:140,215-216).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <utility>

#include "dipole/bhtree.hpp"
#include "dipole_b200.h"

namespace dipole {
namespace b200 {

static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 must be three packed doubles");

namespace {

int g_device = -1;

int device_for_new_trees() {
  if (g_device >= 0) return g_device;
  const char* v = std::getenv("DPL_DEVICE");
  return v ? std::atoi(v) : 0;
}

[[noreturn]] void raise(int rc) {
  std::string msg = dpl_last_error();
  if (rc == DPL_ERR_DATA) throw DataError(msg);
  if (rc == DPL_ERR_NUMERICAL) throw NumericalError(msg);
  if (rc == DPL_ERR_USAGE) throw std::invalid_argument(msg);
  throw std::runtime_error("CUDA: " + msg);
}

inline void ck(int rc) {
  if (rc != DPL_OK) raise(rc);
}

dpl_kernel_params engine_params(const KernelParams& p) {
  dpl_kernel_params k{};
  k.epsilon = p.epsilon;
  k.desingularized = p.desingularized ? 1 : 0;
  k.desing_delta = p.desing_delta;
  k.coincident_value = p.coincident_value;
  return k;
}

bool same_params(const dpl_kernel_params& a, const dpl_kernel_params& b) {
  return a.epsilon == b.epsilon && a.desingularized == b.desingularized &&
         a.desing_delta == b.desing_delta && a.coincident_value == b.coincident_value;
}

constexpr std::size_t kQueueLimit = 1 << 16;  // queued adjoint queries per launch

}  // namespace

struct TreeState {
  dpl_tree_t h = nullptr;
  std::mutex mu;  // one engine handle = one host thread at a time
  bool built = false;
  std::size_t n = 0;
  int C = 1;
  int max_leaf = DipoleTree::kDefaultMaxLeafSize, max_depth = DipoleTree::kDefaultMaxDepth;
  std::vector<double> pos, nrm, area, mu_soa;  // the cloud as last built / updated
  std::vector<ChannelKernel> kinds;
  std::vector<TreeNode> nodes;
  std::vector<int> order;
  std::uint64_t generation = 0;  // bumps on build and channel-kernel changes

  explicit TreeState(int device) { ck(dpl_tree_create(device, nullptr, &h)); }
  ~TreeState() {
    if (h) dpl_tree_destroy(h);
  }

  void load_cloud(const OrientedPointCloud& cloud) {
    n = cloud.size();
    pos.resize(3 * n);
    nrm.resize(3 * n);
    area.resize(n);
    mu_soa.assign(n * static_cast<std::size_t>(C), 0.0);
    for (std::size_t i = 0; i < n; ++i) {  // refresh_point_data (bhtree.cpp:20-34)
      const OrientedPoint& p = cloud.points[i];
      for (int a = 0; a < 3; ++a) pos[3 * i + a] = p.position[a], nrm[3 * i + a] = p.normal[a];
      area[i] = p.area;
      mu_soa[i * C] = p.geometry_moment;
      const int k = std::min<int>(C - 1, static_cast<int>(p.appearance_moments.size()));
      for (int c = 1; c <= k; ++c) mu_soa[i * C + c] = p.appearance_moments[c - 1];
    }
  }

  void build_engine() {
    ck(dpl_tree_build(h, pos.data(), nrm.data(), area.data(), mu_soa.data(),
                      static_cast<int64_t>(n), C, max_leaf, max_depth));
    int64_t nn = 0;
    ck(dpl_tree_node_count(h, &nn));
    std::vector<double> geo(5 * nn);
    std::vector<int32_t> topo(6 * nn), ord(n);
    ck(dpl_tree_export(h, geo.data(), topo.data(), ord.data(), nullptr));
    nodes.assign(nn, TreeNode{});
    for (int64_t i = 0; i < nn; ++i) {
      TreeNode& nd = nodes[i];
      nd.centroid = Vec3(geo[5 * i], geo[5 * i + 1], geo[5 * i + 2]);
      nd.area = geo[5 * i + 3];
      nd.radius = geo[5 * i + 4];
      nd.begin = topo[6 * i], nd.end = topo[6 * i + 1];
      nd.child_begin = topo[6 * i + 2], nd.child_count = topo[6 * i + 3];
      nd.parent = topo[6 * i + 4];
      nd.leaf = topo[6 * i + 5] != 0;
    }
    order.assign(ord.begin(), ord.end());
    kinds.assign(C, ChannelKernel::Dipole);  // build resets the kernels (bhtree.cpp:165)
    built = true;
    ++generation;
  }

  void push_kinds() {
    std::vector<uint8_t> k(C);
    for (int c = 0; c < C; ++c) k[c] = kinds[c] == ChannelKernel::Radial ? DPL_RADIAL : DPL_DIPOLE;
    ck(dpl_tree_set_channel_kernels(h, k.data(), C));
  }

  void require_built() const {
    if (!built) throw std::logic_error("DipoleTree: not built");
  }
};

struct BufferState {
  std::shared_ptr<TreeState> tree;
  std::uint64_t generation = 0;
  dpl_gradbuf_t dev = nullptr;
  GradientBuffer* owner = nullptr;
  // queued per-query adjoints sharing one (params, beta)
  std::vector<double> q_xs;
  std::vector<float> q_dout, q_dgrad;
  bool q_grad = false;
  dpl_kernel_params q_kp{};
  double q_beta = 0;
  std::size_t q_n = 0;
  // host views of the device accumulators
  std::vector<Vec3> node_v, point_n;
  std::vector<double> node_s, point_mu;
  bool views_valid = false;
  bool device_zero = true;

  ~BufferState() {
    if (dev) dpl_gradbuf_destroy(dev);
  }

  void check_tree(const std::shared_ptr<TreeState>& t) const {
    if (tree != t || generation != t->generation)
      throw DataError("GradientBuffer: made by another tree, or before the tree was rebuilt");
  }

  void run_queue_locked() {  // tree->mu held
    if (!q_n) return;
    ck(dpl_adjoint(tree->h, &q_kp, q_beta, q_xs.data(), static_cast<int64_t>(q_n),
                   q_dout.data(), q_grad ? q_dgrad.data() : nullptr, dev));
    q_xs.clear(), q_dout.clear(), q_dgrad.clear();
    q_n = 0;
    q_grad = false;
    device_zero = false;
  }

  void materialize() {
    if (views_valid) return;
    std::lock_guard<std::mutex> lk(tree->mu);
    run_queue_locked();
    const std::size_t nn = tree->nodes.size(), n = tree->n, C = tree->C;
    node_v.assign(nn * C, Vec3::Zero());
    node_s.assign(nn * C, 0.0);
    point_mu.assign(n * C, 0.0);
    point_n.assign(n, Vec3::Zero());
    double de = 0.0;
    if (!device_zero)
      ck(dpl_gradbuf_export(dev, reinterpret_cast<double*>(node_v.data()), node_s.data(),
                            point_mu.data(), reinterpret_cast<double*>(point_n.data()), &de));
    if (owner) owner->d_epsilon = de;
    views_valid = true;
  }
};

template <typename T>
const std::vector<T>& DeviceMirror<T>::view() const {
  static const std::vector<T> empty;
  if (!owner_) return empty;
  owner_->materialize();
  const void* v = nullptr;
  switch (field_) {
    case 0: v = &owner_->node_v; break;
    case 1: v = &owner_->node_s; break;
    case 2: v = &owner_->point_mu; break;
    default: v = &owner_->point_n; break;
  }
  return *static_cast<const std::vector<T>*>(v);
}

template class DeviceMirror<Vec3>;
template class DeviceMirror<double>;

}  // namespace b200

using b200::BufferState;
using b200::ck;
using b200::TreeState;

// ---------------------------------------------------------------- GradientBuffer
GradientBuffer::GradientBuffer() = default;
GradientBuffer::~GradientBuffer() = default;

GradientBuffer::GradientBuffer(GradientBuffer&& o) noexcept
    : d_epsilon(o.d_epsilon), dirty(o.dirty), state_(std::move(o.state_)) {
  bind();
}

GradientBuffer& GradientBuffer::operator=(GradientBuffer&& o) noexcept {
  d_epsilon = o.d_epsilon;
  dirty = o.dirty;
  state_ = std::move(o.state_);
  bind();
  return *this;
}

void GradientBuffer::bind() {
  BufferState* s = state_.get();
  node_v.owner_ = node_s.owner_ = point_mu.owner_ = point_n.owner_ = nullptr;
  node_v.owner_ = s;
  node_s.owner_ = s;
  point_mu.owner_ = s;
  point_n.owner_ = s;
  if (s) s->owner = this;
}

void GradientBuffer::reset() {  // bhtree.cpp:11-18
  d_epsilon = 0.0;
  dirty = false;
  if (!state_) return;
  std::lock_guard<std::mutex> lk(state_->tree->mu);
  state_->q_xs.clear(), state_->q_dout.clear(), state_->q_dgrad.clear();
  state_->q_n = 0;
  ck(dpl_gradbuf_zero(state_->dev));
  state_->device_zero = true;
  state_->views_valid = false;
}

// ---------------------------------------------------------------- DipoleTree
DipoleTree::DipoleTree() : s_(std::make_shared<TreeState>(b200::device_for_new_trees())) {}
DipoleTree::~DipoleTree() = default;
DipoleTree::DipoleTree(DipoleTree&&) noexcept = default;
DipoleTree& DipoleTree::operator=(DipoleTree&&) noexcept = default;

DipoleTree::DipoleTree(const DipoleTree& o) : DipoleTree() { *this = o; }

DipoleTree& DipoleTree::operator=(const DipoleTree& o) {
  if (this == &o) return *this;
  auto s = std::make_shared<TreeState>(b200::device_for_new_trees());
  const TreeState& src = *o.s_;
  if (src.built) {
    s->C = src.C, s->max_leaf = src.max_leaf, s->max_depth = src.max_depth;
    s->pos = src.pos, s->nrm = src.nrm, s->area = src.area, s->mu_soa = src.mu_soa;
    s->n = src.n;
    s->build_engine();  // same cloud -> the same tree (deterministic build)
    s->kinds = src.kinds;
    s->push_kinds();
  }
  s_ = std::move(s);
  return *this;
}

void DipoleTree::set_device(int device) { b200::g_device = device; }

void DipoleTree::build(const OrientedPointCloud& cloud, int max_leaf_size, int max_depth) {
  if (cloud.empty()) throw DataError("DipoleTree::build: empty cloud");
  TreeState& s = *s_;
  std::lock_guard<std::mutex> lk(s.mu);
  s.C = 1 + cloud.k_appearance;
  s.max_leaf = std::max(1, max_leaf_size);
  s.max_depth = std::max(0, max_depth);
  s.load_cloud(cloud);
  s.build_engine();
}

void DipoleTree::update_moments(const OrientedPointCloud& cloud) {
  TreeState& s = *s_;
  s.require_built();
  if (cloud.size() != s.n || 1 + cloud.k_appearance != s.C)
    throw DataError("DipoleTree::update_moments: cloud/tree size mismatch");
  std::lock_guard<std::mutex> lk(s.mu);
  s.load_cloud(cloud);
  ck(dpl_tree_update_moments(s.h, s.pos.data(), s.nrm.data(), s.area.data(), s.mu_soa.data(),
                             static_cast<int64_t>(s.n), s.C));
}

void DipoleTree::set_channel_kernels(std::vector<ChannelKernel> kernels) {
  TreeState& s = *s_;
  if (static_cast<int>(kernels.size()) != s.C)
    throw DataError("DipoleTree::set_channel_kernels: channel count mismatch");
  std::lock_guard<std::mutex> lk(s.mu);
  s.kinds = std::move(kernels);
  if (s.built) {
    s.push_kinds();
    ++s.generation;  // device buffers are laid out by kernel kind
  }
}

const std::vector<ChannelKernel>& DipoleTree::channel_kernels() const { return s_->kinds; }
int DipoleTree::channels() const { return s_->C; }
std::size_t DipoleTree::point_count() const { return s_->n; }
const std::vector<TreeNode>& DipoleTree::nodes() const { return s_->nodes; }
const std::vector<int>& DipoleTree::point_order() const { return s_->order; }

void DipoleTree::dump(const std::string& path) const {
  s_->require_built();
  std::lock_guard<std::mutex> lk(s_->mu);
  ck(dpl_tree_dump(s_->h, path.c_str()));
}

// ---- single queries: one launch each, all through the gradient kernel
namespace {
struct OneQuery {
  std::vector<float> v, g;
  long visited = 0;
};

OneQuery run_one(TreeState& s, const Vec3& x, const KernelParams& params, double beta,
                 bool count) {
  s.require_built();
  OneQuery r;
  r.v.resize(s.C);
  r.g.resize(3 * static_cast<std::size_t>(s.C));
  const double xs[3] = {x[0], x[1], x[2]};
  const dpl_kernel_params kp = b200::engine_params(params);
  dpl_counters cnt{};
  std::lock_guard<std::mutex> lk(s.mu);
  ck(dpl_primal(s.h, &kp, beta, xs, 1, r.v.data(), r.g.data(), count ? &cnt : nullptr));
  r.visited = static_cast<long>(cnt.visited);
  return r;
}
}  // namespace

void DipoleTree::primal(const Vec3& x, const KernelParams& params, double beta_bh,
                        std::span<double> out, long* visited) const {
  OneQuery r = run_one(*s_, x, params, beta_bh, visited != nullptr);
  for (int c = 0; c < s_->C && c < static_cast<int>(out.size()); ++c) out[c] = r.v[c];
  if (visited) *visited = r.visited;
}

double DipoleTree::primal_channel(const Vec3& x, const KernelParams& params, double beta_bh,
                                  int channel, long* visited) const {
  if (channel < 0 || channel >= s_->C) throw std::out_of_range("primal_channel: channel");
  OneQuery r = run_one(*s_, x, params, beta_bh, visited != nullptr);
  if (visited) *visited = r.visited;
  return r.v[channel];
}

void DipoleTree::primal_with_gradient(const Vec3& x, const KernelParams& params, double beta_bh,
                                      std::span<double> out, std::span<Vec3> grad_out,
                                      long* visited) const {
  OneQuery r = run_one(*s_, x, params, beta_bh, visited != nullptr);
  for (int c = 0; c < s_->C; ++c) {
    if (c < static_cast<int>(out.size())) out[c] = r.v[c];
    if (c < static_cast<int>(grad_out.size()))
      grad_out[c] = Vec3(r.g[3 * c], r.g[3 * c + 1], r.g[3 * c + 2]);
  }
  if (visited) *visited = r.visited;
}

void DipoleTree::adjoint(const Vec3& x, const KernelParams& params, double beta_bh,
                         std::span<const double> d_out, std::span<const Vec3> d_grad,
                         GradientBuffer& buf) const {
  TreeState& s = *s_;
  s.require_built();
  if (!buf.state_) throw std::invalid_argument("adjoint: buffer not made by make_buffer()");
  BufferState& b = *buf.state_;
  b.check_tree(s_);
  const int C = s.C;
  const dpl_kernel_params kp = b200::engine_params(params);
  if (b.q_n && (!b200::same_params(kp, b.q_kp) || beta_bh != b.q_beta)) {
    std::lock_guard<std::mutex> lk(s.mu);
    b.run_queue_locked();
  }
  b.q_kp = kp;
  b.q_beta = beta_bh;
  b.q_xs.insert(b.q_xs.end(), {x[0], x[1], x[2]});
  for (int c = 0; c < C; ++c)
    b.q_dout.push_back(c < static_cast<int>(d_out.size()) ? static_cast<float>(d_out[c]) : 0.f);
  if (!d_grad.empty() && !b.q_grad) {  // the batch gains query gradients: earlier rows are 0
    b.q_grad = true;
    b.q_dgrad.assign(b.q_n * 3 * C, 0.f);
  }
  if (b.q_grad)
    for (int c = 0; c < C; ++c)
      for (int a = 0; a < 3; ++a)
        b.q_dgrad.push_back(c < static_cast<int>(d_grad.size()) ? static_cast<float>(d_grad[c][a])
                                                                  : 0.f);
  ++b.q_n;
  b.views_valid = false;
  buf.dirty = true;
  if (b.q_n >= b200::kQueueLimit) {
    std::lock_guard<std::mutex> lk(s.mu);
    b.run_queue_locked();
  }
}

GradientBuffer DipoleTree::make_buffer() const {
  TreeState& s = *s_;
  s.require_built();
  GradientBuffer buf;
  auto st = std::make_unique<BufferState>();
  st->tree = s_;
  st->generation = s.generation;
  {
    std::lock_guard<std::mutex> lk(s.mu);
    ck(dpl_gradbuf_create(s.h, &st->dev));
  }
  buf.state_ = std::move(st);
  buf.bind();
  return buf;
}

PointGradients DipoleTree::flush_gradients(std::span<GradientBuffer> buffers) const {
  TreeState& s = *s_;
  s.require_built();
  const std::size_t M = s.n;
  const int C = s.C;
  PointGradients out;
  out.channels = C;
  out.moments.assign(M * C, 0.0);
  out.normals.assign(M, Vec3::Zero());
  std::vector<dpl_gradbuf_t> devs;
  for (GradientBuffer& b : buffers) {
    if (!b.state_) continue;
    b.state_->check_tree(s_);
    devs.push_back(b.state_->dev);
  }
  if (!devs.empty()) {
    std::vector<float> mom(M * C), nrm(3 * M);
    double de = 0.0;
    std::lock_guard<std::mutex> lk(s.mu);
    for (GradientBuffer& b : buffers)
      if (b.state_) b.state_->run_queue_locked();
    ck(dpl_flush(s.h, devs.data(), static_cast<int32_t>(devs.size()), mom.data(), nrm.data(), &de));
    std::copy(mom.begin(), mom.end(), out.moments.begin());
    for (std::size_t m = 0; m < M; ++m) out.normals[m] = Vec3(nrm[3 * m], nrm[3 * m + 1], nrm[3 * m + 2]);
    out.d_epsilon = de;
  }
  for (GradientBuffer& b : buffers) {  // flush zeroes the buffers (bhtree.cpp:438)
    b.d_epsilon = 0.0;
    b.dirty = false;
    if (b.state_) b.state_->device_zero = true, b.state_->views_valid = false;
  }
  return out;
}

PointGradients DipoleTree::flush_gradients(GradientBuffer& buffer) const {
  return flush_gradients(std::span<GradientBuffer>(&buffer, 1));
}

// ---- batched overloads
void DipoleTree::primal(std::span<const Vec3> xs, const KernelParams& params, double beta_bh,
                        std::span<double> out, std::span<long> visited) const {
  TreeState& s = *s_;
  s.require_built();
  const std::size_t Q = xs.size(), C = s.C;
  if (out.size() < Q * C) throw std::invalid_argument("primal: out must hold Q x channels");
  std::vector<float> o(Q * C);
  std::vector<dpl_counters> cnt(visited.empty() ? 0 : Q);
  const dpl_kernel_params kp = b200::engine_params(params);
  {
    std::lock_guard<std::mutex> lk(s.mu);
    ck(dpl_primal(s.h, &kp, beta_bh, reinterpret_cast<const double*>(xs.data()),
                  static_cast<int64_t>(Q), o.data(), nullptr, cnt.empty() ? nullptr : cnt.data()));
  }
  std::copy(o.begin(), o.end(), out.begin());
  for (std::size_t i = 0; i < cnt.size() && i < visited.size(); ++i) visited[i] = cnt[i].visited;
}

void DipoleTree::primal_channel(std::span<const Vec3> xs, const KernelParams& params,
                                double beta_bh, int channel, std::span<double> out) const {
  TreeState& s = *s_;
  s.require_built();
  const std::size_t Q = xs.size();
  if (out.size() < Q) throw std::invalid_argument("primal_channel: out must hold Q values");
  std::vector<float> o(Q);
  const dpl_kernel_params kp = b200::engine_params(params);
  {
    std::lock_guard<std::mutex> lk(s.mu);
    ck(dpl_primal_channel(s.h, &kp, beta_bh, reinterpret_cast<const double*>(xs.data()),
                          static_cast<int64_t>(Q), channel, o.data()));
  }
  std::copy(o.begin(), o.end(), out.begin());
}

void DipoleTree::primal_with_gradient(std::span<const Vec3> xs, const KernelParams& params,
                                      double beta_bh, std::span<double> out,
                                      std::span<Vec3> grad_out) const {
  TreeState& s = *s_;
  s.require_built();
  const std::size_t Q = xs.size(), C = s.C;
  if (out.size() < Q * C || grad_out.size() < Q * C)
    throw std::invalid_argument("primal_with_gradient: out / grad_out must hold Q x channels");
  std::vector<float> o(Q * C), g(3 * Q * C);
  const dpl_kernel_params kp = b200::engine_params(params);
  {
    std::lock_guard<std::mutex> lk(s.mu);
    ck(dpl_primal(s.h, &kp, beta_bh, reinterpret_cast<const double*>(xs.data()),
                  static_cast<int64_t>(Q), o.data(), g.data(), nullptr));
  }
  std::copy(o.begin(), o.end(), out.begin());
  for (std::size_t i = 0; i < Q * C; ++i) grad_out[i] = Vec3(g[3 * i], g[3 * i + 1], g[3 * i + 2]);
}

void DipoleTree::adjoint(std::span<const Vec3> xs, const KernelParams& params, double beta_bh,
                         std::span<const double> d_out, std::span<const Vec3> d_grad,
                         GradientBuffer& buf) const {
  TreeState& s = *s_;
  s.require_built();
  if (!buf.state_) throw std::invalid_argument("adjoint: buffer not made by make_buffer()");
  BufferState& b = *buf.state_;
  b.check_tree(s_);
  const std::size_t Q = xs.size(), C = s.C;
  if (d_out.size() < Q * C || (!d_grad.empty() && d_grad.size() < Q * C))
    throw std::invalid_argument("adjoint: d_out / d_grad must hold Q x channels");
  std::vector<float> dout(d_out.begin(), d_out.begin() + Q * C);
  std::vector<float> dg;
  if (!d_grad.empty()) {
    dg.resize(3 * Q * C);
    for (std::size_t i = 0; i < Q * C; ++i)
      for (int a = 0; a < 3; ++a) dg[3 * i + a] = static_cast<float>(d_grad[i][a]);
  }
  const dpl_kernel_params kp = b200::engine_params(params);
  std::lock_guard<std::mutex> lk(s.mu);
  b.run_queue_locked();
  ck(dpl_adjoint(s.h, &kp, beta_bh, reinterpret_cast<const double*>(xs.data()),
                 static_cast<int64_t>(Q), dout.data(), dg.empty() ? nullptr : dg.data(), b.dev));
  b.device_zero = false;
  b.views_valid = false;
  buf.dirty = true;
}

}  // namespace dipole
