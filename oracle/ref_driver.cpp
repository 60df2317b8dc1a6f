// C-ABI driver around the UNMODIFIED reference library (test infrastructure).
//
// Built only into oracle/_ref/libdipole_ref.so together with the reference's
// own sources (oracle/Makefile, target `ref`). It is the "reference" arm of
// bench.py (--impl reference / cpu_baseline kind "reference") and the
// generator of the golden vectors under tests/golden/. Every entry point calls
// the reference's public API exactly as its own callers do:
//   * batched forward queries: parallel_for over DipoleTree::primal /
//     primal_channel / primal_with_gradient (proj/src/util.cpp:7-26,
//     proj/src/bhtree.cpp:188-334), workers = hardware_concurrency by default;
//   * adjoint: one GradientBuffer per worker (make_buffer, bhtree.cpp:336-343),
//     DipoleTree::adjoint per query (:345-417), then flush_gradients(span)
//     (:419-459) — the reference's own multi-worker contract (bhtree.hpp:38-40);
//   * render step: render_ray + render_ray_backward per ray
//     (proj/src/renderer.cpp:106-231) on a SceneModel prepared by
//     SceneModel::prepare (proj/src/fields.cpp:7-18).
// Nothing here is on the product path; the product never links this file.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "dipole/bhtree.hpp"
#include "dipole/fields.hpp"
#include "dipole/kernels.hpp"
#include "dipole/meshing.hpp"
#include "dipole/optimizer.hpp"
#include "dipole/oracles.hpp"
#include "dipole/renderer.hpp"

using namespace dipole;

namespace {

thread_local std::string g_err;

struct RefParams {  // mirrors dpl_kernel_params in include/dipole_b200.h
  double epsilon;
  int32_t desingularized;
  int32_t pad;
  double desing_delta;
  double coincident_value;
};

KernelParams to_kp(const RefParams* p) {
  KernelParams k;
  k.epsilon = p->epsilon;
  k.desingularized = p->desingularized != 0;
  k.desing_delta = p->desing_delta;
  k.coincident_value = p->coincident_value;
  return k;
}

OrientedPointCloud make_cloud(const double* pos, const double* nrm, const double* area,
                              const double* mu, int64_t n, int32_t C) {
  OrientedPointCloud cloud;
  cloud.k_appearance = C - 1;
  cloud.points.resize(n);
  for (int64_t i = 0; i < n; ++i) {
    OrientedPoint& p = cloud.points[i];
    p.position = Vec3(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]);
    p.normal = Vec3(nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2]);
    p.area = area[i];
    p.geometry_moment = mu[i * C];
    p.appearance_moments.assign(mu + i * C + 1, mu + i * C + C);
  }
  cloud.snapshot_initial_normals();
  return cloud;
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const DataError& e) {
    g_err = e.what();
    return 2;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // namespace

struct ref_tree {
  OrientedPointCloud cloud;
  DipoleTree tree;
};

struct ref_model {
  SceneModel model;
  std::vector<double> d_head_w;  // head weight gradient of the last ref_render_step
};

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_hardware_concurrency() { return default_workers(); }

int ref_kernel_coeffs(double r, const RefParams* p, int order, double* out7) {
  return guard([&] {
    RadialCoeffs k = kernel_coeffs(r, to_kp(p), order);
    double v[7] = {k.W, k.Wp_r, k.dW_de, k.dWp_r_de, k.R, k.Rp_r, k.dR_de};
    std::memcpy(out7, v, sizeof v);
  });
}

double ref_tau(double t) { return tau(t); }
double ref_erf_approx(double x) { return erf_approx(x); }
double ref_normal_hazard(double z) { return normal_hazard(z); }

double ref_mean_knn_spacing(const double* pos, int64_t n, int k) {
  OrientedPointCloud c;
  c.points.resize(n);
  for (int64_t i = 0; i < n; ++i) c.points[i].position = Vec3(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]);
  return c.mean_knn_spacing(k);
}

int ref_tree_build(const double* pos, const double* nrm, const double* area, const double* mu,
                   int64_t n, int32_t C, int32_t max_leaf, int32_t max_depth, ref_tree** out) {
  return guard([&] {
    auto t = std::make_unique<ref_tree>();
    t->cloud = make_cloud(pos, nrm, area, mu, n, C);
    t->tree.build(t->cloud, max_leaf, max_depth);
    *out = t.release();
  });
}

void ref_tree_free(ref_tree* t) { delete t; }

int ref_tree_set_kinds(ref_tree* t, const uint8_t* kinds, int32_t C) {
  return guard([&] {
    std::vector<ChannelKernel> k(C);
    for (int c = 0; c < C; ++c) k[c] = kinds[c] ? ChannelKernel::Radial : ChannelKernel::Dipole;
    t->tree.set_channel_kernels(std::move(k));
  });
}

int ref_tree_update_moments(ref_tree* t, const double* pos, const double* nrm, const double* area,
                            const double* mu, int64_t n, int32_t C) {
  return guard([&] {
    t->cloud = make_cloud(pos, nrm, area, mu, n, C);
    t->tree.update_moments(t->cloud);
  });
}

int64_t ref_tree_node_count(const ref_tree* t) { return (int64_t)t->tree.nodes().size(); }

// geo: nodes x 5 (cx, cy, cz, area, radius); topo: nodes x 6 (begin, end,
// child_begin, child_count, parent, leaf); order: N
void ref_tree_export(const ref_tree* t, double* geo, int32_t* topo, int32_t* order) {
  const auto& nodes = t->tree.nodes();
  for (size_t i = 0; i < nodes.size(); ++i) {
    const TreeNode& nd = nodes[i];
    double g[5] = {nd.centroid.x(), nd.centroid.y(), nd.centroid.z(), nd.area, nd.radius};
    std::memcpy(geo + 5 * i, g, sizeof g);
    int32_t s[6] = {nd.begin, nd.end, nd.child_begin, nd.child_count, nd.parent, nd.leaf ? 1 : 0};
    std::memcpy(topo + 6 * i, s, sizeof s);
  }
  const auto& po = t->tree.point_order();
  for (size_t i = 0; i < po.size(); ++i) order[i] = po[i];
}

int ref_tree_dump(const ref_tree* t, const char* path) {
  return guard([&] { t->tree.dump(path); });
}

// mode 0: primal (out Q x C); mode 1: primal_with_gradient (out Q x C, grad Q x C x 3);
// mode 2: primal_channel(channel) (out Q)
int ref_primal(const ref_tree* t, const RefParams* p, double beta, const double* xs, int64_t q,
               int mode, int channel, double* out, double* grad, int64_t* visited, int workers) {
  return guard([&] {
    KernelParams kp = to_kp(p);
    const int C = t->tree.channels();
    parallel_for(
        q,
        [&](int64_t lo, int64_t hi, int) {
          std::vector<double> o(C);
          std::vector<Vec3> g(C);
          for (int64_t i = lo; i < hi; ++i) {
            Vec3 x(xs[3 * i], xs[3 * i + 1], xs[3 * i + 2]);
            long v = 0;
            long* vp = visited ? &v : nullptr;
            if (mode == 2) {
              out[i] = t->tree.primal_channel(x, kp, beta, channel, vp);
            } else if (mode == 1) {
              t->tree.primal_with_gradient(x, kp, beta, o, g, vp);
              for (int c = 0; c < C; ++c) {
                out[i * C + c] = o[c];
                for (int a = 0; a < 3; ++a) grad[(i * C + c) * 3 + a] = g[c][a];
              }
            } else {
              t->tree.primal(x, kp, beta, o, vp);
              for (int c = 0; c < C; ++c) out[i * C + c] = o[c];
            }
            if (visited) visited[i] = v;
          }
        },
        workers);
  });
}

// Adjoint of a query batch: per-worker buffers, then one flush. d_grad may be
// NULL (no query-gradient adjoints). Outputs: moments N x C, normals N x 3, d_eps.
int ref_adjoint(const ref_tree* t, const RefParams* p, double beta, const double* xs, int64_t q,
                const double* d_out, const double* d_grad, int workers, double* moments,
                double* normals, double* d_eps) {
  return guard([&] {
    KernelParams kp = to_kp(p);
    const int C = t->tree.channels();
    if (workers <= 0) workers = default_workers();
    workers = (int)std::max<int64_t>(1, std::min<int64_t>(workers, q));
    std::vector<GradientBuffer> bufs;
    for (int w = 0; w < workers; ++w) bufs.push_back(t->tree.make_buffer());
    parallel_for(
        q,
        [&](int64_t lo, int64_t hi, int w) {
          std::vector<Vec3> dg;
          for (int64_t i = lo; i < hi; ++i) {
            Vec3 x(xs[3 * i], xs[3 * i + 1], xs[3 * i + 2]);
            std::span<const double> dout(d_out + i * C, C);
            if (d_grad) {
              dg.resize(C);
              for (int c = 0; c < C; ++c)
                dg[c] = Vec3(d_grad[(i * C + c) * 3], d_grad[(i * C + c) * 3 + 1],
                             d_grad[(i * C + c) * 3 + 2]);
              t->tree.adjoint(x, kp, beta, dout, dg, bufs[w]);
            } else {
              t->tree.adjoint(x, kp, beta, dout, {}, bufs[w]);
            }
          }
        },
        workers);
    PointGradients pg = t->tree.flush_gradients(bufs);
    std::memcpy(moments, pg.moments.data(), pg.moments.size() * sizeof(double));
    for (size_t m = 0; m < pg.normals.size(); ++m)
      for (int a = 0; a < 3; ++a) normals[3 * m + a] = pg.normals[m][a];
    *d_eps = pg.d_epsilon;
  });
}

// The same adjoint with caller-held buffers, so a benchmark can time the
// per-query traversal and the (per-step, query-count independent) buffer
// setup + flush_gradients separately: ref_bufs_create = make_buffer per worker
// (bhtree.cpp:336-343), ref_adjoint_into = parallel_for over DipoleTree::adjoint
// into bufs[w] (:345-417), ref_bufs_flush = flush_gradients(span) (:419-459).
struct ref_bufs {
  std::vector<GradientBuffer> b;
};

int ref_bufs_create(const ref_tree* t, int workers, ref_bufs** out) {
  return guard([&] {
    auto r = std::make_unique<ref_bufs>();
    for (int w = 0; w < std::max(1, workers); ++w) r->b.push_back(t->tree.make_buffer());
    *out = r.release();
  });
}

void ref_bufs_free(ref_bufs* b) { delete b; }

int ref_adjoint_into(const ref_tree* t, const RefParams* p, double beta, const double* xs,
                     int64_t q, const double* d_out, ref_bufs* bufs) {
  return guard([&] {
    KernelParams kp = to_kp(p);
    const int C = t->tree.channels();
    const int workers = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)bufs->b.size(), q));
    parallel_for(
        q,
        [&](int64_t lo, int64_t hi, int w) {
          for (int64_t i = lo; i < hi; ++i) {
            Vec3 x(xs[3 * i], xs[3 * i + 1], xs[3 * i + 2]);
            t->tree.adjoint(x, kp, beta, std::span<const double>(d_out + i * C, C), {},
                            bufs->b[w]);
          }
        },
        workers);
  });
}

int ref_bufs_flush(const ref_tree* t, ref_bufs* bufs, double* moments, double* normals,
                   double* d_eps) {
  return guard([&] {
    PointGradients pg = t->tree.flush_gradients(bufs->b);
    if (moments) std::memcpy(moments, pg.moments.data(), pg.moments.size() * sizeof(double));
    if (normals)
      for (size_t m = 0; m < pg.normals.size(); ++m)
        for (int a = 0; a < 3; ++a) normals[3 * m + a] = pg.normals[m][a];
    if (d_eps) *d_eps = pg.d_epsilon;
  });
}

// Exact O(NQ) naive oracles (proj/src/oracles.cpp:23-59).
int ref_naive_sum(const ref_tree* t, const RefParams* p, const double* xs, int64_t q, int channel,
                  int kind, int with_grad, double* out, double* grad, int workers) {
  return guard([&] {
    KernelParams kp = to_kp(p);
    ChannelKernel k = kind ? ChannelKernel::Radial : ChannelKernel::Dipole;
    parallel_for(
        q,
        [&](int64_t lo, int64_t hi, int) {
          for (int64_t i = lo; i < hi; ++i) {
            Vec3 x(xs[3 * i], xs[3 * i + 1], xs[3 * i + 2]);
            out[i] = naive_dipole_sum(t->cloud, x, kp, channel, k);
            if (with_grad) {
              Vec3 g = naive_dipole_gradient(t->cloud, x, kp, channel, k);
              for (int a = 0; a < 3; ++a) grad[3 * i + a] = g[a];
            }
          }
        },
        workers);
  });
}

int ref_naive_adjoint(const ref_tree* t, const RefParams* p, const double* xs, int64_t q,
                      const double* d_out, const double* d_grad, const uint8_t* kinds,
                      double* moments, double* normals, double* d_eps) {
  return guard([&] {
    const int C = t->tree.channels();
    std::vector<AdjointQuerySpec> specs(q);
    for (int64_t i = 0; i < q; ++i) {
      specs[i].x = Vec3(xs[3 * i], xs[3 * i + 1], xs[3 * i + 2]);
      specs[i].d_out.assign(d_out + i * C, d_out + i * C + C);
      if (d_grad) {
        specs[i].d_grad.resize(C);
        for (int c = 0; c < C; ++c)
          specs[i].d_grad[c] = Vec3(d_grad[(i * C + c) * 3], d_grad[(i * C + c) * 3 + 1],
                                    d_grad[(i * C + c) * 3 + 2]);
      }
    }
    std::vector<ChannelKernel> k(C);
    for (int c = 0; c < C; ++c) k[c] = kinds[c] ? ChannelKernel::Radial : ChannelKernel::Dipole;
    PointGradients pg = naive_adjoint(t->cloud, specs, to_kp(p), k);
    std::memcpy(moments, pg.moments.data(), pg.moments.size() * sizeof(double));
    for (size_t m = 0; m < pg.normals.size(); ++m)
      for (int a = 0; a < 3; ++a) normals[3 * m + a] = pg.normals[m][a];
    *d_eps = pg.d_epsilon;
  });
}

// ---- render step (configs 3 / 5) -------------------------------------------
// A SceneModel as SceneModel::prepare builds it: channel 0 Dipole, 1..K
// Radial, direct-rgb head (the reference default, scene.hpp:59).
int ref_model_create(const double* pos, const double* nrm, const double* area, const double* mu,
                     int64_t n, int32_t C, double epsilon, double lambda, double beta,
                     const double* background, ref_model** out) {
  return guard([&] {
    auto m = std::make_unique<ref_model>();
    m->model.cloud = make_cloud(pos, nrm, area, mu, n, C);
    m->model.kernel.epsilon = epsilon;
    m->model.lambda_scale = lambda;
    m->model.beta_bh = beta;
    m->model.background = Vec3(background[0], background[1], background[2]);
    m->model.head.variant = HeadVariant::DirectRgb;
    m->model.prepare();
    *out = m.release();
  });
}

void ref_model_free(ref_model* m) { delete m; }

// ---- DPCK checkpoint (optimizer.cpp:330-356) ---------------------------------
int ref_model_save_checkpoint(ref_model* m, int32_t iter, const char* path) {
  return guard([&] { save_checkpoint(m->model, iter, path); });
}

// ---- query generators ----------------------------------------
// sample_grid (meshing.cpp:33-59) on the model: values (r2 x r1 x r0), box used
int ref_sample_grid(ref_model* m, const int32_t* res, const double* lo, const double* hi,
                    int workers, double* values, double* lo_out, double* hi_out) {
  return guard([&] {
    FieldGrid g = sample_grid(m->model, {res[0], res[1], res[2]}, Vec3(lo[0], lo[1], lo[2]),
                              Vec3(hi[0], hi[1], hi[2]), workers > 0 ? workers : default_workers());
    std::memcpy(values, g.values.data(), g.values.size() * sizeof(double));
    for (int a = 0; a < 3; ++a) lo_out[a] = g.lo[a], hi_out[a] = g.hi[a];
  });
}

// sample_ray (renderer.cpp:46-86) per ray; t / delta R x max_s
int ref_sample_rays(ref_model* m, const double* rays, int64_t R, double t_near, double t_far,
                    const int32_t* counts5, int32_t max_s, double* t, double* delta,
                    int32_t* count, uint8_t* bracketed) {
  return guard([&] {
    RenderConfig cfg;
    cfg.t_near = t_near;
    cfg.t_far = t_far;
    cfg.probe_count = counts5[0];
    cfg.sparse_before = counts5[1];
    cfg.dense_at = counts5[2];
    cfg.sparse_after = counts5[3];
    cfg.uniform_count = counts5[4];
    parallel_for(
        R,
        [&](std::int64_t r0, std::int64_t r1, int) {
          for (std::int64_t r = r0; r < r1; ++r) {
            Ray ray;
            ray.origin = Vec3(rays[6 * r], rays[6 * r + 1], rays[6 * r + 2]);
            ray.dir = Vec3(rays[6 * r + 3], rays[6 * r + 4], rays[6 * r + 5]);
            RaySamples s = sample_ray(m->model, ray, cfg);
            if ((int)s.t.size() > max_s) throw DataError("ref_sample_rays: max_s too small");
            for (std::size_t j = 0; j < s.t.size(); ++j)
              t[r * max_s + j] = s.t[j], delta[r * max_s + j] = s.delta[j];
            count[r] = (int32_t)s.t.size();
            bracketed[r] = s.bracketed ? 1 : 0;
          }
        },
        default_workers());
  });
}

double ref_model_epsilon(const ref_model* m) { return m->model.kernel.epsilon; }

// Forward + backward of a ray batch: per ray render_ray (tape) then
// render_ray_backward with d_rgb = d_rgb_scale * (rgb - target) — the L2 loss
// gradient supplied by the harness — into per-worker buffers, then flush.
// samples: t (R x S) and delta (R x S). Outputs rgb (R x 3), flushed
// moments (N x C), normals (N x 3), d_eps, d_lambda, d_bg (3).
int ref_render_step(ref_model* mm, const double* rays, const double* ts, const double* deltas,
                    int64_t R, int32_t S, const double* target, double d_rgb_scale, int workers,
                    double* rgb, double* moments, double* normals, double* d_eps,
                    double* d_lambda, double* d_bg) {
  return guard([&] {
    SceneModel& model = mm->model;
    if (workers <= 0) workers = default_workers();
    workers = (int)std::max<int64_t>(1, std::min<int64_t>(workers, R));
    std::vector<GradientBuffer> bufs;
    std::vector<RenderGrads> rgs(workers);
    for (int w = 0; w < workers; ++w) {
      bufs.push_back(model.tree.make_buffer());
      rgs[w].resize_for(model.head);
    }
    parallel_for(
        R,
        [&](int64_t lo, int64_t hi, int w) {
          RayTape tape;
          for (int64_t i = lo; i < hi; ++i) {
            Ray ray;
            ray.origin = Vec3(rays[6 * i], rays[6 * i + 1], rays[6 * i + 2]);
            ray.dir = Vec3(rays[6 * i + 3], rays[6 * i + 4], rays[6 * i + 5]);
            RaySamples smp;
            smp.t.assign(ts + i * S, ts + i * S + S);
            smp.delta.assign(deltas + i * S, deltas + i * S + S);
            RayResult res = render_ray(model, ray, smp, {}, &tape, 0);
            for (int a = 0; a < 3; ++a) rgb[3 * i + a] = res.rgb[a];
            Vec3 d_rgb = d_rgb_scale * (res.rgb - Vec3(target[3 * i], target[3 * i + 1],
                                                        target[3 * i + 2]));
            render_ray_backward(model, tape, d_rgb, {}, bufs[w], rgs[w]);
          }
        },
        workers);
    PointGradients pg = model.tree.flush_gradients(bufs);
    std::memcpy(moments, pg.moments.data(), pg.moments.size() * sizeof(double));
    for (size_t m = 0; m < pg.normals.size(); ++m)
      for (int a = 0; a < 3; ++a) normals[3 * m + a] = pg.normals[m][a];
    *d_eps = pg.d_epsilon;
    double dl = 0;
    Vec3 db = Vec3::Zero();
    for (auto& g : rgs) {
      dl += g.d_lambda;
      db += g.d_background;
    }
    *d_lambda = dl;
    for (int a = 0; a < 3; ++a) d_bg[a] = db[a];
    mm->d_head_w.assign(model.head.mlp.w.size(), 0.0);
    for (auto& g : rgs)
      for (size_t k = 0; k < g.d_head_w.size() && k < mm->d_head_w.size(); ++k)
        mm->d_head_w[k] += g.d_head_w[k];
  });
}

// tiny-MLP radiance head (radiance.hpp: RadianceHead, HeadVariant::TinyMlp)
// with the caller's weights (layer-major rows x cols then bias, radiance.cpp:44-57)
int ref_model_set_mlp_head(ref_model* mm, const int32_t* sizes, int32_t n_sizes, const double* w,
                           int64_t n_w) {
  return guard([&] {
    RadianceHead& h = mm->model.head;
    h.variant = HeadVariant::TinyMlp;
    h.k_appearance = mm->model.cloud.k_appearance;
    h.mlp.sizes.assign(sizes, sizes + n_sizes);
    h.mlp.w.assign(w, w + n_w);
    if (h.mlp.sizes.front() != h.mlp_input_dim() || h.mlp.sizes.back() != h.output_dim())
      throw DataError("ref_model_set_mlp_head: layer sizes do not match the head");
  });
}

int ref_model_head_grads(const ref_model* mm, double* out) {
  return guard([&] { std::memcpy(out, mm->d_head_w.data(), mm->d_head_w.size() * sizeof(double)); });
}

// Adam::step (proj/src/optimizer.cpp:65-81) on a flat parameter group.
struct ref_adam {
  Adam adam;
};
ref_adam* ref_adam_create() { return new ref_adam(); }
void ref_adam_free(ref_adam* a) { delete a; }
int ref_adam_step(ref_adam* a, double* params, const double* grads, int64_t n, double lr) {
  return guard([&] {
    a->adam.step(std::span<double>(params, n), std::span<const double>(grads, n), lr);
  });
}

}  // extern "C"
