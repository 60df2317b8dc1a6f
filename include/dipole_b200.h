/* dipole_b200.h — C-ABI of the B200-native Barnes-Hut dipole-sum engine.
 *
 * This is the drop-in boundary for the reference's hot path
 * (`dipole::DipoleTree`, proj/include/dipole/bhtree.hpp:51-130, and the render
 * step proj/include/dipole/renderer.hpp:86-106). The reference is a C++20
 * library with no FFI; a maintainer swapping the CPU tree for this engine binds
 * these symbols from C++ (include/dipole_b200.hpp re-exposes the reference
 * class API on top of them) or from Python via ctypes.
 *
 * Conventions
 *  - Every function returns an int status: 0 ok, 1 usage, 2 data
 *    (reference DataError, util.hpp:35), 3 numerical (NumericalError), 4 CUDA.
 *    dpl_last_error() returns the message of the calling thread's last failure.
 *  - Array arguments may be HOST or DEVICE pointers (detected per call with
 *    cudaPointerGetAttributes). Host arrays are staged through the handle's
 *    stream; device arrays are used in place. Results are complete when the
 *    call returns for host outputs; device outputs are ordered on the handle's
 *    stream (dpl_tree_sync() waits).
 *  - A handle is not thread-safe (as the reference: build / update_moments /
 *    flush need exclusive access). One handle = one GPU + stream.
 *  - Layouts are row-major: positions N x 3, moments N x C with channel 0 the
 *    geometry moment and 1..C-1 the appearance moments (bhtree.cpp:31-32).
 *  - There is no CPU fallback: every entry point runs sm_100a kernels.
 */
#ifndef DIPOLE_B200_H_
#define DIPOLE_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DPL_OK 0
#define DPL_ERR_USAGE 1
#define DPL_ERR_DATA 2
#define DPL_ERR_NUMERICAL 3
#define DPL_ERR_CUDA 4

/* ChannelKernel (bhtree.hpp:13) */
#define DPL_DIPOLE 0
#define DPL_RADIAL 1

typedef struct dpl_tree_s* dpl_tree_t;
typedef struct dpl_gradbuf_s* dpl_gradbuf_t;
typedef struct dpl_tape_s* dpl_tape_t;

/* KernelParams (kernels.hpp:24-29); epsilon <= 0 selects the singular kernel */
typedef struct {
  double epsilon;
  int32_t desingularized;
  int32_t reserved;
  double desing_delta;
  double coincident_value;
} dpl_kernel_params;

/* Counters of one query, replaying the reference's decisions (visited is
 * bhtree.cpp:201): nodes popped, far-field accepts (area > 0) with t < 6.5 and
 * t >= 6.5, leaf-point interactions with t < 6.5 and t >= 6.5. */
typedef struct {
  int64_t visited, far_near, far_far, pt_near, pt_far;
} dpl_counters;

const char* dpl_last_error(void);
int dpl_version(void);
/* Number of kernel launches this process has issued through the library. */
int64_t dpl_launch_count(void);

/* ---- tree lifecycle: DipoleTree::build / update_moments / set_channel_kernels */
/* stream: a cudaStream_t, or NULL for a library-owned BLOCKING stream
 * (cudaStreamDefault flags): it orders against the legacy default stream, so
 * device arrays produced there (e.g. by torch) are complete before the tree's
 * kernels read them. */
int dpl_tree_create(int device, void* stream, dpl_tree_t* out);
int dpl_tree_destroy(dpl_tree_t tree);
int dpl_tree_set_stream(dpl_tree_t tree, void* stream);
int dpl_tree_sync(dpl_tree_t tree);
/* Host-async mode (default off). When on, dpl_primal / dpl_primal_channel /
 * dpl_adjoint calls on large HOST batches return as soon as their work is
 * queued: inputs are copied host->device on a copy stream (the next call's
 * H2D overlaps the current kernels) and host outputs device->host on a second
 * copy stream. Host inputs must stay unchanged and host outputs unread until
 * dpl_tree_sync() or dpl_flush() (which synchronizes everything) returns; use
 * pinned host memory for real overlap. Off: every call is synchronous. */
int dpl_tree_set_host_async(dpl_tree_t tree, int on);
/* Host-async mode: start uploading the NEXT primal's host query batch now (on
 * the H2D copy stream, e.g. while the current adjoint runs); the next
 * dpl_primal / dpl_primal_channel / dpl_primal_grad0 given the same host
 * pointer and count uses it instead of uploading. The batch must stay
 * unchanged until that call. No-op outside host-async mode. */
int dpl_tree_prefetch(dpl_tree_t tree, const double* xs, int64_t q);

/* DipoleTree::build (bhtree.cpp:158-169): GPU Morton-digit sort + level-by-level
 * BFS numbering reproduces build_structure (:36-105) bit-exactly; geometry
 * (:107-134) and moments (:136-156) follow. Channel kernels reset to Dipole.
 * max_depth <= 42 (the reference's default is 20, bhtree.hpp:54); a deeper
 * request returns DPL_ERR_USAGE. */
int dpl_tree_build(dpl_tree_t tree, const double* pos, const double* nrm, const double* area,
                   const double* mu, int64_t n, int32_t channels, int32_t max_leaf_size,
                   int32_t max_depth);
/* DipoleTree::update_moments (bhtree.cpp:171-176): refreshes point data
 * (positions too, as refresh_point_data does) and node moments. */
int dpl_tree_update_moments(dpl_tree_t tree, const double* pos, const double* nrm,
                            const double* area, const double* mu, int64_t n, int32_t channels);
/* DipoleTree::set_channel_kernels (bhtree.cpp:178-182); kinds[c] in {DPL_DIPOLE, DPL_RADIAL}. */
int dpl_tree_set_channel_kernels(dpl_tree_t tree, const uint8_t* kinds, int32_t channels);

int dpl_tree_channels(dpl_tree_t tree, int32_t* channels);
int dpl_tree_point_count(dpl_tree_t tree, int64_t* n);
int dpl_tree_node_count(dpl_tree_t tree, int64_t* nodes);
/* nodes() / point_order() / point_leaf (bhtree.hpp:69-70,119): geo nodes x 5
 * (cx, cy, cz, area, radius), topo nodes x 6 (begin, end, child_begin,
 * child_count, parent, leaf), order N, leaf_of N. Any pointer may be NULL. */
int dpl_tree_export(dpl_tree_t tree, double* geo, int32_t* topo, int32_t* point_order,
                    int32_t* point_leaf);
/* Node moments (moments_v_ nodes x C x 3, moments_s_ nodes x C), fp32 as stored. */
int dpl_tree_export_moments(dpl_tree_t tree, float* moments_v, float* moments_s);
/* DipoleTree::dump "DPLT" v1 byte format (bhtree.cpp:465-494). */
int dpl_tree_dump(dpl_tree_t tree, const char* path);

/* ---- DPCK checkpoints (optimizer.cpp:294-388) -------------- */
typedef struct {
  int32_t iter;
  int32_t head_variant; /* 0 direct-rgb, 1 tiny-mlp (HeadVariant, radiance.hpp) */
  int32_t with_albedo;
  int32_t reserved;
  double lambda_scale, epsilon, background[3], beta_bh;
} dpl_checkpoint_meta;
/* save_checkpoint (:330-356): the tree's current cloud (positions, normals,
 * areas, moments as last built / updated), the initial normals (N x 3; NULL =
 * the current normals), the head's MLP (n_sizes = 0 for direct-rgb) and the
 * scalars. Byte-identical to the reference's file for the same model. */
int dpl_checkpoint_save(dpl_tree_t tree, const char* path, const dpl_checkpoint_meta* meta,
                        const double* initial_normals, const int32_t* mlp_sizes, int32_t n_sizes,
                        const double* mlp_w, int64_t n_w);
/* load_checkpoint (:358-388), host side. Call with NULL arrays to read the
 * counts (n, k_appearance, n_sizes, n_w), then with buffers: pos / nrm /
 * initial_normals n x 3, area n, mu n x (1 + k_appearance), sizes, w.
 * DataError on a bad magic / version / truncated file. */
int dpl_checkpoint_read(const char* path, dpl_checkpoint_meta* meta, int64_t* n,
                        int32_t* k_appearance, int32_t* n_sizes, int64_t* n_w, double* pos,
                        double* nrm, double* area, double* mu, double* initial_normals,
                        int32_t* sizes, double* w);

/* ---- forward queries -------------------------------------------------------
 * DipoleTree::primal / primal_with_gradient (bhtree.cpp:188-234,276-334) for a
 * batch of q query points xs (q x 3, fp64 like Vec3). out: q x C fp32.
 * grad: NULL (values only) or q x C x 3. counters: NULL or q records.
 * Opening decisions are evaluated in fp64 exactly as the reference does
 * (d = centroid - x; (dx*dx + dy*dy) + dz*dz > (beta^2 * r) * r), so the
 * far-field/leaf sets match the reference's; interaction arithmetic is fp32. */
int dpl_primal(dpl_tree_t tree, const dpl_kernel_params* params, double beta_bh,
               const double* xs, int64_t q, float* out, float* grad, dpl_counters* counters);
/* DipoleTree::primal_channel (bhtree.cpp:236-274): one channel, out q. */
int dpl_primal_channel(dpl_tree_t tree, const dpl_kernel_params* params, double beta_bh,
                       const double* xs, int64_t q, int32_t channel, float* out);
/* Same as dpl_primal but only the gradient of the FIRST channel is produced
 * (grad0: q x 3); this is what the render step consumes (renderer.cpp:125-127). */
int dpl_primal_grad0(dpl_tree_t tree, const dpl_kernel_params* params, double beta_bh,
                     const double* xs, int64_t q, float* out, float* grad0);

/* ---- query generators -------------------------------------- */
/* sample_grid (meshing.cpp:33-59) with geometry_field(x) = 0.5 -
 * primal_channel(x, 0) (fields.cpp:27-29): res[3] >= 2 per axis (DataError
 * otherwise); node (i, j, k) = lo + (i/(r0-1), j/(r1-1), k/(r2-1)) * (hi - lo)
 * in fp64 (FieldGrid::node, :25-30); values[(k * r1 + j) * r0 + i]. When
 * |hi - lo| == 0 the box is the cloud's bounding box padded by 5%; lo_out /
 * hi_out (may be NULL) receive the box used. */
int dpl_sample_grid(dpl_tree_t tree, const dpl_kernel_params* params, double beta_bh,
                    const int32_t* res, const double* lo, const double* hi, float* values,
                    double* lo_out, double* hi_out);

/* The sampler fields of RenderConfig (renderer.hpp:33-41). */
typedef struct {
  double t_near, t_far;
  int32_t probe_count, sparse_before, dense_at, sparse_after, uniform_count, reserved;
} dpl_ray_sampler;

/* sample_ray (renderer.cpp:46-86) for R rays (origin xyz, dir xyz: R x 6 fp64):
 * value-only probes f = 0.5 - primal_channel(o + t dir, 0) at t_near + span i /
 * (n - 1), the first sign change brackets the surface, then sparse / dense /
 * sparse samples around it (or uniform samples). Outputs per ray: t and delta
 * (R x max_samples, first count[r] valid, ascending), count, bracketed.
 * DataError when t_near >= t_far. */
int dpl_sample_rays(dpl_tree_t tree, const dpl_kernel_params* params, double beta_bh,
                    const double* rays, int64_t R, const dpl_ray_sampler* cfg, int32_t max_samples,
                    double* t, double* delta, int32_t* count, uint8_t* bracketed);

/* ---- adjoint (two-stage) ---------------------------------------------------
 * GradientBuffer (bhtree.hpp:40-49): device fp64 accumulators node_v, node_s,
 * point_mu, point_n, d_epsilon. */
int dpl_gradbuf_create(dpl_tree_t tree, dpl_gradbuf_t* out);
int dpl_gradbuf_destroy(dpl_gradbuf_t buf);
int dpl_gradbuf_zero(dpl_gradbuf_t buf);
/* The accumulators of a buffer in the reference's GradientBuffer layout
 * (bhtree.hpp:40-49): node_v nodes x C x 3, node_s nodes x C (a channel of the
 * other kind reads 0), point_mu N x C and point_n N x 3 in cloud order,
 * d_epsilon. Any pointer may be NULL. Synchronous (host outputs). */
int dpl_gradbuf_export(dpl_gradbuf_t buf, double* node_v, double* node_s, double* point_mu,
                       double* point_n, double* d_epsilon);
/* DipoleTree::adjoint (bhtree.cpp:345-417) for q queries: d_out q x C,
 * d_grad NULL or q x C x 3 (radial channels ignore d_grad, as the reference).
 * Warp-aggregated accumulation into node / leaf-point buffers; no per-point
 * ancestor walk here. xs == NULL reuses the queries of the immediately
 * preceding dpl_primal on this handle (same q; its device copy, so a host
 * batch crosses PCIe once per primal -> adjoint pair); usage error otherwise. */
int dpl_adjoint(dpl_tree_t tree, const dpl_kernel_params* params, double beta_bh,
                const double* xs, int64_t q, const float* d_out, const float* d_grad,
                dpl_gradbuf_t buf);
/* DipoleTree::flush_gradients (bhtree.cpp:419-463): sums nbuf buffers, pushes
 * node accumulators down to points (top-down, O(nodes*C + N*C)), zeroes the
 * buffers. moments N x C, normals N x 3 (fp32, any may be NULL), d_epsilon.
 * Host-async mode with host outputs: d_epsilon is returned at once, the
 * moments / normals arrive on the D2H copy stream while later calls run and
 * are complete after dpl_tree_sync (otherwise: complete on return). */
int dpl_flush(dpl_tree_t tree, dpl_gradbuf_t* bufs, int32_t nbuf, float* moments,
              float* normals, double* d_epsilon);

/* flush_gradients split for a cross-rank sum: every rank holds
 * the bit-identical tree, so per-point gradients in TREE order line up across
 * ranks and can be all-reduced chunk by chunk while later chunks are computed.
 *  - dpl_flush_begin: sums the buffers into bufs[0], node push-down, returns
 *    this rank's d_epsilon;
 *  - dpl_flush_rows: rows (hi - lo) x (C + 3) fp32, DEVICE memory, for the
 *    sorted points [lo, hi): [d moments (C) | d normal (3)] of point_order[j]
 *    (stream-ordered on the handle's stream, returns without waiting);
 *  - dpl_flush_end: rows N x (C + 3) (device, summed over ranks by the caller)
 *    -> moments N x C / normals N x 3 in the original order; zeroes the
 *    buffers (reset(), bhtree.cpp:438).
 * With one rank the three calls give exactly dpl_flush's results. */
int dpl_flush_begin(dpl_tree_t tree, dpl_gradbuf_t* bufs, int32_t nbuf, double* d_epsilon);
int dpl_flush_rows(dpl_tree_t tree, dpl_gradbuf_t buf0, int64_t lo, int64_t hi, float* rows);
int dpl_flush_end(dpl_tree_t tree, dpl_gradbuf_t* bufs, int32_t nbuf, const float* rows,
                  float* moments, float* normals);

/* ---- render step (renderer.cpp:106-231) ------------------------------------
 * Rays are (origin, dir) fp64 (R x 6). Samples per ray: S; when ts is NULL the
 * stratified sampler t_j = t_near + (t_far - t_near) * ((j + u_j) / S) with
 * u_j = dpl_uniform(seed, ray * S + j) is used (identical bits in the oracle);
 * otherwise ts / deltas are R x S fp64 (RaySamples, renderer.hpp:43-47).
 * The head is direct-rgb (radiance.cpp:133-145): rgb = logistic(D_1..3). */
typedef struct {
  double lambda_scale;   /* SceneModel::lambda_scale (fields.hpp:17) */
  double beta_bh;        /* SceneModel::beta_bh */
  double background[3];  /* SceneModel::background */
  double t_near, t_far;  /* sampler range (used when ts == NULL) */
  uint64_t seed;         /* sampler seed (used when ts == NULL) */
} dpl_render_params;

int dpl_tape_create(dpl_tape_t* out);
int dpl_tape_destroy(dpl_tape_t tape);
/* render_ray for R rays (tape recorded on device). rgb: R x 3 fp32 output. */
int dpl_render_forward(dpl_tree_t tree, const dpl_kernel_params* params,
                       const dpl_render_params* rp, const double* rays, int64_t R, int32_t S,
                       const double* ts, const double* deltas, float* rgb, dpl_tape_t tape);
/* render_ray_backward with d_weight = 0: d_rgb R x 3 fp32; emits the adjoint
 * queries into buf; d_lambda / d_background (3) are summed over rays (fp64). */
int dpl_render_backward(dpl_tree_t tree, const dpl_kernel_params* params,
                        const dpl_render_params* rp, dpl_tape_t tape, const float* d_rgb,
                        dpl_gradbuf_t buf, double* d_lambda, double* d_background);
/* Tiny-MLP radiance head (HeadVariant::TinyMlp, radiance.hpp)
 * for the render step: sizes run from 22 + (C - 1) inputs (x, sh(omega), normal,
 * appearance) to 3 outputs; w: the reference's flat fp64 layout (per layer rows
 * x cols weights then the bias, radiance.cpp:44-57). n_sizes = 0 restores the
 * direct-rgb head. The layers run on the tensor cores (dpl_gemm_f32's kernel). */
int dpl_tree_set_mlp_head(dpl_tree_t tree, const int32_t* sizes, int32_t n_sizes, const double* w,
                          int64_t n_w);
/* The tiny-MLP head's tensor-core GEMM (tcgen05.mma kind::tf32 with a 3-term
 * hi/lo split, A in TMEM, TMEM accumulators; fp32-class accuracy), exported for
 * tests and host code: D[i][j] = sum_l A[i][l] B[j][l] (d: m x n, row stride
 * ldd), with A read as a[i * lda + l] when a_kcontig else a[l * lda + i], B
 * likewise. flags bit 0: stage B through a pre-split image (bulk async copies,
 * the path the head's weights take). Device pointers; stream NULL = the legacy
 * default stream; synchronous. */
int dpl_gemm_f32(int device, void* stream, int32_t m, int32_t n, int32_t k, const float* a,
                 int64_t lda, int32_t a_kcontig, const float* b, int64_t ldb, int32_t b_kcontig,
                 float* d, int64_t ldd, int32_t flags);
/* RenderGrads::d_head_w accumulated (fp64) by dpl_render_backward since the
 * last call; the accumulator is reset. */
int dpl_head_grads(dpl_tree_t tree, double* d_w, int64_t n_w);
/* The sampler's uniform draw, exported so host code can reproduce it. */
double dpl_uniform(uint64_t seed, uint64_t counter);

/* ---- SceneModel::prepare's eps default (fields.cpp:10-11) -------------------
 * OrientedPointCloud::mean_knn_spacing(k) (pointcloud.cpp:51-65): mean over
 * points of the distances to their k nearest other points; exact kNN on a GPU
 * uniform grid, fp64 distances as the reference computes them. pos: n x 3
 * (host or device). eps = 1.5 * result. */
int dpl_mean_knn_spacing(int device, const double* pos, int64_t n, int32_t k, double* out);

/* ---- Trainer::step point update (optimizer.cpp:161-205) ---------------------
 * Adam (fp64 state, optimizer.cpp:65-81) on the geometry moments, appearance
 * moments and raw normals with flushed gradients g_moments (N x C) and
 * g_normals (N x 3) (fp32, original point order, host or device); normals
 * renormalised when changed (:196-200); then update_moments (bhtree.cpp:171-176).
 * Positions and areas stay fixed, as in the reference trainer. */
typedef struct dpl_point_adam_s* dpl_point_adam_t;
int dpl_point_adam_create(dpl_tree_t tree, dpl_point_adam_t* out);
int dpl_point_adam_destroy(dpl_point_adam_t opt);
int dpl_point_adam_step(dpl_tree_t tree, dpl_point_adam_t opt, const float* g_moments,
                        const float* g_normals, double lr, double beta1, double beta2,
                        double eps);
/* Current cloud parameters (original order, fp64): normals N x 3, moments N x C. */
int dpl_tree_get_points(dpl_tree_t tree, double* normals, double* moments);

/* ---- Sharded point update for G ranks ----------
 * Each rank owns the points [lo, hi) of the original order: it reduce-scatters
 * the flushed gradients, calls dpl_point_adam_step_range with its slice
 * (g_moments (hi - lo) x C, g_normals (hi - lo) x 3; one Adam step per call,
 * no update_moments), all-gathers the updated slices read with
 * dpl_tree_get_points_range, writes the other ranks' slices with
 * dpl_tree_set_points_range, then calls dpl_tree_refresh_moments — the same
 * parameters and node moments as dpl_point_adam_step on the summed gradients.
 * Arrays: host or device, fp64 parameters, original point order. */
int dpl_point_adam_step_range(dpl_tree_t tree, dpl_point_adam_t opt, const float* g_moments,
                              const float* g_normals, int64_t lo, int64_t hi, double lr,
                              double beta1, double beta2, double eps);
int dpl_tree_get_points_range(dpl_tree_t tree, int64_t lo, int64_t hi, double* normals,
                              double* moments);
int dpl_tree_set_points_range(dpl_tree_t tree, int64_t lo, int64_t hi, const double* normals,
                              const double* moments);
/* update_moments (bhtree.cpp:171-176) from the tree's current parameters. */
int dpl_tree_refresh_moments(dpl_tree_t tree);

/* ---- Adam (optimizer.cpp:65-81) on device parameter groups ------------------ */
/* In-place Adam on n fp32 params with fp32 grads and fp32 m/v state; step t is
 * the 1-based iteration after increment. */
int dpl_adam_step(dpl_tree_t tree, float* params, const float* grads, float* m, float* v,
                  int64_t n, double lr, double beta1, double beta2, double eps, int64_t t);

/* ---- debugging: guard zones ---------------------------------------------------
 * With DPL_GUARD=1 in the environment (read once), every device buffer the
 * engine allocates gets 4 KB guard zones before and after it, filled with a
 * byte pattern. dpl_guard_check synchronizes the device and verifies every
 * live buffer's zones (and reports zones found overwritten when buffers were
 * released): NumericalError naming the buffer sizes on a hit. live_buffers
 * (may be NULL) receives the number of guarded buffers checked. */
int dpl_guard_check(int64_t* live_buffers);
/* Positive control of the detector: writes 4 bytes past the end of a fresh
 * guarded buffer and requires dpl_guard_check to report it (DPL_GUARD=1). */
int dpl_guard_selftest(void);

/* ---- measurement -----------------------------------------------------------
 * Per-phase CUDA-event timing on the handle's stream (phases: 0 query Morton
 * sort, 1 forward traversal, 2 adjoint traversal, 3 flush, 4 render per-ray
 * kernels, 5 moment refresh). read() synchronises, returns the summed ms and
 * call counts since the previous read, and clears. */
int dpl_profile_enable(dpl_tree_t tree, int on);
int dpl_profile_read(dpl_tree_t tree, double* ms /* 6 */, int64_t* counts /* 6 */);
/* FFMA / DFMA throughput microbenchmarks (register operands, 8 chains/thread):
 * the measured FP32 / FP64 pipe peaks used as roofline denominators. */
int dpl_peak_fp32(int device, double* tflops);
int dpl_peak_fp64(int device, double* tflops);

#ifdef __cplusplus
}
#endif

#endif /* DIPOLE_B200_H_ */
