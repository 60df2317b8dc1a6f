/* dipole_oracle.h — CPU restatement of the reference hot path, in plain C.
 *
 * TEST INFRASTRUCTURE ONLY. This is the checker the parity tests, smoke() and
 * bench.py's cpu_baseline leg compare the CUDA path against; it is never
 * linked into, called by, or substituted for the product library
 * (paper_2405_16788_b200/libdipole_b200.so). Every function cites the
 * reference file:line it restates (paths relative to /root/reference/proj).
 * It is pinned against the reference itself (oracle/_ref, built from the
 * unmodified sources) and against the golden vectors in tests/golden/.
 *
 * All arithmetic is fp64 with no FMA contraction (-ffp-contract=off), in the
 * reference's operation order, so trees are bitwise identical and sums agree
 * to rounding.
 */
#ifndef DIPOLE_ORACLE_H_
#define DIPOLE_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double epsilon;
  int32_t desingularized;
  int32_t reserved;
  double desing_delta;
  double coincident_value;
} ora_params;

typedef struct {
  int64_t visited, far_near, far_far, pt_near, pt_far;
} ora_counters;

typedef struct ora_tree ora_tree;

double ora_erf(double x);
double ora_tau(double t);
double ora_normal_hazard(double z);
/* out7 = {W, Wp_r, dW_de, dWp_r_de, R, Rp_r, dR_de} */
void ora_kernel_coeffs(double r, const ora_params* p, int order, double* out7);

ora_tree* ora_tree_build(const double* pos, const double* nrm, const double* area,
                         const double* mu, int64_t n, int32_t C, int32_t max_leaf,
                         int32_t max_depth);
void ora_tree_free(ora_tree* t);
int ora_tree_update_moments(ora_tree* t, const double* pos, const double* nrm, const double* area,
                            const double* mu, int64_t n, int32_t C);
int ora_tree_set_kinds(ora_tree* t, const uint8_t* kinds, int32_t C);
int64_t ora_tree_node_count(const ora_tree* t);
void ora_tree_export(const ora_tree* t, double* geo, int32_t* topo, int32_t* order,
                     int32_t* leaf_of);
void ora_tree_export_moments(const ora_tree* t, double* mv, double* ms);

/* mode 0 primal, 1 primal_with_gradient, 2 primal_channel(channel) */
void ora_primal(const ora_tree* t, const ora_params* p, double beta, const double* xs, int64_t q,
                int mode, int channel, double* out, double* grad, ora_counters* counters,
                int threads);
void ora_adjoint(const ora_tree* t, const ora_params* p, double beta, const double* xs, int64_t q,
                 const double* d_out, const double* d_grad, int threads, double* moments,
                 double* normals, double* d_eps);

void ora_naive_sum(const ora_tree* t, const ora_params* p, const double* xs, int64_t q,
                   int channel, int kind, double* out, double* grad);
void ora_naive_adjoint(const ora_tree* t, const ora_params* p, const double* xs, int64_t q,
                       const double* d_out, const double* d_grad, double* moments,
                       double* normals, double* d_eps);

void ora_primal_ex(const ora_tree* t, const ora_params* p, double beta, const double* xs,
                   int64_t q, int mode, int channel, double* out, double* grad,
                   ora_counters* counters, int threads, double* out_abs, double* grad_abs);
/* Test-only: the same primal / adjoint / render step, plus for every flushed output a
 * bound on the sum of |terms| it accumulated (the tolerance scale where the
 * reference's sum cancels). */
void ora_adjoint_ex(const ora_tree* t, const ora_params* p, double beta, const double* xs,
                    int64_t q, const double* d_out, const double* d_grad, int threads,
                    double* moments, double* normals, double* d_eps, double* mom_abs,
                    double* nrm_abs, double* deps_abs);
void ora_render_step_ex(const ora_tree* t, const ora_params* p, double beta, double lambda,
                        const double* background, const double* rays, int64_t R, int32_t S,
                        const double* ts, const double* deltas, const double* target,
                        double scale, int threads, double* rgb, double* moments, double* normals,
                        double* d_eps, double* d_lambda, double* d_bg, double* mom_abs,
                        double* nrm_abs, double* deps_abs);
double ora_uniform(uint64_t seed, uint64_t counter);
void ora_stratified_samples(int64_t R, int32_t S, double t_near, double t_far, uint64_t seed,
                            int64_t ray_offset, double* ts, double* deltas);
/* render_ray + render_ray_backward for R rays, direct-rgb head, loss gradient
 * d_rgb = scale * (rgb - target). Requires channel 0 Dipole and >= 3 appearance
 * channels. */
void ora_render_step(const ora_tree* t, const ora_params* p, double beta, double lambda,
                     const double* background, const double* rays, int64_t R, int32_t S,
                     const double* ts, const double* deltas, const double* target, double scale,
                     int threads, double* rgb, double* moments, double* normals, double* d_eps,
                     double* d_lambda, double* d_bg);

double ora_mean_knn_spacing(const double* pos, int64_t n, int k);

/* sample_grid (meshing.cpp:33-59): values r2 x r1 x r0 of 0.5 - primal_channel(x, 0);
 * returns 2 (DataError) for a resolution below 2. pos: the cloud (bounding box). */
int ora_sample_grid(const ora_tree* t, const ora_params* p, double beta, const int32_t* res,
                    const double* lo, const double* hi, const double* pos, int64_t n,
                    int threads, double* values, double* lo_out, double* hi_out);
/* sample_ray (renderer.cpp:46-86) for R rays (origin, dir); counts5 = {probe_count,
 * sparse_before, dense_at, sparse_after, uniform_count}; t / delta R x max_s. */
void ora_sample_rays(const ora_tree* t, const ora_params* p, double beta, const double* rays,
                     int64_t R, double t_near, double t_far, const int32_t* counts5,
                     int32_t max_s, int threads, double* ts, double* delta, int32_t* count,
                     uint8_t* bracketed);

void ora_adam_step(double* params, const double* grads, double* m, double* v, int64_t n,
                   double lr, double beta1, double beta2, double eps, int64_t t);

#ifdef __cplusplus
}
#endif

#endif
