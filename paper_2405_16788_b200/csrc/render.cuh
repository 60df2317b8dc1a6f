// render.cuh — render-step kernels (render.cu).
#pragma once

#include "tree.cuh"

namespace dpl {

double host_uniform(uint64_t seed, uint64_t counter);
void render_samples(cudaStream_t s, const double* rays, int64_t R, int S, const double* ts_in,
                    double t_near, double t_far, uint64_t seed, double* ts_out, double* xs);
// vals: RS x vstride forward values (channel 0 = geometry); head_raw: RS x 3
// tiny-MLP outputs, or null for the direct-rgb head (channels 1..3 of vals)
void render_composite(cudaStream_t s, const double* rays, int64_t R, int S, const double* ts,
                      const double* deltas, double t_near, const float* vals, int vstride,
                      const float* head_raw, const float* g0, double lambda, const double* bg,
                      double* tape, float* rgb);
// d_out: RS x dstride adjoint inputs; d_raw: RS x 3 head output adjoints for the
// tiny-MLP (null: written into d_out channels 1..3, the direct-rgb head)
// (ts, deltas, vals, head_raw, g0: the forward's inputs, re-read per sample;
// tape: T_j, p_j per sample and sum_j p_j per ray from render_composite)
void render_backward_rays(cudaStream_t s, const double* rays, int64_t R, int S, const double* ts,
                          const double* deltas, double t_near, const float* vals, int vstride,
                          const float* head_raw, const float* g0, const double* tape,
                          const float* d_rgb, double lambda, const double* bg, float* d_out,
                          int dstride, float* d_raw, float* d_grad0, double* sums);
// tiny-MLP input adjoint -> tree adjoint inputs for samples [q0, q0 + q): appearance
// channels into d_out (stride C), the implicit-normal term into d_grad0
// (renderer.cpp:206-211, 226-227)
void render_mlp_scatter(cudaStream_t s, const float* dX, int din, int64_t q0, int64_t q, int K,
                        const float* g0, float* d_out, int C, float* d_grad0);

}  // namespace dpl
