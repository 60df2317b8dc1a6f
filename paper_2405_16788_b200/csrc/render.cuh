// render.cuh — render-step kernels (render.cu).
#pragma once

#include "tree.cuh"

namespace dpl {

double host_uniform(uint64_t seed, uint64_t counter);
void render_samples(cudaStream_t s, const double* rays, int64_t R, int S, const double* ts_in,
                    double t_near, double t_far, uint64_t seed, double* ts_out, double* xs);
void render_composite(cudaStream_t s, const double* rays, int64_t R, int S, const double* ts,
                      const double* deltas, double t_near, const float* vals, const float* g0, double lambda,
                      const double* bg, double* tape, float* rgb);
void render_backward_rays(cudaStream_t s, const double* rays, int64_t R, int S,
                          const double* tape, const float* d_rgb, double lambda, const double* bg,
                          float* d_out, float* d_grad0, double* sums);

}  // namespace dpl
