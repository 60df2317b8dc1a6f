// sampling.cuh — query generators around the forward kernels: the mesh-
// extraction grid (sample_grid, meshing.cpp:33-59) and the probe-then-refine
// ray sampler (sample_ray, renderer.cpp:46-86). Geometry values are
// f = 0.5 - primal_channel(x, 0) (geometry_field, fields.cpp:27-29).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace dpl {

struct RaySampler {
  double t_near, t_far;
  int probe_count, sparse_before, dense_at, sparse_after, uniform_count;
};

// grid nodes [start, start + n) of the flat (k * r1 + j) * r0 + i order
void grid_nodes(const double lo[3], const double hi[3], const int res[3], int64_t start, int64_t n,
                double* xs, cudaStream_t s);
// a[i] = i
void iota32(int32_t* a, int64_t n, cudaStream_t s);
// out[i] = 0.5f - v[i]
void half_minus(const float* v, int64_t n, float* out, cudaStream_t s);

// probe round: queries for n_act active rays x kcount probes starting at probe i0
void probe_points(const double* rays, const int32_t* act, int64_t n_act, int i0, int kcount,
                  const RaySampler& c, double* xs, cudaStream_t s);
// scan the round's values in probe order; bracket[r] = probe index of the first
// sign change, -1 while none, -2 when the probes ran out; appends still-active
// rays to next_act (count in *n_next)
void probe_scan(const float* v, const int32_t* act, int64_t n_act, int i0, int kcount,
                const RaySampler& c, float* prev_f, int32_t* bracket, int32_t* next_act,
                int* n_next, cudaStream_t s);
// samples per ray from the bracket (or uniform), t / delta R x max_s
void emit_samples(const int32_t* bracket, int64_t R, const RaySampler& c, int max_s, double* t,
                  double* delta, int32_t* count, uint8_t* bracketed, cudaStream_t s);

}  // namespace dpl
