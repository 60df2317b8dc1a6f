// sampling.cu — grid and ray-probe query generators (see sampling.cuh). All
// positions follow the reference's fp64 expression order (no FMA).
#include "dpl_internal.cuh"
#include "sampling.cuh"

namespace dpl {

namespace {

inline unsigned grid_for(int64_t n, int b) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + b - 1) / b, 148 * 64));
}

// FieldGrid::node (meshing.cpp:25-30): lo + f.cwiseProduct(hi - lo)
__global__ void k_grid_nodes(double lo0, double lo1, double lo2, double hi0, double hi1, double hi2,
                             int r0, int r1, int r2, int64_t start, int64_t n, double* xs) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = start + q;
    const int i = (int)(g % r0);
    const int j = (int)((g / r0) % r1);
    const int k = (int)(g / ((int64_t)r0 * r1));
    const double f0 = r0 > 1 ? __ddiv_rn((double)i, (double)(r0 - 1)) : 0.0;
    const double f1 = r1 > 1 ? __ddiv_rn((double)j, (double)(r1 - 1)) : 0.0;
    const double f2 = r2 > 1 ? __ddiv_rn((double)k, (double)(r2 - 1)) : 0.0;
    xs[3 * q] = __dadd_rn(lo0, __dmul_rn(f0, __dsub_rn(hi0, lo0)));
    xs[3 * q + 1] = __dadd_rn(lo1, __dmul_rn(f1, __dsub_rn(hi1, lo1)));
    xs[3 * q + 2] = __dadd_rn(lo2, __dmul_rn(f2, __dsub_rn(hi2, lo2)));
  }
}

__global__ void k_iota32(int32_t* a, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (int32_t)i;
}

__global__ void k_half_minus(const float* __restrict__ v, int64_t n, float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = 0.5f - v[i];
}

// probe i of a ray: t = t_near + span * i / (n - 1) (renderer.cpp:59)
__device__ __forceinline__ double probe_t(const RaySampler& c, int i) {
  const int n = c.probe_count < 2 ? 2 : c.probe_count;
  const double span = __dsub_rn(c.t_far, c.t_near);
  return __dadd_rn(c.t_near, __ddiv_rn(__dmul_rn(span, (double)i), (double)(n - 1)));
}

__global__ void k_probe_points(const double* __restrict__ rays, const int32_t* __restrict__ act,
                               int64_t n_act, int i0, int kcount, RaySampler c, double* xs) {
  const int64_t total = n_act * kcount;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = q / kcount;
    const int k = (int)(q - a * kcount);
    const double* r = rays + 6 * (size_t)act[a];
    const double t = probe_t(c, i0 + k);
    // ray.origin + t * ray.dir (renderer.cpp:61)
    xs[3 * q] = __dadd_rn(r[0], __dmul_rn(t, r[3]));
    xs[3 * q + 1] = __dadd_rn(r[1], __dmul_rn(t, r[4]));
    xs[3 * q + 2] = __dadd_rn(r[2], __dmul_rn(t, r[5]));
  }
}

// first sign change of f over the probes, in order (renderer.cpp:62-68)
__global__ void k_probe_scan(const float* __restrict__ v, const int32_t* __restrict__ act,
                             int64_t n_act, int i0, int kcount, RaySampler c, float* prev_f,
                             int32_t* bracket, int32_t* next_act, int* n_next) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n_act) return;
  const int32_t ray = act[a];
  const int n = c.probe_count < 2 ? 2 : c.probe_count;
  float pf = prev_f[ray];
  int32_t br = -1;
  for (int k = 0; k < kcount; ++k) {
    const int i = i0 + k;
    const float f = 0.5f - v[a * kcount + k];
    if (i > 0 && ((pf > 0.f && f <= 0.f) || (pf <= 0.f && f > 0.f))) {
      br = i;
      break;
    }
    pf = f;
  }
  if (br < 0 && i0 + kcount >= n) br = -2;  // probes exhausted: uniform samples
  prev_f[ray] = pf;
  bracket[ray] = br;
  if (br == -1) next_act[atomicAdd(n_next, 1)] = ray;
}

// RaySamples (renderer.cpp:69-85)
__global__ void k_emit(const int32_t* __restrict__ bracket, int64_t R, RaySampler c, int max_s,
                       double* t, double* delta, int32_t* count, uint8_t* bracketed) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  double* tr = t + (size_t)r * max_s;
  double* dr = delta + (size_t)r * max_s;
  const double span = __dsub_rn(c.t_far, c.t_near);
  if (span < 1e-9) {  // :50-54
    tr[0] = 0.5 * __dadd_rn(c.t_near, c.t_far);
    dr[0] = __dsub_rn(tr[0], c.t_near);
    for (int j = 1; j < max_s; ++j) tr[j] = dr[j] = 0.0;
    count[r] = 1;
    bracketed[r] = 0;
    return;
  }
  int m = 0;
  auto emit = [&](double lo, double hi, int cnt) {
    for (int i = 0; i < cnt; ++i)
      tr[m++] = __dadd_rn(lo, __ddiv_rn(__dmul_rn(__dsub_rn(hi, lo), (double)i + 0.5), (double)cnt));
  };
  const int br = bracket[r];
  if (br < 1) {
    emit(c.t_near, c.t_far, c.uniform_count > 1 ? c.uniform_count : 1);
  } else {
    const double lo = probe_t(c, br - 1), hi = probe_t(c, br);
    emit(c.t_near, lo, c.sparse_before);
    emit(lo, hi, c.dense_at > 1 ? c.dense_at : 1);
    emit(hi, c.t_far, c.sparse_after);
  }
  for (int j = 0; j < m; ++j) dr[j] = __dsub_rn(tr[j], j == 0 ? c.t_near : tr[j - 1]);
  for (int j = m; j < max_s; ++j) tr[j] = dr[j] = 0.0;  // deterministic padding
  count[r] = m;
  bracketed[r] = br >= 1 ? 1 : 0;
}

}  // namespace

void grid_nodes(const double lo[3], const double hi[3], const int res[3], int64_t start, int64_t n,
                double* xs, cudaStream_t s) {
  k_grid_nodes<<<grid_for(n, 256), 256, 0, s>>>(lo[0], lo[1], lo[2], hi[0], hi[1], hi[2], res[0],
                                                res[1], res[2], start, n, xs);
  count_launch();
}

void iota32(int32_t* a, int64_t n, cudaStream_t s) {
  k_iota32<<<grid_for(n, 256), 256, 0, s>>>(a, n);
  count_launch();
}

void half_minus(const float* v, int64_t n, float* out, cudaStream_t s) {
  k_half_minus<<<grid_for(n, 256), 256, 0, s>>>(v, n, out);
  count_launch();
}

void probe_points(const double* rays, const int32_t* act, int64_t n_act, int i0, int kcount,
                  const RaySampler& c, double* xs, cudaStream_t s) {
  k_probe_points<<<grid_for(n_act * kcount, 256), 256, 0, s>>>(rays, act, n_act, i0, kcount, c, xs);
  count_launch();
}

void probe_scan(const float* v, const int32_t* act, int64_t n_act, int i0, int kcount,
                const RaySampler& c, float* prev_f, int32_t* bracket, int32_t* next_act,
                int* n_next, cudaStream_t s) {
  k_probe_scan<<<(unsigned)((n_act + 127) / 128), 128, 0, s>>>(v, act, n_act, i0, kcount, c,
                                                               prev_f, bracket, next_act, n_next);
  count_launch();
}

void emit_samples(const int32_t* bracket, int64_t R, const RaySampler& c, int max_s, double* t,
                  double* delta, int32_t* count, uint8_t* bracketed, cudaStream_t s) {
  k_emit<<<(unsigned)((R + 127) / 128), 128, 0, s>>>(bracket, R, c, max_s, t, delta, count,
                                                      bracketed);
  count_launch();
}

}  // namespace dpl
