// render.cu — K11/K12: the ray-sample render step on top of K6 / K7.
//
// Restates render_ray (proj/src/renderer.cpp:106-171, no lights) and
// render_ray_backward (:173-231) with the direct-rgb head
// (proj/src/radiance.cpp:133-145, 160-174):
//   forward  x_j = o + t_j dir (fp64, as the reference), K6 gives D_0..3 and
//            grad D_0; per ray: f = 1/2 - D_0, grad f = -grad D_0,
//            s = dir . grad f, sigma = lambda h(lambda f) |s| (h = phi / Phi,
//            kernels.cpp:93-98), r_j = logistic(D_1..3),
//            p_j = T_j (1 - exp(-sigma_j delta_j)), rgb = sum p_j r_j + T bg;
//   backward dp_j = d_rgb . (r_j - bg); a reverse suffix scan gives d sigma_j;
//            d_out_0 = -d_f, d_grad_0 = -d grad f, d_out_{1..3} = p d_rgb r(1-r),
//            which feed K7 (the tree adjoint) for all samples at once.
// The per-ray scans are sequential in fp64 (tiny next to the traversals).
#include <algorithm>

#include "render.cuh"

namespace dpl {

__host__ __device__ inline double uniform_u(uint64_t seed, uint64_t counter) {
  uint64_t z = seed + (counter + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * 0x1.0p-53;
}

double host_uniform(uint64_t seed, uint64_t counter) { return uniform_u(seed, counter); }

// sample positions (and generated t) for every (ray, sample)
__global__ void k_samples(const double* __restrict__ rays, int64_t R, int S,
                          const double* __restrict__ ts_in, double t_near, double t_far,
                          uint64_t seed, int64_t ray_offset, double* ts_out, double* xs) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= R * S) return;
  int64_t r = g / S;
  int j = (int)(g % S);
  double t;
  if (ts_in) {
    t = ts_in[g];
  } else {
    double u = uniform_u(seed, (uint64_t)(ray_offset + r) * (uint64_t)S + (uint64_t)j);
    double span = __dsub_rn(t_far, t_near);
    t = __dadd_rn(t_near, __dmul_rn(span, __ddiv_rn(__dadd_rn((double)j, u), (double)S)));
  }
  ts_out[g] = t;
  const double* o = rays + 6 * r;
  xs[3 * g] = __dadd_rn(o[0], __dmul_rn(t, o[3]));
  xs[3 * g + 1] = __dadd_rn(o[1], __dmul_rn(t, o[4]));
  xs[3 * g + 2] = __dadd_rn(o[2], __dmul_rn(t, o[5]));
}

// normal_hazard (kernels.cpp:93-98)
__device__ __forceinline__ double hazard(double z) {
  if (z > -6.0) {
    double pdf = exp(-0.5 * z * z) * 0.3989422804014326779;
    double cdf = 0.5 * erfc(-z * 0.7071067811865475244);
    return pdf / cdf;
  }
  double z2 = z * z;
  return -z / (1.0 - 1.0 / z2 + 3.0 / (z2 * z2) - 15.0 / (z2 * z2 * z2));
}

__device__ __forceinline__ double logistic_d(double x) {  // radiance.cpp:30-38
  if (x >= 0) return 1.0 / (1.0 + exp(-x));
  double e = exp(x);
  return e / (1.0 + e);
}

// Per-sample inputs of the composite, re-read (not taped) by the backward:
// f = 1/2 - D_0, s = dir . grad f, the head colours and delta — the same
// expressions in both kernels, so the backward sees the forward's exact values.
struct SampleIn {
  double f, s, h0, h1, h2, delta;
};
__device__ __forceinline__ SampleIn sample_in(const double* dir, int64_t g, double t, double prev,
                                              const double* __restrict__ deltas,
                                              const float* __restrict__ vals, int vstride,
                                              const float* __restrict__ head_raw,
                                              const float* __restrict__ g0) {
  SampleIn a;
  a.delta = deltas ? deltas[g] : t - prev;  // delta_0 = t_0 - t_near (renderer.hpp:324)
  a.f = 0.5 - (double)vals[(int64_t)vstride * g];
  const double gx = -(double)g0[3 * g], gy = -(double)g0[3 * g + 1], gz = -(double)g0[3 * g + 2];
  a.s = (dir[0] * gx + dir[1] * gy) + dir[2] * gz;
  // head rgb: logistic of the direct-rgb channels 1..3 (radiance.cpp:133-145)
  // or of the tiny-MLP's raw outputs (:153-154)
  const float* hr = head_raw ? head_raw + 3 * g : vals + (int64_t)vstride * g + 1;
  a.h0 = logistic_d(hr[0]), a.h1 = logistic_d(hr[1]), a.h2 = logistic_d(hr[2]);
  return a;
}

// one thread per ray: composite (renderer.cpp:120-168). The tape keeps only
// the sequential state per sample — T_j and p_j — plus sum_j p_j per ray
// (tape + 2 RS); everything else is recomputed from the forward's outputs.
__global__ void k_composite(const double* __restrict__ rays, int64_t R, int S,
                            const double* __restrict__ ts, const double* __restrict__ deltas,
                            double t_near,
                            const float* __restrict__ vals /* RS x vstride */, int vstride,
                            const float* __restrict__ head_raw /* RS x 3 or null */,
                            const float* __restrict__ g0 /* RS x 3 */, double lambda, double bg0,
                            double bg1, double bg2, double* tape /* RS x 2 + R */, float* rgb_out) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= R) return;
  const double* dir = rays + 6 * r + 3;
  double trans = 1.0, c0 = 0, c1 = 0, c2 = 0, prev = t_near, sum_p = 0;
#pragma unroll 4
  for (int j = 0; j < S; ++j) {
    int64_t g = r * S + j;
    double t = ts[g];
    const SampleIn a = sample_in(dir, g, t, prev, deltas, vals, vstride, head_raw, g0);
    prev = t;
    double sigma = lambda * hazard(lambda * a.f) * fabs(a.s);
    double E = exp(-sigma * a.delta);
    double p = trans * (1.0 - E);
    c0 += p * a.h0, c1 += p * a.h1, c2 += p * a.h2;
    sum_p += p;
    reinterpret_cast<double2*>(tape)[g] = make_double2(trans, p);
    trans *= E;
  }
  tape[2 * R * S + r] = sum_p;
  rgb_out[3 * r] = (float)(c0 + trans * bg0);
  rgb_out[3 * r + 1] = (float)(c1 + trans * bg1);
  rgb_out[3 * r + 2] = (float)(c2 + trans * bg2);
}

// one thread per ray: render_ray_backward up to the tree adjoint (:184-228)
__global__ void k_backward_ray(const double* __restrict__ rays, int64_t R, int S,
                               const double* __restrict__ ts, const double* __restrict__ deltas,
                               double t_near, const float* __restrict__ vals, int vstride,
                               const float* __restrict__ head_raw, const float* __restrict__ g0,
                               const double* __restrict__ tape, const float* __restrict__ d_rgb,
                               double lambda, double bg0, double bg1, double bg2,
                               float* d_out /* RS x dstride */, int dstride,
                               float* d_raw /* RS x 3: head raw-output adjoint, or null */,
                               float* d_grad0 /* RS x 3 */,
                               double* sums /* d_lambda, d_bg0..2 */) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double dl = 0, db0 = 0, db1 = 0, db2 = 0;
  if (r < R) {
    const double* dir = rays + 6 * r + 3;
    double dr0 = d_rgb[3 * r], dr1 = d_rgb[3 * r + 1], dr2 = d_rgb[3 * r + 2];
    const double sum_p = tape[2 * R * S + r];  // summed in sample order by the composite
    db0 = (1.0 - sum_p) * dr0, db1 = (1.0 - sum_p) * dr1, db2 = (1.0 - sum_p) * dr2;
    double suffix = 0;
#pragma unroll 4
    for (int j = S - 1; j >= 0; --j) {
      int64_t g = r * S + j;
      const double t = ts[g];
      const double prev = j > 0 ? ts[g - 1] : t_near;
      const SampleIn a = sample_in(dir, g, t, prev, deltas, vals, vstride, head_raw, g0);
      const double2 tp = reinterpret_cast<const double2*>(tape)[g];
      double dp = (dr0 * (a.h0 - bg0) + dr1 * (a.h1 - bg1)) + dr2 * (a.h2 - bg2);
      double trans = tp.x, p = tp.y;
      double E = trans > 0 ? 1.0 - p / trans : 0.0;
      double dsig = a.delta * (trans * E * dp - suffix);
      suffix += p * dp;
      // hazard chain rule (:213-221)
      double f = a.f, s = a.s;
      double u = lambda * f;
      double haz = hazard(u);
      double dhaz = -u * haz - haz * haz;
      double abs_s = fabs(s);
      double sgn_s = s > 0 ? 1.0 : (s < 0 ? -1.0 : 0.0);
      double d_f = dsig * lambda * lambda * abs_s * dhaz;
      dl += dsig * (haz * abs_s + lambda * abs_s * dhaz * f);
      double k = dsig * lambda * haz * sgn_s;
      d_out[(int64_t)dstride * g] = (float)(-d_f);
      d_grad0[3 * g] = (float)(-k * dir[0]);
      d_grad0[3 * g + 1] = (float)(-k * dir[1]);
      d_grad0[3 * g + 2] = (float)(-k * dir[2]);
      // head backward d_raw = d_radiance * rgb (1 - rgb) (radiance.cpp:166): the
      // direct-rgb head's channel adjoints, or the tiny-MLP's output adjoint
      float* dr = d_raw ? d_raw + 3 * g : d_out + (int64_t)dstride * g + 1;
      dr[0] = (float)(p * dr0 * a.h0 * (1.0 - a.h0));
      dr[1] = (float)(p * dr1 * a.h1 * (1.0 - a.h1));
      dr[2] = (float)(p * dr2 * a.h2 * (1.0 - a.h2));
    }
  }
  // warp-reduce the ray sums, one fp64 atomic per warp and quantity
  for (int o = 16; o > 0; o >>= 1) {
    dl += __shfl_xor_sync(0xffffffffu, dl, o);
    db0 += __shfl_xor_sync(0xffffffffu, db0, o);
    db1 += __shfl_xor_sync(0xffffffffu, db1, o);
    db2 += __shfl_xor_sync(0xffffffffu, db2, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(sums, dl);
    atomicAdd(sums + 1, db0);
    atomicAdd(sums + 2, db1);
    atomicAdd(sums + 3, db2);
  }
}

// d_grad_f += (d_normal - n (n . d_normal)) / |grad f| (renderer.cpp:206-211);
// d_grad[0] = -d_grad_f, d_out[1 + k] = d_appearance[k] (:226-229)
__global__ void k_mlp_scatter(const float* __restrict__ dX, int din, int64_t q0, int64_t q, int K,
                              const float* __restrict__ g0, float* __restrict__ d_out, int C,
                              float* __restrict__ d_grad0) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = q0 + i;
    const float* r = dX + i * din;
    for (int k = 0; k < K; ++k) d_out[g * C + 1 + k] = r[22 + k];
    const double gx = -(double)g0[3 * g], gy = -(double)g0[3 * g + 1], gz = -(double)g0[3 * g + 2];
    const double gn = sqrt((gx * gx + gy * gy) + gz * gz);
    if (gn > 1e-12) {
      const double nx = gx / gn, ny = gy / gn, nz = gz / gn;
      const double dnx = r[19], dny = r[20], dnz = r[21];
      const double dot = (nx * dnx + ny * dny) + nz * dnz;
      d_grad0[3 * g] -= (float)((dnx - nx * dot) / gn);
      d_grad0[3 * g + 1] -= (float)((dny - ny * dot) / gn);
      d_grad0[3 * g + 2] -= (float)((dnz - nz * dot) / gn);
    }
  }
}

void render_mlp_scatter(cudaStream_t s, const float* dX, int din, int64_t q0, int64_t q, int K,
                        const float* g0, float* d_out, int C, float* d_grad0) {
  const unsigned b = (unsigned)std::max<int64_t>(1, std::min<int64_t>((q + 255) / 256, 148 * 32));
  k_mlp_scatter<<<b, 256, 0, s>>>(dX, din, q0, q, K, g0, d_out, C, d_grad0);
  count_launch();
}

void render_samples(cudaStream_t s, const double* rays, int64_t R, int S, const double* ts_in,
                    double t_near, double t_far, uint64_t seed, double* ts_out, double* xs) {
  int64_t tot = R * S;
  k_samples<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(rays, R, S, ts_in, t_near, t_far, seed, 0,
                                                         ts_out, xs);
  count_launch();
}

void render_composite(cudaStream_t s, const double* rays, int64_t R, int S, const double* ts,
                      const double* deltas, double t_near, const float* vals, int vstride,
                      const float* head_raw, const float* g0, double lambda, const double* bg,
                      double* tape, float* rgb) {
  k_composite<<<(unsigned)((R + 127) / 128), 128, 0, s>>>(rays, R, S, ts, deltas, t_near, vals,
                                                         vstride, head_raw, g0, lambda, bg[0],
                                                         bg[1], bg[2], tape, rgb);
  count_launch();
}

void render_backward_rays(cudaStream_t s, const double* rays, int64_t R, int S, const double* ts,
                          const double* deltas, double t_near, const float* vals, int vstride,
                          const float* head_raw, const float* g0, const double* tape,
                          const float* d_rgb, double lambda, const double* bg, float* d_out,
                          int dstride, float* d_raw, float* d_grad0, double* sums) {
  k_backward_ray<<<(unsigned)((R + 127) / 128), 128, 0, s>>>(
      rays, R, S, ts, deltas, t_near, vals, vstride, head_raw, g0, tape, d_rgb, lambda, bg[0],
      bg[1], bg[2], d_out, dstride, d_raw, d_grad0, sums);
  count_launch();
}

}  // namespace dpl
