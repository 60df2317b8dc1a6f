// coeffs.cuh — fp32 radial coefficients of the regularized dipole kernel.
//
// Device restatement of kernel_coeffs (proj/src/kernels.cpp:100-153). With
// t = r/eps, u = t^2, e = exp(-u) and g = tau(t)/t^3 every coefficient is
// written in a cancellation-free form:
//   W     = g / eps^3                       R     = W * r
//   Wp_r  = h / eps^5,  h = ((4/sqrt pi) e - 3 g) / u
//   Rp_r  = ((4/sqrt pi) e - 2 g) / (eps^3 r)
//   dW_de = -(4/sqrt pi) e / eps^4          dR_de = dW_de * r
//   dWp_r_de = (8/sqrt pi) e / eps^6        (the reference's two-term form, simplified)
// For t < 1, g, h and 2 - 2P come from all-positive series in u (the erf
// series of kernels.cpp:12-24 with its n = 0 term cancelled analytically), so
// fp32 keeps full relative precision down to t = 0. For t >= 6.5 the
// reference sets tau = 1, tau' = tau'' = 0 (kernels.cpp:50-55); so do we.
#pragma once

#include "dpl_internal.cuh"

namespace dpl {

struct Co {
  float W, R, Wp_r, Rp_r, dW_de, dWp_r_de, dR_de;
  bool near;  // t < 6.5 (epsilon derivatives non-zero)
};

__device__ __forceinline__ float horner_P(float u) {  // sum_{n>=1} 2^n u^(n-1) / (2n+1)!!
  float s = 7.447646152e-08f;
  s = fmaf(s, u, 7.820028460e-07f);
  s = fmaf(s, u, 7.429027037e-06f);
  s = fmaf(s, u, 6.314672981e-05f);
  s = fmaf(s, u, 4.736004736e-04f);
  s = fmaf(s, u, 3.078403078e-03f);
  s = fmaf(s, u, 1.693121693e-02f);
  s = fmaf(s, u, 7.619047619e-02f);
  s = fmaf(s, u, 2.666666667e-01f);
  return fmaf(s, u, 6.666666667e-01f);
}
__device__ __forceinline__ float horner_H(float u) {  // sum_{n>=2} 3 2^n u^(n-2) / (2n+1)!!
  float s = 1.942864214e-08f;
  s = fmaf(s, u, 2.234293846e-07f);
  s = fmaf(s, u, 2.346008538e-06f);
  s = fmaf(s, u, 2.228708111e-05f);
  s = fmaf(s, u, 1.894401894e-04f);
  s = fmaf(s, u, 1.420801421e-03f);
  s = fmaf(s, u, 9.235209235e-03f);
  s = fmaf(s, u, 5.079365079e-02f);
  s = fmaf(s, u, 2.285714286e-01f);
  return fmaf(s, u, 8.000000000e-01f);
}
__device__ __forceinline__ float horner_Q(float u) {  // 2 - 2 P(u)
  float s = -1.489529230e-07f;
  s = fmaf(s, u, -1.564005692e-06f);
  s = fmaf(s, u, -1.485805407e-05f);
  s = fmaf(s, u, -1.262934596e-04f);
  s = fmaf(s, u, -9.472009472e-04f);
  s = fmaf(s, u, -6.156806157e-03f);
  s = fmaf(s, u, -3.386243386e-02f);
  s = fmaf(s, u, -1.523809524e-01f);
  s = fmaf(s, u, -5.333333333e-01f);
  return fmaf(s, u, 6.666666667e-01f);
}

#define DPL_2_SQRTPI 1.1283791670955126f
#define DPL_4_SQRTPI 2.2567583341910252f
#define DPL_8_SQRTPI 4.5135166683820505f

// ORDER 0: W, R. ORDER 1: + Wp_r, Rp_r. ORDER 2: + epsilon derivatives.
// r2 > 0 is the fp32 squared distance (rounded from the exact fp64 one),
// except r2 == 0 for coincident points under the regularized kernel.
template <int ORDER>
__device__ __forceinline__ Co coeffs(float r2, const KParams& kp) {
  Co c;
  c.Wp_r = c.Rp_r = c.dW_de = c.dWp_r_de = c.dR_de = 0.f;
  c.near = false;
  if (kp.mode == KM_REGULARIZED) {
    float inv_r = rsqrt_pos(r2);  // r2 == 0 (coincidence) is handled by the near branch
    float r = r2 * inv_r;
    float t = r * kp.inv_eps;
    if (r2 > 0.f && t >= 6.5f) {  // tau = 1 (kernels.cpp:50-55); products of rsqrt, no divide
      const float inv_r2 = inv_r * inv_r;
      c.R = inv_r2;
      c.W = inv_r2 * inv_r;
      if (ORDER >= 1) {
        c.Wp_r = -3.0f * c.W * inv_r2;
        c.Rp_r = -2.0f * inv_r2 * inv_r2;
      }
      return c;
    }
    if (r2 == 0.f) r = 0.f, t = 0.f;
    c.near = true;
    float u = t * t;
    float e = expf(-u);
    float g, h = 0.f, q = 0.f;
    if (t < 1.0f) {
      float ke = DPL_2_SQRTPI * e;
      g = ke * horner_P(u);
      if (ORDER >= 1) {
        h = -ke * horner_H(u);
        q = ke * horner_Q(u);
      }
    } else {
      float tau = erff(t) - DPL_2_SQRTPI * t * e;
      g = tau / (t * u);
      if (ORDER >= 1) {
        h = (DPL_4_SQRTPI * e - 3.0f * g) / u;
        q = DPL_4_SQRTPI * e - 2.0f * g;
      }
    }
    c.W = g * kp.inv_eps3;
    c.R = c.W * r;
    if (ORDER >= 1) {
      c.Wp_r = h * kp.inv_eps5;
      c.Rp_r = r > 0.f ? q * kp.inv_eps3 / r : 0.f;
    }
    if (ORDER >= 2) {
      c.dW_de = -DPL_4_SQRTPI * e * kp.inv_eps4;
      c.dR_de = c.dW_de * r;
      c.dWp_r_de = DPL_8_SQRTPI * e * kp.inv_eps6;
    }
    return c;
  }
  if (kp.mode == KM_SINGULAR) {  // kernels.cpp:112-121; callers guarantee r2 > 0
    float inv_r = rsqrtf(r2);
    float inv_r2 = inv_r * inv_r;
    c.R = inv_r2;
    c.W = inv_r * inv_r2;
    if (ORDER >= 1) {
      c.Wp_r = -3.0f * c.W * inv_r2;
      c.Rp_r = -2.0f * inv_r2 * inv_r2;
    }
    return c;
  }
  // desingularized, kernels.cpp:102-111: s = r^2 + delta^2
  float s = r2 + kp.delta2;
  float s32 = s * sqrtf(s);
  float r = sqrtf(r2);
  c.W = 1.0f / s32;
  c.R = r * c.W;
  if (ORDER >= 1) {
    c.Wp_r = -3.0f / (s32 * s);
    c.Rp_r = r > 0.f ? (c.W - 3.0f * r2 / (s32 * s)) / r : 0.f;
  }
  return c;
}

}  // namespace dpl
