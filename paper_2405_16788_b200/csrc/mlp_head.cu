// mlp_head.cu — tiny-MLP radiance head for the batched render step (see
// mlp_head.cuh). Reference: Mlp::forward / Mlp::backward and
// RadianceHead::eval / backward (radiance.cpp:59-180).
#include <algorithm>
#include <cstdlib>

#include "mlp_head.cuh"
#include "tc_gemm.cuh"

#include "../../include/dipole_b200.h"

namespace dpl {

namespace {

inline unsigned blocks_for(int64_t n, int b) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + b - 1) / b, 148 * 32));
}

// real spherical harmonics up to degree 3 (sh_encode, radiance.cpp:7-28)
__device__ __forceinline__ void sh_encode(double x, double y, double z, float* o) {
  const double x2 = x * x, y2 = y * y, z2 = z * z;
  o[0] = 0.28209479177387814f;
  o[1] = (float)(0.4886025119029199 * y);
  o[2] = (float)(0.4886025119029199 * z);
  o[3] = (float)(0.4886025119029199 * x);
  o[4] = (float)(1.0925484305920792 * x * y);
  o[5] = (float)(1.0925484305920792 * y * z);
  o[6] = (float)(0.31539156525252005 * (3.0 * z2 - 1.0));
  o[7] = (float)(1.0925484305920792 * x * z);
  o[8] = (float)(0.5462742152960396 * (x2 - y2));
  o[9] = (float)(0.5900435899266435 * y * (3.0 * x2 - y2));
  o[10] = (float)(2.890611442640554 * x * y * z);
  o[11] = (float)(0.4570457994644658 * y * (5.0 * z2 - 1.0));
  o[12] = (float)(0.3731763325901154 * z * (5.0 * z2 - 3.0));
  o[13] = (float)(0.4570457994644658 * x * (5.0 * z2 - 1.0));
  o[14] = (float)(1.445305721320277 * z * (x2 - y2));
  o[15] = (float)(0.5900435899266435 * x * (x2 - 3.0 * y2));
}

// head input rows (RadianceHead::eval, radiance.cpp:146-152; n_hat and omega_head
// as render_ray builds them, renderer.cpp:111,128-130)
__global__ void k_inputs(const double* __restrict__ rays, int S, const double* __restrict__ xs,
                         const float* __restrict__ vals, int C, const float* __restrict__ g0,
                         int64_t q0, int64_t q, int K, float* __restrict__ X, int ldx) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = q0 + i;
    const double* dir = rays + 6 * (g / S) + 3;
    const double ox = -dir[0], oy = -dir[1], oz = -dir[2];
    float* row = X + i * ldx;
    row[0] = (float)xs[3 * g], row[1] = (float)xs[3 * g + 1], row[2] = (float)xs[3 * g + 2];
    sh_encode(ox, oy, oz, row + 3);
    const double gx = -(double)g0[3 * g], gy = -(double)g0[3 * g + 1], gz = -(double)g0[3 * g + 2];
    const double gn = sqrt((gx * gx + gy * gy) + gz * gz);
    if (gn > 1e-12) {
      row[19] = (float)(gx / gn), row[20] = (float)(gy / gn), row[21] = (float)(gz / gn);
    } else {
      row[19] = (float)ox, row[20] = (float)oy, row[21] = (float)oz;
    }
    for (int k = 0; k < K; ++k) row[22 + k] = vals[g * C + 1 + k];
  }
}

// y = y + bias (+ ReLU unless last), row-major q x rows
__global__ void k_bias_act(float* __restrict__ y, const float* __restrict__ b, int64_t q, int rows,
                           int relu) {
  const int64_t n = q * rows;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = y[i] + b[i % rows];
    y[i] = relu ? fmaxf(v, 0.f) : v;
  }
}

// Narrow layers (<= 4 output rows: the rgb layer) are HBM-bound, not GEMM-shaped:
// a 128-row MMA tile would be 97 % padding, so their two backward products run
// on the FP32 pipe at memory speed.
// d_in[q][c] = gate(act[q][c]) * sum_r delta[q][r] W[r][c]   (Mlp::backward, radiance.cpp:105-112)
template <int R>
__global__ void k_narrow_dx(const float* __restrict__ delta, const float* __restrict__ W,
                            const float* __restrict__ gate, int64_t q, int cols,
                            float* __restrict__ out) {
  const int c4n = cols >> 2;
  const int64_t n4 = q * c4n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t qi = i / c4n;
    const int c4 = (int)(i - qi * c4n);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float d = __ldg(delta + qi * R + r);
      const float4 w = __ldg(reinterpret_cast<const float4*>(W + (size_t)r * cols) + c4);
      v.x = fmaf(d, w.x, v.x), v.y = fmaf(d, w.y, v.y), v.z = fmaf(d, w.z, v.z), v.w = fmaf(d, w.w, v.w);
    }
    if (gate) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(gate + qi * cols) + c4);
      v.x = a.x > 0.f ? v.x : 0.f, v.y = a.y > 0.f ? v.y : 0.f;
      v.z = a.z > 0.f ? v.z : 0.f, v.w = a.w > 0.f ? v.w : 0.f;
    }
    reinterpret_cast<float4*>(out + qi * cols)[c4] = v;
  }
}

// dW[r][c] += sum_q delta[q][r] in[q][c], db[r] += sum_q delta[q][r] (fp64
// accumulators, RenderGrads::d_head_w): thread = input column, a block walks
// a contiguous slice of the samples, fp32 partial sums of at most 1024 samples
// per fp64 atomic
template <int R>
__global__ void k_narrow_dw(const float* __restrict__ delta, const float* __restrict__ in,
                            int64_t q, int cols, int ldin, double* __restrict__ dW,
                            double* __restrict__ db) {
  const int64_t per = (q + gridDim.x - 1) / gridDim.x;
  const int64_t q0 = (int64_t)blockIdx.x * per, q1 = q0 + per < q ? q0 + per : q;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    for (int64_t b0 = q0; b0 < q1; b0 += 1024) {
      const int64_t b1 = b0 + 1024 < q1 ? b0 + 1024 : q1;
      float acc[R], sb[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = sb[r] = 0.f;
      for (int64_t qi = b0; qi < b1; ++qi) {
        const float x = __ldg(in + qi * ldin + c);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const float d = __ldg(delta + qi * R + r);
          acc[r] = fmaf(d, x, acc[r]);
          sb[r] += d;
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (acc[r] != 0.f) atomicAdd(dW + (size_t)r * cols + c, (double)acc[r]);
        if (c == 0 && sb[r] != 0.f) atomicAdd(db + r, (double)sb[r]);
      }
    }
  }
}

__global__ void k_to_f32(const double* __restrict__ a, int64_t n, float* __restrict__ b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (float)a[i];
}

}  // namespace

MlpHead::~MlpHead() = default;

int MlpHead::widest() const {
  int w = 0;
  for (int s : sizes) w = std::max(w, s);
  return w;
}

void mlp_set(MlpHead& m, const Tree& t, const int* sizes, int n_sizes, const double* w,
             size_t n_w) {
  if (n_sizes == 0) {
    m.active = false;
    m.sizes.clear();
    return;
  }
  m.K = t.C - 1;
  m.sizes.assign(sizes, sizes + n_sizes);
  if (n_sizes < 2 || m.sizes.front() != 22 + m.K || m.sizes.back() != 3)
    throw Error(DPL_ERR_DATA, "mlp head: sizes must run from 22 + K inputs to 3 outputs");
  m.offs.clear();
  size_t n = 0;
  for (int l = 0; l + 1 < n_sizes; ++l) {
    m.offs.push_back(n);
    n += (size_t)m.sizes[l + 1] * m.sizes[l] + m.sizes[l + 1];
  }
  if (n != n_w) throw Error(DPL_ERR_DATA, "mlp head: weight count does not match the sizes");
  m.n_w = n;
  m.device = t.device;
  // fp32 weights: the host fp64 array goes up once, converted on the device
  DevBuf w64;
  w64.reserve(n * 8);
  DPL_CUDA(cudaMemcpyAsync(w64.p, w, n * 8, cudaMemcpyHostToDevice, t.stream));
  m.w32.reserve(n * 4);
  k_to_f32<<<blocks_for(n, 256), 256, 0, t.stream>>>(w64.as<double>(), n, m.w32.as<float>());
  count_launch();
  m.dw64.reserve(n * 8);
  DPL_CUDA(cudaMemsetAsync(m.dw64.p, 0, n * 8, t.stream));
  // tensor-core B images of every layer's W and W^T (weights change only here)
  m.img_fwd.clear(), m.img_bwd.clear();
  size_t ib = 0;
  for (int l = 0; l + 1 < n_sizes; ++l) {
    const int rows = m.sizes[l + 1], cols = m.sizes[l];
    m.img_fwd.push_back(ib);
    ib += tc_b_image_bytes(rows, cols);
    m.img_bwd.push_back(ib);
    ib += tc_b_image_bytes(cols, rows);
  }
  m.img.reserve(ib);
  for (int l = 0; l + 1 < n_sizes; ++l) {
    const int rows = m.sizes[l + 1], cols = m.sizes[l];
    const float* W = m.w32.as<float>() + m.offs[l];
    tc_b_image(W, cols, true, rows, cols, m.img.as<uint8_t>() + m.img_fwd[l], t.stream);
    tc_b_image(W, cols, false, cols, rows, m.img.as<uint8_t>() + m.img_bwd[l], t.stream);
  }
  DPL_CUDA(cudaStreamSynchronize(t.stream));
  m.active = true;
  ++m.version;
}

void mlp_inputs(cudaStream_t s, const double* rays, int S, const double* xs, const float* vals,
                int C, const float* g0, int64_t q0, int64_t q, int K, float* X, int ldx) {
  k_inputs<<<blocks_for(q, 256), 256, 0, s>>>(rays, S, xs, vals, C, g0, q0, q, K, X, ldx);
  count_launch();
}

// layer l: out (q x rows) = in (q x cols) . W^T + b, ReLU except on the last layer
static void layer_fwd(MlpHead& m, cudaStream_t s, int l, const float* in, int64_t q, float* out) {
  const int rows = m.sizes[l + 1], cols = m.sizes[l];
  const int lda = l == 0 ? m.ldx() : cols;  // the input rows X are padded to 16 bytes
  const float* W = m.w32.as<float>() + m.offs[l];
  const bool last = l + 2 == (int)m.sizes.size();
  TcGemm g;
  g.M = (int)q, g.N = rows, g.K = cols;
  g.A = in, g.lda = lda;              // in[q][cols]
  g.B = W, g.ldb = cols;              // W[rows][cols]
  g.b_image = m.img.as<uint8_t>() + m.img_fwd[l];
  g.D = out, g.ldd = rows;
  g.bias = W + (size_t)rows * cols;
  g.epi = last ? TC_BIAS : TC_BIAS_RELU;
  tc_gemm(g, m.device, s);
}

void mlp_forward(MlpHead& m, cudaStream_t s, const float* X, int64_t q, float* raw, float* keep) {
  const int L = (int)m.sizes.size() - 1;
  const size_t wide = (size_t)m.widest();
  const float* in = X;
  if (keep) {  // layer-major block: act[l] at keep + q * (sizes[1] + .. + sizes[l-1])
    float* p = keep;
    for (int l = 0; l < L; ++l) {
      float* out = l + 1 == L ? raw : p;
      layer_fwd(m, s, l, in, q, out);
      in = out;
      p += (size_t)q * m.sizes[l + 1];
    }
    return;
  }
  m.ws.reserve(2 * (size_t)q * wide * 4);
  float* buf[2] = {m.ws.as<float>(), m.ws.as<float>() + (size_t)q * wide};
  for (int l = 0; l < L; ++l) {
    float* out = l + 1 == L ? raw : buf[l & 1];
    layer_fwd(m, s, l, in, q, out);
    in = out;
  }
}

void mlp_backward(MlpHead& m, cudaStream_t s, const float* X, int64_t q, const float* d_raw,
                  float* dX, const float* kept) {
  const int L = (int)m.sizes.size() - 1;
  // recompute the chunk's activations (Mlp::Tape), then walk back (:95-119)
  size_t acts = 0;
  for (int l = 1; l <= L; ++l) acts += (size_t)m.sizes[l];
  const size_t wide = (size_t)m.widest();
  m.ws.reserve(((kept ? 0 : (size_t)q * acts) + 2 * (size_t)q * wide) * 4);
  std::vector<float*> act(L + 1);
  act[0] = const_cast<float*>(X);
  float* p = kept ? const_cast<float*>(kept) : m.ws.as<float>();
  for (int l = 1; l <= L; ++l) {
    act[l] = p;  // act[L] (the raw outputs) is never read by the backward
    p += (size_t)q * m.sizes[l];
  }
  float* dbuf[2];
  dbuf[0] = kept ? m.ws.as<float>() : p;
  dbuf[1] = dbuf[0] + (size_t)q * wide;
  if (!kept)
    for (int l = 0; l < L; ++l) layer_fwd(m, s, l, act[l], q, act[l + 1]);
  // delta: d loss / d (output of layer l), already through that layer's ReLU
  const float* delta = d_raw;
  double* dw = m.dw64.as<double>();
  for (int l = L - 1; l >= 0; --l) {
    const int rows = m.sizes[l + 1], cols = m.sizes[l];
    const float* W = m.w32.as<float>() + m.offs[l];
    // narrow output (the rgb layer): both products at memory speed on the FP32 pipe
    if (rows == 3 && (cols & 3) == 0) {
      const int ldin = l == 0 ? m.ldx() : cols;
      k_narrow_dw<3><<<std::max(1, 148 * 8 / ((cols + 255) / 256)), std::min(256, cols), 0, s>>>(
          delta, act[l], q, cols, ldin, dw + m.offs[l], dw + m.offs[l] + (size_t)rows * cols);
      float* out = l == 0 ? dX : dbuf[l & 1];
      k_narrow_dx<3><<<blocks_for(q * (cols >> 2), 256), 256, 0, s>>>(
          delta, W, l > 0 ? act[l] : nullptr, q, cols, out);
      count_launch(2);
      delta = out;
      continue;
    }
    // dW (rows x cols) += delta^T . in over the chunk's samples (split-K, fp64
    // accumulation into RenderGrads::d_head_w)
    TcGemm gw;
    gw.M = rows, gw.N = cols, gw.K = (int)q;
    gw.A = delta, gw.lda = rows, gw.a_kcontig = false;   // A[r][q] = delta[q][r]
    gw.B = act[l], gw.ldb = l == 0 ? m.ldx() : cols, gw.b_kcontig = false;  // B[c][q] = in[q][c]
    gw.D64 = dw + m.offs[l], gw.ldd = cols;
    gw.epi = TC_ACC64;
    // one wave of CTAs: the M x N tiles times the K slices ~ the SM count
    const int tiles = ((rows + 127) / 128) * ((cols + 127) / 128);
    gw.split_k = (int)std::max<int64_t>(1, std::min<int64_t>(2 * 148 / tiles, q / 1024));
    // db = column sums of delta, summed by the same CTAs as A's row sums
    gw.bias_grad = dw + m.offs[l] + (size_t)rows * cols;
    tc_gemm(gw, m.device, s);
    // d_in (q x cols) = delta . W, through the ReLU of the layer below (its
    // output is act[l], Mlp::backward's gate, radiance.cpp:105-107)
    TcGemm gi;
    gi.M = (int)q, gi.N = cols, gi.K = rows;
    gi.A = delta, gi.lda = rows;                      // delta[q][rows]
    gi.B = W, gi.ldb = cols, gi.b_kcontig = false;    // B[c][r] = W[r][c]
    gi.b_image = m.img.as<uint8_t>() + m.img_bwd[l];
    gi.D = l == 0 ? dX : dbuf[l & 1], gi.ldd = cols;
    if (l > 0) {
      gi.epi = TC_GATE;
      gi.aux = act[l], gi.ldaux = cols;
    }
    tc_gemm(gi, m.device, s);
    delta = gi.D;
  }
}

}  // namespace dpl
