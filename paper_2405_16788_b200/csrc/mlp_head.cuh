// mlp_head.cuh — the tiny-MLP radiance head (radiance.hpp /
// radiance.cpp:40-180) for the batched render step.
//
// Input per sample (RadianceHead::eval, radiance.cpp:146-154): x (3),
// sh_encode(omega_head) (16), implicit normal (3), appearance channels (K).
// Dense ReLU layers, linear last layer, rgb = logistic(raw). Weights keep the
// reference's flat layout (per layer: rows x cols matrix, then the bias).
// The layers run on the tensor cores through tc_gemm.cuh (tcgen05, TMEM
// accumulators, 3xTF32 for fp32-class accuracy) with bias / ReLU / ReLU-gate
// fused into the epilogue; the weight gradient accumulates in fp64 like
// RenderGrads::d_head_w.
#pragma once

#include <vector>

#include "tree.cuh"

namespace dpl {

constexpr int kShDim = 16;

struct MlpHead {
  bool active = false;
  int device = 0;
  int K = 0;                 // appearance channels (= tree C - 1)
  std::vector<int> sizes;    // sizes[0] = 22 + K, back() = 3
  std::vector<size_t> offs;  // layer offsets into the flat weights
  size_t n_w = 0;
  DevBuf w32;   // fp32 weights, reference layout
  DevBuf dw64;  // fp64 weight gradient accumulator
  DevBuf ws;    // activations / deltas of one chunk
  // per layer: pre-split tensor-core images of W (forward: B[r][c] = W[r][c])
  // and of W^T (input gradient: B[c][r] = W[r][c]), built by mlp_set
  std::vector<size_t> img_fwd, img_bwd;  // byte offsets into img
  DevBuf img;
  uint64_t version = 0;  // bumped by mlp_set (kept activations belong to one set of weights)
  // fp32 activations per sample that a backward needs (outputs of layers 1..L-1... L)
  size_t acts_per_sample() const {
    size_t a = 0;
    for (size_t l = 1; l < sizes.size(); ++l) a += (size_t)sizes[l];
    return a;
  }
  ~MlpHead();
  int din() const { return sizes.empty() ? 0 : sizes.front(); }
  // row stride of the input rows X: din rounded up to 4 floats, so the first
  // layer's A rows are 16-byte aligned (the tensor-core GEMM's cp.async path)
  int ldx() const { return (din() + 3) & ~3; }
  int widest() const;
};

// set (or, with n_sizes == 0, clear) the head; w: host fp64, reference layout
void mlp_set(MlpHead& m, const Tree& t, const int* sizes, int n_sizes, const double* w, size_t n_w);

// X rows (fp32, q x din) from the render tape: x (fp64 positions), omega_head =
// -dir, n_hat from the channel-0 gradient (renderer.cpp:124-130), appearance
// = channels 1..K of vals (q x C)
void mlp_inputs(cudaStream_t s, const double* rays, int S, const double* xs, const float* vals,
                int C, const float* g0, int64_t q0, int64_t q, int K, float* X, int ldx);

// raw outputs (q x 3, fp32) of the samples [q0, q0 + q). keep != nullptr: the
// chunk's activations (q x acts_per_sample floats, layer-major) are written
// there for the backward — with 180 GB of HBM the render tape can hold them
// (34 GB for 8.4M samples of a 4 x 256 head) instead of recomputing the forward.
void mlp_forward(MlpHead& m, cudaStream_t s, const float* X, int64_t q, float* raw,
                 float* keep = nullptr);

// backward of a chunk: d_raw (q x 3) -> d_X (q x din); accumulates dW (fp64).
// kept: the activations mlp_forward stored for this chunk, or nullptr to
// recompute them (Mlp::Tape, radiance.cpp:59-93)
void mlp_backward(MlpHead& m, cudaStream_t s, const float* X, int64_t q, const float* d_raw,
                  float* dX, const float* kept = nullptr);

}  // namespace dpl
