// tc_gemm.cuh — fp32-accurate GEMM on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulator in TMEM) for the tiny-MLP head.
//
//   D[m][n] (op)= sum_k A[m][k] B[n][k]
//
// A is M x K and B is N x K; each operand is read from global memory either
// K-contiguous (X[row * ld + k]) or row-contiguous (X[k * ld + row]) and split
// into tf32 hi + lo parts: three MMAs per k-step (hi.hi + hi.lo + lo.hi), so
// each product carries ~2^-21 relative error (fp32-class, the 1e-4 parity bar
// with margin). A goes to tensor memory, B to shared memory in the canonical
// K-major SWIZZLE_128B layout — staged by the threads, or bulk-copied from a
// pre-split image (tc_b_image, for operands reused across calls such as
// weights). The epilogue is fused (bias, ReLU, ReLU gate, fp64 accumulation of
// split-K partial sums).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace dpl {

enum TcEpi : int {
  TC_STORE = 0,      // D = acc
  TC_BIAS_RELU = 1,  // D = max(acc + bias[n], 0)
  TC_BIAS = 2,       // D = acc + bias[n]
  TC_GATE = 3,       // D = aux[m][n] > 0 ? acc : 0   (ReLU backward)
  TC_ACC64 = 4,      // D64[m][n] += acc (fp64 atomics; split-K over gridDim.z)
};

struct TcGemm {
  int M = 0, N = 0, K = 0;
  const float* A = nullptr;
  int64_t lda = 0;
  bool a_kcontig = true;  // A[m * lda + k] (else A[k * lda + m])
  const float* B = nullptr;
  int64_t ldb = 0;
  bool b_kcontig = true;  // B[n * ldb + k] (else B[k * ldb + n])
  const uint8_t* b_image = nullptr;  // pre-split B (tc_b_image of the same N, K): used instead of B
  float* D = nullptr;     // D[m * ldd + n]
  double* D64 = nullptr;  // TC_ACC64 target, D64[m * ldd + n]
  int64_t ldd = 0;
  const float* bias = nullptr;  // N
  const float* aux = nullptr;   // TC_GATE: aux[m * ldaux + n]
  int64_t ldaux = 0;
  int epi = TC_STORE;
  int split_k = 1;  // TC_ACC64 only: K is cut into split_k slices (blockIdx.z)
  double* bias_grad = nullptr;  // TC_ACC64 only: += row sums of A (sum_k A[m][k])
};

void tc_gemm(const TcGemm& g, int device, cudaStream_t s);

// pre-split, pre-swizzled image of a B operand (N x K, read like TcGemm::B)
size_t tc_b_image_bytes(int N, int K);
void tc_b_image(const float* B, int64_t ldb, bool kcontig, int N, int K, uint8_t* img,
                cudaStream_t s);

}  // namespace dpl
