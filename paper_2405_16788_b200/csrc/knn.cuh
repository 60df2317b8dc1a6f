// knn.cuh — mean k-NN spacing (eps default) on the GPU.
#pragma once

#include "tree.cuh"

namespace dpl {

// pos_dev: n x 3 fp64 device array; ws: 3 scratch buffers
double mean_knn_spacing(cudaStream_t st, const double* pos_dev, int64_t n, int k, DevBuf* ws);

}  // namespace dpl
