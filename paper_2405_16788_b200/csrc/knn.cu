// knn.cu — OrientedPointCloud::mean_knn_spacing on the GPU (SceneModel's
// default eps = 1.5 x this, proj/src/fields.cpp:10-11; pointcloud.cpp:51-65).
//
// For every point: the k nearest OTHER points (the reference takes the k+1
// nearest including the point itself and drops the first), distances
// sqrt((dx*dx + dy*dy) + dz*dz) in fp64 without FMA — the same values the
// reference's kd-tree produces. Exact kNN over a uniform grid: points are
// bucketed by cell (CUB radix sort), each query scans rings of cells until
// the ring lower bound exceeds its current k+1-th distance. The per-point
// sums of the k distances (ascending) are reduced in fp64; only the order of
// the final sum differs from the reference's sequential loop (ulp level).
#include <cub/cub.cuh>

#include "knn.cuh"

namespace dpl {

constexpr int KNN_MAX = 32;

__global__ void k_cell_ids(const double* __restrict__ pos, int64_t n, double lx, double ly,
                           double lz, double inv_h, int gx, int gy, int gz, uint32_t* cell,
                           int32_t* idx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int cx = min(gx - 1, max(0, (int)((pos[3 * i] - lx) * inv_h)));
  int cy = min(gy - 1, max(0, (int)((pos[3 * i + 1] - ly) * inv_h)));
  int cz = min(gz - 1, max(0, (int)((pos[3 * i + 2] - lz) * inv_h)));
  cell[i] = (uint32_t)((cz * gy + cy) * gx + cx);
  idx[i] = (int32_t)i;
}

__global__ void k_cell_starts(const uint32_t* __restrict__ cell_sorted, int64_t n,
                              int32_t* start, int32_t* end) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t c = cell_sorted[i];
  if (i == 0 || cell_sorted[i - 1] != c) start[c] = (int32_t)i;
  if (i == n - 1 || cell_sorted[i + 1] != c) end[c] = (int32_t)(i + 1);
}

__global__ void k_knn_sum(const double* __restrict__ pos, const int32_t* __restrict__ idx_sorted,
                          const int32_t* __restrict__ cstart, const int32_t* __restrict__ cend,
                          int64_t n, int kk, double lx, double ly, double lz, double h,
                          double inv_h, int gx, int gy, int gz, double* sums, int32_t* counts) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double qx = pos[3 * i], qy = pos[3 * i + 1], qz = pos[3 * i + 2];
  const int cx = min(gx - 1, max(0, (int)((qx - lx) * inv_h)));
  const int cy = min(gy - 1, max(0, (int)((qy - ly) * inv_h)));
  const int cz = min(gz - 1, max(0, (int)((qz - lz) * inv_h)));
  double best[KNN_MAX];  // ascending squared distances
  int nb = 0;
  const int maxring = max(gx, max(gy, gz));
  for (int ring = 0; ring <= maxring; ++ring) {
    for (int z = cz - ring; z <= cz + ring; ++z) {
      if (z < 0 || z >= gz) continue;
      for (int y = cy - ring; y <= cy + ring; ++y) {
        if (y < 0 || y >= gy) continue;
        const bool edge_yz = (z == cz - ring || z == cz + ring || y == cy - ring || y == cy + ring);
        for (int x = cx - ring; x <= cx + ring; x += (edge_yz ? 1 : 2 * ring)) {
          if (x >= 0 && x < gx) {
            const int c = (z * gy + y) * gx + x;
            for (int s = cstart[c]; s < cend[c]; ++s) {
              const int64_t j = idx_sorted[s];
              const double dx = __dsub_rn(pos[3 * j], qx), dy = __dsub_rn(pos[3 * j + 1], qy),
                           dz = __dsub_rn(pos[3 * j + 2], qz);
              const double d2 =
                  __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
              if (nb < kk || d2 < best[nb - 1]) {
                int w = nb < kk ? nb++ : kk - 1;
                while (w > 0 && best[w - 1] > d2) best[w] = best[w - 1], --w;
                best[w] = d2;
              }
            }
          }
          if (ring == 0) break;
        }
      }
    }
    // every unvisited point lies at least ring * h away along some axis
    const double reach = ring * h;
    if (nb == kk && best[kk - 1] <= reach * reach) break;
  }
  double s = 0.0;
  for (int j = 1; j < nb; ++j) s = __dadd_rn(s, __dsqrt_rn(best[j]));
  sums[i] = s;
  counts[i] = nb > 0 ? nb - 1 : 0;
}

double mean_knn_spacing(cudaStream_t st, const double* pos_dev, int64_t n, int k, DevBuf* ws) {
  if (n < 2) return 0.0;
  const int kk = (int)std::min<int64_t>(k + 1, n);
  if (kk > KNN_MAX) throw Error(1, "mean_knn_spacing: k > 31 not supported");
  // bounding box on the host (positions are copied back once; n x 24 bytes)
  std::vector<double> hp(n * 3);
  DPL_CUDA(cudaMemcpyAsync(hp.data(), pos_dev, n * 24, cudaMemcpyDeviceToHost, st));
  DPL_CUDA(cudaStreamSynchronize(st));
  double lo[3], hi[3];
  for (int a = 0; a < 3; ++a) lo[a] = hi[a] = hp[a];
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], hp[3 * i + a]);
      hi[a] = std::max(hi[a], hp[3 * i + a]);
    }
  double ext = std::max(hi[0] - lo[0], std::max(hi[1] - lo[1], hi[2] - lo[2]));
  if (!(ext > 0)) ext = 1.0;
  // ~2 points per cell for a volume fill; clamp the grid to 2^30 cells
  double h = ext / std::cbrt((double)n / 2.0);
  int g[3];
  for (;;) {
    for (int a = 0; a < 3; ++a) g[a] = std::max(1, (int)((hi[a] - lo[a]) / h) + 1);
    if ((double)g[0] * g[1] * g[2] <= (double)(1 << 28)) break;
    h *= 1.25;
  }
  const int64_t cells = (int64_t)g[0] * g[1] * g[2];
  DevBuf& b0 = ws[0];
  DevBuf& b1 = ws[1];
  DevBuf& b2 = ws[2];
  b0.reserve(n * 16 + 256);
  uint32_t* cell = b0.as<uint32_t>();
  uint32_t* cell_s = cell + n;
  int32_t* idx = reinterpret_cast<int32_t*>(cell_s + n);
  int32_t* idx_s = idx + n;
  b1.reserve(cells * 8 + 16);
  int32_t* cs = b1.as<int32_t>();
  int32_t* ce = cs + cells;
  const int B = 256;
  const unsigned grid = (unsigned)((n + B - 1) / B);
  k_cell_ids<<<grid, B, 0, st>>>(pos_dev, n, lo[0], lo[1], lo[2], 1.0 / h, g[0], g[1], g[2], cell,
                                 idx);
  count_launch();
  size_t tb = 0;
  int bits = 1;
  while ((1ll << bits) < cells) ++bits;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, cell, cell_s, idx, idx_s, (int)n, 0, bits, st);
  b2.reserve(std::max<size_t>(tb, (size_t)n * 12) + 256);
  DPL_CUDA(cub::DeviceRadixSort::SortPairs(b2.p, tb, cell, cell_s, idx, idx_s, (int)n, 0, bits, st));
  count_launch(3);
  DPL_CUDA(cudaMemsetAsync(cs, 0, cells * 4, st));
  DPL_CUDA(cudaMemsetAsync(ce, 0, cells * 4, st));
  k_cell_starts<<<grid, B, 0, st>>>(cell_s, n, cs, ce);
  count_launch();
  double* sums = reinterpret_cast<double*>(b2.p);  // sort temp no longer needed
  int32_t* cnts = reinterpret_cast<int32_t*>(sums + n);
  k_knn_sum<<<grid, B, 0, st>>>(pos_dev, idx_s, cs, ce, n, kk, lo[0], lo[1], lo[2], h, 1.0 / h,
                                  g[0], g[1], g[2], sums, cnts);
  count_launch();
  DPL_CUDA(cudaGetLastError());
  std::vector<double> hs(n);
  std::vector<int32_t> hc(n);
  DPL_CUDA(cudaMemcpyAsync(hs.data(), sums, n * 8, cudaMemcpyDeviceToHost, st));
  DPL_CUDA(cudaMemcpyAsync(hc.data(), cnts, n * 4, cudaMemcpyDeviceToHost, st));
  DPL_CUDA(cudaStreamSynchronize(st));
  double s = 0;
  int64_t c = 0;
  for (int64_t i = 0; i < n; ++i) s += hs[i], c += hc[i];  // point order, as the reference
  return c ? s / (double)c : 0.0;
}

}  // namespace dpl
