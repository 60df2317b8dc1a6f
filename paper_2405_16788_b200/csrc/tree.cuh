// tree.cuh — host-side handle of one device-resident dipole tree.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "dpl_internal.cuh"

namespace dpl {

// Grow-only device allocation.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  bool guarded = false;  // allocated with guard zones (DPL_GUARD=1)
  void reserve(size_t b);
  void release();
  void swap(DevBuf& o);  // exchanges the allocations (and their guard registrations)
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
  ~DevBuf() { release(); }
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// DPL_GUARD=1: guard zones around every DevBuf (tree.cu)
int guard_check_all(std::string& msg);
int guard_live_count();

struct Tree {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;

  int64_t n = 0, nodes = 0;
  int C = 0, max_leaf = 8, max_depth = 20;
  std::vector<int64_t> level_off;  // BFS level offsets, size levels + 1
  std::vector<uint8_t> kinds;      // per channel, 0 Dipole, 1 Radial
  int Cd = 0, Cr = 0, PR = 0, F4 = 1;  // dipole / radial channel counts, radial pad, row float4s
  std::vector<int> dip_ch, rad_ch, slot_of;
  double root_lo[3] = {0, 0, 0}, root_hi[3] = {0, 0, 0};
  uint64_t version = 0;    // bumped by build / update_points (invalidates interaction lists)
  double thr_beta = -1.0;  // beta the thresholds were computed for (NaN-safe compare)
  bool thr_valid = false;

  // original-order point data (fp64, device)
  DevBuf pos64, nrm64, area64, mu64;
  // structure
  DevBuf order, leaf_of, pt_leaf;  // int32: sorted->orig, orig->leaf, sorted->leaf
  DevBuf node_ctr64, node_area64, node_rad64;  // double3 / double / double
  DevBuf node_dec, node_topo, node_parent, node_geo, node_flag;
  DevBuf node_sumv, node_sums;  // fp64 unnormalised moment sums (nodes x Cd x 3, nodes x Cr)
  DevBuf node_row, node_rec;  // fp32 payload rows (nodes x F4 float4), packed node records
  // sorted point data
  DevBuf pt_pos64, pt_geo, pt_row, pt_nrm, pt_mud, pt_rec;
  // tf32 hi / lo split of node_row / pt_row for the TMEM forward (DPL_FORWARD_TMEM)
  DevBuf node_row_split, pt_row_split;  // [row][hi | lo]
  DevBuf chmap;  // int32 [Cd dip ids | Cr rad ids]
  // scratch
  DevBuf scratch[8];

  // optional per-phase CUDA-event timing (dpl_profile_*)
  bool prof = false;
  struct Rec {
    int phase;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> ev_pool;
  cudaEvent_t take_event();

  TreeView view() const;
  void set_layout();  // from kinds: Cd, Cr, channel maps, upload
};

void tree_build(Tree& t, const double* pos, const double* nrm, const double* area,
                const double* mu, int64_t n, int C, int max_leaf, int max_depth);
void tree_update_points(Tree& t, const double* pos, const double* nrm, const double* area,
                        const double* mu);  // device pointers, original order
void tree_compute_moments(Tree& t);
// DPL_FORWARD_TMEM set: the tensor-memory forward (forward_tm.cu) is selected and
// tree_compute_moments also writes the split rows
bool forward_tmem_enabled();
void tree_refresh_sorted_positions(Tree& t);  // pt_pos64 / pt_geo from pos64 / area64
void tree_set_kinds(Tree& t, const uint8_t* kinds);
void tree_ensure_thresholds(Tree& t, double beta);
void tree_point_bbox(Tree& t, double lo[3], double hi[3]);  // current positions, synchronous
void tree_export(Tree& t, double* geo, int32_t* topo, int32_t* order, int32_t* leaf_of);
// fp64 normalised moments for all channels, both representations (dump)
void tree_full_moments(Tree& t, std::vector<double>& mv, std::vector<double>& ms);

KParams make_kparams(const double epsilon, int desingularized, double delta);

// profiling phases
enum Phase : int { PH_SORT = 0, PH_FORWARD = 1, PH_ADJOINT = 2, PH_FLUSH = 3, PH_RENDER = 4,
                   PH_MOMENTS = 5, PH_COUNT = 6 };

// RAII: records an event pair on the tree's stream around a phase when profiling
struct PhaseTimer {
  Tree& t;
  int phase;
  cudaEvent_t a = nullptr;
  PhaseTimer(Tree& tr, int ph);
  ~PhaseTimer();
};

}  // namespace dpl
