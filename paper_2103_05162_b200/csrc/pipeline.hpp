// Host-side pieces of the device pipeline shared between translation units.
#pragma once

#include <cfloat>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

#include "bvh.cuh"
#include "engine.hpp"

namespace tcb {

// Device-side counters / small reductions of one run (one memset per run).
struct DevCounters {
  unsigned long long pairs;
  unsigned long long dists;
  long long clusters;
  long long cores;
  long long noise;
  unsigned long long key_and;  // AND / OR over the keys of the current sort
  unsigned long long key_or;
  uint32_t bounds_ord[6];      // order-preserving encodings: min xyz, max xyz
  int32_t nonfinite;
  int32_t count_a;             // generic device-side counts (cells, prims ...)
  int32_t count_b;
  int32_t pad;
  unsigned long long probe[8];  // -DTCB_PROBE builds only (make probe): work counters
};

#ifdef TCB_PROBE
#define TCB_PROBE_ONLY(...) __VA_ARGS__
#else
#define TCB_PROBE_ONLY(...)
#endif

// Stream-ordered scratch allocations released at scope exit (pool_alloc: the
// library's private per-device pool, so repeat calls reuse HBM instead of
// re-mapping it).
class Scratch {
 public:
  explicit Scratch(cudaStream_t s) : stream_(s) {}
  ~Scratch();
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  void* alloc(size_t bytes);
  template <typename T>
  T* alloc_n(int64_t count) {
    return static_cast<T*>(alloc(static_cast<size_t>(count > 0 ? count : 1) * sizeof(T)));
  }
  cudaStream_t stream() const { return stream_; }

 private:
  cudaStream_t stream_;
  std::vector<void*> ptrs_;
};

// Small pinned host staging buffer (thread-local) for device->host reads that
// size later launches.
void* pinned_staging(size_t bytes);

// Timing events for the stages of one run.
class StageClock {
 public:
  explicit StageClock(cudaStream_t s);
  ~StageClock();
  void mark(int stage_begin);  // record an event that opens `stage_begin`
  void finish();               // record the closing event
  // Elapsed ms of each stage (call after the stream is synchronized).
  void collect(double* stage_ms) const;

 private:
  cudaStream_t stream_;
  cudaEvent_t ev_[kNumStages + 1];
  int stage_of_[kNumStages + 1];
  int count_ = 0;
};

// ---- BVH construction (build.cu) ----

// Primitive source for the build: either points (degenerate boxes, read from
// the row-major coords) or explicit boxes.
struct PrimSource {
  const float* coords = nullptr;  // points mode: n*D floats
  const float4* lo = nullptr;     // boxes mode
  const float4* hi = nullptr;
  const int32_t* aux = nullptr;   // leaf payload per primitive (nullptr: primitive index)
  int64_t count = 0;
};

struct BuiltBvh {
  DeviceBvh tree;
  float4* leaf_pt = nullptr;          // points mode only: rank -> (x, y, z, id bits)
  const uint64_t* codes = nullptr;    // sorted Morton codes (leaf rank order)
  const uint32_t* scene_ord = nullptr;  // Morton scene box (order-preserving bits, 6)
  int sort_passes = 0;
};

// Builds the LBVH of bvh.cpp:10-124 (scene bounds over centroids, Morton,
// stable (code, index) sort, Karras topology, refit). Checks the points for
// non-finite coordinates when validate_finite (throws InvalidArgument).
// stream_ordered: no host synchronization (the sort passes are planned on the
// device, see radix_sort_pairs_prefix_async); a non-finite coordinate only
// sets d_ctr->nonfinite, which the traversal kernels honour by doing nothing
// and the caller must check or report.
template <int D>
BuiltBvh build_bvh(const PrimSource& src, bool validate_finite, DevCounters* d_ctr,
                   Scratch& scratch, StageClock* clock, bool stream_ordered = false);

// Raw point bounds into d_ctr->bounds_ord + finiteness flag (resets both).
template <int D>
void launch_point_bounds(const float* coords, int64_t n, DevCounters* d_ctr, cudaStream_t s);

// ---- traversal / finalize (dbscan.cu) ----
// FDBSCAN core pass / main pass: flags and parent are indexed by LEAF RANK.
template <int D>
void fdbscan_core_pass(const BuiltBvh& b, int64_t n, double eps2, int minpts,
                       uint8_t* flags, DevCounters* d_ctr, cudaStream_t s);
// force_core (minpts == 2) uses the contained-subtree pass (k_fd_main_fof) and
// allocates its run-coverage scratch from `scratch`.
// key[rank]: the element's key; roots are the minimum-key element of a set.
template <int D>
void fdbscan_main_pass(const BuiltBvh& b, const int32_t* key, int64_t n, double eps2,
                       bool force_core, uint8_t* flags, int32_t* parent, DevCounters* d_ctr,
                       Scratch& scratch);
// out[rank] = keys[order[rank]]
void gather_rank_keys(const int32_t* keys, const int32_t* order, int64_t n, int32_t* out,
                      cudaStream_t s);
// Moves per-point bytes between input order and leaf-rank order:
// to_rank: dst[r] = src[order[r]]; else dst[order[r]] = src[r].
void permute_flags(const uint8_t* src, const int32_t* order, int64_t n, uint8_t* dst,
                   bool to_rank, cudaStream_t s);
void init_union_find(int32_t* parent, uint8_t* flags, int64_t n, cudaStream_t s);
// Throws InvalidArgument when any of the n caller keys is negative (syncs).
void check_keys_nonnegative(const int32_t* keys, int64_t n, Scratch& scratch);
// FDBSCAN finalize in rank space: labels[order[rank]] = key of the rank's
// root (or -1), core flags likewise, through destination buckets
// (k_fin_bucket, then k_fin_window / k_fin_scatter, dbscan.cu): whole-sector
// output writes. With a sink, the output is written in 8 contiguous ranges,
// each handed to the sink once final.
void finalize_labels_bucketed(int32_t* parent, uint8_t* flags, const int32_t* key,
                              const int32_t* order, int64_t n, int32_t* labels,
                              uint8_t* core_out, DevCounters* d_ctr, Scratch& scratch,
                              bool force_core, const ChunkSink* sink = nullptr);

// ---- whole FDBSCAN pipeline over the point BVH (engine.cu) ----
// d_keys (optional): unique int32 key per point; labels are then the key of
// each cluster's minimum-key core instead of its minimum index.
template <int D>
void run_fdbscan(const float* d_coords, int64_t n, float eps, int minpts, int32_t* d_labels,
                 uint8_t* d_core, DevCounters* ctr, Scratch& scratch, StageClock& clock,
                 const int32_t* d_keys = nullptr, const ChunkSink* sink = nullptr);

// ---- DenseBox (grid.cu) ----
struct GridParams;  // cell side, origin, extents (grid.cu)
// build_grid (dense_grid.cpp:23-77) on the device plus the primitive counts of
// make_mixed_primitives (dense_grid.cpp:79-98). Cells are in cell-id order,
// members of a cell in index order (perm), exactly the reference's grid.
struct DeviceGrid {
  const GridParams* params = nullptr;
  const uint64_t* ids = nullptr;    // sorted cell id per sorted position
  const int32_t* perm = nullptr;    // sorted position -> point index
  uint64_t* spare_keys = nullptr;   // n-entry sort buffers free for reuse
  int32_t* spare_vals = nullptr;
  void* sort_tmp = nullptr;
  void* scan_tmp = nullptr;
  int32_t* cell_of_sorted = nullptr;  // sorted position -> cell
  int32_t* cell_begin = nullptr;      // num_cells (first sorted position)
  float4* sorted_pt = nullptr;        // (x, y, z, point index bits) in sorted order
  int32_t num_cells = 0;
  int32_t* cell_end = nullptr;
  uint8_t* cell_dense = nullptr;
  int32_t* prim_off = nullptr;        // first primitive of each cell
  int32_t num_prims = 0, num_dense = 0;
};
// stop_if_no_dense: return right after the cell sort (num_dense = 0, only
// params / ids / perm / sort buffers set) when no cell holds minpts points.
template <int D>
DeviceGrid build_device_grid(const float* d_coords, int64_t n, float eps, int minpts,
                             DevCounters* ctr, Scratch& scratch, bool stop_if_no_dense = false);
// Primitive boxes and payloads (point index, or ~cell for a DenseBox).
template <int D>
void build_mixed_prims(const DeviceGrid& g, int64_t n, Scratch& scratch, float4** lo,
                       float4** hi, int32_t** aux);
template <int D>
void run_densebox(const float* d_coords, int64_t n, float eps, int minpts,
                  int32_t* d_labels, uint8_t* d_core, DevCounters* d_ctr,
                  Scratch& scratch, StageClock& clock, double* dense_fraction);

// ---- brute force (bruteforce.cu) ----
template <int D>
void run_bruteforce(const float* d_coords, int64_t n, float eps, int minpts,
                    int32_t* d_labels, uint8_t* d_core, DevCounters* d_ctr,
                    Scratch& scratch);

#ifdef __CUDACC__
// One atomic per block (not per warp): ~1k same-address atomics instead of
// ~1e5 serialized ones at the L2 slice.
template <int D>
__device__ __forceinline__ void publish_bounds(float* mn, float* mx, bool bad, DevCounters* ctr) {
  __shared__ float red[32];
  auto fmin_op = [](float a, float b) { return fminf(a, b); };
  auto fmax_op = [](float a, float b) { return fmaxf(a, b); };
#pragma unroll
  for (int k = 0; k < D; ++k) {
    float lo = block_reduce(mn[k], fmin_op, FLT_MAX, red);
    if (threadIdx.x == 0) atomicMin(&ctr->bounds_ord[k], f2ord(lo));
    float hi = block_reduce(mx[k], fmax_op, -FLT_MAX, red);
    if (threadIdx.x == 0) atomicMax(&ctr->bounds_ord[3 + k], f2ord(hi));
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&ctr->nonfinite, 1);
}

__device__ __forceinline__ void publish_and_or(uint64_t a, uint64_t o, DevCounters* ctr) {
  __shared__ unsigned long long red64[32];
  auto and_op = [](unsigned long long x, unsigned long long y) { return x & y; };
  auto or_op = [](unsigned long long x, unsigned long long y) { return x | y; };
  unsigned long long ra = block_reduce<unsigned long long>(a, and_op, ~0ull, red64);
  if (threadIdx.x == 0) atomicAnd(&ctr->key_and, ra);
  unsigned long long ro = block_reduce<unsigned long long>(o, or_op, 0ull, red64);
  if (threadIdx.x == 0) atomicOr(&ctr->key_or, ro);
}

#endif

inline unsigned grid_for(int64_t work, int block, int64_t max_blocks = 148 * 64);

inline unsigned grid_for(int64_t work, int block, int64_t max_blocks) {
  int64_t b = (work + block - 1) / block;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return static_cast<unsigned>(b);
}

}  // namespace tcb
