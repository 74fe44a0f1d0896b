// FDBSCAN passes over the point BVH, and label finalization.
//
//   k_fd_core   fdbscan_mark_cores (dbscan.cpp:36-58): one thread per leaf
//               rank (Morton order, so a warp's queries are spatial
//               neighbours and walk nearly the same nodes), unmasked query,
//               early exit once minpts neighbours (self included) are seen.
//   k_fd_main   fdbscan_main_phase (dbscan.cpp:60-88): rank-masked query so
//               every unordered within-eps pair is found exactly once, each
//               pair resolved on the spot with the lock-free union-find; no
//               neighbour list is ever stored.
//   k_finalize  UnionFind::flatten + finalize_labels + the stats loop
//               (union_find.hpp:77-86, dbscan.cpp:202-219, :274-282).
//
// For point leaves the leaf box test IS the exact distance test (the box is
// degenerate and box_distance_sq reduces to distance_sq term by term, the
// subtraction merely negated), so a visited leaf is a within-eps neighbour
// and its distance is not recomputed.
#include <cmath>

#include "device_common.cuh"
#include "pipeline.hpp"

namespace tcb {

namespace {

constexpr int kQueryBlock = 128;

template <int D>
__device__ __forceinline__ void load_query(const float4* leaf_pt, int64_t r, float* p,
                                           int32_t* id) {
  float4 q = leaf_pt[r];
  p[0] = q.x;
  p[1] = q.y;
  if (D == 3) p[2] = q.z;
  *id = __float_as_int(q.w);
}

__device__ __forceinline__ void flush_counter(unsigned long long* dst, unsigned long long v) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

// fdbscan_mark_cores query (dbscan.cpp:36-58): unmasked, early exit once
// minpts neighbours (self included) are seen.
template <int D>
struct CoreQuery {
  const float4* __restrict__ nodes;
  const float4* __restrict__ leaf_pt;
  BallTest bt;
  int minpts;
  uint8_t* __restrict__ flags;
  int32_t* stack;  // per-thread traversal stack, kept outside the struct
  unsigned long long dists = 0;
  float p[3];
  int32_t id, node;
  int count, top;
  __device__ bool begin(int64_t r) {
    load_query<D>(leaf_pt, r, p, &id);
    id = static_cast<int32_t>(r);  // flags are kept in rank space
    count = 0;
    node = 0;
    top = 0;
    return true;
  }
  __device__ bool step() {
    auto visit = [&](int32_t, int32_t, const float*, const float*) -> bool {
      ++dists;
      return ++count < minpts;  // early exit (dbscan.cpp:48-53)
    };
    return bvh_step<D>(nodes, p, bt, 0, node, top, stack, visit);
  }
  __device__ void end() {
    if (count >= minpts) flags[id] = 1;
  }
};

template <int D>
__global__ void __launch_bounds__(kQueryBlock)
k_fd_core(const float4* __restrict__ nodes, const float4* __restrict__ leaf_pt, int64_t m,
          BallTest bt, int minpts, uint8_t* __restrict__ flags, DevCounters* ctr, bool persistent) {
  int32_t stack[kStackDepth];
  CoreQuery<D> q{nodes, leaf_pt, bt, minpts, flags, stack};
  if (persistent)
    run_query_queue(m, &ctr->queue[0], q);
  else
    run_query_direct(m, q);
  flush_counter(&ctr->dists, q.dists);
}

// fdbscan_main_phase (dbscan.cpp:60-88): one thread per leaf rank r (Morton
// order, so a warp's queries are spatial neighbours walking nearly the same
// nodes), top-down query masked at r so each unordered within-eps pair is met
// exactly once, and resolved on the spot — no neighbour list is stored.
template <int D, bool kForceCore>
__global__ void __launch_bounds__(kQueryBlock)
k_fd_main(const float4* __restrict__ nodes, const float4* __restrict__ leaf_pt, int64_t m,
          BallTest bt, const uint8_t* __restrict__ flags, int32_t* __restrict__ parent,
          const int32_t* __restrict__ key, DevCounters* ctr) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  unsigned long long pairs = 0;
  if (r < m) {
    float p[3];
    int32_t id;
    load_query<D>(leaf_pt, r, p, &id);
    const int32_t rank = static_cast<int32_t>(r);
    const bool core_r = kForceCore ? true : flags[rank] != 0;
    int32_t hint = rank;
    bool settled = false;
    auto visit = [&](int32_t s, int32_t, const float*, const float*) -> bool {
      if (s == rank) return true;
      ++pairs;
      if (kForceCore)
        uf_unite_hinted_keyed(parent, key, rank, s, hint);  // all pairs core-core (dbscan.hpp:85-89)
      else
        resolve_pair_keyed(rank, s, core_r, flags, parent, key, hint, settled);
      return true;
    };
    bvh_query<D>(nodes, p, bt, rank, visit);
  }
  flush_counter(&ctr->pairs, pairs);
  flush_counter(&ctr->dists, pairs);
}

__global__ void k_permute(const uint8_t* __restrict__ src, const int32_t* __restrict__ order,
                          int64_t n, uint8_t* __restrict__ dst, bool to_rank) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (to_rank)
      dst[r] = src[order[r]];
    else
      dst[order[r]] = src[r];
  }
}

__global__ void k_init_uf(int32_t* __restrict__ parent, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    parent[i] = static_cast<int32_t>(i);
}

// minpts == 2: a point is core iff some other point lies within eps, i.e.
// iff it shares a union-find set with another point. Flatten, and mark every
// non-root point and the root it hangs under (the reference sets both flags
// per pair instead, dbscan.hpp:85-88; the final flags are the same).
__global__ void __launch_bounds__(256)
k_flatten_mark(int32_t* __restrict__ parent, uint8_t* __restrict__ flags, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t p = ld_relaxed(parent + i);
    if (p == static_cast<int32_t>(i)) continue;
    int32_t q;
    while (p != (q = ld_relaxed(parent + p))) p = q;
    st_relaxed(parent + i, p);
    flags[i] = 1;
    if (!flags[p]) flags[p] = 1;
  }
}

// Rank-space finalize (FDBSCAN): flatten over ranks; outputs scattered back
// to input order through key[rank] = original index. The representative of a
// set is its minimum-key rank, so label = key[root] = minimum original index.
__global__ void __launch_bounds__(256)
k_finalize_ranks(int32_t* __restrict__ parent, const uint8_t* __restrict__ flags,
                 const int32_t* __restrict__ key, int64_t n, int32_t* __restrict__ labels,
                 uint8_t* __restrict__ core_out, DevCounters* ctr) {
  long long noise = 0, clusters = 0, cores = 0;
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < n;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t p = ld_relaxed(parent + s);
    int32_t q;
    while (p != (q = ld_relaxed(parent + p))) p = q;
    st_relaxed(parent + s, p);
    const bool core = flags[s] != 0;
    const int32_t i = key[s];
    const int32_t lab = (core || p != s) ? key[p] : -1;  // dbscan.cpp:215
    labels[i] = lab;
    core_out[i] = core ? 1 : 0;
    noise += lab == -1;
    clusters += lab == i;
    cores += core;
  }
  noise = warp_sum(noise);
  clusters = warp_sum(clusters);
  cores = warp_sum(cores);
  if ((threadIdx.x & 31) == 0) {
    if (noise) atomicAdd(reinterpret_cast<unsigned long long*>(&ctr->noise), noise);
    if (clusters) atomicAdd(reinterpret_cast<unsigned long long*>(&ctr->clusters), clusters);
    if (cores) atomicAdd(reinterpret_cast<unsigned long long*>(&ctr->cores), cores);
  }
}

__global__ void __launch_bounds__(256)
k_finalize(int32_t* __restrict__ parent, const uint8_t* __restrict__ flags, int64_t n,
           int32_t* __restrict__ labels, uint8_t* __restrict__ core_out, DevCounters* ctr) {
  long long noise = 0, clusters = 0, cores = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t p = ld_relaxed(parent + i);
    int32_t q;
    while (p != (q = ld_relaxed(parent + p))) p = q;
    st_relaxed(parent + i, p);
    const bool core = flags[i] != 0;
    const int32_t lab = (core || p != i) ? p : -1;  // dbscan.cpp:215
    labels[i] = lab;
    core_out[i] = core ? 1 : 0;
    noise += lab == -1;
    clusters += lab == static_cast<int32_t>(i);
    cores += core;
  }
  noise = warp_sum(noise);
  clusters = warp_sum(clusters);
  cores = warp_sum(cores);
  if ((threadIdx.x & 31) == 0) {
    if (noise) atomicAdd(reinterpret_cast<unsigned long long*>(&ctr->noise), noise);
    if (clusters) atomicAdd(reinterpret_cast<unsigned long long*>(&ctr->clusters), clusters);
    if (cores) atomicAdd(reinterpret_cast<unsigned long long*>(&ctr->cores), cores);
  }
}

}  // namespace

template <int D>
void fdbscan_core_pass(const BuiltBvh& b, int64_t n, double eps2, int minpts,
                       uint8_t* flags, DevCounters* d_ctr, cudaStream_t s) {
  note_launch(), k_fd_core<D><<<query_grid(k_fd_core<D>, n), kQueryBlock, 0, s>>>(
      b.tree.nodes, b.leaf_pt, n, BallTest::make(eps2), minpts, flags, d_ctr, query_mode() == 1);
  TCB_CUDA(cudaGetLastError());
}

template <int D>
void fdbscan_main_pass(const BuiltBvh& b, int64_t n, double eps2, bool force_core,
                       uint8_t* flags, int32_t* parent, DevCounters* d_ctr,
                       cudaStream_t s) {
  const BallTest bt = BallTest::make(eps2);
  auto launch = [&](auto kernel) {
    note_launch(), kernel<<<grid_for(n, kQueryBlock, INT32_MAX), kQueryBlock, 0, s>>>(
        b.tree.nodes, b.leaf_pt, n, bt, flags, parent, b.tree.leaf_order, d_ctr);
  };
  if (force_core)
    launch(k_fd_main<D, true>);
  else
    launch(k_fd_main<D, false>);
  TCB_CUDA(cudaGetLastError());
}

void permute_flags(const uint8_t* src, const int32_t* order, int64_t n, uint8_t* dst, bool to_rank,
                   cudaStream_t s) {
  note_launch(), k_permute<<<grid_for(n, 256), 256, 0, s>>>(src, order, n, dst, to_rank);
  TCB_CUDA(cudaGetLastError());
}

void init_union_find(int32_t* parent, uint8_t* flags, int64_t n, cudaStream_t s) {
  note_launch(), k_init_uf<<<grid_for(n, 256), 256, 0, s>>>(parent, n);
  TCB_CUDA(cudaMemsetAsync(flags, 0, static_cast<size_t>(n), s));
  TCB_CUDA(cudaGetLastError());
}

void finalize_labels_ranks(int32_t* parent, uint8_t* flags, const int32_t* key, int64_t n,
                           int32_t* labels, uint8_t* core_out, DevCounters* d_ctr, cudaStream_t s,
                           bool force_core) {
  if (force_core) note_launch(), k_flatten_mark<<<grid_for(n, 256), 256, 0, s>>>(parent, flags, n);
  note_launch(), k_finalize_ranks<<<grid_for(n, 256), 256, 0, s>>>(parent, flags, key, n, labels,
                                                                   core_out, d_ctr);
  TCB_CUDA(cudaGetLastError());
}

void finalize_labels(int32_t* parent, uint8_t* flags, int64_t n, int32_t* labels,
                     uint8_t* core_out, DevCounters* d_ctr, cudaStream_t s, bool force_core) {
  if (force_core) note_launch(), k_flatten_mark<<<grid_for(n, 256), 256, 0, s>>>(parent, flags, n);
  note_launch(), k_finalize<<<grid_for(n, 256), 256, 0, s>>>(parent, flags, n, labels, core_out, d_ctr);
  TCB_CUDA(cudaGetLastError());
}

template void fdbscan_core_pass<2>(const BuiltBvh&, int64_t, double, int, uint8_t*,
                                   DevCounters*, cudaStream_t);
template void fdbscan_core_pass<3>(const BuiltBvh&, int64_t, double, int, uint8_t*,
                                   DevCounters*, cudaStream_t);
template void fdbscan_main_pass<2>(const BuiltBvh&, int64_t, double, bool, uint8_t*,
                                   int32_t*, DevCounters*, cudaStream_t);
template void fdbscan_main_pass<3>(const BuiltBvh&, int64_t, double, bool, uint8_t*,
                                   int32_t*, DevCounters*, cudaStream_t);

}  // namespace tcb
