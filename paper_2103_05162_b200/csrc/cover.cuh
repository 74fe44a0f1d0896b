// Covered runs of contained subtrees (shared by the point and the DenseBox
// passes). A traversal that finds a subtree whose every leaf is a neighbour
// records the run [first, last] of leaf ranks as reach[first] =
// max(reach[first], last) (reach initialised to -1); afterwards every rank l
// covered by a run (first < l <= last for some run) is joined with l - 1 by
// `join(l)` — both lie in one run, so both are neighbours of that run's query.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "device_common.cuh"
#include "engine.hpp"

namespace tcb {

namespace cover_detail {
namespace {  // internal linkage: this header is compiled into several TUs
// ---- covered runs: rank l joins l - 1 iff some recorded run [f, t] has
// f < l <= t, i.e. iff max(reach[0 .. l-1]) >= l. A max-scan in three
// kernels over tiles of kCoverTile ranks: tile maxima, a one-block scan of
// those, then the tile-local scan that performs the unions.
constexpr int kCoverThreads = 256;
constexpr int kCoverItems = 8;
constexpr int kCoverTile = kCoverThreads * kCoverItems;

__device__ __forceinline__ void load_tile(const int32_t* __restrict__ reach, int64_t n,
                                          int64_t base, int32_t* v) {
  const int64_t i0 = base + threadIdx.x * kCoverItems;
  if (i0 + kCoverItems <= n) {
    const int4 a = __ldg(reinterpret_cast<const int4*>(reach + i0));
    const int4 b = __ldg(reinterpret_cast<const int4*>(reach + i0) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
#pragma unroll
    for (int k = 0; k < kCoverItems; ++k) v[k] = i0 + k < n ? reach[i0 + k] : -1;
  }
}

__global__ void __launch_bounds__(kCoverThreads)
k_cover_tiles(const int32_t* __restrict__ reach, int64_t n, int32_t* __restrict__ tile_max) {
  __shared__ int32_t red[32];
  int32_t v[kCoverItems];
  load_tile(reach, n, blockIdx.x * static_cast<int64_t>(kCoverTile), v);
  int32_t mx = v[0];
#pragma unroll
  for (int k = 1; k < kCoverItems; ++k) mx = max(mx, v[k]);
  mx = block_reduce(mx, [](int32_t a, int32_t b) { return max(a, b); }, -1, red);
  if (threadIdx.x == 0) tile_max[blockIdx.x] = mx;
}

// Exclusive max-scan of the tile maxima, one block (each thread a contiguous
// chunk).
__global__ void __launch_bounds__(1024)
k_cover_carry(int32_t* __restrict__ tile_max, int64_t tiles) {
  __shared__ int32_t part[1024];
  const int64_t per = (tiles + blockDim.x - 1) / blockDim.x;
  const int64_t b = threadIdx.x * per, e = min(b + per, tiles);
  int32_t mx = -1;
  for (int64_t t = b; t < e; ++t) mx = max(mx, tile_max[t]);
  part[threadIdx.x] = mx;
  __syncthreads();
  for (int o = 1; o < static_cast<int>(blockDim.x); o <<= 1) {
    int32_t x = threadIdx.x >= static_cast<unsigned>(o) ? part[threadIdx.x - o] : -1;
    __syncthreads();
    part[threadIdx.x] = max(part[threadIdx.x], x);
    __syncthreads();
  }
  int32_t run = threadIdx.x > 0 ? part[threadIdx.x - 1] : -1;
  for (int64_t t = b; t < e; ++t) {
    const int32_t x = tile_max[t];
    tile_max[t] = run;
    run = max(run, x);
  }
}

template <class Join>
__global__ void __launch_bounds__(kCoverThreads)
k_cover_unite(const int32_t* __restrict__ reach, int64_t n, const int32_t* __restrict__ carry,
              Join join) {
  __shared__ int32_t warp_max[kCoverThreads / 32];
  const int64_t base = blockIdx.x * static_cast<int64_t>(kCoverTile);
  int32_t v[kCoverItems];
  load_tile(reach, n, base, v);
  int32_t mine = v[0];
#pragma unroll
  for (int k = 1; k < kCoverItems; ++k) mine = max(mine, v[k]);
  // exclusive max over the threads before this one (warp scan + warp totals)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int32_t inc = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t x = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc = max(inc, x);
  }
  if (lane == 31) warp_max[w] = inc;
  __syncthreads();
  int32_t run = max(carry[blockIdx.x], __shfl_up_sync(0xffffffffu, inc, 1));
  if (lane == 0) run = carry[blockIdx.x];
  for (int k = 0; k < w; ++k) run = max(run, warp_max[k]);
  const int64_t i0 = base + threadIdx.x * kCoverItems;
#pragma unroll
  for (int k = 0; k < kCoverItems; ++k) {
    const int64_t l = i0 + k;
    if (l < n && run >= l && l > 0) join(static_cast<int32_t>(l));
    run = max(run, v[k]);
  }
}

}  // namespace
}  // namespace cover_detail

// rank space (FDBSCAN): ranks are union-find elements, roots chosen by key
struct KeyedJoin {
  int32_t* parent;
  const int32_t* key;
  uint8_t* mark = nullptr;  // see uf_unite_keyed
  __device__ __forceinline__ void operator()(int32_t a) const {
    const int32_t pa = ld_relaxed(parent + a), pb = ld_relaxed(parent + a - 1);
    if (pa != pb && pa != a - 1 && pb != a) uf_unite_keyed(parent, key, a, a - 1, mark);
  }
};

// DenseBox: primitive ranks mapped to their first query slot (slot-space
// union-find keyed by point id, see k_queries in grid.cu)
struct SlotJoin {
  int32_t* parent;
  const int32_t* key;
  const int32_t* qoff;
  uint8_t* mark = nullptr;
  __device__ __forceinline__ void operator()(int32_t l) const {
    const int32_t a = __ldg(qoff + l), b = __ldg(qoff + l - 1);
    const int32_t pa = ld_relaxed(parent + a), pb = ld_relaxed(parent + b);
    if (pa != pb && pa != b && pb != a) uf_unite_keyed(parent, key, a, b, mark);
  }
};

inline int64_t cover_tiles(int64_t n) {
  return (n + cover_detail::kCoverTile - 1) / cover_detail::kCoverTile;
}

void note_launch();

template <class Join>
inline void launch_cover_joins(const int32_t* reach, int64_t n, int32_t* tile_max, Join join,
                               cudaStream_t s) {
  using namespace cover_detail;
  const int64_t tiles = cover_tiles(n);
  const unsigned tgrid = static_cast<unsigned>(tiles);
  note_launch(), k_cover_tiles<<<tgrid, kCoverThreads, 0, s>>>(reach, n, tile_max);
  note_launch(), k_cover_carry<<<1, 1024, 0, s>>>(tile_max, tiles);
  note_launch(), k_cover_unite<<<tgrid, kCoverThreads, 0, s>>>(reach, n, tile_max, join);
  TCB_CUDA(cudaGetLastError());
}

}  // namespace tcb
