// Device stages of the Morton-range multi-GPU path, exposed
// through the additive C ABI (treeclust_gpu.h). The collectives between them
// (bounds all-reduce, splitter all-gather, point / halo / flag all-to-all,
// cross-shard edge all-gather) are issued by the caller's communicator
// (paper_2103_05162_b200/shard.py drives them through torch.distributed).
//
//   tcg_morton_codes_device   Morton codes of a shard's points against the
//                             GLOBAL scene box (same fp64 quantization as the
//                             tree build, geometry.hpp:132-156)
//   tcg_near_boxes_device     which points lie within eps of any box of a
//                             peer's region (halo selection): an LBVH over
//                             the peer's boxes + an early-exit ball query
//   tcg_core_flags_device     exact core flags (|N_eps| >= minpts, self
//                             included) of every point of own + ghost set
//   tcg_cluster_given_core_device
//                             main pass + finalize with core flags supplied
//                             by the caller (owners' exact flags for ghosts)
#include <cuda_runtime.h>

#include <cmath>
#include <memory>
#include <limits>

#include "device_common.cuh"
#include "engine.hpp"
#include "pipeline.hpp"
#include "treeclust_gpu.h"

#define TC_EXPORT extern "C" __attribute__((visibility("default")))

namespace tcb {
namespace {

template <int D>
__global__ void __launch_bounds__(256)
k_codes(const float* __restrict__ coords, int64_t n, float3 lo, float3 hi,
        unsigned long long* __restrict__ codes) {
  constexpr int bits = D == 2 ? 31 : 21;
  constexpr uint64_t cells = 1ull << bits;
  const double cells_d = static_cast<double>(cells);
  const float l[3] = {lo.x, lo.y, lo.z}, h[3] = {hi.x, hi.y, hi.z};
  double w[3];
#pragma unroll
  for (int k = 0; k < D; ++k) w[k] = __dsub_rn(static_cast<double>(h[k]), static_cast<double>(l[k]));
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint64_t q[3] = {0, 0, 0};
#pragma unroll
    for (int k = 0; k < D; ++k) q[k] = quantize(coords[i * D + k], l[k], w[k], cells_d, cells);
    codes[i] = D == 2 ? (spread2(q[0]) | (spread2(q[1]) << 1))
                      : (spread3(q[0]) | (spread3(q[1]) << 1) | (spread3(q[2]) << 2));
  }
}

template <int D>
__global__ void __launch_bounds__(256)
k_pack_boxes(const float* __restrict__ lo, const float* __restrict__ hi, int64_t nb,
             float4* __restrict__ lo4, float4* __restrict__ hi4) {
  for (int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; b < nb;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    lo4[b] = make_float4(lo[b * D], lo[b * D + 1], D == 3 ? lo[b * D + 2] : 0.f, 0.f);
    hi4[b] = make_float4(hi[b * D], hi[b * D + 1], D == 3 ? hi[b * D + 2] : 0.f, 0.f);
  }
}

template <int D>
__global__ void __launch_bounds__(128)
k_near(const float4* __restrict__ nodes, const float* __restrict__ coords, int64_t n, BallTest bt,
       uint8_t* __restrict__ mask) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  float p[3] = {coords[i * D], coords[i * D + 1], D == 3 ? coords[i * D + 2] : 0.f};
  bool hit = false;
  auto visit = [&](int32_t, int32_t, const float*, const float*) -> bool {
    hit = true;
    return false;
  };
  bvh_query<D>(nodes, p, bt, 0, visit);
  mask[i] = hit ? 1 : 0;
}

template <int D>
void near_boxes(const float* d_coords, int64_t n, float eps, const float* d_lo, const float* d_hi,
                int64_t nb, uint8_t* d_mask, cudaStream_t st) {
  Scratch scratch(st);
  if (nb == 0) {
    TCB_CUDA(cudaMemsetAsync(d_mask, 0, static_cast<size_t>(n), st));
    return;
  }
  DevCounters* ctr = scratch.alloc_n<DevCounters>(1);
  TCB_CUDA(cudaMemsetAsync(ctr, 0, sizeof(DevCounters), st));
  float4* lo4 = scratch.alloc_n<float4>(nb);
  float4* hi4 = scratch.alloc_n<float4>(nb);
  note_launch(), k_pack_boxes<D><<<grid_for(nb, 256), 256, 0, st>>>(d_lo, d_hi, nb, lo4, hi4);
  PrimSource src;
  src.lo = lo4;
  src.hi = hi4;
  src.count = nb;
  BuiltBvh b = build_bvh<D>(src, false, ctr, scratch, nullptr);
  const BallTest bt = BallTest::make(static_cast<double>(eps) * static_cast<double>(eps));
  note_launch(), k_near<D><<<grid_for(n, 128, INT32_MAX), 128, 0, st>>>(b.tree.nodes, d_coords, n, bt,
                                                                        d_mask);
  TCB_CUDA(cudaGetLastError());
}

template <int D>
void core_flags(const float* d_coords, int64_t n, float eps, int minpts, uint8_t* d_core,
                cudaStream_t st) {
  Scratch scratch(st);
  DevCounters* ctr = scratch.alloc_n<DevCounters>(1);
  TCB_CUDA(cudaMemsetAsync(ctr, 0, sizeof(DevCounters), st));
  PrimSource src;
  src.coords = d_coords;
  src.count = n;
  BuiltBvh b = build_bvh<D>(src, true, ctr, scratch, nullptr);
  uint8_t* flags = scratch.alloc_n<uint8_t>(n);  // rank space
  TCB_CUDA(cudaMemsetAsync(flags, 0, static_cast<size_t>(n), st));
  const double eps2 = static_cast<double>(eps) * static_cast<double>(eps);
  fdbscan_core_pass<D>(b, n, eps2, minpts, flags, ctr, st);
  permute_flags(flags, b.tree.leaf_order, n, d_core, /*to_rank=*/false, st);
}

template <int D>
void given_core(const float* d_coords, int64_t n, float eps, const uint8_t* d_core_in,
                int32_t* d_labels, uint8_t* d_core_out, cudaStream_t st, tc_cluster_stats* stats) {
  Scratch scratch(st);
  DevCounters* ctr = scratch.alloc_n<DevCounters>(1);
  TCB_CUDA(cudaMemsetAsync(ctr, 0, sizeof(DevCounters), st));
  PrimSource src;
  src.coords = d_coords;
  src.count = n;
  BuiltBvh b = build_bvh<D>(src, true, ctr, scratch, nullptr);
  int32_t* parent = scratch.alloc_n<int32_t>(n);
  uint8_t* flags = scratch.alloc_n<uint8_t>(n);
  init_union_find(parent, flags, n, st);
  permute_flags(d_core_in, b.tree.leaf_order, n, flags, /*to_rank=*/true, st);
  const double eps2 = static_cast<double>(eps) * static_cast<double>(eps);
  fdbscan_main_pass<D>(b, b.tree.leaf_order, n, eps2, /*force_core=*/false, flags, parent, ctr,
                       scratch);
  finalize_labels_bucketed(parent, flags, b.tree.leaf_order, b.tree.leaf_order, n, d_labels,
                           d_core_out, ctr, scratch, /*force_core=*/false);
  if (stats) {
    DevCounters h;
    TCB_CUDA(cudaMemcpyAsync(&h, ctr, sizeof h, cudaMemcpyDeviceToHost, st));
    TCB_CUDA(cudaStreamSynchronize(st));
    *stats = tc_cluster_stats{};
    stats->pair_resolutions = h.pairs;
    stats->distance_evaluations = h.dists;
    stats->cluster_count = h.clusters;
    stats->core_count = h.cores;
    stats->noise_count = h.noise;
  }
}

// ---- local context: one point BVH of a shard's own + ghost set serving the
// core pass, the ghost-flag exchange (done by the caller) and the main pass
struct LocalCtx {
  cudaStream_t st;
  Scratch scratch;
  DevCounters* ctr = nullptr;
  BuiltBvh b;
  const int32_t* key = nullptr;  // rank -> caller key
  int64_t n = 0;
  int dim = 0;
  double eps2 = 0.0;
  explicit LocalCtx(cudaStream_t s) : st(s), scratch(s) {}
};

template <int D>
void local_build(LocalCtx& c, const float* d_coords, const int32_t* d_keys) {
  check_keys_nonnegative(d_keys, c.n, c.scratch);
  c.ctr = c.scratch.alloc_n<DevCounters>(1);
  TCB_CUDA(cudaMemsetAsync(c.ctr, 0, sizeof(DevCounters), c.st));
  PrimSource src;
  src.coords = d_coords;
  src.count = c.n;
  c.b = build_bvh<D>(src, true, c.ctr, c.scratch, nullptr);
  int32_t* k = c.scratch.alloc_n<int32_t>(c.n);
  gather_rank_keys(d_keys, c.b.tree.leaf_order, c.n, k, c.st);
  c.key = k;
}

template <int D>
void local_core(LocalCtx& c, int minpts, uint8_t* d_core) {
  Scratch tmp(c.st);
  uint8_t* flags = tmp.alloc_n<uint8_t>(c.n);  // rank space
  TCB_CUDA(cudaMemsetAsync(flags, 0, static_cast<size_t>(c.n), c.st));
  fdbscan_core_pass<D>(c.b, c.n, c.eps2, minpts, flags, c.ctr, c.st);
  permute_flags(flags, c.b.tree.leaf_order, c.n, d_core, /*to_rank=*/false, c.st);
}

template <int D>
void local_cluster(LocalCtx& c, const uint8_t* d_core_in, int32_t* d_labels, uint8_t* d_core_out) {
  Scratch tmp(c.st);
  int32_t* parent = tmp.alloc_n<int32_t>(c.n);
  uint8_t* flags = tmp.alloc_n<uint8_t>(c.n);
  init_union_find(parent, flags, c.n, c.st);
  permute_flags(d_core_in, c.b.tree.leaf_order, c.n, flags, /*to_rank=*/true, c.st);
  fdbscan_main_pass<D>(c.b, c.key, c.n, c.eps2, /*force_core=*/false, flags, parent, c.ctr, tmp);
  finalize_labels_bucketed(parent, flags, c.key, c.b.tree.leaf_order, c.n, d_labels, d_core_out,
                           c.ctr, tmp, /*force_core=*/false);
}

__global__ void k_unite_pairs(const int32_t* __restrict__ edges, int64_t m, int32_t* parent) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < m;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    uf_unite(parent, edges[2 * e], edges[2 * e + 1]);
}

__global__ void k_flatten_all(int32_t* parent, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t p = ld_relaxed(parent + i), q;
    while (p != (q = ld_relaxed(parent + p))) p = q;
    st_relaxed(parent + i, p);
  }
}

// ---- redistribution: owner by Morton range + packed rows in owner order ----
// owner = number of splitters <= code (torch.bucketize(right=True)); a row is
// dim coordinate words, the global id (2 words) and the code (2 words).
constexpr int kRouteThreads = 256;
constexpr int kMaxRanks = 1024;

__device__ __forceinline__ int route_owner(const int64_t* s_split, int nsplit, int64_t code) {
  int lo = 0, hi = nsplit;  // first splitter > code
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (s_split[mid] <= code) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kRouteThreads)
k_route_count(const int64_t* __restrict__ codes, int64_t n, const int64_t* __restrict__ split,
              int nsplit, unsigned long long* __restrict__ counts) {
  __shared__ int64_t s_split[kMaxRanks];
  __shared__ unsigned int s_cnt[kMaxRanks];
  for (int i = threadIdx.x; i < nsplit; i += blockDim.x) s_split[i] = split[i];
  for (int i = threadIdx.x; i <= nsplit; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    atomicAdd(&s_cnt[route_owner(s_split, nsplit, codes[i])], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i <= nsplit; i += blockDim.x)
    if (s_cnt[i]) atomicAdd(counts + i, static_cast<unsigned long long>(s_cnt[i]));
}

// cursor[o] = exclusive prefix of counts (one block)
__global__ void k_route_offsets(const unsigned long long* __restrict__ counts, int world,
                                unsigned long long* __restrict__ cursor) {
  if (threadIdx.x == 0) {
    unsigned long long acc = 0;
    for (int o = 0; o < world; ++o) {
      cursor[o] = acc;
      acc += counts[o];
    }
  }
}

template <int D>
__global__ void __launch_bounds__(kRouteThreads)
k_route_scatter(const float* __restrict__ coords, const int64_t* __restrict__ gid,
                const int64_t* __restrict__ codes, int64_t n, const int64_t* __restrict__ split,
                int nsplit, unsigned long long* __restrict__ cursor, int32_t* __restrict__ rows) {
  __shared__ int64_t s_split[kMaxRanks];
  __shared__ unsigned int s_cnt[kMaxRanks];
  __shared__ unsigned long long s_base[kMaxRanks];
  for (int i = threadIdx.x; i < nsplit; i += blockDim.x) s_split[i] = split[i];
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t b0 = blockIdx.x * static_cast<int64_t>(blockDim.x); b0 < n; b0 += stride) {
    for (int i = threadIdx.x; i <= nsplit; i += blockDim.x) s_cnt[i] = 0;
    __syncthreads();
    const int64_t i = b0 + threadIdx.x;
    int o = 0;
    unsigned loc = 0;
    int64_t code = 0;
    if (i < n) {
      code = codes[i];
      o = route_owner(s_split, nsplit, code);
      loc = atomicAdd(&s_cnt[o], 1u);
    }
    __syncthreads();
    for (int k = threadIdx.x; k <= nsplit; k += blockDim.x)
      if (s_cnt[k]) s_base[k] = atomicAdd(cursor + k, static_cast<unsigned long long>(s_cnt[k]));
    __syncthreads();
    if (i < n) {
      int32_t* row = rows + static_cast<int64_t>(s_base[o] + loc) * (D + 4);
#pragma unroll
      for (int k = 0; k < D; ++k) row[k] = __float_as_int(coords[i * D + k]);
      const int64_t g = gid[i];
      row[D] = static_cast<int32_t>(g & 0xffffffff);
      row[D + 1] = static_cast<int32_t>(g >> 32);
      row[D + 2] = static_cast<int32_t>(code & 0xffffffff);
      row[D + 3] = static_cast<int32_t>(code >> 32);
    }
    __syncthreads();
  }
}

// rows (dim coordinate words, gid, code) -> contiguous coordinates, global
// ids and codes (codes optional): the inverse of k_route_scatter's packing
template <int D>
__global__ void __launch_bounds__(256)
k_unpack_rows(const int32_t* __restrict__ rows, int64_t n, float* __restrict__ coords,
              int64_t* __restrict__ gid, int64_t* __restrict__ codes) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t* row = rows + i * (D + 4);
#pragma unroll
    for (int k = 0; k < D; ++k) coords[i * D + k] = __int_as_float(row[k]);
    gid[i] = static_cast<int64_t>(static_cast<uint32_t>(row[D])) |
             (static_cast<int64_t>(row[D + 1]) << 32);
    if (codes)
      codes[i] = static_cast<int64_t>(static_cast<uint32_t>(row[D + 2])) |
                 (static_cast<int64_t>(row[D + 3]) << 32);
  }
}

// ---- region boxes: tight boxes of Morton-prefix cells of a shard's points --
// The cell of a point is code >> shift, with the shift chosen on the device so
// that the shard's code range spans at most 2^kCellBits cells; each occupied
// cell's box is reduced with order-preserving atomics, then the occupied ones
// are compacted. Every point lies in the box of its cell: the boxes cover the
// shard, which is all the eps-halo selection needs (tcg_near_peers_device).
// 4096 cells: a block reduces its points' boxes in shared memory (96 KB in
// 3D) and merges each touched cell into the global boxes once — 37M global
// atomics per pass become a few million (a 65536-cell table took 2.1 ms on
// 37M points, almost all of it in contended global atomics). The cells are
// Morton-prefix blocks of the shard's own range, so a coarse cell's tight
// box stays inside the shard's region and the halo is as thin as before.
constexpr int kCellBits = 12;

__global__ void k_code_range(const int64_t* __restrict__ codes, int64_t n,
                             unsigned long long* range) {
  unsigned long long mn = ~0ull, mx = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long c = static_cast<unsigned long long>(codes[i]);
    mn = c < mn ? c : mn;
    mx = c > mx ? c : mx;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, mn, o);
    const unsigned long long b = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(range, mn);
    atomicMax(range + 1, mx);
  }
}

template <int D>
__global__ void __launch_bounds__(1024)
k_cell_boxes(const float* __restrict__ coords, const int64_t* __restrict__ codes, int64_t n,
             const unsigned long long* __restrict__ range, uint32_t* __restrict__ cell_ord) {
  const unsigned long long lo = range[0], hi = range[1];
  int shift = 0;
  while (((hi >> shift) - (lo >> shift)) >= (1ull << kCellBits)) ++shift;
  extern __shared__ uint32_t s_box[];  // [cell][lo D | hi D]
  constexpr int kWords = (1 << kCellBits) * 2 * D;
  for (int w = threadIdx.x; w < kWords; w += blockDim.x) s_box[w] = (w % (2 * D)) < D ? ~0u : 0u;
  __syncthreads();
  // a contiguous chunk per block (consecutive points share cells more often)
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per, b1 = b0 + per < n ? b0 + per : n;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
    const uint64_t c = (static_cast<unsigned long long>(codes[i]) >> shift) - (lo >> shift);
    uint32_t* b = s_box + c * (2 * D);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const uint32_t v = f2ord(coords[i * D + k]);
      atomicMin(b + k, v);
      atomicMax(b + D + k, v);
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < (1 << kCellBits); c += blockDim.x) {
    const uint32_t* b = s_box + c * (2 * D);
    if (b[0] > b[D]) continue;  // untouched here
    uint32_t* g = cell_ord + static_cast<int64_t>(c) * (2 * D);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      atomicMin(g + k, b[k]);
      atomicMax(g + D + k, b[D + k]);
    }
  }
}

template <int D>
__global__ void __launch_bounds__(256)
k_cell_compact(const uint32_t* __restrict__ cell_ord, float* __restrict__ box_lo,
               float* __restrict__ box_hi, unsigned long long* __restrict__ count) {
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       c < (int64_t{1} << kCellBits); c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t* b = cell_ord + c * (2 * D);
    if (b[0] > b[D]) continue;  // no point in this cell
    const unsigned long long k = atomicAdd(count, 1ull);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      box_lo[k * D + j] = ord2f(b[j]);
      box_hi[k * D + j] = ord2f(b[D + j]);
    }
  }
}

__global__ void k_fill_u32(uint32_t* p, int64_t n, uint32_t a, uint32_t b, int period, int half) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = (i % period) < half ? a : b;
}

// ---- halo: the set of peers (bit j = peer j) whose region boxes lie within
// eps of each point, from one traversal of an LBVH over all peers' boxes ----
template <int D>
__global__ void __launch_bounds__(128)
k_near_peers(const float4* __restrict__ nodes, const float* __restrict__ coords, int64_t n,
             BallTest bt, unsigned long long* __restrict__ mask) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  float p[3] = {coords[i * D], coords[i * D + 1], D == 3 ? coords[i * D + 2] : 0.f};
  unsigned long long m = 0;
  auto visit = [&](int32_t, int32_t owner, const float*, const float*) -> bool {
    if (static_cast<uint32_t>(owner) < 64u) m |= 1ull << owner;  // (owners >= 64 unsupported)
    return true;
  };
  bvh_query<D>(nodes, p, bt, 0, visit);
  mask[i] = m;
}

template <int D>
void near_peers(const float* d_coords, int64_t n, float eps, const float* d_lo, const float* d_hi,
                const int32_t* d_owner, int64_t nb, unsigned long long* d_mask, cudaStream_t st) {
  Scratch scratch(st);
  if (nb == 0) {
    TCB_CUDA(cudaMemsetAsync(d_mask, 0, static_cast<size_t>(n) * 8, st));
    return;
  }
  DevCounters* ctr = scratch.alloc_n<DevCounters>(1);
  TCB_CUDA(cudaMemsetAsync(ctr, 0, sizeof(DevCounters), st));
  float4* lo4 = scratch.alloc_n<float4>(nb);
  float4* hi4 = scratch.alloc_n<float4>(nb);
  note_launch(), k_pack_boxes<D><<<grid_for(nb, 256), 256, 0, st>>>(d_lo, d_hi, nb, lo4, hi4);
  PrimSource src;
  src.lo = lo4;
  src.hi = hi4;
  src.aux = d_owner;
  src.count = nb;
  BuiltBvh b = build_bvh<D>(src, false, ctr, scratch, nullptr);
  const BallTest bt = BallTest::make(static_cast<double>(eps) * static_cast<double>(eps));
  note_launch(), k_near_peers<D><<<grid_for(n, 128, INT32_MAX), 128, 0, st>>>(b.tree.nodes,
                                                                              d_coords, n, bt,
                                                                              d_mask);
  TCB_CUDA(cudaGetLastError());
}

template <typename Fn>
tc_status run_guarded(Fn&& fn) {
  try {
    fn();
    return TC_OK;
  } catch (const InvalidArgument&) {
    return TC_ERR_INVALID_ARGUMENT;
  } catch (...) {
    cudaGetLastError();
    return TC_ERR_INTERNAL;
  }
}

bool bad_shape(const void* p, int64_t n, int dim) {
  return !p || n < 0 || n > std::numeric_limits<int32_t>::max() || (dim != 2 && dim != 3);
}

}  // namespace
}  // namespace tcb

using namespace tcb;

TC_EXPORT tc_status tcg_morton_codes_device(const float* d_coords, int64_t n, int dim,
                                            const float* lo, const float* hi, uint64_t* d_codes,
                                            void* stream) {
  if (bad_shape(d_coords, n, dim) || !lo || !hi || !d_codes) return TC_ERR_INVALID_ARGUMENT;
  return run_guarded([&] {
    reset_launch_count();
    const float3 l = make_float3(lo[0], lo[1], dim == 3 ? lo[2] : 0.f);
    const float3 h = make_float3(hi[0], hi[1], dim == 3 ? hi[2] : 0.f);
    auto st = static_cast<cudaStream_t>(stream);
    auto* out = reinterpret_cast<unsigned long long*>(d_codes);
    if (n == 0) return;
    if (dim == 2)
      note_launch(), k_codes<2><<<grid_for(n, 256), 256, 0, st>>>(d_coords, n, l, h, out);
    else
      note_launch(), k_codes<3><<<grid_for(n, 256), 256, 0, st>>>(d_coords, n, l, h, out);
    TCB_CUDA(cudaGetLastError());
  });
}

TC_EXPORT tc_status tcg_near_boxes_device(const float* d_coords, int64_t n, int dim, float eps,
                                          const float* d_box_lo, const float* d_box_hi,
                                          int64_t num_boxes, uint8_t* d_mask, void* stream) {
  if (bad_shape(d_coords, n, dim) || !d_mask || num_boxes < 0 || !(eps > 0.f))
    return TC_ERR_INVALID_ARGUMENT;
  return run_guarded([&] {
    reset_launch_count();
    if (n == 0) return;
    auto st = static_cast<cudaStream_t>(stream);
    if (dim == 2)
      near_boxes<2>(d_coords, n, eps, d_box_lo, d_box_hi, num_boxes, d_mask, st);
    else
      near_boxes<3>(d_coords, n, eps, d_box_lo, d_box_hi, num_boxes, d_mask, st);
  });
}

TC_EXPORT tc_status tcg_core_flags_device(const float* d_coords, int64_t n, int dim, float eps,
                                          int minpts, uint8_t* d_core, void* stream) {
  if (bad_shape(d_coords, n, dim) || n < 1 || !d_core || !(eps > 0.f) || !std::isfinite(eps) ||
      minpts < 2)
    return TC_ERR_INVALID_ARGUMENT;
  return run_guarded([&] {
    auto st = static_cast<cudaStream_t>(stream);
    reset_launch_count();
    if (dim == 2)
      core_flags<2>(d_coords, n, eps, minpts, d_core, st);
    else
      core_flags<3>(d_coords, n, eps, minpts, d_core, st);
  });
}

TC_EXPORT tc_status tcg_cluster_given_core_device(const float* d_coords, int64_t n, int dim,
                                                  float eps, const uint8_t* d_core_in,
                                                  int32_t* d_labels, uint8_t* d_core_out,
                                                  void* stream, tc_cluster_stats* stats) {
  if (bad_shape(d_coords, n, dim) || n < 1 || !d_core_in || !d_labels || !d_core_out ||
      !(eps > 0.f) || !std::isfinite(eps))
    return TC_ERR_INVALID_ARGUMENT;
  return run_guarded([&] {
    auto st = static_cast<cudaStream_t>(stream);
    reset_launch_count();
    if (dim == 2)
      given_core<2>(d_coords, n, eps, d_core_in, d_labels, d_core_out, st, stats);
    else
      given_core<3>(d_coords, n, eps, d_core_in, d_labels, d_core_out, st, stats);
  });
}

struct tcg_local : tcb::LocalCtx {
  using LocalCtx::LocalCtx;
};

TC_EXPORT tc_status tcg_local_create(const float* d_coords, const int32_t* d_keys, int64_t n,
                                     int dim, float eps, void* stream, tcg_local** out) {
  if (bad_shape(d_coords, n, dim) || n < 1 || !d_keys || !out || !(eps > 0.f) ||
      !std::isfinite(eps))
    return TC_ERR_INVALID_ARGUMENT;
  tcg_local* c = nullptr;
  const tc_status st = run_guarded([&] {
    reset_launch_count();
    auto ctx = std::make_unique<tcg_local>(static_cast<cudaStream_t>(stream));
    ctx->n = n;
    ctx->dim = dim;
    ctx->eps2 = static_cast<double>(eps) * static_cast<double>(eps);
    if (dim == 2)
      local_build<2>(*ctx, d_coords, d_keys);
    else
      local_build<3>(*ctx, d_coords, d_keys);
    c = ctx.release();
  });
  if (st == TC_OK) *out = c;
  return st;
}

TC_EXPORT tc_status tcg_local_core_flags(tcg_local* ctx, int minpts, uint8_t* d_core) {
  if (!ctx || !d_core || minpts < 2) return TC_ERR_INVALID_ARGUMENT;
  return run_guarded([&] {
    reset_launch_count();
    if (ctx->dim == 2)
      local_core<2>(*ctx, minpts, d_core);
    else
      local_core<3>(*ctx, minpts, d_core);
  });
}

TC_EXPORT tc_status tcg_local_cluster(tcg_local* ctx, const uint8_t* d_core_in, int32_t* d_labels,
                                      uint8_t* d_core_out) {
  if (!ctx || !d_core_in || !d_labels || !d_core_out) return TC_ERR_INVALID_ARGUMENT;
  return run_guarded([&] {
    reset_launch_count();
    if (ctx->dim == 2)
      local_cluster<2>(*ctx, d_core_in, d_labels, d_core_out);
    else
      local_cluster<3>(*ctx, d_core_in, d_labels, d_core_out);
  });
}

TC_EXPORT void tcg_local_free(tcg_local* ctx) { delete ctx; }

TC_EXPORT tc_status tcg_shard_route_device(const float* d_coords, const int64_t* d_gid,
                                           const int64_t* d_codes, int64_t n, int dim,
                                           const int64_t* d_splitters, int num_splitters,
                                           int32_t* d_rows, int64_t* d_counts, void* stream) {
  if ((n > 0 && (!d_coords || !d_gid || !d_codes || !d_rows)) || n < 0 ||
      n > std::numeric_limits<int32_t>::max() || (dim != 2 && dim != 3) || !d_counts ||
      num_splitters < 0 || num_splitters >= kMaxRanks || (num_splitters > 0 && !d_splitters))
    return TC_ERR_INVALID_ARGUMENT;
  return run_guarded([&] {
    reset_launch_count();
    auto st = static_cast<cudaStream_t>(stream);
    auto* counts = reinterpret_cast<unsigned long long*>(d_counts);
    const int world = num_splitters + 1;
    TCB_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * world, st));
    if (n == 0) return;
    Scratch scratch(st);
    auto* cursor = scratch.alloc_n<unsigned long long>(world);
    const unsigned g = grid_for(n, kRouteThreads, 148 * 8);
    note_launch(), k_route_count<<<g, kRouteThreads, 0, st>>>(d_codes, n, d_splitters,
                                                             num_splitters, counts);
    note_launch(), k_route_offsets<<<1, 32, 0, st>>>(counts, world, cursor);
    if (dim == 2)
      note_launch(), k_route_scatter<2><<<g, kRouteThreads, 0, st>>>(
          d_coords, d_gid, d_codes, n, d_splitters, num_splitters, cursor, d_rows);
    else
      note_launch(), k_route_scatter<3><<<g, kRouteThreads, 0, st>>>(
          d_coords, d_gid, d_codes, n, d_splitters, num_splitters, cursor, d_rows);
    TCB_CUDA(cudaGetLastError());
  });
}

TC_EXPORT tc_status tcg_shard_unpack_rows_device(const int32_t* d_rows, int64_t n, int dim,
                                                 float* d_coords, int64_t* d_gid,
                                                 int64_t* d_codes, void* stream) {
  if ((n > 0 && (!d_rows || !d_coords || !d_gid)) || n < 0 || (dim != 2 && dim != 3))
    return TC_ERR_INVALID_ARGUMENT;
  return run_guarded([&] {
    reset_launch_count();
    if (n == 0) return;
    auto st = static_cast<cudaStream_t>(stream);
    const unsigned g = grid_for(n, 256, 148 * 16);
    if (dim == 2)
      note_launch(), k_unpack_rows<2><<<g, 256, 0, st>>>(d_rows, n, d_coords, d_gid, d_codes);
    else
      note_launch(), k_unpack_rows<3><<<g, 256, 0, st>>>(d_rows, n, d_coords, d_gid, d_codes);
    TCB_CUDA(cudaGetLastError());
  });
}

TC_EXPORT tc_status tcg_shard_region_boxes_device(const float* d_coords, const int64_t* d_codes,
                                                  int64_t n, int dim, float* d_box_lo,
                                                  float* d_box_hi, int64_t* d_num_boxes,
                                                  void* stream) {
  if ((n > 0 && (!d_coords || !d_codes)) || n < 0 || (dim != 2 && dim != 3) || !d_box_lo ||
      !d_box_hi || !d_num_boxes)
    return TC_ERR_INVALID_ARGUMENT;
  return run_guarded([&] {
    reset_launch_count();
    auto st = static_cast<cudaStream_t>(stream);
    auto* count = reinterpret_cast<unsigned long long*>(d_num_boxes);
    TCB_CUDA(cudaMemsetAsync(count, 0, sizeof(int64_t), st));
    if (n == 0) return;
    Scratch scratch(st);
    auto* range = scratch.alloc_n<unsigned long long>(2);
    note_launch(), k_fill_u32<<<1, 32, 0, st>>>(reinterpret_cast<uint32_t*>(range), 4,
                                                 0xffffffffu, 0u, 4, 2);
    const int64_t words = (int64_t{1} << kCellBits) * 2 * dim;
    auto* cell_ord = scratch.alloc_n<uint32_t>(words);
    note_launch(), k_fill_u32<<<grid_for(words, 256), 256, 0, st>>>(cell_ord, words, 0xffffffffu,
                                                                     0u, 2 * dim, dim);
    note_launch(), k_code_range<<<grid_for(n, 256, 148 * 8), 256, 0, st>>>(d_codes, n, range);
    const unsigned g = grid_for(n, 1024, 148 * 2);
    const unsigned gc = grid_for(int64_t{1} << kCellBits, 256);
    const size_t smem = sizeof(uint32_t) * (size_t{1} << kCellBits) * 2 * dim;
    if (dim == 2) {
      TCB_CUDA(cudaFuncSetAttribute(k_cell_boxes<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
      note_launch(), k_cell_boxes<2><<<g, 1024, smem, st>>>(d_coords, d_codes, n, range, cell_ord);
      note_launch(), k_cell_compact<2><<<gc, 256, 0, st>>>(cell_ord, d_box_lo, d_box_hi, count);
    } else {
      TCB_CUDA(cudaFuncSetAttribute(k_cell_boxes<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
      note_launch(), k_cell_boxes<3><<<g, 1024, smem, st>>>(d_coords, d_codes, n, range, cell_ord);
      note_launch(), k_cell_compact<3><<<gc, 256, 0, st>>>(cell_ord, d_box_lo, d_box_hi, count);
    }
    TCB_CUDA(cudaGetLastError());
  });
}

TC_EXPORT tc_status tcg_near_peers_device(const float* d_coords, int64_t n, int dim, float eps,
                                          const float* d_box_lo, const float* d_box_hi,
                                          const int32_t* d_box_owner, int64_t num_boxes,
                                          uint64_t* d_mask, void* stream) {
  if (bad_shape(d_coords, n, dim) || !d_mask || num_boxes < 0 || !(eps > 0.f) ||
      (num_boxes > 0 && (!d_box_lo || !d_box_hi || !d_box_owner)))
    return TC_ERR_INVALID_ARGUMENT;
  return run_guarded([&] {
    reset_launch_count();
    if (n == 0) return;
    auto st = static_cast<cudaStream_t>(stream);
    auto* mask = reinterpret_cast<unsigned long long*>(d_mask);
    if (dim == 2)
      near_peers<2>(d_coords, n, eps, d_box_lo, d_box_hi, d_box_owner, num_boxes, mask, st);
    else
      near_peers<3>(d_coords, n, eps, d_box_lo, d_box_hi, d_box_owner, num_boxes, mask, st);
  });
}

TC_EXPORT tc_status tcg_union_edges_device(const int32_t* d_edges, int64_t m, int32_t n,
                                           int32_t* d_root, void* stream) {
  if ((!d_edges && m > 0) || m < 0 || n < 1 || !d_root) return TC_ERR_INVALID_ARGUMENT;
  return run_guarded([&] {
    reset_launch_count();
    auto st = static_cast<cudaStream_t>(stream);
    Scratch scratch(st);
    uint8_t* tmp = scratch.alloc_n<uint8_t>(n);
    init_union_find(d_root, tmp, n, st);
    if (m > 0) note_launch(), k_unite_pairs<<<grid_for(m, 256), 256, 0, st>>>(d_edges, m, d_root);
    note_launch(), k_flatten_all<<<grid_for(n, 256), 256, 0, st>>>(d_root, n);
    TCB_CUDA(cudaGetLastError());
  });
}
