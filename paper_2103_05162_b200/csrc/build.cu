// LBVH construction on the device (reference: bvh.cpp:10-124).
//
//   k_centroid_bounds   scene Aabb over primitive centroids (bvh.cpp:15-21),
//                       fused with the finiteness check of PointSet::validate
//                       (geometry.hpp:29-37)
//   k_morton            fp64 quantization + interleave (geometry.hpp:132-156),
//                       fused AND/OR reduction of the codes for the sort
//   radix_sort_pairs    stable (code, index) order (bvh.cpp:27-32)
//   k_karras            Karras-2012 split search per internal node
//                       (bvh.cpp:49-86); also writes child payloads, the
//                       children's max leaf rank and parent links
//   k_refit             bottom-up boxes with atomic arrival flags
//                       (bvh.cpp:88-124); points mode also gathers the
//                       Morton-ordered query points (bvh.cpp:34-39)
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstring>

#include "device_common.cuh"
#include "pipeline.hpp"
#include "primitives.cuh"

namespace tcb {

namespace {

__global__ void k_reset_build(DevCounters* ctr) {
  int t = threadIdx.x;
  if (t < 3) ctr->bounds_ord[t] = 0xffffffffu;
  else if (t < 6) ctr->bounds_ord[t] = 0u;
  else if (t == 6) ctr->key_and = ~0ull;
  else if (t == 7) ctr->key_or = 0ull;
  else if (t == 8) ctr->nonfinite = 0;
}

// Primitive box accessors. Points: degenerate box at the point.
template <int D>
struct PointBoxes {
  const float* coords;
  __device__ __forceinline__ void box(int64_t i, float* lo, float* hi) const {
#pragma unroll
    for (int k = 0; k < D; ++k) lo[k] = hi[k] = coords[i * D + k];
  }
};

template <int D>
struct ExplicitBoxes {
  const float4* lo4;
  const float4* hi4;
  __device__ __forceinline__ void box(int64_t i, float* lo, float* hi) const {
    float4 a = lo4[i], b = hi4[i];
    lo[0] = a.x;
    lo[1] = a.y;
    hi[0] = b.x;
    hi[1] = b.y;
    if (D == 3) {
      lo[2] = a.z;
      hi[2] = b.z;
    }
  }
};

// Aabb::centroid (geometry.hpp:67-69): 0.5f * (min + max) in fp32.
template <int D>
__device__ __forceinline__ void centroid(const float* lo, const float* hi, float* c) {
#pragma unroll
  for (int k = 0; k < D; ++k) c[k] = __fmul_rn(0.5f, __fadd_rn(lo[k], hi[k]));
}

template <int D, class Src>
__global__ void __launch_bounds__(256)
k_centroid_bounds(Src src, int64_t m, bool check_finite, DevCounters* ctr) {
  float mn[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, mx[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
  bool bad = false;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float lo[3], hi[3], c[3];
    src.box(i, lo, hi);
    if (check_finite) {
#pragma unroll
      for (int k = 0; k < D; ++k) bad |= !isfinite(lo[k]);
    }
    centroid<D>(lo, hi, c);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      mn[k] = fminf(mn[k], c[k]);
      mx[k] = fmaxf(mx[k], c[k]);
    }
  }
  publish_bounds<D>(mn, mx, bad, ctr);
}

template <int D, class Src>
__global__ void __launch_bounds__(256)
k_morton(Src src, int64_t m, DevCounters* ctr, uint64_t* __restrict__ keys,
         int32_t* __restrict__ vals) {
  constexpr int bits = D == 2 ? 31 : 21;  // morton_bits_per_axis (geometry.hpp:130)
  constexpr uint64_t cells = 1ull << bits;
  const double cells_d = static_cast<double>(cells);
  float lo_s[3], w_lo[3];
  double w[3];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    lo_s[k] = ord2f(ctr->bounds_ord[k]);
    float hi_s = ord2f(ctr->bounds_ord[3 + k]);
    w[k] = __dsub_rn(static_cast<double>(hi_s), static_cast<double>(lo_s[k]));
    w_lo[k] = lo_s[k];
  }
  uint64_t acc_and = ~0ull, acc_or = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float lo[3], hi[3], c[3];
    src.box(i, lo, hi);
    centroid<D>(lo, hi, c);
    uint64_t code;
    if (D == 2) {
      uint64_t x = quantize(c[0], w_lo[0], w[0], cells_d, cells);
      uint64_t y = quantize(c[1], w_lo[1], w[1], cells_d, cells);
      code = spread2(x) | (spread2(y) << 1);
    } else {
      uint64_t x = quantize(c[0], w_lo[0], w[0], cells_d, cells);
      uint64_t y = quantize(c[1], w_lo[1], w[1], cells_d, cells);
      uint64_t z = quantize(c[2], w_lo[2], w[2], cells_d, cells);
      code = spread3(x) | (spread3(y) << 1) | (spread3(z) << 2);
    }
    keys[i] = code;
    vals[i] = static_cast<int32_t>(i);
    acc_and &= code;
    acc_or |= code;
  }
  publish_and_or(acc_and, acc_or, ctr);
}

// Bvh::delta (bvh.cpp:49-56): common prefix of (code, index) keys.
__device__ __forceinline__ int key_delta(const uint64_t* __restrict__ codes, int64_t m,
                                         int64_t i, int64_t j) {
  if (j < 0 || j >= m) return -1;
  uint64_t ci = codes[i], cj = codes[j];
  if (ci != cj) return __clzll(static_cast<long long>(ci ^ cj));
  return 64 + __clz(static_cast<int>(static_cast<uint32_t>(i) ^ static_cast<uint32_t>(j)));
}

// Leaves in Morton rank order (bvh.cpp:34-39): leaf_lo[s] / leaf_hi[s] =
// box of primitive order[s]; in points mode both alias one array whose w
// component carries the point id (the query points of the traversals).
template <int D, class Src>
__global__ void __launch_bounds__(256)
k_gather_leaves(Src src, const int32_t* __restrict__ order, int64_t m, float4* __restrict__ leaf_lo,
                float4* __restrict__ leaf_hi) {
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < m;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t prim = order[s];
    float lo[3], hi[3];
    src.box(prim, lo, hi);
    leaf_lo[s] = make_float4(lo[0], lo[1], D == 3 ? lo[2] : 0.f, __int_as_float(prim));
    if (leaf_hi != leaf_lo) leaf_hi[s] = make_float4(hi[0], hi[1], D == 3 ? hi[2] : 0.f, 0.f);
  }
}

// Subtrees of at most kDirectRange leaves get their boxes straight from the
// contiguous leaf run (k_small_boxes); only larger nodes are refit bottom-up.
constexpr int kDirectRange = 32;

template <int D>
__global__ void __launch_bounds__(256)
k_karras(const float4* __restrict__ leaf_lo, const float4* __restrict__ leaf_hi,
         const uint64_t* __restrict__ codes, const int32_t* __restrict__ order,
         const int32_t* __restrict__ prim_aux, int64_t m, float4* __restrict__ nodes,
         int4* __restrict__ node_info, int32_t* __restrict__ leaf_up,
         int32_t* __restrict__ starts, int32_t* __restrict__ num_starts) {
  using T = NodeTraits<D>;
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= m - 1) return;
  const int d = key_delta(codes, m, i, i + 1) > key_delta(codes, m, i, i - 1) ? 1 : -1;
  const int delta_min = key_delta(codes, m, i, i - d);
  int64_t lmax = 2;
  while (key_delta(codes, m, i, i + lmax * d) > delta_min) lmax *= 2;
  int64_t l = 0;
  for (int64_t t = lmax / 2; t >= 1; t /= 2)
    if (key_delta(codes, m, i, i + (l + t) * d) > delta_min) l += t;
  const int64_t j = i + l * d;
  const int delta_node = key_delta(codes, m, i, j);
  int64_t s = 0, t = l;
  do {
    t = (t + 1) / 2;
    if (key_delta(codes, m, i, i + (s + t) * d) > delta_node) s += t;
  } while (t > 1);
  const int64_t gamma = i + s * d + (d < 0 ? d : 0);
  const int64_t lo = i < j ? i : j, hi = i < j ? j : i;

  float* f = reinterpret_cast<float*>(nodes + i * T::kVec);
  // A leaf child's box goes straight into its slot here (bvh.cpp:34-39's
  // gather fused in), so the refit only ever waits on internal children.
  auto leaf_child = [&](int64_t rank, int slot, int32_t& link, int32_t& aux) {
    link = ~static_cast<int32_t>(rank);
    const int32_t prim = order[rank];
    aux = prim_aux ? prim_aux[prim] : prim;
    const float4 a = leaf_lo[rank], c = leaf_hi[rank];
    const float blo[3] = {a.x, a.y, a.z}, bhi[3] = {c.x, c.y, c.z};
#pragma unroll
    for (int k = 0; k < D; ++k) {
      f[slot * 2 * D + k] = blo[k];
      f[slot * 2 * D + D + k] = bhi[k];
    }
  };
  int32_t left, right, aux_l, aux_r;
  // Own info (delta = prefix length shared by the whole range, the range);
  // the parent link of each child is written here, by its parent.
  node_info[i].y = delta_node;
  node_info[i].z = static_cast<int32_t>(lo);
  node_info[i].w = static_cast<int32_t>(hi);
  const int32_t up_left = static_cast<int32_t>(i) | kUpLeftBit;
  const int32_t up_right = static_cast<int32_t>(i);
  if (lo == gamma) {
    leaf_child(gamma, 0, left, aux_l);
    leaf_up[gamma] = up_left;
  } else {
    left = static_cast<int32_t>(gamma);
    aux_l = static_cast<int32_t>(gamma);  // max leaf rank of [lo, gamma]
    node_info[gamma].x = up_left;
  }
  if (hi == gamma + 1) {
    leaf_child(gamma + 1, 1, right, aux_r);
    leaf_up[gamma + 1] = up_right;
  } else {
    right = static_cast<int32_t>(gamma + 1);
    aux_r = static_cast<int32_t>(hi);  // max leaf rank of [gamma+1, hi]
    node_info[gamma + 1].x = up_right;
  }
  *reinterpret_cast<int4*>(f + T::kIntOff) = make_int4(left, right, aux_l, aux_r);
  if (i == 0) node_info[0].x = kNoParent;
  // refit climbers start at the large nodes whose two children are leaves or
  // small subtrees (both slots are complete before k_refit runs)
  const bool start = (hi - lo + 1 > kDirectRange) && (gamma - lo + 1 <= kDirectRange) &&
                     (hi - gamma <= kDirectRange);
  const uint32_t mask = __ballot_sync(__activemask(), start);
  if (mask) {
    const int leader = __ffs(mask) - 1;
    int32_t base = 0;
    if ((threadIdx.x & 31) == leader) base = atomicAdd(num_starts, __popc(mask));
    base = __shfl_sync(__activemask(), base, leader);
    if (start) starts[base + __popc(mask & ((1u << (threadIdx.x & 31)) - 1))] = static_cast<int32_t>(i);
  }
}

// Box of every non-root internal node with <= kDirectRange leaves, reduced
// directly over its contiguous leaf run, into its slot of the parent.
template <int D>
__global__ void __launch_bounds__(256)
k_small_boxes(const float4* __restrict__ leaf_lo, const float4* __restrict__ leaf_hi,
              const int4* __restrict__ node_info, int64_t m, float4* __restrict__ nodes) {
  using T = NodeTraits<D>;
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x + 1; c < m - 1;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int4 info = node_info[c];
    if (info.w - info.z + 1 > kDirectRange) continue;
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int32_t s = info.z; s <= info.w; ++s) {
      const float4 a = __ldg(leaf_lo + s), b = __ldg(leaf_hi + s);
      lo[0] = fminf(lo[0], a.x);
      lo[1] = fminf(lo[1], a.y);
      lo[2] = fminf(lo[2], a.z);
      hi[0] = fmaxf(hi[0], b.x);
      hi[1] = fmaxf(hi[1], b.y);
      hi[2] = fmaxf(hi[2], b.z);
    }
    float* pf = reinterpret_cast<float*>(nodes + static_cast<int64_t>(up_parent(info.x)) * T::kVec);
    float* slot = pf + (up_is_left(info.x) ? 0 : 2 * D);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      slot[k] = lo[k];
      slot[D + k] = hi[k];
    }
  }
}

// Bottom-up refit (bvh.cpp:88-124) of the nodes above kDirectRange leaves.
// Climbers start at the large nodes whose children are leaves or small
// subtrees (slots filled by k_karras / k_small_boxes, which run first; k_karras
// lists them). A finished node writes its box (union of its two slots) into its
// slot of the parent; if the sibling is a leaf or small the climber continues,
// otherwise the two climbers meet at an arrival counter and the second one
// continues. Only that meeting needs ordering: the writer's slot store must be
// visible before its arrival (release fence, issued once per warp step for all
// lanes that need it); the second arriver reads the sibling slot through L2
// (ld.cg), after the atomic that observed the sibling's arrival.
template <int D>
__global__ void __launch_bounds__(256)
k_refit(const int32_t* __restrict__ starts, const int32_t* __restrict__ num_starts,
        float4* nodes, const int4* __restrict__ node_info, int32_t* __restrict__ arrivals) {
  using T = NodeTraits<D>;
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int32_t count = *num_starts;
  if (blockIdx.x * static_cast<int64_t>(blockDim.x) >= count) return;  // whole block idle
  bool active = t < count;
  int32_t c = active ? starts[t] : 0;
  while (__any_sync(0xffffffffu, active)) {
    bool fence = false;
    int32_t p = 0;
    if (active) {
      if (c == 0) {  // the root's own box is never tested (bvh.hpp:55-58)
        active = false;
      } else {
        const float* cf = reinterpret_cast<const float*>(nodes + static_cast<int64_t>(c) * T::kVec);
        float lo[3], hi[3];
#pragma unroll
        for (int k = 0; k < D; ++k) {
          lo[k] = fminf(__ldcg(cf + k), __ldcg(cf + 2 * D + k));
          hi[k] = fmaxf(__ldcg(cf + D + k), __ldcg(cf + 3 * D + k));
        }
        p = up_parent(node_info[c].x);
        float* pf = reinterpret_cast<float*>(nodes + static_cast<int64_t>(p) * T::kVec);
        const int2 pl = *reinterpret_cast<const int2*>(pf + T::kIntOff);
        const bool is_left = pl.x == c;
        float* slot = pf + (is_left ? 0 : 2 * D);
#pragma unroll
        for (int k = 0; k < D; ++k) {
          __stcg(slot + k, lo[k]);
          __stcg(slot + D + k, hi[k]);
        }
        const int32_t sibling = is_left ? pl.y : pl.x;
        bool ready = sibling < 0;  // a leaf: its slot is already in place
        if (!ready) {
          const int4 si = node_info[sibling];
          ready = si.w - si.z + 1 <= kDirectRange;  // filled by k_small_boxes
        }
        if (ready)
          c = p;
        else
          fence = true;  // meet the sibling's climber
      }
    }
    if (__any_sync(0xffffffffu, fence)) __threadfence();
    if (fence) {
      if (atomicAdd(arrivals + p, 1) == 0)
        active = false;
      else
        c = p;
    }
  }
}

// 1-leaf tree: pseudo root with the leaf on the left and an empty box right.
template <int D, class Src>
__global__ void k_single_leaf(Src src, const int32_t* __restrict__ prim_aux, float4* nodes,
                              float4* leaf_pt, int4* node_info, int32_t* leaf_up) {
  node_info[0] = make_int4(kNoParent, 0, 0, 0);
  leaf_up[0] = kUpLeftBit;
  using T = NodeTraits<D>;
  float lo[3], hi[3];
  src.box(0, lo, hi);
  float* f = reinterpret_cast<float*>(nodes);
  for (int k = 0; k < D; ++k) {
    f[k] = lo[k];
    f[D + k] = hi[k];
    f[2 * D + k] = INFINITY;
    f[3 * D + k] = -INFINITY;
  }
  int32_t aux = prim_aux ? prim_aux[0] : 0;
  int4* ip = reinterpret_cast<int4*>(f + T::kIntOff);
  *ip = make_int4(~0, ~0, aux, aux);
  if (leaf_pt) leaf_pt[0] = make_float4(lo[0], lo[1], D == 3 ? lo[2] : 0.f, __int_as_float(0));
}

template <int D, class Src>
BuiltBvh build_impl(const Src& boxes, const PrimSource& src, bool validate_finite,
                    bool points_mode, DevCounters* d_ctr, Scratch& scratch,
                    StageClock* clock) {
  cudaStream_t st = scratch.stream();
  const int64_t m = src.count;
  BuiltBvh out;
  out.tree.num_leaves = static_cast<int32_t>(m);
  const int64_t num_nodes = std::max<int64_t>(1, m - 1);
  out.tree.nodes = scratch.alloc_n<float4>(num_nodes * NodeTraits<D>::kVec);
  if (points_mode) out.leaf_pt = scratch.alloc_n<float4>(m);

  // Reset the per-build reductions (bounds, key AND/OR, finiteness flag).
  note_launch(), k_reset_build<<<1, 32, 0, st>>>(d_ctr);

  const unsigned g = grid_for(m, 256, 148 * 8);
  note_launch(), k_centroid_bounds<D><<<g, 256, 0, st>>>(boxes, m, validate_finite, d_ctr);
  uint64_t* keys = scratch.alloc_n<uint64_t>(m);
  int32_t* vals = scratch.alloc_n<int32_t>(m);
  note_launch(), k_morton<D><<<g, 256, 0, st>>>(boxes, m, d_ctr, keys, vals);
  TCB_CUDA(cudaGetLastError());

  // One small read-back: finiteness + key AND/OR decide the sort passes.
  auto* h = static_cast<unsigned char*>(pinned_staging(64));
  TCB_CUDA(cudaMemcpyAsync(h, &d_ctr->key_and, 16, cudaMemcpyDeviceToHost, st));
  TCB_CUDA(cudaMemcpyAsync(h + 16, &d_ctr->nonfinite, 4, cudaMemcpyDeviceToHost, st));
  TCB_CUDA(cudaStreamSynchronize(st));
  unsigned long long key_and, key_or;
  int32_t nonfinite;
  std::memcpy(&key_and, h, 8);
  std::memcpy(&key_or, h + 8, 8);
  std::memcpy(&nonfinite, h + 16, 4);
  if (validate_finite && nonfinite) throw InvalidArgument{"PointSet: non-finite coordinate"};

  if (clock) clock->mark(kStSort);
  uint64_t* keys_alt = scratch.alloc_n<uint64_t>(m);
  int32_t* vals_alt = scratch.alloc_n<int32_t>(m);
  void* sort_tmp = scratch.alloc(radix_sort_scratch_bytes(m));
  bool in_alt = radix_sort_pairs(keys, vals, keys_alt, vals_alt, m, key_and, key_or,
                                 sort_tmp, st, &out.sort_passes);
  const uint64_t* codes = in_alt ? keys_alt : keys;
  int32_t* order = in_alt ? vals_alt : vals;
  out.tree.leaf_order = order;

  if (clock) clock->mark(kStTopo);
  float4* leaf_pt = out.leaf_pt;
  out.codes = codes;
  out.node_info = scratch.alloc_n<int4>(std::max<int64_t>(1, m - 1));
  out.leaf_up = scratch.alloc_n<int32_t>(m);
  uint32_t* scene = scratch.alloc_n<uint32_t>(8);
  TCB_CUDA(cudaMemcpyAsync(scene, &d_ctr->bounds_ord[0], 6 * sizeof(uint32_t),
                           cudaMemcpyDeviceToDevice, st));
  out.scene_ord = scene;
  if (m == 1) {
    note_launch(), k_single_leaf<D><<<1, 1, 0, st>>>(boxes, src.aux, out.tree.nodes, leaf_pt,
                                                     out.node_info, out.leaf_up);
  } else {
    int32_t* arrivals = scratch.alloc_n<int32_t>(m);  // [m-1] = start count
    int32_t* starts = scratch.alloc_n<int32_t>(m / 2 + 1);
    TCB_CUDA(cudaMemsetAsync(arrivals, 0, sizeof(int32_t) * m, st));
    const unsigned gn = grid_for(m - 1, 256, INT32_MAX);
    // sorted leaf boxes (points mode: the query points themselves)
    float4* leaf_lo = points_mode ? leaf_pt : scratch.alloc_n<float4>(m);
    float4* leaf_hi = points_mode ? leaf_pt : scratch.alloc_n<float4>(m);
    note_launch(), k_gather_leaves<D><<<grid_for(m, 256), 256, 0, st>>>(boxes, order, m, leaf_lo,
                                                                         leaf_hi);
    note_launch(), k_karras<D><<<gn, 256, 0, st>>>(leaf_lo, leaf_hi, codes, order, src.aux, m,
                                                   out.tree.nodes, out.node_info, out.leaf_up,
                                                   starts, arrivals + (m - 1));
    note_launch(), k_small_boxes<D><<<grid_for(m, 256), 256, 0, st>>>(leaf_lo, leaf_hi,
                                                                       out.node_info, m,
                                                                       out.tree.nodes);
    note_launch(), k_refit<D><<<grid_for(m / 2 + 1, 256, INT32_MAX), 256, 0, st>>>(
        starts, arrivals + (m - 1), out.tree.nodes, out.node_info, arrivals);
  }
  TCB_CUDA(cudaGetLastError());
  return out;
}

}  // namespace

namespace {

// compute_bounds (geometry.hpp:95-101): raw point min/max (not centroids)
// plus the finiteness check of PointSet::validate.
template <int D>
__global__ void __launch_bounds__(256)
k_point_bounds(const float* __restrict__ coords, int64_t n, DevCounters* ctr) {
  float mn[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, mx[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
  bool bad = false;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      float v = coords[i * D + k];
      bad |= !isfinite(v);
      mn[k] = fminf(mn[k], v);
      mx[k] = fmaxf(mx[k], v);
    }
  }
  publish_bounds<D>(mn, mx, bad, ctr);
}

}  // namespace

template <int D>
void launch_point_bounds(const float* coords, int64_t n, DevCounters* ctr, cudaStream_t s) {
  note_launch(), k_reset_build<<<1, 32, 0, s>>>(ctr);
  note_launch(), k_point_bounds<D><<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(coords, n, ctr);
  TCB_CUDA(cudaGetLastError());
}

template void launch_point_bounds<2>(const float*, int64_t, DevCounters*, cudaStream_t);
template void launch_point_bounds<3>(const float*, int64_t, DevCounters*, cudaStream_t);

template <int D>
BuiltBvh build_bvh(const PrimSource& src, bool validate_finite, DevCounters* d_ctr,
                   Scratch& scratch, StageClock* clock) {
  if (src.coords) {
    PointBoxes<D> b{src.coords};
    return build_impl<D>(b, src, validate_finite, true, d_ctr, scratch, clock);
  }
  ExplicitBoxes<D> b{src.lo, src.hi};
  return build_impl<D>(b, src, validate_finite, false, d_ctr, scratch, clock);
}

template BuiltBvh build_bvh<2>(const PrimSource&, bool, DevCounters*, Scratch&, StageClock*);
template BuiltBvh build_bvh<3>(const PrimSource&, bool, DevCounters*, Scratch&, StageClock*);

}  // namespace tcb
