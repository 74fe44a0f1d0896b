// Stage-level probes for the parity tests (treeclust_gpu.h, tcg_debug_*):
// each runs ONE device stage on host-provided inputs and copies its result
// back, so a test can compare it with the reference's own accessors:
//   tcg_debug_point_bvh   the device LBVH in the reference's node view
//                         (bvh.hpp:74-79: leaf(r).id, node_left/right/
//                         max_rank/box) — trees must be identical
//   tcg_debug_sort_pairs  the radix sort (stable, (key, index) order)
//   tcg_debug_union_find  concurrent device unite() over an edge list, then
//                         flatten (acceptance.cpp:174-233 compares against a
//                         sequential replay)
//   tcg_debug_grid        the device build_grid (dense_grid.cpp:23-77): perm,
//                         cell_of_point, cells (id, begin, end, dense)
//   tcg_debug_mixed_bvh   the DenseBox tree over make_mixed_primitives
//                         (dense_grid.cpp:79-98) in the reference's node view
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "device_common.cuh"
#include "engine.hpp"
#include "pipeline.hpp"
#include "primitives.cuh"

#define TC_EXPORT extern "C" __attribute__((visibility("default")))

namespace tcb {
namespace {

__global__ void k_unite_edges(const int32_t* __restrict__ edges, int64_t m, int32_t* parent) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < m;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    uf_unite(parent, edges[2 * e], edges[2 * e + 1]);
}

__global__ void k_flatten(int32_t* parent, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t p = ld_relaxed(parent + i), q;
    while (p != (q = ld_relaxed(parent + p))) p = q;
    st_relaxed(parent + i, p);
  }
}

template <int D>
void point_bvh(const float* d_coords, int64_t n, Scratch& scratch, std::vector<float4>& nodes,
               std::vector<int32_t>& order) {
  DevCounters* ctr = scratch.alloc_n<DevCounters>(1);
  TCB_CUDA(cudaMemsetAsync(ctr, 0, sizeof(DevCounters), scratch.stream()));
  PrimSource src;
  src.coords = d_coords;
  src.count = n;
  BuiltBvh b = build_bvh<D>(src, true, ctr, scratch, nullptr);
  const int64_t nn = n > 1 ? n : 1;  // n - 1 internal nodes + the spare slot
  nodes.resize(static_cast<size_t>(nn * NodeTraits<D>::kVec));
  order.resize(static_cast<size_t>(n));
  TCB_CUDA(cudaMemcpyAsync(nodes.data(), b.tree.nodes, nodes.size() * sizeof(float4),
                           cudaMemcpyDeviceToHost, scratch.stream()));
  TCB_CUDA(cudaMemcpyAsync(order.data(), b.tree.leaf_order, order.size() * sizeof(int32_t),
                           cudaMemcpyDeviceToHost, scratch.stream()));
  TCB_CUDA(cudaStreamSynchronize(scratch.stream()));
}

template <typename Fn>
tc_status run_guarded(Fn&& fn) {
  try {
    return fn();
  } catch (const InvalidArgument&) {
    return TC_ERR_INVALID_ARGUMENT;
  } catch (...) {
    cudaGetLastError();
    return TC_ERR_INTERNAL;
  }
}

struct Stream {
  cudaStream_t s = nullptr;
  Stream() { TCB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~Stream() {
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
};

}  // namespace
}  // namespace tcb

using namespace tcb;

namespace tcb {
namespace {

// Our internal nodes are numbered by split (root moved to 0, k_climb); the
// reference numbers them Karras-style: the root is 0, a left child is named
// by the last rank of its range, a right child by the first. Writes the
// reference's node view (bvh.hpp:74-79) of our records.
void karras_view(const std::vector<float4>& nodes, int dim, int64_t m, int32_t* left,
                 int32_t* right, int32_t* max_rank, float* boxes) {
  const int kv = 4;  // NodeTraits<D>::kVec
  struct Item {
    int32_t ours, karras, lo, hi;
  };
  std::vector<Item> todo{{0, 0, 0, static_cast<int32_t>(m - 1)}};
  while (!todo.empty()) {
    const Item it = todo.back();
    todo.pop_back();
    const float* f = reinterpret_cast<const float*>(nodes.data() + static_cast<int64_t>(it.ours) * kv);
    const int32_t* ii = reinterpret_cast<const int32_t*>(f + 4 * dim);
    const int32_t split = ii[0] < 0 ? ~ii[0] : ii[2];  // last rank of the left child
    const int32_t i = it.karras;
    left[i] = ii[0] < 0 ? ii[0] : split;
    right[i] = ii[1] < 0 ? ii[1] : split + 1;
    max_rank[i] = it.hi;
    if (ii[0] >= 0) todo.push_back({ii[0], split, it.lo, split});
    if (ii[1] >= 0) todo.push_back({ii[1], split + 1, split + 1, it.hi});
    // Own box = union of the two child boxes stored in the node.
    for (int k = 0; k < 3; ++k) {
      float lo = 0.f, hi = 0.f;
      if (k < dim) {
        lo = f[k] < f[2 * dim + k] ? f[k] : f[2 * dim + k];
        hi = f[dim + k] > f[3 * dim + k] ? f[dim + k] : f[3 * dim + k];
      }
      boxes[6 * i + k] = lo;
      boxes[6 * i + 3 + k] = hi;
    }
  }
}

template <int D>
void mixed_bvh(const float* d_coords, int64_t n, float eps, int minpts, Scratch& scratch,
               std::vector<float4>& nodes, std::vector<int32_t>& leaf_aux) {
  DevCounters* ctr = scratch.alloc_n<DevCounters>(1);
  TCB_CUDA(cudaMemsetAsync(ctr, 0, sizeof(DevCounters), scratch.stream()));
  const DeviceGrid g = build_device_grid<D>(d_coords, n, eps, minpts, ctr, scratch);
  float4 *lo, *hi;
  int32_t* aux;
  build_mixed_prims<D>(g, n, scratch, &lo, &hi, &aux);
  PrimSource src;
  src.lo = lo;
  src.hi = hi;
  src.aux = aux;
  src.count = g.num_prims;
  BuiltBvh b = build_bvh<D>(src, false, ctr, scratch, nullptr);
  const int64_t m = g.num_prims;
  nodes.resize(static_cast<size_t>(std::max<int64_t>(m, 1) * NodeTraits<D>::kVec));
  std::vector<int32_t> order(static_cast<size_t>(m)), paux(static_cast<size_t>(m));
  cudaStream_t st = scratch.stream();
  TCB_CUDA(cudaMemcpyAsync(nodes.data(), b.tree.nodes, sizeof(float4) * nodes.size(),
                           cudaMemcpyDeviceToHost, st));
  TCB_CUDA(cudaMemcpyAsync(order.data(), b.tree.leaf_order, sizeof(int32_t) * m,
                           cudaMemcpyDeviceToHost, st));
  TCB_CUDA(cudaMemcpyAsync(paux.data(), aux, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, st));
  TCB_CUDA(cudaStreamSynchronize(st));
  leaf_aux.resize(static_cast<size_t>(m));
  for (int64_t r = 0; r < m; ++r) leaf_aux[r] = paux[order[r]];
}

}  // namespace
}  // namespace tcb

TC_EXPORT tc_status tcg_debug_point_bvh(const float* coords, int64_t n, int dim,
                                        int32_t* leaf_ids, int32_t* left, int32_t* right,
                                        int32_t* max_rank, float* boxes) {
  if (!coords || n < 1 || (dim != 2 && dim != 3)) return TC_ERR_INVALID_ARGUMENT;
  return run_guarded([&] {
    Stream st;
    std::vector<float4> nodes;
    std::vector<int32_t> order;
    {
      Scratch scratch(st.s);
      float* d = scratch.alloc_n<float>(n * dim);
      TCB_CUDA(cudaMemcpyAsync(d, coords, sizeof(float) * n * dim, cudaMemcpyHostToDevice, st.s));
      if (dim == 2)
        point_bvh<2>(d, n, scratch, nodes, order);
      else
        point_bvh<3>(d, n, scratch, nodes, order);
    }
    std::memcpy(leaf_ids, order.data(), sizeof(int32_t) * n);
    if (n == 1) return TC_OK;
    karras_view(nodes, dim, n, left, right, max_rank, boxes);
    return TC_OK;
  });
}

TC_EXPORT tc_status tcg_debug_sort_pairs(const uint64_t* keys, int64_t n, uint64_t* keys_out,
                                         int32_t* vals_out) {
  if (!keys || n < 1) return TC_ERR_INVALID_ARGUMENT;
  return run_guarded([&] {
    Stream st;
    Scratch scratch(st.s);
    uint64_t* k = scratch.alloc_n<uint64_t>(n);
    uint64_t* k2 = scratch.alloc_n<uint64_t>(n);
    int32_t* v = scratch.alloc_n<int32_t>(n);
    int32_t* v2 = scratch.alloc_n<int32_t>(n);
    std::vector<int32_t> iota(static_cast<size_t>(n));
    uint64_t a = ~0ull, o = 0;
    for (int64_t i = 0; i < n; ++i) {
      iota[i] = static_cast<int32_t>(i);
      a &= keys[i];
      o |= keys[i];
    }
    TCB_CUDA(cudaMemcpyAsync(k, keys, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, st.s));
    TCB_CUDA(cudaMemcpyAsync(v, iota.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st.s));
    void* tmp = scratch.alloc(radix_sort_scratch_bytes(n));
    bool alt = radix_sort_pairs(k, v, k2, v2, n, a, o, tmp, st.s);
    TCB_CUDA(cudaMemcpyAsync(keys_out, alt ? k2 : k, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, st.s));
    TCB_CUDA(cudaMemcpyAsync(vals_out, alt ? v2 : v, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st.s));
    TCB_CUDA(cudaStreamSynchronize(st.s));
    return TC_OK;
  });
}

TC_EXPORT tc_status tcg_debug_union_find(const int32_t* edges, int64_t m, int32_t n,
                                         int32_t* parent_out) {
  if (!edges || !parent_out || n < 1 || m < 0) return TC_ERR_INVALID_ARGUMENT;
  return run_guarded([&] {
    Stream st;
    Scratch scratch(st.s);
    int32_t* e = scratch.alloc_n<int32_t>(2 * m);
    int32_t* parent = scratch.alloc_n<int32_t>(n);
    uint8_t* flags = scratch.alloc_n<uint8_t>(n);
    if (m) TCB_CUDA(cudaMemcpyAsync(e, edges, sizeof(int32_t) * 2 * m, cudaMemcpyHostToDevice, st.s));
    init_union_find(parent, flags, n, st.s);
    if (m) note_launch(), k_unite_edges<<<grid_for(m, 256), 256, 0, st.s>>>(e, m, parent);
    note_launch(), k_flatten<<<grid_for(n, 256), 256, 0, st.s>>>(parent, n);
    TCB_CUDA(cudaGetLastError());
    TCB_CUDA(cudaMemcpyAsync(parent_out, parent, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st.s));
    TCB_CUDA(cudaStreamSynchronize(st.s));
    return TC_OK;
  });
}

TC_EXPORT tc_status tcg_debug_grid(const float* coords, int64_t n, int dim, float eps, int minpts,
                                   int32_t* perm, int32_t* cell_of_point, uint64_t* cell_id,
                                   int32_t* cell_begin, int32_t* cell_end, uint8_t* cell_dense,
                                   int64_t cap, int64_t* num_cells) {
  if (!coords || n < 1 || (dim != 2 && dim != 3) || !perm || !cell_of_point || !num_cells ||
      !(eps > 0.f) || minpts < 2)
    return TC_ERR_INVALID_ARGUMENT;
  return run_guarded([&] {
    Stream st;
    Scratch scratch(st.s);
    float* d = scratch.alloc_n<float>(n * dim);
    TCB_CUDA(cudaMemcpyAsync(d, coords, sizeof(float) * n * dim, cudaMemcpyHostToDevice, st.s));
    DevCounters* ctr = scratch.alloc_n<DevCounters>(1);
    TCB_CUDA(cudaMemsetAsync(ctr, 0, sizeof(DevCounters), st.s));
    const DeviceGrid g = dim == 2 ? build_device_grid<2>(d, n, eps, minpts, ctr, scratch)
                                  : build_device_grid<3>(d, n, eps, minpts, ctr, scratch);
    const int64_t m = g.num_cells;
    std::vector<int32_t> cos(static_cast<size_t>(n)), cb(static_cast<size_t>(m));
    std::vector<uint64_t> ids(static_cast<size_t>(n));
    TCB_CUDA(cudaMemcpyAsync(perm, g.perm, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st.s));
    TCB_CUDA(cudaMemcpyAsync(cos.data(), g.cell_of_sorted, sizeof(int32_t) * n,
                             cudaMemcpyDeviceToHost, st.s));
    TCB_CUDA(cudaMemcpyAsync(ids.data(), g.ids, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, st.s));
    TCB_CUDA(cudaMemcpyAsync(cb.data(), g.cell_begin, sizeof(int32_t) * m, cudaMemcpyDeviceToHost,
                             st.s));
    if (m <= cap && cell_end && cell_dense) {
      TCB_CUDA(cudaMemcpyAsync(cell_end, g.cell_end, sizeof(int32_t) * m, cudaMemcpyDeviceToHost,
                               st.s));
      TCB_CUDA(cudaMemcpyAsync(cell_dense, g.cell_dense, m, cudaMemcpyDeviceToHost, st.s));
    }
    TCB_CUDA(cudaStreamSynchronize(st.s));
    for (int64_t s2 = 0; s2 < n; ++s2) cell_of_point[perm[s2]] = cos[s2];
    if (m <= cap && cell_id && cell_begin) {
      for (int64_t c = 0; c < m; ++c) {
        cell_begin[c] = cb[c];
        cell_id[c] = ids[cb[c]];
      }
    }
    *num_cells = m;
    return TC_OK;
  });
}

TC_EXPORT tc_status tcg_debug_mixed_bvh(const float* coords, int64_t n, int dim, float eps,
                                        int minpts, uint8_t* leaf_kind, int32_t* leaf_id,
                                        int32_t* left, int32_t* right, int32_t* max_rank,
                                        float* boxes, int64_t cap, int64_t* num_leaves) {
  if (!coords || n < 1 || (dim != 2 && dim != 3) || !num_leaves || !(eps > 0.f) || minpts < 2)
    return TC_ERR_INVALID_ARGUMENT;
  return run_guarded([&] {
    Stream st;
    std::vector<float4> nodes;
    std::vector<int32_t> leaf_aux;
    {
      Scratch scratch(st.s);
      float* d = scratch.alloc_n<float>(n * dim);
      TCB_CUDA(cudaMemcpyAsync(d, coords, sizeof(float) * n * dim, cudaMemcpyHostToDevice, st.s));
      if (dim == 2)
        mixed_bvh<2>(d, n, eps, minpts, scratch, nodes, leaf_aux);
      else
        mixed_bvh<3>(d, n, eps, minpts, scratch, nodes, leaf_aux);
    }
    const int64_t m = static_cast<int64_t>(leaf_aux.size());
    *num_leaves = m;
    if (m > cap || !leaf_kind || !leaf_id) return TC_OK;
    for (int64_t r = 0; r < m; ++r) {  // payload: point index, or ~cell for a DenseBox
      leaf_kind[r] = leaf_aux[r] < 0 ? 1 : 0;
      leaf_id[r] = leaf_aux[r] < 0 ? ~leaf_aux[r] : leaf_aux[r];
    }
    if (m > 1 && left && right && max_rank && boxes)
      karras_view(nodes, dim, m, left, right, max_rank, boxes);
    return TC_OK;
  });
}
