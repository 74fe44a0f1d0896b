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
