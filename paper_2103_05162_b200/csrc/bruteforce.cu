// TC_ALGO_BRUTEFORCE on the device: the O(n^2) reference semantics of
// dbscan_bruteforce (oracle.cpp:10-60), bounded by the oracle cap.
//
// The reference expands clusters breadth-first in index order, so its output
// is fully deterministic and has a closed form, which is what we compute:
//   core[i]   = |{j : d(i,j) <= eps}| >= minpts            (self included)
//   label of a core point = minimum index of its core component
//   label of a non-core point = minimum such label over the cores within eps
//                               (the first cluster expanded that reaches it),
//                               or -1 when no core is within eps.
// Distances use the exact fp64 chain of geometry.hpp:72-79. Points are staged
// through shared memory tiles; n <= cap keeps this a small kernel.
#include <cfloat>
#include <cstring>

#include "device_common.cuh"
#include "pipeline.hpp"

namespace tcb {

namespace {

constexpr int kBfBlock = 256;

template <int D>
__device__ __forceinline__ void load_pt(const float* coords, int64_t i, float* p) {
#pragma unroll
  for (int k = 0; k < D; ++k) p[k] = coords[i * D + k];
}

template <int D>
__global__ void __launch_bounds__(kBfBlock)
k_bf_core(const float* __restrict__ coords, int64_t n, double eps2, int minpts,
          uint8_t* __restrict__ core) {
  __shared__ float tile[kBfBlock * 3];
  const int64_t i = blockIdx.x * static_cast<int64_t>(kBfBlock) + threadIdx.x;
  float p[3] = {0.f, 0.f, 0.f};
  if (i < n) load_pt<D>(coords, i, p);
  int64_t count = 0;
  for (int64_t base = 0; base < n; base += kBfBlock) {
    int64_t j = base + threadIdx.x;
    if (j < n) load_pt<D>(coords, j, tile + threadIdx.x * 3);
    __syncthreads();
    const int lim = static_cast<int>(n - base < kBfBlock ? n - base : kBfBlock);
    if (i < n)
      for (int t = 0; t < lim; ++t) count += dist2<D>(p, tile + t * 3) <= eps2;
    __syncthreads();
  }
  if (i < n) core[i] = count >= minpts ? 1 : 0;
}

template <int D>
__global__ void __launch_bounds__(kBfBlock)
k_bf_union(const float* __restrict__ coords, int64_t n, double eps2,
           const uint8_t* __restrict__ core, int32_t* __restrict__ parent) {
  __shared__ float tile[kBfBlock * 3];
  __shared__ uint8_t tcore[kBfBlock];
  const int64_t i = blockIdx.x * static_cast<int64_t>(kBfBlock) + threadIdx.x;
  float p[3] = {0.f, 0.f, 0.f};
  const bool ci = i < n && core[i];
  if (i < n) load_pt<D>(coords, i, p);
  for (int64_t base = 0; base < n; base += kBfBlock) {
    int64_t j = base + threadIdx.x;
    if (j < n) {
      load_pt<D>(coords, j, tile + threadIdx.x * 3);
      tcore[threadIdx.x] = core[j];
    }
    __syncthreads();
    const int lim = static_cast<int>(n - base < kBfBlock ? n - base : kBfBlock);
    if (ci)
      for (int t = 0; t < lim; ++t)
        if (base + t > i && tcore[t] && dist2<D>(p, tile + t * 3) <= eps2)
          uf_unite(parent, static_cast<int32_t>(i), static_cast<int32_t>(base + t));
    __syncthreads();
  }
}

template <int D>
__global__ void __launch_bounds__(kBfBlock)
k_bf_label(const float* __restrict__ coords, int64_t n, double eps2,
           const uint8_t* __restrict__ core, const int32_t* __restrict__ root,
           int32_t* __restrict__ labels, DevCounters* ctr) {
  __shared__ float tile[kBfBlock * 3];
  __shared__ int32_t troot[kBfBlock];
  const int64_t i = blockIdx.x * static_cast<int64_t>(kBfBlock) + threadIdx.x;
  float p[3] = {0.f, 0.f, 0.f};
  const bool ci = i < n && core[i];
  if (i < n) load_pt<D>(coords, i, p);
  int32_t best = ci ? root[i] : INT32_MAX;
  for (int64_t base = 0; base < n; base += kBfBlock) {
    int64_t j = base + threadIdx.x;
    if (j < n) {
      load_pt<D>(coords, j, tile + threadIdx.x * 3);
      troot[threadIdx.x] = core[j] ? root[j] : -1;
    }
    __syncthreads();
    const int lim = static_cast<int>(n - base < kBfBlock ? n - base : kBfBlock);
    if (i < n && !ci)
      for (int t = 0; t < lim; ++t)
        if (troot[t] >= 0 && troot[t] < best && dist2<D>(p, tile + t * 3) <= eps2)
          best = troot[t];
    __syncthreads();
  }
  long long noise = 0, clusters = 0, cores = 0;
  if (i < n) {
    int32_t lab = best == INT32_MAX ? -1 : best;
    labels[i] = lab;
    noise = lab == -1;
    clusters = lab == static_cast<int32_t>(i);
    cores = ci;
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

__global__ void k_bf_flatten(int32_t* __restrict__ parent, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t p = ld_relaxed(parent + i);
    int32_t q;
    while (p != (q = ld_relaxed(parent + p))) p = q;
    st_relaxed(parent + i, p);
  }
}

}  // namespace

template <int D>
void run_bruteforce(const float* d_coords, int64_t n, float eps, int minpts, int32_t* d_labels,
                    uint8_t* d_core, DevCounters* ctr, Scratch& scratch) {
  cudaStream_t st = scratch.stream();
  launch_point_bounds<D>(d_coords, n, ctr, st);  // PointSet::validate
  auto* h = static_cast<int32_t*>(pinned_staging(64));
  TCB_CUDA(cudaMemcpyAsync(h, &ctr->nonfinite, 4, cudaMemcpyDeviceToHost, st));
  TCB_CUDA(cudaStreamSynchronize(st));
  if (*h) throw InvalidArgument{"PointSet: non-finite coordinate"};

  const double eps2 = static_cast<double>(eps) * static_cast<double>(eps);
  int32_t* parent = scratch.alloc_n<int32_t>(n);
  uint8_t* tmp_flags = scratch.alloc_n<uint8_t>(n);
  init_union_find(parent, tmp_flags, n, st);
  const unsigned g = grid_for(n, kBfBlock, INT32_MAX);
  note_launch(), k_bf_core<D><<<g, kBfBlock, 0, st>>>(d_coords, n, eps2, minpts, d_core);
  note_launch(), k_bf_union<D><<<g, kBfBlock, 0, st>>>(d_coords, n, eps2, d_core, parent);
  note_launch(), k_bf_flatten<<<grid_for(n, 256), 256, 0, st>>>(parent, n);
  note_launch(), k_bf_label<D><<<g, kBfBlock, 0, st>>>(d_coords, n, eps2, d_core, parent, d_labels, ctr);
  TCB_CUDA(cudaGetLastError());
}

template void run_bruteforce<2>(const float*, int64_t, float, int, int32_t*, uint8_t*,
                                DevCounters*, Scratch&);
template void run_bruteforce<3>(const float*, int64_t, float, int, int32_t*, uint8_t*,
                                DevCounters*, Scratch&);

}  // namespace tcb
