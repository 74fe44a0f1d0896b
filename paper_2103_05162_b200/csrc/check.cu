// Device-side parity checker: the border-validity part
// of check_equivalence (oracle.cpp:72-116) over the GPU point BVH. A border
// point (non-core, non-noise) is valid iff some core point within eps carries
// the same label. Returns the smallest invalid index (the reference scans
// borders in index order and reports the first).
#include <climits>
#include <cstring>

#include "check.hpp"
#include "device_common.cuh"
#include "pipeline.hpp"

namespace tcb {

namespace {

template <int D>
__global__ void __launch_bounds__(128)
k_border_check(const float4* __restrict__ nodes, const float4* __restrict__ leaf_pt, int64_t m,
               BallTest bt, const int32_t* __restrict__ labels, const uint8_t* __restrict__ core,
               unsigned long long* __restrict__ bad) {
  int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= m) return;
  float4 q = leaf_pt[r];
  const int32_t i = __float_as_int(q.w);
  if (core[i] || labels[i] == -1) return;
  const int32_t li = labels[i];
  float p[3] = {q.x, q.y, q.z};
  bool ok = false;
  auto visit = [&](int32_t, int32_t j, const float*, const float*) -> bool {
    if (core[j] && labels[j] == li) {
      ok = true;
      return false;
    }
    return true;
  };
  bvh_query<D>(nodes, p, bt, 0, visit);
  if (!ok) atomicMin(bad, static_cast<unsigned long long>(i));
}

template <int D>
int64_t first_bad_border_impl(const float* d_coords, int64_t n, float eps,
                              const int32_t* d_labels, const uint8_t* d_core, cudaStream_t st) {
  Scratch scratch(st);
  DevCounters* ctr = scratch.alloc_n<DevCounters>(1);
  TCB_CUDA(cudaMemsetAsync(ctr, 0, sizeof(DevCounters), st));
  PrimSource src;
  src.coords = d_coords;
  src.count = n;
  BuiltBvh b = build_bvh<D>(src, true, ctr, scratch, nullptr);
  unsigned long long* bad = scratch.alloc_n<unsigned long long>(1);
  TCB_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st));
  const double eps2 = static_cast<double>(eps) * static_cast<double>(eps);
  note_launch(), k_border_check<D><<<grid_for(n, 128, INT32_MAX), 128, 0, st>>>(b.tree.nodes, b.leaf_pt, n,
                                                                 BallTest::make(eps2), d_labels, d_core, bad);
  TCB_CUDA(cudaGetLastError());
  unsigned long long h = 0;
  TCB_CUDA(cudaMemcpyAsync(&h, bad, sizeof h, cudaMemcpyDeviceToHost, st));
  TCB_CUDA(cudaStreamSynchronize(st));
  return h == ~0ull ? -1 : static_cast<int64_t>(h);
}

}  // namespace

int64_t first_bad_border(const float* d_coords, int64_t n, int dim, float eps,
                         const int32_t* d_labels, const uint8_t* d_core, cudaStream_t st) {
  return dim == 2 ? first_bad_border_impl<2>(d_coords, n, eps, d_labels, d_core, st)
                  : first_bad_border_impl<3>(d_coords, n, eps, d_labels, d_core, st);
}

}  // namespace tcb
