// Device-side parity checker: check_equivalence
// (REF oracle.cpp:120-163) on device buffers, so the parity gates at 37M-497M
// points cost milliseconds instead of host loops.
//
//   k_eq_flags      core flags / noise sets: smallest diverging index
//                   (oracle.cpp:136-142 scan in index order and report the
//                   first)
//   k_eq_insert     core partition: per clustering, a hash table label ->
//                   smallest core index carrying it (the entry the reference's
//                   sequential emplace keeps, oracle.cpp:144-152)
//   k_eq_verify     a core i diverges iff the other clustering's label of the
//                   first core sharing i's label differs from its own; the
//                   smallest such i is exactly the index the sequential scan
//                   fails at
//   k_border_check  borders_valid (oracle.cpp:72-116): a border point is valid
//                   iff some core within eps carries its label; queried over
//                   the GPU point BVH, smallest invalid index reported
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

// slot 0: core flags, 1: noise, 2: core partition, 3: border A, 4: border B
struct EqState {
  unsigned long long first[5];
  unsigned long long cores;
};

__global__ void k_eq_flags(const int32_t* __restrict__ la, const uint8_t* __restrict__ ca,
                           const int32_t* __restrict__ lb, const uint8_t* __restrict__ cb,
                           int64_t n, EqState* st) {
  unsigned long long cores = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const bool a = ca[i] != 0, b = cb[i] != 0;
    if (a != b) atomicMin(&st->first[0], static_cast<unsigned long long>(i));
    if ((la[i] == -1) != (lb[i] == -1)) atomicMin(&st->first[1], static_cast<unsigned long long>(i));
    cores += a;
  }
  cores = warp_sum(cores);
  if ((threadIdx.x & 31) == 0 && cores) atomicAdd(&st->cores, cores);
}

constexpr unsigned long long kEmpty = ~0ull;

__device__ __forceinline__ uint64_t label_hash(int32_t v) {
  uint64_t z = static_cast<uint32_t>(v) * 0x9e3779b97f4a7c15ull;
  return z ^ (z >> 29);
}

// Open addressing, linear probing; keys are the label as an unsigned 32-bit
// value (kEmpty never collides with one), values the smallest core index.
__device__ __forceinline__ uint64_t table_slot(unsigned long long* keys, uint64_t mask, int32_t v,
                                               bool insert) {
  const unsigned long long k = static_cast<uint32_t>(v);
  for (uint64_t s = label_hash(v) & mask;; s = (s + 1) & mask) {
    unsigned long long cur = keys[s];
    if (cur == kEmpty && insert) cur = atomicCAS(keys + s, kEmpty, k);
    if (cur == k || (cur == kEmpty && insert)) return s;
    if (cur == kEmpty) return ~0ull;  // absent (never happens for an inserted label)
  }
}

__global__ void k_eq_insert(const int32_t* __restrict__ la, const uint8_t* __restrict__ ca,
                            const int32_t* __restrict__ lb, int64_t n, uint64_t mask,
                            unsigned long long* ka, unsigned int* va, unsigned long long* kb,
                            unsigned int* vb) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!ca[i]) continue;
    atomicMin(va + table_slot(ka, mask, la[i], true), static_cast<unsigned>(i));
    atomicMin(vb + table_slot(kb, mask, lb[i], true), static_cast<unsigned>(i));
  }
}

__global__ void k_eq_verify(const int32_t* __restrict__ la, const uint8_t* __restrict__ ca,
                            const int32_t* __restrict__ lb, int64_t n, uint64_t mask,
                            unsigned long long* ka, const unsigned int* __restrict__ va,
                            unsigned long long* kb, const unsigned int* __restrict__ vb,
                            EqState* st) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!ca[i]) continue;
    const unsigned ja = va[table_slot(ka, mask, la[i], false)];
    const unsigned jb = vb[table_slot(kb, mask, lb[i], false)];
    if (lb[ja] != lb[i] || la[jb] != la[i])
      atomicMin(&st->first[2], static_cast<unsigned long long>(i));
  }
}

template <int D>
void border_checks(const float* d_coords, int64_t n, float eps, const int32_t* const* labels,
                   const uint8_t* const* core, int count, unsigned long long* bad,
                   Scratch& scratch) {
  cudaStream_t st = scratch.stream();
  DevCounters* ctr = scratch.alloc_n<DevCounters>(1);
  TCB_CUDA(cudaMemsetAsync(ctr, 0, sizeof(DevCounters), st));
  PrimSource src;
  src.coords = d_coords;
  src.count = n;
  BuiltBvh b = build_bvh<D>(src, true, ctr, scratch, nullptr);
  const BallTest bt = BallTest::make(static_cast<double>(eps) * static_cast<double>(eps));
  for (int k = 0; k < count; ++k) {
    note_launch(), k_border_check<D><<<grid_for(n, 128, INT32_MAX), 128, 0, st>>>(
        b.tree.nodes, b.leaf_pt, n, bt, labels[k], core[k], bad + k);
    TCB_CUDA(cudaGetLastError());
  }
}

void border_checks_dim(const float* d_coords, int64_t n, int dim, float eps,
                       const int32_t* const* labels, const uint8_t* const* core, int count,
                       unsigned long long* bad, Scratch& scratch) {
  if (dim == 2)
    border_checks<2>(d_coords, n, eps, labels, core, count, bad, scratch);
  else
    border_checks<3>(d_coords, n, eps, labels, core, count, bad, scratch);
}

}  // namespace

int64_t first_bad_border(const float* d_coords, int64_t n, int dim, float eps,
                         const int32_t* d_labels, const uint8_t* d_core, cudaStream_t st) {
  Scratch scratch(st);
  auto* bad = scratch.alloc_n<unsigned long long>(1);
  TCB_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st));
  border_checks_dim(d_coords, n, dim, eps, &d_labels, &d_core, 1, bad, scratch);
  unsigned long long h = 0;
  TCB_CUDA(cudaMemcpyAsync(&h, bad, sizeof h, cudaMemcpyDeviceToHost, st));
  TCB_CUDA(cudaStreamSynchronize(st));
  return h == kEmpty ? -1 : static_cast<int64_t>(h);
}

EqVerdict check_equivalence_device(const float* d_coords, int64_t n, int dim, float eps,
                                   const int32_t* la, const uint8_t* ca, const int32_t* lb,
                                   const uint8_t* cb, cudaStream_t st) {
  Scratch scratch(st);
  auto* state = scratch.alloc_n<EqState>(1);
  TCB_CUDA(cudaMemsetAsync(state, 0xff, sizeof(EqState::first), st));
  TCB_CUDA(cudaMemsetAsync(&state->cores, 0, sizeof(unsigned long long), st));
  const unsigned g = grid_for(n, 256, 148 * 16);
  note_launch(), k_eq_flags<<<g, 256, 0, st>>>(la, ca, lb, cb, n, state);
  TCB_CUDA(cudaGetLastError());
  EqState h;
  TCB_CUDA(cudaMemcpyAsync(&h, state, sizeof h, cudaMemcpyDeviceToHost, st));
  TCB_CUDA(cudaStreamSynchronize(st));
  EqVerdict v;
  auto done = [&](int check, unsigned long long at) {
    v.check = check;
    v.at = static_cast<int64_t>(at);
    return v;
  };
  if (h.first[0] != kEmpty) return done(1, h.first[0]);
  if (h.first[1] != kEmpty) return done(2, h.first[1]);
  if (h.cores > 0) {
    uint64_t slots = 2;
    while (slots < 2 * h.cores) slots <<= 1;
    auto* ka = scratch.alloc_n<unsigned long long>(static_cast<int64_t>(slots));
    auto* kb = scratch.alloc_n<unsigned long long>(static_cast<int64_t>(slots));
    auto* va = scratch.alloc_n<unsigned int>(static_cast<int64_t>(slots));
    auto* vb = scratch.alloc_n<unsigned int>(static_cast<int64_t>(slots));
    TCB_CUDA(cudaMemsetAsync(ka, 0xff, slots * sizeof(unsigned long long), st));
    TCB_CUDA(cudaMemsetAsync(kb, 0xff, slots * sizeof(unsigned long long), st));
    TCB_CUDA(cudaMemsetAsync(va, 0xff, slots * sizeof(unsigned int), st));
    TCB_CUDA(cudaMemsetAsync(vb, 0xff, slots * sizeof(unsigned int), st));
    note_launch(), k_eq_insert<<<g, 256, 0, st>>>(la, ca, lb, n, slots - 1, ka, va, kb, vb);
    note_launch(), k_eq_verify<<<g, 256, 0, st>>>(la, ca, lb, n, slots - 1, ka, va, kb, vb, state);
    TCB_CUDA(cudaGetLastError());
  }
  const int32_t* labels[2] = {la, lb};
  const uint8_t* core[2] = {ca, cb};
  border_checks_dim(d_coords, n, dim, eps, labels, core, 2, &state->first[3], scratch);
  TCB_CUDA(cudaMemcpyAsync(&h, state, sizeof h, cudaMemcpyDeviceToHost, st));
  TCB_CUDA(cudaStreamSynchronize(st));
  for (int k = 2; k < 5; ++k)
    if (h.first[k] != kEmpty) return done(k + 1, h.first[k]);
  return done(0, 0);
}

const char* equivalence_message(int check) {
  switch (check) {
    case 0: return "PASS";
    case 1: return "core flags differ";
    case 2: return "noise sets differ";
    case 3: return "core partitions differ";
    case 4: return "first clustering has an invalid border label";
    case 5: return "second clustering has an invalid border label";
  }
  return "unknown";
}

}  // namespace tcb
