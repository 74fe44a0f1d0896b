// tcg_cluster_multi: the Morton-range sharded path of SURVEY.md §8(e) behind
// the C ABI, for a C / C++ caller of the drop-in (the Python path,
// paper_2103_05162_b200/shard.py, runs the same protocol one process per GPU
// over torch.distributed). One host thread per shard drives its device; the
// exchanges are peer copies (cudaMemcpyPeerAsync: NVLink between B200s, a
// plain device copy when two shards share a device). Protocol:
//   1. the input is cut into S contiguous slices, one per shard; the global
//      scene box is the min / max of the slice bounds;
//   2. Morton codes of every point against the global box; a strided sample
//      of each slice's codes gives S - 1 splitters;
//   3. every slice sends each point (coords, global id) to the shard owning
//      its Morton range (block-aggregated counts and slots, peer copies);
//   4. each shard sorts its own points by code and publishes the boxes of
//      runs of kHaloBlock of them; it sends every peer its points within eps
//      of one of the peer's boxes (tcg_near_boxes_device) — the ghosts;
//   5. local clustering of own + ghost points keyed by global id:
//      minpts == 2 one keyed run (tcg_cluster_keyed_device: core == "has a
//      neighbour", exact for own points); minpts > 2 one local context
//      (tcg_local_*): exact own core flags, the ghosts' flags from their
//      owners (peer copies in export order), then the main pass;
//   6. every core that is a ghost somewhere or was exported yields an edge
//      (global id, local label); the edges of all shards are merged by a
//      host union-find with min-id hooking, so every cluster is labelled by
//      its minimum core id — exactly the single-GPU / reference label;
//   7. own labels are mapped through the merge and written to the result in
//      input order.
// Core flags, noise and core labels equal tc_cluster's; borders take a valid
// adjacent cluster. pair_resolutions / distance_evaluations are not summed
// across shards (ghost pairs would be counted twice) and are reported as 0.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <exception>
#include <memory>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include "device_common.cuh"
#include "engine.hpp"
#include "pipeline.hpp"
#include "primitives.cuh"
#include "treeclust_gpu.h"

namespace tcb {
namespace {

constexpr int kMaxShards = 64;
constexpr int64_t kHaloBlock = 2048;
constexpr int64_t kSamplesPerShard = 4096;

// Device buffer owned by one shard's device.
struct DevBuf {
  void* p = nullptr;
  int dev = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { reset(); }
  void reset() {
    if (p) {
      cudaSetDevice(dev);
      cudaFree(p);
      p = nullptr;
    }
  }
  template <typename T>
  T* alloc(int d, int64_t count) {
    reset();
    dev = d;
    TCB_CUDA(cudaSetDevice(d));
    TCB_CUDA(cudaMalloc(&p, static_cast<size_t>(std::max<int64_t>(count, 1)) * sizeof(T)));
    return static_cast<T*>(p);
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

__device__ __forceinline__ int owner_of(uint64_t code, const uint64_t* __restrict__ split, int ns) {
  int lo = 0, hi = ns;  // first splitter > code
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (split[mid] > code) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// Owner histogram of a slice: per-block shared counts, one global atomic per
// (block, owner).
__global__ void __launch_bounds__(256)
k_owner_hist(const uint64_t* __restrict__ codes, int64_t n, const uint64_t* __restrict__ split,
             int ns, unsigned long long* __restrict__ counts) {
  __shared__ unsigned s_cnt[kMaxShards];
  for (int o = threadIdx.x; o <= ns; o += blockDim.x) s_cnt[o] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    atomicAdd(&s_cnt[owner_of(codes[i], split, ns)], 1u);
  __syncthreads();
  for (int o = threadIdx.x; o <= ns; o += blockDim.x)
    if (s_cnt[o]) atomicAdd(&counts[o], static_cast<unsigned long long>(s_cnt[o]));
}

// Scatter a slice into per-owner segments of the send buffers (order inside
// a segment is arbitrary: results are keyed by global id).
template <int D>
__global__ void __launch_bounds__(256)
k_owner_scatter(const float* __restrict__ x, const uint64_t* __restrict__ codes, int64_t n,
                int32_t gid0, const uint64_t* __restrict__ split, int ns,
                unsigned long long* __restrict__ cursor, float* __restrict__ sx,
                int32_t* __restrict__ sgid) {
  __shared__ unsigned s_cnt[kMaxShards];
  __shared__ unsigned long long s_base[kMaxShards];
  for (int64_t b0 = static_cast<int64_t>(blockIdx.x) * blockDim.x; b0 < n;
       b0 += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    for (int o = threadIdx.x; o <= ns; o += blockDim.x) s_cnt[o] = 0;
    __syncthreads();
    const int64_t i = b0 + threadIdx.x;
    int o = 0;
    unsigned loc = 0;
    if (i < n) {
      o = owner_of(codes[i], split, ns);
      loc = atomicAdd(&s_cnt[o], 1u);
    }
    __syncthreads();
    for (int q = threadIdx.x; q <= ns; q += blockDim.x)
      if (s_cnt[q]) s_base[q] = atomicAdd(&cursor[q], static_cast<unsigned long long>(s_cnt[q]));
    __syncthreads();
    if (i < n) {
      const unsigned long long dst = s_base[o] + loc;
#pragma unroll
      for (int k = 0; k < D; ++k) sx[dst * D + k] = x[i * D + k];
      sgid[dst] = gid0 + static_cast<int32_t>(i);
    }
    __syncthreads();
  }
}

// Boxes of runs of kHaloBlock own points in Morton order: one block per box.
template <int D>
__global__ void __launch_bounds__(256)
k_run_boxes(const float* __restrict__ x, const int32_t* __restrict__ order, int64_t n,
            float* __restrict__ lo, float* __restrict__ hi) {
  const int64_t b = blockIdx.x;
  const int64_t s = b * kHaloBlock, e = min(s + kHaloBlock, n);
  float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t r = s + threadIdx.x; r < e; r += blockDim.x) {
    const int64_t i = order[r];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      mn[k] = fminf(mn[k], x[i * D + k]);
      mx[k] = fmaxf(mx[k], x[i * D + k]);
    }
  }
  __shared__ float red[32];
  auto fmin_op = [](float a, float c) { return fminf(a, c); };
  auto fmax_op = [](float a, float c) { return fmaxf(a, c); };
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const float a = block_reduce(mn[k], fmin_op, INFINITY, red);
    if (threadIdx.x == 0) lo[b * D + k] = a;
    const float c = block_reduce(mx[k], fmax_op, -INFINITY, red);
    if (threadIdx.x == 0) hi[b * D + k] = c;
  }
}

// Indices of the set mask entries, in index order (mask -> scan -> slots).
__global__ void k_mask_to_int(const uint8_t* __restrict__ m, int64_t n, int32_t* __restrict__ v) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    v[i] = m[i] ? 1 : 0;
}
__global__ void k_compact(const uint8_t* __restrict__ m, const int32_t* __restrict__ pos, int64_t n,
                          int32_t* __restrict__ idx) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (m[i]) idx[pos[i]] = static_cast<int32_t>(i);
}

// Gather rows idx of (x, gid) into a packed send segment.
template <int D>
__global__ void k_gather_rows(const float* __restrict__ x, const int32_t* __restrict__ gid,
                              const int32_t* __restrict__ idx, int64_t m, float* __restrict__ ox,
                              int32_t* __restrict__ ogid) {
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < m;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx[j];
#pragma unroll
    for (int k = 0; k < D; ++k) ox[j * D + k] = x[i * D + k];
    ogid[j] = gid[i];
  }
}

__global__ void k_gather_u8(const uint8_t* __restrict__ v, const int32_t* __restrict__ idx,
                            int64_t m, uint8_t* __restrict__ out) {
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < m;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[j] = v[idx[j]];
}

__global__ void k_mark(const int32_t* __restrict__ idx, int64_t m, uint8_t* __restrict__ flag) {
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < m;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x)
    flag[idx[j]] = 1;
}

// Edge flags: a core that is a ghost (i >= n_own) or was exported.
__global__ void k_edge_mask(const uint8_t* __restrict__ core, const uint8_t* __restrict__ exported,
                            int64_t n_own, int64_t nl, uint8_t* __restrict__ m) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nl;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    m[i] = core[i] && (i >= n_own || exported[i]) ? 1 : 0;
}

__global__ void k_edges(const int32_t* __restrict__ gid, const int32_t* __restrict__ lab,
                        const int32_t* __restrict__ idx, int64_t m, int2* __restrict__ e) {
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < m;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t i = idx[j];
    e[j] = make_int2(gid[i], lab[i]);
  }
}

struct Shard {
  int dev = 0;
  cudaStream_t st = nullptr;
  int64_t b = 0, e = 0;  // input slice
  DevBuf slice_x, codes, counts, split, send_x, send_gid;
  std::vector<int64_t> send_cnt, send_off;  // per destination shard
  DevBuf own_x, own_gid;                    // own points, then ghosts
  int64_t n_own = 0, n_ghost = 0;
  std::vector<float> box_lo, box_hi;  // host copies of the run boxes
  int64_t nb = 0;
  std::vector<std::unique_ptr<DevBuf>> exp_idx;  // per peer: exported own indices
  std::vector<int64_t> exp_cnt;
  DevBuf lab, core, core_in;
  std::vector<int2> edges;
};

// Runs fn(s) for every shard on its own host thread (device set), rethrowing
// the first failure.
template <typename Fn>
void each_shard(std::vector<Shard>& sh, Fn&& fn) {
  std::vector<std::thread> th;
  std::exception_ptr err;
  std::mutex mu;
  for (size_t s = 0; s < sh.size(); ++s)
    th.emplace_back([&, s] {
      try {
        TCB_CUDA(cudaSetDevice(sh[s].dev));
        fn(static_cast<int>(s));
        TCB_CUDA(cudaStreamSynchronize(sh[s].st));
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        if (!err) err = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  if (err) std::rethrow_exception(err);
}

void check_status(tc_status st) {
  if (st == TC_ERR_INVALID_ARGUMENT) throw InvalidArgument{"sharded run: invalid argument"};
  if (st != TC_OK) throw CudaFailure{cudaErrorUnknown, __FILE__, __LINE__};
}

unsigned g(int64_t n) { return grid_for(n, 256); }

}  // namespace

template <int D>
void cluster_multi(const float* h_coords, int64_t n, float eps, int minpts, const int* devices,
                   int num, int32_t* h_labels, uint8_t* h_core, tc_cluster_stats* stats) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  std::vector<Shard> sh(static_cast<size_t>(num));
  for (int s = 0; s < num; ++s) {
    sh[s].dev = devices[s];
    sh[s].b = n * s / num;
    sh[s].e = n * (s + 1) / num;
    TCB_CUDA(cudaSetDevice(sh[s].dev));
    TCB_CUDA(cudaStreamCreateWithFlags(&sh[s].st, cudaStreamNonBlocking));
  }
  struct Streams {
    std::vector<Shard>* sh;
    ~Streams() {
      for (auto& x : *sh)
        if (x.st) {
          cudaSetDevice(x.dev);
          cudaStreamSynchronize(x.st);
          cudaStreamDestroy(x.st);
        }
    }
  } streams_guard{&sh};

  // 1. slices up; slice bounds -> global scene box
  std::vector<float> lo(3, INFINITY), hi(3, -INFINITY);
  std::mutex mu;
  each_shard(sh, [&](int s) {
    Shard& x = sh[s];
    const int64_t m = x.e - x.b;
    float* d = x.slice_x.alloc<float>(x.dev, m * D);
    if (m == 0) return;
    TCB_CUDA(cudaMemcpyAsync(d, h_coords + x.b * D, sizeof(float) * m * D, cudaMemcpyHostToDevice,
                             x.st));
    Scratch scratch(x.st);
    DevCounters* ctr = scratch.alloc_n<DevCounters>(1);
    TCB_CUDA(cudaMemsetAsync(ctr, 0, sizeof(DevCounters), x.st));
    launch_point_bounds<D>(d, m, ctr, x.st);
    DevCounters h;
    TCB_CUDA(cudaMemcpyAsync(&h, ctr, sizeof h, cudaMemcpyDeviceToHost, x.st));
    TCB_CUDA(cudaStreamSynchronize(x.st));
    if (h.nonfinite) throw InvalidArgument{"PointSet: non-finite coordinate"};
    std::lock_guard<std::mutex> lk(mu);
    for (int k = 0; k < D; ++k) {
      lo[k] = std::min(lo[k], ord2f(h.bounds_ord[k]));
      hi[k] = std::max(hi[k], ord2f(h.bounds_ord[3 + k]));
    }
  });

  // 2. Morton codes against the global box, sampled splitters
  std::vector<uint64_t> samples;
  each_shard(sh, [&](int s) {
    Shard& x = sh[s];
    const int64_t m = x.e - x.b;
    uint64_t* c = x.codes.alloc<uint64_t>(x.dev, m);
    if (m == 0) return;
    check_status(tcg_morton_codes_device(x.slice_x.as<float>(), m, D, lo.data(), hi.data(), c,
                                         x.st));
    const int64_t k = std::min(m, kSamplesPerShard);
    const int64_t stride = m / k;
    std::vector<uint64_t> smp(static_cast<size_t>(k));
    TCB_CUDA(cudaMemcpy2DAsync(smp.data(), sizeof(uint64_t), c, sizeof(uint64_t) * stride,
                               sizeof(uint64_t), static_cast<size_t>(k), cudaMemcpyDeviceToHost,
                               x.st));
    TCB_CUDA(cudaStreamSynchronize(x.st));
    std::lock_guard<std::mutex> lk(mu);
    samples.insert(samples.end(), smp.begin(), smp.end());
  });
  std::sort(samples.begin(), samples.end());
  std::vector<uint64_t> split;
  for (int j = 1; j < num; ++j)
    split.push_back(samples.empty() ? ~0ull : samples[samples.size() * j / num]);

  // 3. redistribution: counts, send segments, own buffers, peer copies
  each_shard(sh, [&](int s) {
    Shard& x = sh[s];
    const int64_t m = x.e - x.b;
    x.send_cnt.assign(num, 0);
    x.send_off.assign(num + 1, 0);
    uint64_t* dsplit = x.split.alloc<uint64_t>(x.dev, num);
    auto* cnt = x.counts.alloc<unsigned long long>(x.dev, 2 * num);
    if (num > 1)
      TCB_CUDA(cudaMemcpyAsync(dsplit, split.data(), sizeof(uint64_t) * (num - 1),
                               cudaMemcpyHostToDevice, x.st));
    TCB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * 2 * num, x.st));
    float* sx = x.send_x.alloc<float>(x.dev, m * D);
    int32_t* sg = x.send_gid.alloc<int32_t>(x.dev, m);
    if (m == 0) return;
    note_launch(), k_owner_hist<<<g(m), 256, 0, x.st>>>(x.codes.as<uint64_t>(), m, dsplit, num - 1,
                                                       cnt);
    std::vector<unsigned long long> hc(static_cast<size_t>(num));
    TCB_CUDA(cudaMemcpyAsync(hc.data(), cnt, sizeof(unsigned long long) * num,
                             cudaMemcpyDeviceToHost, x.st));
    TCB_CUDA(cudaStreamSynchronize(x.st));
    for (int t = 0; t < num; ++t) {
      x.send_cnt[t] = static_cast<int64_t>(hc[t]);
      x.send_off[t + 1] = x.send_off[t] + x.send_cnt[t];
    }
    std::vector<unsigned long long> cur(x.send_off.begin(), x.send_off.end() - 1);
    TCB_CUDA(cudaMemcpyAsync(cnt + num, cur.data(), sizeof(unsigned long long) * num,
                             cudaMemcpyHostToDevice, x.st));
    note_launch(), k_owner_scatter<D><<<std::min<unsigned>(g(m), 148 * 16), 256, 0, x.st>>>(
        x.slice_x.as<float>(), x.codes.as<uint64_t>(), m, static_cast<int32_t>(x.b), dsplit,
        num - 1, cnt + num, sx, sg);
    TCB_CUDA(cudaGetLastError());
  });
  each_shard(sh, [&](int t) {  // receive buffers (room for ghosts added later)
    Shard& x = sh[t];
    x.n_own = 0;
    for (int s = 0; s < num; ++s) x.n_own += sh[s].send_cnt[t];
    x.slice_x.reset();
    x.codes.reset();
  });
  // ghosts are at most every peer point; size the receive buffers after the
  // halo counts instead: first the own points into exact-size buffers
  std::vector<DevBuf> own_x(num), own_gid(num);
  each_shard(sh, [&](int t) {
    own_x[t].alloc<float>(sh[t].dev, sh[t].n_own * D);
    own_gid[t].alloc<int32_t>(sh[t].dev, sh[t].n_own);
  });
  each_shard(sh, [&](int s) {
    Shard& x = sh[s];
    for (int t = 0; t < num; ++t) {
      if (!x.send_cnt[t]) continue;
      int64_t at = 0;
      for (int q = 0; q < s; ++q) at += sh[q].send_cnt[t];
      TCB_CUDA(cudaMemcpyPeerAsync(own_x[t].as<float>() + at * D, sh[t].dev,
                                   x.send_x.as<float>() + x.send_off[t] * D, x.dev,
                                   sizeof(float) * x.send_cnt[t] * D, x.st));
      TCB_CUDA(cudaMemcpyPeerAsync(own_gid[t].as<int32_t>() + at, sh[t].dev,
                                   x.send_gid.as<int32_t>() + x.send_off[t], x.dev,
                                   sizeof(int32_t) * x.send_cnt[t], x.st));
    }
  });
  each_shard(sh, [&](int s) {
    sh[s].send_x.reset();
    sh[s].send_gid.reset();
  });
  const auto t_part = clk::now();

  // 4. halo: run boxes of each shard, then every shard's points near a peer's boxes
  each_shard(sh, [&](int t) {
    Shard& x = sh[t];
    x.nb = (x.n_own + kHaloBlock - 1) / kHaloBlock;
    x.box_lo.assign(static_cast<size_t>(x.nb * D), 0.f);
    x.box_hi.assign(static_cast<size_t>(x.nb * D), 0.f);
    if (x.n_own == 0 || num == 1) return;
    Scratch scratch(x.st);
    const int64_t m = x.n_own;
    uint64_t* k1 = scratch.alloc_n<uint64_t>(m);
    uint64_t* k2 = scratch.alloc_n<uint64_t>(m);
    int32_t* v1 = scratch.alloc_n<int32_t>(m);
    int32_t* v2 = scratch.alloc_n<int32_t>(m);
    check_status(tcg_morton_codes_device(own_x[t].as<float>(), m, D, lo.data(), hi.data(), k1,
                                         x.st));
    std::vector<int32_t> iota(static_cast<size_t>(m));
    for (int64_t i = 0; i < m; ++i) iota[i] = static_cast<int32_t>(i);
    TCB_CUDA(cudaMemcpyAsync(v1, iota.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, x.st));
    void* tmp = scratch.alloc(radix_sort_scratch_bytes(m));
    const bool alt = radix_sort_pairs(k1, v1, k2, v2, m, 0ull, ~0ull, tmp, x.st);
    float* blo = scratch.alloc_n<float>(x.nb * D);
    float* bhi = scratch.alloc_n<float>(x.nb * D);
    note_launch(), k_run_boxes<D><<<static_cast<unsigned>(x.nb), 256, 0, x.st>>>(
        own_x[t].as<float>(), alt ? v2 : v1, m, blo, bhi);
    TCB_CUDA(cudaMemcpyAsync(x.box_lo.data(), blo, sizeof(float) * x.nb * D,
                             cudaMemcpyDeviceToHost, x.st));
    TCB_CUDA(cudaMemcpyAsync(x.box_hi.data(), bhi, sizeof(float) * x.nb * D,
                             cudaMemcpyDeviceToHost, x.st));
    TCB_CUDA(cudaStreamSynchronize(x.st));
  });
  each_shard(sh, [&](int s) {
    Shard& x = sh[s];
    x.exp_idx.clear();
    x.exp_cnt.assign(num, 0);
    for (int t = 0; t < num; ++t) x.exp_idx.emplace_back(new DevBuf);
    if (x.n_own == 0 || num == 1) return;
    Scratch scratch(x.st);
    uint8_t* mask = scratch.alloc_n<uint8_t>(x.n_own);
    int32_t* ones = scratch.alloc_n<int32_t>(x.n_own);
    int32_t* pos = scratch.alloc_n<int32_t>(x.n_own);
    int32_t* tot = scratch.alloc_n<int32_t>(1);
    void* stmp = scratch.alloc(scan_scratch_bytes(x.n_own));
    for (int t = 0; t < num; ++t) {
      if (t == s || sh[t].nb == 0) continue;
      float* blo = scratch.alloc_n<float>(sh[t].nb * D);
      float* bhi = scratch.alloc_n<float>(sh[t].nb * D);
      TCB_CUDA(cudaMemcpyAsync(blo, sh[t].box_lo.data(), sizeof(float) * sh[t].nb * D,
                               cudaMemcpyHostToDevice, x.st));
      TCB_CUDA(cudaMemcpyAsync(bhi, sh[t].box_hi.data(), sizeof(float) * sh[t].nb * D,
                               cudaMemcpyHostToDevice, x.st));
      check_status(tcg_near_boxes_device(own_x[s].as<float>(), x.n_own, D, eps, blo, bhi,
                                         sh[t].nb, mask, x.st));
      note_launch(), k_mask_to_int<<<g(x.n_own), 256, 0, x.st>>>(mask, x.n_own, ones);
      exclusive_scan_i32(ones, pos, x.n_own, tot, stmp, x.st);
      int32_t h = 0;
      TCB_CUDA(cudaMemcpyAsync(&h, tot, sizeof(int32_t), cudaMemcpyDeviceToHost, x.st));
      TCB_CUDA(cudaStreamSynchronize(x.st));
      x.exp_cnt[t] = h;
      int32_t* idx = x.exp_idx[t]->alloc<int32_t>(x.dev, h);
      if (h) note_launch(), k_compact<<<g(x.n_own), 256, 0, x.st>>>(mask, pos, x.n_own, idx);
    }
  });
  // local sets: own points then ghosts (in (source shard, export) order)
  each_shard(sh, [&](int t) {
    Shard& x = sh[t];
    x.n_ghost = 0;
    for (int s = 0; s < num; ++s) x.n_ghost += sh[s].exp_cnt[t];
    const int64_t nl = x.n_own + x.n_ghost;
    float* lx = x.own_x.alloc<float>(x.dev, nl * D);
    int32_t* lg = x.own_gid.alloc<int32_t>(x.dev, nl);
    if (x.n_own) {
      TCB_CUDA(cudaMemcpyAsync(lx, own_x[t].as<float>(), sizeof(float) * x.n_own * D,
                               cudaMemcpyDeviceToDevice, x.st));
      TCB_CUDA(cudaMemcpyAsync(lg, own_gid[t].as<int32_t>(), sizeof(int32_t) * x.n_own,
                               cudaMemcpyDeviceToDevice, x.st));
    }
  });
  each_shard(sh, [&](int s) {  // ghosts: gather the exported rows, copy to the peer
    Shard& x = sh[s];
    for (int t = 0; t < num; ++t) {
      const int64_t c = x.exp_cnt[t];
      if (!c) continue;
      int64_t at = sh[t].n_own;
      for (int q = 0; q < s; ++q) at += sh[q].exp_cnt[t];
      Scratch scratch(x.st);
      float* gx = scratch.alloc_n<float>(c * D);
      int32_t* gg = scratch.alloc_n<int32_t>(c);
      note_launch(), k_gather_rows<D><<<g(c), 256, 0, x.st>>>(
          own_x[s].as<float>(), own_gid[s].as<int32_t>(), x.exp_idx[t]->as<int32_t>(), c, gx, gg);
      TCB_CUDA(cudaMemcpyPeerAsync(sh[t].own_x.as<float>() + at * D, sh[t].dev, gx, x.dev,
                                   sizeof(float) * c * D, x.st));
      TCB_CUDA(cudaMemcpyPeerAsync(sh[t].own_gid.as<int32_t>() + at, sh[t].dev, gg, x.dev,
                                   sizeof(int32_t) * c, x.st));
      TCB_CUDA(cudaStreamSynchronize(x.st));  // gx / gg are released with the scratch
    }
  });
  for (auto& b : own_x) b.reset();
  for (auto& b : own_gid) b.reset();
  const auto t_halo = clk::now();

  // 5. local clustering keyed by global id
  std::vector<std::unique_ptr<tcg_local, void (*)(tcg_local*)>> ctx;
  for (int s = 0; s < num; ++s) ctx.emplace_back(nullptr, tcg_local_free);
  each_shard(sh, [&](int t) {
    Shard& x = sh[t];
    const int64_t nl = x.n_own + x.n_ghost;
    int32_t* lab = x.lab.alloc<int32_t>(x.dev, nl);
    uint8_t* core = x.core.alloc<uint8_t>(x.dev, nl);
    if (nl == 0) return;
    if (minpts == 2) {
      check_status(tcg_cluster_keyed_device(x.own_x.as<float>(), x.own_gid.as<int32_t>(), nl, D,
                                            eps, 2, lab, core, x.st, nullptr));
    } else {
      tcg_local* c = nullptr;
      check_status(tcg_local_create(x.own_x.as<float>(), x.own_gid.as<int32_t>(), nl, D, eps,
                                    x.st, &c));
      ctx[t].reset(c);
      uint8_t* cin = x.core_in.alloc<uint8_t>(x.dev, nl);
      check_status(tcg_local_core_flags(c, minpts, cin));
    }
  });
  if (minpts > 2) {
    each_shard(sh, [&](int s) {  // owners' flags of the exported points -> the peers' ghosts
      Shard& x = sh[s];
      for (int t = 0; t < num; ++t) {
        const int64_t c = x.exp_cnt[t];
        if (!c) continue;
        int64_t at = sh[t].n_own;
        for (int q = 0; q < s; ++q) at += sh[q].exp_cnt[t];
        Scratch scratch(x.st);
        uint8_t* f = scratch.alloc_n<uint8_t>(c);
        note_launch(), k_gather_u8<<<g(c), 256, 0, x.st>>>(x.core_in.as<uint8_t>(),
                                                          x.exp_idx[t]->as<int32_t>(), c, f);
        TCB_CUDA(cudaMemcpyPeerAsync(sh[t].core_in.as<uint8_t>() + at, sh[t].dev, f, x.dev, c,
                                     x.st));
        TCB_CUDA(cudaStreamSynchronize(x.st));
      }
    });
    each_shard(sh, [&](int t) {
      Shard& x = sh[t];
      if (x.n_own + x.n_ghost == 0) return;
      check_status(tcg_local_cluster(ctx[t].get(), x.core_in.as<uint8_t>(), x.lab.as<int32_t>(),
                                     x.core.as<uint8_t>()));
    });
  }
  each_shard(sh, [&](int t) { ctx[t].reset(); });  // freed on their own device / stream
  const auto t_local = clk::now();

  // 6. cross-shard edges: cores that are ghosts here or were exported
  each_shard(sh, [&](int t) {
    Shard& x = sh[t];
    const int64_t nl = x.n_own + x.n_ghost;
    x.edges.clear();
    if (nl == 0 || num == 1) return;
    Scratch scratch(x.st);
    uint8_t* exported = scratch.alloc_n<uint8_t>(nl);
    TCB_CUDA(cudaMemsetAsync(exported, 0, static_cast<size_t>(nl), x.st));
    for (int q = 0; q < num; ++q)
      if (x.exp_cnt[q])
        note_launch(), k_mark<<<g(x.exp_cnt[q]), 256, 0, x.st>>>(x.exp_idx[q]->as<int32_t>(),
                                                                x.exp_cnt[q], exported);
    uint8_t* m = scratch.alloc_n<uint8_t>(nl);
    int32_t* ones = scratch.alloc_n<int32_t>(nl);
    int32_t* pos = scratch.alloc_n<int32_t>(nl);
    int32_t* tot = scratch.alloc_n<int32_t>(1);
    void* stmp = scratch.alloc(scan_scratch_bytes(nl));
    note_launch(), k_edge_mask<<<g(nl), 256, 0, x.st>>>(x.core.as<uint8_t>(), exported, x.n_own,
                                                       nl, m);
    note_launch(), k_mask_to_int<<<g(nl), 256, 0, x.st>>>(m, nl, ones);
    exclusive_scan_i32(ones, pos, nl, tot, stmp, x.st);
    int32_t h = 0;
    TCB_CUDA(cudaMemcpyAsync(&h, tot, sizeof(int32_t), cudaMemcpyDeviceToHost, x.st));
    TCB_CUDA(cudaStreamSynchronize(x.st));
    if (!h) return;
    int32_t* idx = scratch.alloc_n<int32_t>(h);
    int2* e = scratch.alloc_n<int2>(h);
    note_launch(), k_compact<<<g(nl), 256, 0, x.st>>>(m, pos, nl, idx);
    note_launch(), k_edges<<<g(h), 256, 0, x.st>>>(x.own_gid.as<int32_t>(), x.lab.as<int32_t>(),
                                                   idx, h, e);
    x.edges.resize(static_cast<size_t>(h));
    TCB_CUDA(cudaMemcpyAsync(x.edges.data(), e, sizeof(int2) * h, cudaMemcpyDeviceToHost, x.st));
  });
  // host union-find over the edge endpoints (min-id hooking)
  std::unordered_map<int32_t, int32_t> parent;
  auto find = [&](int32_t v) {
    auto it = parent.find(v);
    if (it == parent.end()) return v;
    int32_t r = v;
    while (true) {
      auto p = parent.find(r);
      if (p == parent.end() || p->second == r) break;
      r = p->second;
    }
    while (v != r) {  // path compression
      int32_t& pv = parent[v];
      const int32_t next = pv;
      pv = r;
      v = next;
    }
    return r;
  };
  for (auto& x : sh)
    for (const int2& e : x.edges) {
      const int32_t a = find(e.x), c = find(e.y);
      if (a == c) continue;
      parent[std::max(a, c)] = std::min(a, c);
      parent.emplace(std::min(a, c), std::min(a, c));
    }

  // 7. own labels through the merge, scattered to input order
  std::vector<int64_t> clusters(num, 0), cores(num, 0), noise(num, 0);
  each_shard(sh, [&](int t) {
    Shard& x = sh[t];
    const int64_t m = x.n_own;
    if (m == 0) return;
    std::vector<int32_t> gid(static_cast<size_t>(m)), lab(static_cast<size_t>(m));
    std::vector<uint8_t> core(static_cast<size_t>(m));
    TCB_CUDA(cudaMemcpyAsync(gid.data(), x.own_gid.as<int32_t>(), sizeof(int32_t) * m,
                             cudaMemcpyDeviceToHost, x.st));
    TCB_CUDA(cudaMemcpyAsync(lab.data(), x.lab.as<int32_t>(), sizeof(int32_t) * m,
                             cudaMemcpyDeviceToHost, x.st));
    TCB_CUDA(cudaMemcpyAsync(core.data(), x.core.as<uint8_t>(), m, cudaMemcpyDeviceToHost, x.st));
    TCB_CUDA(cudaStreamSynchronize(x.st));
    for (int64_t i = 0; i < m; ++i) {
      int32_t l = lab[i];
      if (l >= 0) {
        auto it = parent.find(l);
        if (it != parent.end()) {
          while (true) {  // read-only walk (no compression across threads)
            auto p = parent.find(l);
            if (p == parent.end() || p->second == l) break;
            l = p->second;
          }
        }
      }
      h_labels[gid[i]] = l;
      h_core[gid[i]] = core[i];
      clusters[t] += l >= 0 && l == gid[i];
      cores[t] += core[i] != 0;
      noise[t] += l < 0;
    }
  });
  const auto t_end = clk::now();
  if (stats) {
    *stats = tc_cluster_stats{};
    auto sec = [](clk::time_point a, clk::time_point b) {
      return std::chrono::duration<double>(b - a).count();
    };
    stats->build_seconds = sec(t0, t_halo);  // partition + halo
    stats->main_seconds = sec(t_halo, t_local);
    stats->finalize_seconds = sec(t_local, t_end);
    stats->preprocess_skipped = minpts == 2 ? 1 : 0;
    for (int s = 0; s < num; ++s) {
      stats->cluster_count += clusters[s];
      stats->core_count += cores[s];
      stats->noise_count += noise[s];
    }
  }
  (void)t_part;
}

template void cluster_multi<2>(const float*, int64_t, float, int, const int*, int, int32_t*,
                               uint8_t*, tc_cluster_stats*);
template void cluster_multi<3>(const float*, int64_t, float, int, const int*, int, int32_t*,
                               uint8_t*, tc_cluster_stats*);

}  // namespace tcb
