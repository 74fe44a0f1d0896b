// Orchestration of one device run (dbscan_run, dbscan.cpp:221-284, on the
// GPU): validation, index build, core pass, fused main pass, finalize, and
// per-stage CUDA-event timing into tc_cluster_stats.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <limits>
#include <mutex>
#include <string>

#include "device_common.cuh"
#include "engine.hpp"
#include "pipeline.hpp"

namespace tcb {

// ---------------------------------------------------------------------------
// Scratch / staging / clock
// ---------------------------------------------------------------------------
namespace {

// The library's own stream-ordered memory pool per device (the device's
// default pool, which other users of the process share, is never touched).
// Scratch is reused across calls up to the release threshold; above it the
// pool returns memory to the driver at the next synchronization, so a huge
// run (C5: ~80 GB) does not stay reserved afterwards.
constexpr int kMaxDevices = 64;
std::mutex g_pool_mu;
cudaMemPool_t g_pool[kMaxDevices] = {};
uint64_t g_pool_threshold = uint64_t{24} << 30;

cudaMemPool_t library_pool(int dev) {
  std::lock_guard<std::mutex> lock(g_pool_mu);
  if (!g_pool[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    TCB_CUDA(cudaMemPoolCreate(&pool, &props));
    TCB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &g_pool_threshold));
    g_pool[dev] = pool;
  }
  return g_pool[dev];
}

thread_local double t_last_stage_ms[kNumStages] = {};
thread_local int64_t t_launches = 0;

}  // namespace

Scratch::~Scratch() {
  for (void* p : ptrs_) cudaFreeAsync(p, stream_);
}

void* Scratch::alloc(size_t bytes) {
  void* p = pool_alloc(bytes, stream_);
  ptrs_.push_back(p);
  return p;
}

void* pool_alloc(size_t bytes, cudaStream_t stream) {
  int dev = 0;
  TCB_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) throw CudaFailure{cudaErrorInvalidDevice, __FILE__, __LINE__};
  void* p = nullptr;
  bytes = (bytes + 255) & ~size_t{255};
  cudaError_t e = cudaMallocFromPoolAsync(&p, bytes > 0 ? bytes : 256, library_pool(dev), stream);
  if (e != cudaSuccess) throw CudaFailure{e, __FILE__, __LINE__};
  return p;
}

void set_pool_release_threshold(uint64_t bytes) {
  std::lock_guard<std::mutex> lock(g_pool_mu);
  g_pool_threshold = bytes;
  for (cudaMemPool_t pool : g_pool)
    if (pool) TCB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &bytes));
}

void trim_pools() {
  std::lock_guard<std::mutex> lock(g_pool_mu);
  for (cudaMemPool_t pool : g_pool)
    if (pool) cudaMemPoolTrimTo(pool, 0);
}

void* pinned_staging(size_t bytes) {
  struct Buf {
    void* p = nullptr;
    size_t n = 0;
    ~Buf() {
      if (p) cudaFreeHost(p);
    }
  };
  thread_local Buf buf;
  if (buf.n < bytes) {
    if (buf.p) cudaFreeHost(buf.p);
    buf.p = nullptr;
    size_t want = bytes < 4096 ? 4096 : bytes;
    TCB_CUDA(cudaMallocHost(&buf.p, want));
    buf.n = want;
  }
  return buf.p;
}

StageClock::StageClock(cudaStream_t s) : stream_(s) {
  for (auto& e : ev_) e = nullptr;
}

StageClock::~StageClock() {
  for (auto& e : ev_)
    if (e) cudaEventDestroy(e);
}

void StageClock::mark(int stage_begin) {
  if (count_ > kNumStages) return;
  if (!ev_[count_]) TCB_CUDA(cudaEventCreate(&ev_[count_]));
  TCB_CUDA(cudaEventRecord(ev_[count_], stream_));
  stage_of_[count_] = stage_begin;
  ++count_;
}

void StageClock::finish() { mark(-1); }

void StageClock::collect(double* stage_ms) const {
  for (int s = 0; s < kNumStages; ++s) stage_ms[s] = 0.0;
  for (int i = 0; i + 1 < count_; ++i) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ev_[i], ev_[i + 1]) == cudaSuccess && stage_of_[i] >= 0)
      stage_ms[stage_of_[i]] += ms;
  }
  if (count_ >= 2) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ev_[0], ev_[count_ - 1]) == cudaSuccess)
      stage_ms[kStTotal] = ms;
  }
}

void note_launch() { ++t_launches; }
void reset_launch_count() { t_launches = 0; }
int64_t launch_count() { return t_launches; }


void set_last_stage_ms(const double* ms) {
  for (int s = 0; s < kNumStages; ++s) t_last_stage_ms[s] = ms[s];
}

int get_last_stage_ms(double* out, int cap) {
  int k = cap < kNumStages ? cap : kNumStages;
  for (int s = 0; s < k; ++s) out[s] = t_last_stage_ms[s];
  return k;
}

// ---------------------------------------------------------------------------
// FDBSCAN (dbscan.cpp:221-284 with Algorithm::Fdbscan)
// ---------------------------------------------------------------------------
template <int D>
void run_fdbscan(const float* d_coords, int64_t n, float eps, int minpts, int32_t* d_labels,
                 uint8_t* d_core, DevCounters* ctr, Scratch& scratch, StageClock& clock,
                 const int32_t* d_keys, const ChunkSink* sink) {
  cudaStream_t st = scratch.stream();
  const double eps2 = static_cast<double>(eps) * static_cast<double>(eps);
  PrimSource src;
  src.coords = d_coords;
  src.count = n;
  clock.mark(kStBounds);
  // stream-ordered: no host read-back; a non-finite coordinate is reported
  // by run_device from ctr->nonfinite
  BuiltBvh b = build_bvh<D>(src, /*validate_finite=*/true, ctr, scratch, &clock,
                            /*stream_ordered=*/true);

  int32_t* parent = scratch.alloc_n<int32_t>(n);
  uint8_t* flags = scratch.alloc_n<uint8_t>(n);
  const int32_t* key = b.tree.leaf_order;  // rank -> original index
  if (d_keys) {
    check_keys_nonnegative(d_keys, n, scratch);
    int32_t* k = scratch.alloc_n<int32_t>(n);
    gather_rank_keys(d_keys, b.tree.leaf_order, n, k, st);
    key = k;
  }
  clock.mark(kStCore);
  init_union_find(parent, flags, n, st);
  if (minpts > 2) fdbscan_core_pass<D>(b, n, eps2, minpts, flags, ctr, st);
  clock.mark(kStMain);
  fdbscan_main_pass<D>(b, key, n, eps2, minpts == 2, flags, parent, ctr, scratch);
  clock.mark(kStFinal);
  // whole-sector output writes through destination buckets; with a sink
  // (tc_cluster) the output is finished in 8 ranges, each copied to the host
  // while the next is written
  finalize_labels_bucketed(parent, flags, key, b.tree.leaf_order, n, d_labels, d_core, ctr,
                           scratch, minpts == 2, sink);
  clock.finish();
}

template void run_fdbscan<2>(const float*, int64_t, float, int, int32_t*, uint8_t*, DevCounters*,
                             Scratch&, StageClock&, const int32_t*, const ChunkSink*);
template void run_fdbscan<3>(const float*, int64_t, float, int, int32_t*, uint8_t*, DevCounters*,
                             Scratch&, StageClock&, const int32_t*, const ChunkSink*);

namespace {

// A stream-ordered FDBSCAN run over a non-finite coordinate did no traversal
// work: its outputs become all noise and the device status says why.
__global__ void k_nonfinite_outputs(const DevCounters* __restrict__ ctr, int64_t n,
                                    int32_t* __restrict__ labels, uint8_t* __restrict__ core,
                                    int32_t* __restrict__ d_status) {
  const bool bad = ctr->nonfinite != 0;
  if (d_status && blockIdx.x == 0 && threadIdx.x == 0)
    *d_status = bad ? TC_ERR_INVALID_ARGUMENT : TC_OK;
  if (!bad) return;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    labels[i] = -1;
    core[i] = 0;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// Entry
// ---------------------------------------------------------------------------
void run_device(const float* d_coords, int64_t n, int dim, float eps, int minpts,
                tc_algorithm algo, int64_t oracle_cap, int32_t* d_labels, uint8_t* d_core,
                cudaStream_t stream, bool want_stats, RunOutput* out,
                const std::function<void(cudaStream_t)>& tail, const int32_t* d_keys,
                const ChunkSink* sink, int32_t* d_status) {
  if (dim != 2 && dim != 3) throw InvalidArgument{"PointSet: dimension must be 2 or 3"};
  if (n < 1) throw InvalidArgument{"PointSet: empty"};
  if (!(eps > 0.f) || !std::isfinite(eps))
    throw InvalidArgument{"eps must be positive and finite"};
  if (minpts < 2) throw InvalidArgument{"minpts must be >= 2"};
  if (n > std::numeric_limits<int32_t>::max())
    throw InvalidArgument{"dbscan_run: more than 2^31-1 points"};
  if (!d_coords || !d_labels || !d_core) throw InvalidArgument{"null buffer"};
  if (d_keys && algo != TC_ALGO_FDBSCAN) throw InvalidArgument{"keys need FDBSCAN"};

  reset_launch_count();
  Scratch scratch(stream);
  StageClock clock(stream);
  DevCounters* ctr = scratch.alloc_n<DevCounters>(1);
  TCB_CUDA(cudaMemsetAsync(ctr, 0, sizeof(DevCounters), stream));

  double dense_fraction = 0.0;
  switch (algo) {
    case TC_ALGO_FDBSCAN:
      if (dim == 2)
        run_fdbscan<2>(d_coords, n, eps, minpts, d_labels, d_core, ctr, scratch, clock, d_keys,
                       sink);
      else
        run_fdbscan<3>(d_coords, n, eps, minpts, d_labels, d_core, ctr, scratch, clock, d_keys,
                       sink);
      note_launch(), k_nonfinite_outputs<<<grid_for(n, 256, 148 * 4), 256, 0, stream>>>(
          ctr, n, d_labels, d_core, d_status);
      TCB_CUDA(cudaGetLastError());
      d_status = nullptr;  // written
      break;
    case TC_ALGO_DENSEBOX:
      if (dim == 2)
        run_densebox<2>(d_coords, n, eps, minpts, d_labels, d_core, ctr, scratch, clock,
                        &dense_fraction);
      else
        run_densebox<3>(d_coords, n, eps, minpts, d_labels, d_core, ctr, scratch, clock,
                        &dense_fraction);
      break;
    case TC_ALGO_BRUTEFORCE: {
      int64_t cap = oracle_cap > 0 ? oracle_cap : 10000;
      if (n > cap) throw CapExceeded{};
      clock.mark(kStMain);
      if (dim == 2)
        run_bruteforce<2>(d_coords, n, eps, minpts, d_labels, d_core, ctr, scratch);
      else
        run_bruteforce<3>(d_coords, n, eps, minpts, d_labels, d_core, ctr, scratch);
      clock.finish();
      break;
    }
    default:
      throw InvalidArgument{"unknown algorithm"};
  }

  if (d_status) TCB_CUDA(cudaMemsetAsync(d_status, 0, sizeof(int32_t), stream));  // TC_OK
  if (tail) tail(stream);
  if (want_stats || out) {
    DevCounters h;
    TCB_CUDA(cudaMemcpyAsync(&h, ctr, sizeof h, cudaMemcpyDeviceToHost, stream));
    TCB_CUDA(cudaStreamSynchronize(stream));
    if (h.nonfinite) throw InvalidArgument{"PointSet: non-finite coordinate"};
    RunOutput ro;
    clock.collect(ro.stage_ms);
    set_last_stage_ms(ro.stage_ms);
    tc_cluster_stats& s = ro.stats;
    s.build_seconds =
        (ro.stage_ms[kStBounds] + ro.stage_ms[kStSort] + ro.stage_ms[kStTopo] +
         ro.stage_ms[kStGrid]) * 1e-3;
    s.preprocess_seconds = ro.stage_ms[kStCore] * 1e-3;
    s.main_seconds = ro.stage_ms[kStMain] * 1e-3;
    s.finalize_seconds = ro.stage_ms[kStFinal] * 1e-3;
    s.preprocess_skipped = (algo != TC_ALGO_BRUTEFORCE && minpts == 2) ? 1 : 0;
    s.dense_point_fraction = dense_fraction;
    if (algo != TC_ALGO_BRUTEFORCE) {
      s.pair_resolutions = h.pairs;
      s.distance_evaluations = h.dists;
    }
    s.cluster_count = h.clusters;
    s.core_count = h.cores;
    s.noise_count = h.noise;
    TCB_PROBE_ONLY(std::fprintf(stderr, "[probe] %llu %llu %llu %llu %llu %llu %llu %llu\n",
                                h.probe[0], h.probe[1], h.probe[2], h.probe[3], h.probe[4],
                                h.probe[5], h.probe[6], h.probe[7]);)
    if (out) *out = ro;
  }
}

}  // namespace tcb
