// Host-side interface between the C ABI (capi.cpp) and the device pipeline.
// No torch types, no exceptions across the ABI: every entry returns tc_status.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <functional>

#include "treeclust.h"

namespace tcb {

// Internal exceptions thrown inside the engine and mapped to tc_status at the
// ABI (mirrors `guarded`, capi.cpp:30-43).
struct InvalidArgument {
  const char* what;
};
struct CapExceeded {};
struct CudaFailure {
  cudaError_t err;
  const char* file;
  int line;
};

#define TCB_CUDA(expr)                                              \
  do {                                                              \
    cudaError_t _e = (expr);                                        \
    if (_e != cudaSuccess) throw ::tcb::CudaFailure{_e, __FILE__, __LINE__}; \
  } while (0)

// Per-stage device milliseconds (see tcg_last_stage_ms in treeclust_gpu.h).
enum Stage { kStBounds = 0, kStSort, kStTopo, kStGrid, kStCore, kStMain, kStFinal, kStTotal, kNumStages };

struct RunOutput {
  tc_cluster_stats stats{};
  double stage_ms[kNumStages]{};
};

// Called with [i0, i1) once labels/core flags of those points are final
// (enqueued on the given stream): lets tc_cluster overlap the device->host
// copy of early chunks with the finalize of later ones.
using ChunkSink = std::function<void(int64_t i0, int64_t i1, cudaStream_t)>;

// Full device pipeline. d_coords/d_labels/d_core are device pointers.
// want_stats: synchronize at the end and fill `out`.
// FDBSCAN never synchronizes the host before that end (the build's sort is
// planned on the device); a non-finite coordinate turns the outputs into
// all noise, sets *d_status (device int, optional) to TC_ERR_INVALID_ARGUMENT
// and, with want_stats / out, throws InvalidArgument after the final sync.
// `tail` (optional) is invoked after the last kernel is enqueued and before
// the final synchronization, e.g. to enqueue the device->host result copies.
void run_device(const float* d_coords, int64_t n, int dim, float eps, int minpts,
                tc_algorithm algo, int64_t oracle_cap, int32_t* d_labels,
                uint8_t* d_core, cudaStream_t stream, bool want_stats,
                RunOutput* out,
                const std::function<void(cudaStream_t)>& tail = nullptr,
                const int32_t* d_keys = nullptr, const ChunkSink* sink = nullptr,
                int32_t* d_status = nullptr);

// Stream-ordered allocation from the library's private per-device pool (the
// process's default pool is left alone); release with cudaFreeAsync.
void* pool_alloc(size_t bytes, cudaStream_t stream);
// Bytes the private pools keep reserved across calls (default 24 GiB), and an
// immediate release of everything unused.
void set_pool_release_threshold(uint64_t bytes);
void trim_pools();

// Kernel-launch accounting (thread-local; reset at the start of run_device).
void note_launch();
void reset_launch_count();
int64_t launch_count();

// Thread-local copy of the last run's stage times.
void set_last_stage_ms(const double* ms);
int get_last_stage_ms(double* out, int cap);

// ---- Morton-range sharded path behind the C ABI (multi.cu) ----
// num shards, shard s on CUDA device devices[s] (devices may repeat); host
// coords in, host labels / core flags out in input order.
template <int D>
void cluster_multi(const float* h_coords, int64_t n, float eps, int minpts, const int* devices,
                   int num, int32_t* h_labels, uint8_t* h_core, tc_cluster_stats* stats);

}  // namespace tcb
