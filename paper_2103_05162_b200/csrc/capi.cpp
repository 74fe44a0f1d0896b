// The C ABI (include/treeclust.h, include/treeclust_gpu.h).
//
// Mirrors the reference's capi.cpp contract: opaque handles owned by the
// library, output handles written only on success, C++ failures mapped onto
// tc_status exactly like `guarded` (capi.cpp:30-43):
//   invalid argument -> TC_ERR_INVALID_ARGUMENT, I/O (std::runtime_error) ->
//   TC_ERR_IO, allocation / CUDA failure / anything else -> TC_ERR_INTERNAL.
// tc_cluster replaces dbscan_run with the device pipeline (engine.cu); the
// host copy of the points goes up once, labels + core flags come back once.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>

#include "check.hpp"
#include "engine.hpp"
#include "host_data.hpp"
#include "treeclust.h"
#include "treeclust_gpu.h"

#define TC_EXPORT extern "C" __attribute__((visibility("default")))

namespace {

// ---------------------------------------------------------------------------
// Host buffers: page-locked when large (full-rate H2D / D2H), cached across
// calls so repeated tc_cluster calls do not pay for pinning again.
// ---------------------------------------------------------------------------
class HostPool {
 public:
  static HostPool& get() {
    static HostPool* p = new HostPool();  // intentionally leaked (no teardown-order issues)
    return *p;
  }
  void* acquire(size_t bytes, bool* pinned) {
    *pinned = false;
    if (bytes == 0) bytes = 1;
    if (bytes >= kPinMin) {
      size_t key = round(bytes);
      {
        std::lock_guard<std::mutex> lock(mu_);
        auto it = free_.find(key);
        if (it != free_.end()) {
          void* p = it->second;
          free_.erase(it);
          cached_ -= key;
          *pinned = true;
          return p;
        }
      }
      void* p = nullptr;
      if (cudaMallocHost(&p, key) == cudaSuccess) {
        *pinned = true;
        return p;
      }
      cudaGetLastError();  // clear (no device / no driver): fall back to pageable
    }
    void* p = std::malloc(bytes);
    if (!p) throw std::bad_alloc();
    return p;
  }
  void release(void* p, size_t bytes, bool pinned) {
    if (!p) return;
    if (!pinned) {
      std::free(p);
      return;
    }
    size_t key = round(bytes);
    {
      std::lock_guard<std::mutex> lock(mu_);
      if (cached_ + key <= kCacheCap) {
        free_.emplace(key, p);
        cached_ += key;
        return;
      }
    }
    cudaFreeHost(p);
  }
  void trim() {
    std::lock_guard<std::mutex> lock(mu_);
    for (auto& kv : free_) cudaFreeHost(kv.second);
    free_.clear();
    cached_ = 0;
  }

 private:
  static constexpr size_t kPinMin = size_t{1} << 20;
  static constexpr size_t kCacheCap = size_t{4} << 30;  // pinned bytes kept for reuse
  static size_t round(size_t b) { return (b + (size_t{2} << 20) - 1) & ~((size_t{2} << 20) - 1); }
  std::mutex mu_;
  std::multimap<size_t, void*> free_;
  size_t cached_ = 0;
};

template <typename T>
struct HostArray {
  T* ptr = nullptr;
  size_t count = 0;
  bool pinned = false;
  HostArray() = default;
  explicit HostArray(size_t n) : count(n) {
    ptr = static_cast<T*>(HostPool::get().acquire(n * sizeof(T), &pinned));
  }
  HostArray(const HostArray&) = delete;
  HostArray& operator=(const HostArray&) = delete;
  ~HostArray() { HostPool::get().release(ptr, count * sizeof(T), pinned); }
};

}  // namespace

struct tc_dataset {
  int dim = 0;
  int64_t n = 0;
  HostArray<float> coords;
  tc_dataset(int d, int64_t count) : dim(d), n(count), coords(static_cast<size_t>(count) * d) {}
};

struct tc_result {
  int64_t n = 0;
  HostArray<int32_t> labels;
  HostArray<uint8_t> core;
  tc_cluster_stats stats{};
  explicit tc_result(int64_t count)
      : n(count), labels(static_cast<size_t>(count)), core(static_cast<size_t>(count)) {}
};

namespace {

template <typename Fn>
tc_status guarded(Fn&& fn) {
  try {
    return fn();
  } catch (const tcb::InvalidArgument&) {
    return TC_ERR_INVALID_ARGUMENT;
  } catch (const tcb::CapExceeded&) {
    return TC_ERR_CAP_EXCEEDED;
  } catch (const tcb::CudaFailure&) {
    cudaGetLastError();
    return TC_ERR_INTERNAL;
  } catch (const std::invalid_argument&) {
    return TC_ERR_INVALID_ARGUMENT;
  } catch (const std::runtime_error&) {
    return TC_ERR_IO;
  } catch (const std::bad_alloc&) {
    return TC_ERR_INTERNAL;
  } catch (...) {
    return TC_ERR_INTERNAL;
  }
}

tc_status publish(tcb::HostPoints&& pts, tc_dataset** out) {
  tcb::validate_points(pts.dim, pts.coords.data(), static_cast<int64_t>(pts.coords.size()));
  auto ds = std::make_unique<tc_dataset>(pts.dim, pts.size());
  std::memcpy(ds->coords.ptr, pts.coords.data(), pts.coords.size() * sizeof(float));
  *out = ds.release();
  return TC_OK;
}

// TCB_HOST_TIMING=1: host wall-clock marks of tc_cluster on stderr.
struct HostTimer {
  bool on = std::getenv("TCB_HOST_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[tc_cluster] %-22s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// RAII stream + device buffers for one ABI call.
struct DeviceCall {
  cudaStream_t st = nullptr;
  std::vector<void*> bufs;
  DeviceCall() {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
      cudaGetLastError();
      throw tcb::CudaFailure{cudaErrorNoDevice, __FILE__, __LINE__};
    }
    TCB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  }
  ~DeviceCall() {
    for (void* p : bufs) cudaFreeAsync(p, st);
    if (st) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
  }
  template <typename T>
  T* alloc(int64_t count) {
    void* p = tcb::pool_alloc(static_cast<size_t>(std::max<int64_t>(count, 1)) * sizeof(T), st);
    bufs.push_back(p);
    return static_cast<T*>(p);
  }
};

// One algorithm on a dataset already resident on the device.
// FDBSCAN results reach the host chunk by chunk: each finalized chunk is
// copied on a second stream while the next one is computed.
struct ChunkedCopy {
  cudaStream_t cp = nullptr;
  std::vector<cudaEvent_t> events;
  ChunkedCopy() { TCB_CUDA(cudaStreamCreateWithFlags(&cp, cudaStreamNonBlocking)); }
  ~ChunkedCopy() {
    if (cp) {
      cudaStreamSynchronize(cp);
      cudaStreamDestroy(cp);
    }
    for (cudaEvent_t e : events) cudaEventDestroy(e);
  }
};

void device_cluster(DeviceCall& call, const float* d_coords, int64_t n, int dim, float eps,
                    int minpts, tc_algorithm algo, int64_t cap, int32_t* d_labels,
                    uint8_t* d_core, tc_result* res) {
  tcb::RunOutput ro;
  if (res && algo == TC_ALGO_FDBSCAN) {
    ChunkedCopy cc;
    tcb::ChunkSink sink = [&](int64_t i0, int64_t i1, cudaStream_t s) {
      cudaEvent_t e;
      TCB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      cc.events.push_back(e);
      TCB_CUDA(cudaEventRecord(e, s));
      TCB_CUDA(cudaStreamWaitEvent(cc.cp, e, 0));
      TCB_CUDA(cudaMemcpyAsync(res->labels.ptr + i0, d_labels + i0, sizeof(int32_t) * (i1 - i0),
                               cudaMemcpyDeviceToHost, cc.cp));
      TCB_CUDA(cudaMemcpyAsync(res->core.ptr + i0, d_core + i0, static_cast<size_t>(i1 - i0),
                               cudaMemcpyDeviceToHost, cc.cp));
    };
    tcb::run_device(d_coords, n, dim, eps, minpts, algo, cap, d_labels, d_core, call.st, true,
                    &ro, nullptr, nullptr, &sink);
    TCB_CUDA(cudaStreamSynchronize(cc.cp));
    res->stats = ro.stats;
    return;
  }
  tcb::run_device(d_coords, n, dim, eps, minpts, algo, cap, d_labels, d_core, call.st, true, &ro,
                  [&](cudaStream_t s) {
                    if (!res) return;
                    TCB_CUDA(cudaMemcpyAsync(res->labels.ptr, d_labels, sizeof(int32_t) * n,
                                             cudaMemcpyDeviceToHost, s));
                    TCB_CUDA(cudaMemcpyAsync(res->core.ptr, d_core, n, cudaMemcpyDeviceToHost, s));
                  });
  if (res) res->stats = ro.stats;
}

// check_equivalence (oracle.cpp:120-163) on the device, message text as the
// reference's index_message (oracle.cpp:64-68).
struct Equivalence {
  bool pass = true;
  std::string message = "PASS";
};

Equivalence device_equivalence(const float* d_coords, int64_t n, int dim, float eps,
                               const int32_t* la, const uint8_t* ca, const int32_t* lb,
                               const uint8_t* cb, cudaStream_t st) {
  const tcb::EqVerdict v = tcb::check_equivalence_device(d_coords, n, dim, eps, la, ca, lb, cb, st);
  Equivalence r;
  if (v.check != 0) {
    std::ostringstream os;
    os << tcb::equivalence_message(v.check) << " (first divergence at point " << v.at << ")";
    r.pass = false;
    r.message = os.str();
  }
  return r;
}

}  // namespace

// ===========================================================================
// Reference ABI
// ===========================================================================

TC_EXPORT const char* tc_status_string(tc_status status) {
  switch (status) {
    case TC_OK: return "ok";
    case TC_ERR_INVALID_ARGUMENT: return "invalid argument";
    case TC_ERR_IO: return "i/o error";
    case TC_ERR_VERIFY_FAIL: return "verification failed";
    case TC_ERR_CAP_EXCEEDED: return "oracle cap exceeded";
    case TC_ERR_INTERNAL: return "internal error";
  }
  return "unknown status";
}

TC_EXPORT tc_status tc_dataset_create(const float* coords, int64_t n, int dim, tc_dataset** out) {
  if (!coords || !out || n < 1) return TC_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    if (dim != 2 && dim != 3) throw std::invalid_argument("PointSet: dimension must be 2 or 3");
    tcb::validate_points(dim, coords, n * dim);
    auto ds = std::make_unique<tc_dataset>(dim, n);
    std::memcpy(ds->coords.ptr, coords, static_cast<size_t>(n) * dim * sizeof(float));
    *out = ds.release();
    return TC_OK;
  });
}

TC_EXPORT tc_status tc_dataset_load(const char* path, tc_file_format format, tc_dataset** out) {
  if (!path || !out) return TC_ERR_INVALID_ARGUMENT;
  return guarded([&] { return publish(tcb::load_points(path, static_cast<int>(format)), out); });
}

TC_EXPORT tc_status tc_dataset_save(const tc_dataset* ds, const char* path, tc_file_format format) {
  if (!ds || !path) return TC_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    tcb::save_points(path, static_cast<int>(format), ds->dim, ds->coords.ptr, ds->n);
    return TC_OK;
  });
}

TC_EXPORT int64_t tc_dataset_size(const tc_dataset* ds) { return ds ? ds->n : 0; }
TC_EXPORT int tc_dataset_dim(const tc_dataset* ds) { return ds ? ds->dim : 0; }
TC_EXPORT const float* tc_dataset_coords(const tc_dataset* ds) { return ds ? ds->coords.ptr : nullptr; }
TC_EXPORT void tc_dataset_free(tc_dataset* ds) { delete ds; }

TC_EXPORT tc_status tc_generate_blobs(int k, int64_t per_blob, int dim, float separation,
                                      float sigma, uint64_t seed, tc_dataset** out) {
  if (!out) return TC_ERR_INVALID_ARGUMENT;
  return guarded([&] { return publish(tcb::gen_blobs(k, per_blob, dim, separation, sigma, seed), out); });
}

TC_EXPORT tc_status tc_generate_uniform(int64_t n, int dim, const float* lo, const float* hi,
                                        uint64_t seed, tc_dataset** out) {
  if (!out || !lo || !hi) return TC_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    for (int k = 0; k < dim && k < 3; ++k)
      if (!(lo[k] <= hi[k])) throw std::invalid_argument("bounds");
    return publish(tcb::gen_uniform(n, dim, lo, hi, seed), out);
  });
}

TC_EXPORT tc_status tc_generate_lattice(int64_t side, int dim, float spacing, tc_dataset** out) {
  if (!out) return TC_ERR_INVALID_ARGUMENT;
  return guarded([&] { return publish(tcb::gen_lattice(side, dim, spacing), out); });
}

TC_EXPORT tc_status tc_cluster(const tc_dataset* ds, float eps, int minpts, tc_algorithm algorithm,
                               int threads, int64_t oracle_cap, tc_result** out) {
  (void)threads;  // accepted for ABI compatibility; the work runs on the GPU
  if (!ds || !out) return TC_ERR_INVALID_ARGUMENT;
  return guarded([&]() -> tc_status {
    if (algorithm != TC_ALGO_FDBSCAN && algorithm != TC_ALGO_DENSEBOX &&
        algorithm != TC_ALGO_BRUTEFORCE)
      return TC_ERR_INVALID_ARGUMENT;
    if (algorithm == TC_ALGO_BRUTEFORCE) {  // cap before validation (capi.cpp:166-168)
      int64_t cap = oracle_cap > 0 ? oracle_cap : 10000;
      if (ds->n > cap) return TC_ERR_CAP_EXCEEDED;
    }
    if (!(eps > 0.f) || !std::isfinite(eps) || minpts < 2) return TC_ERR_INVALID_ARGUMENT;
    const int64_t n = ds->n;
    HostTimer ht;
    auto res = std::make_unique<tc_result>(n);
    ht.mark("result alloc");
    DeviceCall call;
    float* d_coords = call.alloc<float>(n * ds->dim);
    int32_t* d_labels = call.alloc<int32_t>(n);
    uint8_t* d_core = call.alloc<uint8_t>(n);
    ht.mark("stream + device alloc");
    TCB_CUDA(cudaMemcpyAsync(d_coords, ds->coords.ptr, sizeof(float) * n * ds->dim,
                             cudaMemcpyHostToDevice, call.st));
    device_cluster(call, d_coords, n, ds->dim, eps, minpts, algorithm, oracle_cap, d_labels,
                   d_core, res.get());
    ht.mark("H2D + device + D2H");
    if (algorithm == TC_ALGO_BRUTEFORCE) {  // the reference leaves timers/counters at 0
      tc_cluster_stats& s = res->stats;
      s.build_seconds = s.preprocess_seconds = s.main_seconds = s.finalize_seconds = 0.0;
      s.preprocess_skipped = 0;
      s.pair_resolutions = s.distance_evaluations = 0;
    }
    *out = res.release();
    ht.mark("release");
    return TC_OK;
  });
}

TC_EXPORT tc_status tcg_cluster_multi(const tc_dataset* ds, float eps, int minpts,
                                      tc_algorithm algorithm, const int* devices,
                                      int num_devices, tc_result** out) {
  if (!ds || !out || !devices || num_devices < 1 || num_devices > 64)
    return TC_ERR_INVALID_ARGUMENT;
  return guarded([&]() -> tc_status {
    if (algorithm != TC_ALGO_FDBSCAN && algorithm != TC_ALGO_DENSEBOX)
      return TC_ERR_INVALID_ARGUMENT;
    if (!(eps > 0.f) || !std::isfinite(eps) || minpts < 2) return TC_ERR_INVALID_ARGUMENT;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) count = 0;
    for (int s = 0; s < num_devices; ++s)
      if (devices[s] < 0 || devices[s] >= count) return count ? TC_ERR_INVALID_ARGUMENT
                                                              : TC_ERR_INTERNAL;
    auto res = std::make_unique<tc_result>(ds->n);
    if (ds->dim == 2)
      tcb::cluster_multi<2>(ds->coords.ptr, ds->n, eps, minpts, devices, num_devices,
                            res->labels.ptr, res->core.ptr, &res->stats);
    else
      tcb::cluster_multi<3>(ds->coords.ptr, ds->n, eps, minpts, devices, num_devices,
                            res->labels.ptr, res->core.ptr, &res->stats);
    *out = res.release();
    return TC_OK;
  });
}

TC_EXPORT int64_t tc_result_size(const tc_result* res) { return res ? res->n : 0; }
TC_EXPORT const int32_t* tc_result_labels(const tc_result* res) { return res ? res->labels.ptr : nullptr; }
TC_EXPORT const uint8_t* tc_result_core_flags(const tc_result* res) { return res ? res->core.ptr : nullptr; }

TC_EXPORT tc_status tc_result_stats(const tc_result* res, tc_cluster_stats* out) {
  if (!res || !out) return TC_ERR_INVALID_ARGUMENT;
  *out = res->stats;
  return TC_OK;
}

TC_EXPORT void tc_result_free(tc_result* res) { delete res; }

TC_EXPORT tc_status tc_verify(const tc_dataset* ds, float eps, int minpts, int threads,
                              int64_t oracle_cap, char* report, size_t report_len) {
  (void)threads;
  if (!ds) return TC_ERR_INVALID_ARGUMENT;
  std::string text;
  tc_status status = guarded([&]() -> tc_status {
    const int64_t n = ds->n;
    const int dim = ds->dim;
    const int64_t cap = oracle_cap > 0 ? oracle_cap : 10000;
    DeviceCall call;
    float* d_coords = call.alloc<float>(n * dim);
    TCB_CUDA(cudaMemcpyAsync(d_coords, ds->coords.ptr, sizeof(float) * n * dim,
                             cudaMemcpyHostToDevice, call.st));
    struct Run {
      int32_t* d_labels;
      uint8_t* d_core;
    };
    auto run = [&](tc_algorithm algo) {
      Run r{call.alloc<int32_t>(n), call.alloc<uint8_t>(n)};
      device_cluster(call, d_coords, n, dim, eps, minpts, algo, cap, r.d_labels, r.d_core,
                     nullptr);
      return r;
    };
    auto line = [&](const char* name, const Equivalence& e) {
      text += name;
      text += ": ";
      text += e.pass ? std::string("PASS") : "FAIL \xE2\x80\x94 " + e.message;
      text += '\n';
    };
    auto equiv = [&](const Run& a, const Run& b) {
      return device_equivalence(d_coords, n, dim, eps, a.d_labels, a.d_core, b.d_labels,
                                b.d_core, call.st);
    };
    Run fd = run(TC_ALGO_FDBSCAN);
    Run db = run(TC_ALGO_DENSEBOX);
    bool all = true;
    Equivalence x = equiv(fd, db);
    line("fdbscan vs densebox", x);
    all &= x.pass;
    if (n <= cap) {
      Run bf = run(TC_ALGO_BRUTEFORCE);
      Equivalence a = equiv(fd, bf);
      line("fdbscan vs bruteforce", a);
      Equivalence b = equiv(db, bf);
      line("densebox vs bruteforce", b);
      all &= a.pass && b.pass;
    } else {
      std::ostringstream os;
      os << "bruteforce reference skipped: n=" << n << " exceeds oracle cap " << cap
         << " (cross-algorithm check only)\n";
      text += os.str();
    }
    return all ? TC_OK : TC_ERR_VERIFY_FAIL;
  });
  if (report && report_len > 0) {
    size_t len = std::min(report_len - 1, text.size());
    std::memcpy(report, text.data(), len);
    report[len] = '\0';
  }
  return status;
}

// ===========================================================================
// Additive ABI (treeclust_gpu.h)
// ===========================================================================

TC_EXPORT int tcg_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return c;
}

TC_EXPORT const char* tcg_version(void) { return "treeclust-b200 0.1 (sm_100a)"; }

// Only FDBSCAN without stats enqueues a run with no host synchronization; any
// other call on a capturing stream is refused before it touches the capture.
static bool capture_refused(void* stream, tc_algorithm algorithm, bool stats) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(static_cast<cudaStream_t>(stream), &cs) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cs != cudaStreamCaptureStatusNone && (algorithm != TC_ALGO_FDBSCAN || stats);
}

TC_EXPORT tc_status tcg_cluster_device(const float* d_coords, int64_t n, int dim, float eps,
                                       int minpts, tc_algorithm algorithm, int64_t oracle_cap,
                                       int32_t* d_labels, uint8_t* d_core, void* stream,
                                       tc_cluster_stats* stats) {
  if (capture_refused(stream, algorithm, stats != nullptr)) return TC_ERR_INVALID_ARGUMENT;
  return guarded([&]() -> tc_status {
    tcb::RunOutput ro;
    tcb::run_device(d_coords, n, dim, eps, minpts, algorithm, oracle_cap, d_labels, d_core,
                    static_cast<cudaStream_t>(stream), stats != nullptr,
                    stats ? &ro : nullptr);
    if (stats) *stats = ro.stats;
    return TC_OK;
  });
}

TC_EXPORT tc_status tcg_cluster_device_async(const float* d_coords, int64_t n, int dim, float eps,
                                             int minpts, tc_algorithm algorithm,
                                             int64_t oracle_cap, int32_t* d_labels,
                                             uint8_t* d_core, void* stream, int32_t* d_status) {
  if (capture_refused(stream, algorithm, false)) return TC_ERR_INVALID_ARGUMENT;
  return guarded([&]() -> tc_status {
    tcb::run_device(d_coords, n, dim, eps, minpts, algorithm, oracle_cap, d_labels, d_core,
                    static_cast<cudaStream_t>(stream), false, nullptr, nullptr, nullptr, nullptr,
                    d_status);
    return TC_OK;
  });
}

TC_EXPORT tc_status tcg_cluster_keyed_device(const float* d_coords, const int32_t* d_keys,
                                             int64_t n, int dim, float eps, int minpts,
                                             int32_t* d_labels, uint8_t* d_core, void* stream,
                                             tc_cluster_stats* stats) {
  if (!d_keys) return TC_ERR_INVALID_ARGUMENT;
  return guarded([&]() -> tc_status {
    tcb::RunOutput ro;
    tcb::run_device(d_coords, n, dim, eps, minpts, TC_ALGO_FDBSCAN, 0, d_labels, d_core,
                    static_cast<cudaStream_t>(stream), stats != nullptr, stats ? &ro : nullptr,
                    nullptr, d_keys);
    if (stats) *stats = ro.stats;
    return TC_OK;
  });
}

TC_EXPORT tc_status tcg_binary_info(const char* path, int64_t* n, int* dim) {
  if (!path || !n || !dim) return TC_ERR_INVALID_ARGUMENT;
  return guarded([&]() -> tc_status {
    tcb::binary_info(path, n, dim);
    return TC_OK;
  });
}

TC_EXPORT tc_status tcg_load_binary_device(const char* path, float* d_coords, int64_t n, int dim,
                                           void* stream) {
  if (!path || !d_coords || n < 1 || (dim != 2 && dim != 3)) return TC_ERR_INVALID_ARGUMENT;
  return guarded([&]() -> tc_status {
    tcb::load_binary_device(path, d_coords, n, dim, static_cast<cudaStream_t>(stream));
    return TC_OK;
  });
}

TC_EXPORT int tcg_last_stage_ms(double* out, int cap) {
  if (!out || cap <= 0) return 0;
  return tcb::get_last_stage_ms(out, cap);
}

TC_EXPORT int64_t tcg_last_launch_count(void) { return tcb::launch_count(); }

TC_EXPORT tc_status tcg_generate_hacc_like(int64_t n, double box_len, double halo_frac,
                                           uint64_t seed, tc_dataset** out) {
  if (!out) return TC_ERR_INVALID_ARGUMENT;
  return guarded([&] { return publish(tcb::gen_hacc_like(n, box_len, halo_frac, seed), out); });
}

TC_EXPORT tc_status tcg_generate_taxi_like(int64_t n, uint64_t seed, tc_dataset** out) {
  if (!out) return TC_ERR_INVALID_ARGUMENT;
  return guarded([&] { return publish(tcb::gen_taxi_like(n, seed), out); });
}

TC_EXPORT tc_status tcg_generate_blobs_device(int k, int64_t per_blob, int dim,
                                              float separation, float sigma, uint64_t seed,
                                              float* d_out, void* stream) {
  if (!d_out) return TC_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    tcb::reset_launch_count();
    tcb::gen_blobs_device(k, per_blob, dim, separation, sigma, seed, d_out,
                          static_cast<cudaStream_t>(stream));
    return TC_OK;
  });
}

TC_EXPORT tc_status tcg_generate_uniform_device(int64_t n, int dim, const float* lo,
                                                const float* hi, uint64_t seed, float* d_out,
                                                void* stream) {
  if (!d_out || !lo || !hi) return TC_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    tcb::reset_launch_count();
    tcb::gen_uniform_device(n, dim, lo, hi, seed, d_out, static_cast<cudaStream_t>(stream));
    return TC_OK;
  });
}

TC_EXPORT tc_status tcg_generate_lattice_device(int64_t side, int dim, float spacing,
                                                float* d_out, void* stream) {
  if (!d_out) return TC_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    tcb::reset_launch_count();
    tcb::gen_lattice_device(side, dim, spacing, d_out, static_cast<cudaStream_t>(stream));
    return TC_OK;
  });
}

TC_EXPORT tc_status tcg_generate_hacc_like_device(int64_t n, double box_len, double halo_frac,
                                                  uint64_t seed, float* d_out, void* stream) {
  if (!d_out) return TC_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    tcb::reset_launch_count();
    tcb::gen_hacc_like_device(n, box_len, halo_frac, seed, d_out,
                              static_cast<cudaStream_t>(stream));
    return TC_OK;
  });
}

TC_EXPORT tc_status tcg_generate_taxi_like_device(int64_t n, uint64_t seed, float* d_out,
                                                  void* stream) {
  if (!d_out) return TC_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    tcb::reset_launch_count();
    tcb::gen_taxi_like_device(n, seed, d_out, static_cast<cudaStream_t>(stream));
    return TC_OK;
  });
}

TC_EXPORT tc_status tcg_random_instance(uint64_t seed, int64_t min_n, int64_t max_n, float* eps,
                                        int* minpts, tc_dataset** out) {
  if (!out || !eps || !minpts || min_n < 1 || max_n < min_n) return TC_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    return publish(tcb::gen_random_instance(seed, min_n, max_n, eps, minpts), out);
  });
}

TC_EXPORT tc_status tcg_dataset_create_pinned(const float* coords, int64_t n, int dim,
                                              tc_dataset** out) {
  return tc_dataset_create(coords, n, dim, out);  // large datasets are pinned already
}

TC_EXPORT tc_status tcg_check_equivalence_device(const float* d_coords, int64_t n, int dim,
                                                 float eps, const int32_t* d_labels_a,
                                                 const uint8_t* d_core_a,
                                                 const int32_t* d_labels_b,
                                                 const uint8_t* d_core_b, void* stream,
                                                 int* check, int64_t* at) {
  if (!d_coords || n < 1 || (dim != 2 && dim != 3) || !d_labels_a || !d_core_a || !d_labels_b ||
      !d_core_b || !check || !at || !(eps > 0.f) || !std::isfinite(eps))
    return TC_ERR_INVALID_ARGUMENT;
  return guarded([&]() -> tc_status {
    const tcb::EqVerdict v =
        tcb::check_equivalence_device(d_coords, n, dim, eps, d_labels_a, d_core_a, d_labels_b,
                                      d_core_b, static_cast<cudaStream_t>(stream));
    *check = v.check;
    *at = v.at;
    return TC_OK;
  });
}

TC_EXPORT tc_status tcg_first_bad_border_device(const float* d_coords, int64_t n, int dim,
                                                float eps, const int32_t* d_labels,
                                                const uint8_t* d_core, void* stream,
                                                int64_t* at) {
  if (!d_coords || n < 1 || (dim != 2 && dim != 3) || !d_labels || !d_core || !at ||
      !(eps > 0.f) || !std::isfinite(eps))
    return TC_ERR_INVALID_ARGUMENT;
  return guarded([&]() -> tc_status {
    *at = tcb::first_bad_border(d_coords, n, dim, eps, d_labels, d_core,
                                static_cast<cudaStream_t>(stream));
    return TC_OK;
  });
}

TC_EXPORT tc_status tcg_set_pool_release_threshold(uint64_t bytes) {
  return guarded([&]() -> tc_status {
    tcb::set_pool_release_threshold(bytes);
    return TC_OK;
  });
}

TC_EXPORT void tcg_release_cached_memory(void) {
  HostPool::get().trim();
  tcb::trim_pools();
}
