// LSD radix sort (8-bit digits, reduce-then-scan) and exclusive scan.
//
// Per sorted digit window:
//   k_sort_upsweep    per-tile digit histogram, warp-aggregated with
//                     __match_any_sync (Morton digits are heavily skewed in
//                     clustered data, so plain shared atomics would serialize)
//   k_sort_scan_rows  one CTA per digit scans that digit's row of tile counts
//                     (digit-major layout -> global offsets) and its total
//   k_sort_downsweep  stable in-tile ranking (match_any + per-warp counters),
//                     staging through shared memory so the global writes are
//                     contiguous runs per digit
// Constant digit windows (AND == OR over all keys) are skipped entirely.
#include "primitives.cuh"

#include <algorithm>

#include "device_common.cuh"
#include "engine.hpp"

namespace tcb {

namespace {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / kWarp;
constexpr int kIPT = 16;
constexpr int kTile = kSortThreads * kIPT;  // 4096 keys per tile
constexpr int kRadix = 256;

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Block-wide exclusive scan of one value per thread (blockDim.x == NT).
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* smem_warp,
                                                    uint32_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t s = lane < NT / 32 ? smem_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < NT / 32) smem_warp[lane] = s;  // inclusive per-warp totals
  }
  __syncthreads();
  uint32_t warp_prefix = w > 0 ? smem_warp[w - 1] : 0;
  if (total) *total = smem_warp[NT / 32 - 1];
  uint32_t r = warp_prefix + x - v;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kSortThreads)
k_sort_upsweep(const uint64_t* __restrict__ keys, int64_t n, int shift,
               uint32_t* __restrict__ tile_hist, int num_tiles) {
  __shared__ uint32_t h[kRadix];
  for (int i = threadIdx.x; i < kRadix; i += kSortThreads) h[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile + w * (kIPT * 32);
  uint64_t k[kIPT];
#pragma unroll
  for (int j = 0; j < kIPT; ++j) {
    int64_t idx = base + j * 32 + lane;
    k[j] = idx < n ? __ldcs(keys + idx) : 0;
  }
#pragma unroll
  for (int j = 0; j < kIPT; ++j) {
    int64_t idx = base + j * 32 + lane;
    uint32_t mask = __ballot_sync(0xffffffffu, idx < n);
    if (idx < n) {
      uint32_t d = static_cast<uint32_t>(k[j] >> shift) & (kRadix - 1);
      uint32_t peers = __match_any_sync(mask, d);
      if ((peers & lanemask_lt()) == 0) atomicAdd(&h[d], __popc(peers));
    }
  }
  __syncthreads();
  for (int d = threadIdx.x; d < kRadix; d += kSortThreads)
    tile_hist[static_cast<int64_t>(d) * num_tiles + blockIdx.x] = h[d];
}

constexpr int kScanRowThreads = 1024;

// One CTA per digit: exclusive scan of tile counts along the row, row total
// into totals[d].
__global__ void __launch_bounds__(kScanRowThreads)
k_sort_scan_rows(uint32_t* __restrict__ tile_hist, int num_tiles,
                 uint32_t* __restrict__ totals) {
  __shared__ uint32_t warp_tot[32];
  uint32_t* row = tile_hist + static_cast<int64_t>(blockIdx.x) * num_tiles;
  uint32_t running = 0;
  for (int base = 0; base < num_tiles; base += kScanRowThreads * 4) {
    uint32_t v[4];
    uint32_t s = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int i = base + threadIdx.x * 4 + q;
      v[q] = i < num_tiles ? row[i] : 0;
      s += v[q];
    }
    uint32_t tot;
    uint32_t pre = block_excl_scan<kScanRowThreads>(s, warp_tot, &tot);
    pre += running;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int i = base + threadIdx.x * 4 + q;
      if (i < num_tiles) row[i] = pre;
      pre += v[q];
    }
    running += tot;
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = running;
}

struct DownsweepSmem {
  uint64_t keys[kTile];
  int32_t vals[kTile];
  uint32_t wcnt[kSortWarps][kRadix];
  uint32_t tile_start[kRadix];
  uint32_t global_start[kRadix];
  uint32_t warp_tot[32];
};

__global__ void __launch_bounds__(kSortThreads)
k_sort_downsweep(const uint64_t* __restrict__ keys_in, const int32_t* __restrict__ vals_in,
                 uint64_t* __restrict__ keys_out, int32_t* __restrict__ vals_out,
                 int64_t n, int shift, const uint32_t* __restrict__ tile_hist,
                 const uint32_t* __restrict__ totals, int num_tiles) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  DownsweepSmem& S = *reinterpret_cast<DownsweepSmem*>(smem_raw);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kSortWarps * kRadix; i += kSortThreads)
    (&S.wcnt[0][0])[i] = 0;

  const int64_t tile_base = static_cast<int64_t>(blockIdx.x) * kTile;
  const int64_t base = tile_base + w * (kIPT * 32);
  uint64_t k[kIPT];
  int32_t v[kIPT];
#pragma unroll
  for (int j = 0; j < kIPT; ++j) {
    int64_t idx = base + j * 32 + lane;
    if (idx < n) {
      k[j] = __ldcs(keys_in + idx);
      v[j] = __ldcs(vals_in + idx);
    }
  }
  __syncthreads();

  uint32_t rank[kIPT];
#pragma unroll
  for (int j = 0; j < kIPT; ++j) {
    int64_t idx = base + j * 32 + lane;
    uint32_t mask = __ballot_sync(0xffffffffu, idx < n);
    rank[j] = 0;
    if (idx < n) {
      uint32_t d = static_cast<uint32_t>(k[j] >> shift) & (kRadix - 1);
      uint32_t peers = __match_any_sync(mask, d);
      uint32_t before = S.wcnt[w][d];
      rank[j] = before + __popc(peers & lanemask_lt());
      __syncwarp(mask);
      if ((peers & lanemask_lt()) == 0) S.wcnt[w][d] = before + __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();

  // Per digit (thread d): exclusive prefix over warps, tile count.
  uint32_t tile_count = 0;
  {
    const int d = threadIdx.x;  // kSortThreads == kRadix
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ++ww) {
      uint32_t c = S.wcnt[ww][d];
      S.wcnt[ww][d] = tile_count;
      tile_count += c;
    }
  }
  uint32_t tstart = block_excl_scan<kSortThreads>(tile_count, S.warp_tot, nullptr);
  uint32_t dstart = block_excl_scan<kSortThreads>(totals[threadIdx.x], S.warp_tot, nullptr);
  S.tile_start[threadIdx.x] = tstart;
  S.global_start[threadIdx.x] =
      dstart + tile_hist[static_cast<int64_t>(threadIdx.x) * num_tiles + blockIdx.x];
  __syncthreads();

#pragma unroll
  for (int j = 0; j < kIPT; ++j) {
    int64_t idx = base + j * 32 + lane;
    if (idx < n) {
      uint32_t d = static_cast<uint32_t>(k[j] >> shift) & (kRadix - 1);
      uint32_t pos = S.tile_start[d] + S.wcnt[w][d] + rank[j];
      S.keys[pos] = k[j];
      S.vals[pos] = v[j];
    }
  }
  __syncthreads();

  const int tile_n = static_cast<int>(n - tile_base < kTile ? n - tile_base : kTile);
  for (int p = threadIdx.x; p < tile_n; p += kSortThreads) {
    uint64_t key = S.keys[p];
    uint32_t d = static_cast<uint32_t>(key >> shift) & (kRadix - 1);
    uint32_t out = S.global_start[d] + (p - S.tile_start[d]);
    keys_out[out] = key;
    vals_out[out] = S.vals[p];
  }
}

// ---------------------------------------------------------------------------
// Exclusive scan (reduce-then-scan, 3 kernels)
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 512;
constexpr int kScanIPT = 8;
constexpr int kScanTile = kScanThreads * kScanIPT;

__global__ void __launch_bounds__(kScanThreads)
k_scan_reduce(const int32_t* __restrict__ in, int64_t n, int32_t* __restrict__ partial) {
  __shared__ uint32_t warp_tot[32];
  int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanIPT;
  uint32_t s = 0;
#pragma unroll
  for (int q = 0; q < kScanIPT; ++q)
    if (base + q < n) s += static_cast<uint32_t>(in[base + q]);
  uint32_t tot;
  block_excl_scan<kScanThreads>(s, warp_tot, &tot);
  if (threadIdx.x == 0) partial[blockIdx.x] = static_cast<int32_t>(tot);
}

__global__ void __launch_bounds__(1024)
k_scan_partials(int32_t* __restrict__ partial, int num, int32_t* __restrict__ d_total) {
  __shared__ uint32_t warp_tot[32];
  uint32_t running = 0;
  for (int base = 0; base < num; base += 1024) {
    int i = base + threadIdx.x;
    uint32_t v = i < num ? static_cast<uint32_t>(partial[i]) : 0;
    uint32_t tot;
    uint32_t pre = block_excl_scan<1024>(v, warp_tot, &tot);
    if (i < num) partial[i] = static_cast<int32_t>(pre + running);
    running += tot;
  }
  if (threadIdx.x == 0 && d_total) *d_total = static_cast<int32_t>(running);
}

__global__ void __launch_bounds__(kScanThreads)
k_scan_downsweep(const int32_t* __restrict__ in, int32_t* __restrict__ out, int64_t n,
                 const int32_t* __restrict__ partial) {
  __shared__ uint32_t warp_tot[32];
  int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanIPT;
  uint32_t v[kScanIPT];
  uint32_t s = 0;
#pragma unroll
  for (int q = 0; q < kScanIPT; ++q) {
    v[q] = base + q < n ? static_cast<uint32_t>(in[base + q]) : 0;
    s += v[q];
  }
  uint32_t pre = block_excl_scan<kScanThreads>(s, warp_tot, nullptr) +
                 static_cast<uint32_t>(partial[blockIdx.x]);
#pragma unroll
  for (int q = 0; q < kScanIPT; ++q) {
    if (base + q < n) out[base + q] = static_cast<int32_t>(pre);
    pre += v[q];
  }
}

int64_t num_sort_tiles(int64_t n) { return (n + kTile - 1) / kTile; }

}  // namespace

size_t radix_sort_scratch_bytes(int64_t n) {
  int64_t t = num_sort_tiles(std::max<int64_t>(n, 1));
  return static_cast<size_t>(t) * kRadix * sizeof(uint32_t) + kRadix * sizeof(uint32_t) + 256;
}

bool radix_sort_pairs(uint64_t* keys, int32_t* vals, uint64_t* keys_alt,
                      int32_t* vals_alt, int64_t n, uint64_t and_all,
                      uint64_t or_all, void* scratch, cudaStream_t stream,
                      int* passes_run) {
  int passes = 0;
  bool in_alt = false;
  if (n > 1) {
    const int num_tiles = static_cast<int>(num_sort_tiles(n));
    uint32_t* tile_hist = static_cast<uint32_t*>(scratch);
    uint32_t* totals = tile_hist + static_cast<int64_t>(num_tiles) * kRadix;
    TCB_CUDA(cudaFuncSetAttribute(k_sort_downsweep,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sizeof(DownsweepSmem))));
    const uint64_t varying = and_all ^ or_all;
    for (int shift = 0; shift < 64; shift += 8) {
      if (((varying >> shift) & 0xffull) == 0) continue;  // constant digit window
      const uint64_t* kin = in_alt ? keys_alt : keys;
      const int32_t* vin = in_alt ? vals_alt : vals;
      uint64_t* kout = in_alt ? keys : keys_alt;
      int32_t* vout = in_alt ? vals : vals_alt;
      note_launch(), k_sort_upsweep<<<num_tiles, kSortThreads, 0, stream>>>(kin, n, shift, tile_hist,
                                                             num_tiles);
      note_launch(), k_sort_scan_rows<<<kRadix, kScanRowThreads, 0, stream>>>(tile_hist, num_tiles, totals);
      note_launch(), k_sort_downsweep<<<num_tiles, kSortThreads, sizeof(DownsweepSmem), stream>>>(
          kin, vin, kout, vout, n, shift, tile_hist, totals, num_tiles);
      TCB_CUDA(cudaGetLastError());
      in_alt = !in_alt;
      ++passes;
    }
  }
  if (passes_run) *passes_run = passes;
  return in_alt;
}

size_t scan_scratch_bytes(int64_t n) {
  int64_t blocks = (std::max<int64_t>(n, 1) + kScanTile - 1) / kScanTile;
  return static_cast<size_t>(blocks) * sizeof(int32_t) + 256;
}

void exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, int32_t* d_total,
                        void* scratch, cudaStream_t stream) {
  if (n <= 0) {
    if (d_total) TCB_CUDA(cudaMemsetAsync(d_total, 0, sizeof(int32_t), stream));
    return;
  }
  int blocks = static_cast<int>((n + kScanTile - 1) / kScanTile);
  int32_t* partial = static_cast<int32_t*>(scratch);
  note_launch(), k_scan_reduce<<<blocks, kScanThreads, 0, stream>>>(in, n, partial);
  note_launch(), k_scan_partials<<<1, 1024, 0, stream>>>(partial, blocks, d_total);
  note_launch(), k_scan_downsweep<<<blocks, kScanThreads, 0, stream>>>(in, out, n, partial);
  TCB_CUDA(cudaGetLastError());
}

}  // namespace tcb
