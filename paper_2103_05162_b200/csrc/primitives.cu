// LSD radix sort (8-bit digits, Onesweep-style single pass per digit window
// with decoupled look-back) and a device-wide exclusive scan. Constant digit
// windows (AND == OR over all keys) are skipped entirely.
#include "primitives.cuh"

#include <algorithm>

#include "device_common.cuh"
#include "engine.hpp"
#include "pipeline.hpp"

namespace tcb {

namespace {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / kWarp;
#ifndef TCB_SORT_IPT
#define TCB_SORT_IPT 16
#endif
#ifndef TCB_SORT_MINB  // 3 resident tiles per SM (ptxas caps registers at 85;
#define TCB_SORT_MINB 3   // measured on C2: 2.84 ms vs 3.14 ms uncapped at 2/SM)
#endif
#ifndef TCB_SORT_LOOKBACK
#define TCB_SORT_LOOKBACK 4
#endif
constexpr int kIPT = TCB_SORT_IPT;
constexpr int kLookback = TCB_SORT_LOOKBACK;
constexpr int kTile = kSortThreads * kIPT;  // 4096 keys per tile
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;

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

// ---------------------------------------------------------------------------
// Onesweep LSD radix sort (one kernel per digit window, decoupled look-back).
//
//   k_sort_hist      the global histogram of the first sorted digit window
//                    (block-private shared histogram, one global atomic per
//                    bin per block); each onesweep pass adds the histogram of
//                    the next window from the keys it holds anyway
//   k_sort_onesweep  per digit window: a tile grabs its id from a counter (so
//                    look-back only ever waits on tiles already running),
//                    ranks its keys stably (__match_any_sync + per-warp
//                    counters), publishes its digit counts, looks back over
//                    the predecessors' published counts (flag + 30-bit count
//                    in one word: no fence needed) for its exclusive offsets,
//                    and scatters through shared memory so the global writes
//                    are contiguous runs per digit.
// Per key and window: 12 B read + 12 B written (the reduce-then-scan scheme
// it replaces also re-read the keys for a separate histogram pass).
// ---------------------------------------------------------------------------
constexpr int kMaxPasses = 8;
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagInc = 2u << 30;
constexpr uint32_t kCountMask = (1u << 30) - 1;

struct PassShifts {
  int shift[kMaxPasses];
  int count;
};

}  // namespace

// Device-side pass plan of the stream-ordered sort (radix_sort_pairs_prefix_async).
struct SortPlan {
  int32_t count;               // active passes (slots 0..count-1)
  int32_t shift[kMaxPasses];
  int32_t fix;                 // prefix plan: the low bits vary, the fix-up orders groups
  int32_t src_alt;             // where the last active pass left the pairs
  int32_t pad[5];
};

namespace {

// Histogram of the first sorted digit window only; every onesweep pass builds
// the histogram of the NEXT window from the keys it already holds.
__global__ void __launch_bounds__(kSortThreads)
k_sort_hist(const uint64_t* __restrict__ keys, int64_t n, int shift,
            uint32_t* __restrict__ ghist, const SortPlan* __restrict__ plan) {
  if (plan) {  // stream-ordered sort: the first window comes from the device plan
    if (plan->count == 0) return;
    shift = plan->shift[0];
  }
  __shared__ uint32_t h[kRadix];
  for (int i = threadIdx.x; i < kRadix; i += kSortThreads) h[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    atomicAdd(&h[static_cast<uint32_t>(__ldcs(keys + i) >> shift) & (kRadix - 1)], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < kRadix; i += kSortThreads)
    if (h[i]) atomicAdd(ghist + i, h[i]);
}

struct SortShared {
  uint32_t wcnt[kSortWarps][kRadix];
  uint32_t tile_start[kRadix];
  uint32_t global_start[kRadix];
  uint32_t warp_tot[32];
  uint32_t next_hist[kRadix];
  int tile;
};

struct OnesweepSmem {
  uint64_t keys[kTile];
  int32_t vals[kTile];
  SortShared c;
};

__device__ __forceinline__ uint32_t ld_status(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_status(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// One onesweep tile whose keys / values are in registers: stable ranking,
// digit counts published for the look-back, the next window's histogram,
// scatter through the staging arrays (tile order by digit), contiguous
// global writes. S.wcnt and S.next_hist must be zero on entry.
__device__ __forceinline__ void onesweep_tile(SortShared& S, uint64_t* st_keys, int32_t* st_vals,
                                              const uint64_t (&k)[kIPT], const int32_t (&v)[kIPT],
                                              int tile, int64_t n, int shift, int next_shift,
                                              const uint32_t* __restrict__ ghist,
                                              uint32_t* __restrict__ status,
                                              uint64_t* __restrict__ keys_out,
                                              int32_t* __restrict__ vals_out,
                                              uint32_t* __restrict__ ghist_next) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t tile_base = static_cast<int64_t>(tile) * kTile;
  const int64_t base = tile_base + w * (kIPT * 32);
  if (next_shift >= 0) {
#pragma unroll
    for (int j = 0; j < kIPT; ++j)
      if (base + j * 32 + lane < n)
        atomicAdd(&S.next_hist[static_cast<uint32_t>(k[j] >> next_shift) & (kRadix - 1)], 1u);
  }

  uint32_t rank[kIPT];
#pragma unroll
  for (int j = 0; j < kIPT; ++j) {
    const int64_t idx = base + j * 32 + lane;
    const uint32_t mask = __ballot_sync(0xffffffffu, idx < n);
    rank[j] = 0;
    const uint32_t d = static_cast<uint32_t>(k[j] >> shift) & (kRadix - 1);
    // peers = lanes with the same digit: 8 ballots (one per digit bit)
    // instead of __match_any_sync, which is the slow part of the ranking
    uint32_t peers = mask;
#pragma unroll
    for (int b = 0; b < kRadixBits; ++b) {
      const uint32_t bit = __ballot_sync(0xffffffffu, (d >> b) & 1u);
      peers &= ((d >> b) & 1u) ? bit : ~bit;
    }
    if (idx < n) {
      const uint32_t before = S.wcnt[w][d];
      rank[j] = before + __popc(peers & lanemask_lt());
      __syncwarp(mask);
      if ((peers & lanemask_lt()) == 0) S.wcnt[w][d] = before + __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();

  // thread d owns digit d: warp prefix, tile count, publish, look back
  const int d = threadIdx.x;  // kSortThreads == kRadix
  uint32_t tile_count = 0;
#pragma unroll
  for (int ww = 0; ww < kSortWarps; ++ww) {
    const uint32_t c = S.wcnt[ww][d];
    S.wcnt[ww][d] = tile_count;
    tile_count += c;
  }
  uint32_t* my = status + static_cast<int64_t>(tile) * kRadix + d;
  st_status(my, (tile == 0 ? kFlagInc : kFlagAgg) | tile_count);
  // decoupled look-back, kLookback predecessors per round trip
  uint32_t excl = 0;
  for (int t = tile - 1; t >= 0;) {
    uint32_t sv[kLookback];
#pragma unroll
    for (int j = 0; j < kLookback; ++j)
      sv[j] = t - j >= 0 ? ld_status(status + static_cast<int64_t>(t - j) * kRadix + d)
                         : kFlagInc;  // before tile 0: an inclusive zero
    bool done = false;
    int used = 0;
#pragma unroll
    for (int j = 0; j < kLookback; ++j) {
      if (done || used < j) break;
      if ((sv[j] & ~kCountMask) == 0) break;  // not published yet: retry from here
      excl += sv[j] & kCountMask;
      used = j + 1;
      if (sv[j] & kFlagInc) done = true;
    }
    if (done) break;
    t -= used;
  }
  if (tile > 0) st_status(my, kFlagInc | (excl + tile_count));
  const uint32_t tstart = block_excl_scan<kSortThreads>(tile_count, S.warp_tot, nullptr);
  const uint32_t dbase = block_excl_scan<kSortThreads>(ghist[d], S.warp_tot, nullptr);
  S.tile_start[d] = tstart;
  S.global_start[d] = dbase + excl;
  if (next_shift >= 0 && S.next_hist[d]) atomicAdd(ghist_next + d, S.next_hist[d]);
  __syncthreads();

#pragma unroll
  for (int j = 0; j < kIPT; ++j) {
    const int64_t idx = base + j * 32 + lane;
    if (idx < n) {
      const uint32_t dd = static_cast<uint32_t>(k[j] >> shift) & (kRadix - 1);
      const uint32_t pos = S.tile_start[dd] + S.wcnt[w][dd] + rank[j];
      st_keys[pos] = k[j];
      st_vals[pos] = v[j];
    }
  }
  __syncthreads();

  const int tile_n = static_cast<int>(n - tile_base < kTile ? n - tile_base : kTile);
  for (int p = threadIdx.x; p < tile_n; p += kSortThreads) {
    const uint64_t key = st_keys[p];
    const uint32_t dd = static_cast<uint32_t>(key >> shift) & (kRadix - 1);
    const uint32_t out = S.global_start[dd] + (p - S.tile_start[dd]);
    keys_out[out] = key;
    vals_out[out] = st_vals[p];
  }
}

// kLoop: a block keeps taking tiles until none is left (the guarded
// fallback passes run on a one-block-per-SM grid); otherwise one tile each.
template <bool kLoop>
__global__ void __launch_bounds__(kSortThreads, TCB_SORT_MINB)
k_sort_onesweep(const uint64_t* __restrict__ keys_in, const int32_t* __restrict__ vals_in,
                uint64_t* __restrict__ keys_out, int32_t* __restrict__ vals_out, int64_t n,
                int shift, const uint32_t* __restrict__ ghist, uint32_t* __restrict__ status,
                uint32_t* __restrict__ tile_counter, int next_shift,
                uint32_t* __restrict__ ghist_next, const SortPlan* __restrict__ plan,
                int slot, uint32_t* __restrict__ status_next) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  OnesweepSmem& B = *reinterpret_cast<OnesweepSmem*>(smem_raw);
  SortShared& S = B.c;
  if (plan) {  // stream-ordered sort: inactive slots do nothing
    const int cnt = plan->count;
    if (slot >= cnt) return;
    shift = plan->shift[slot];
    next_shift = slot + 1 < cnt ? plan->shift[slot + 1] : -1;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int num_tiles = static_cast<int>((n + kTile - 1) / kTile);
  // Tiles are taken in counter order, so a block only ever looks back at
  // tiles already owned by running blocks: a grid smaller than the tile count
  // (the guarded fallback passes) loops safely.
  do {
    if (threadIdx.x == 0) S.tile = static_cast<int>(atomicAdd(tile_counter, 1u));
    for (int i = threadIdx.x; i < kSortWarps * kRadix; i += kSortThreads) (&S.wcnt[0][0])[i] = 0;
    S.next_hist[threadIdx.x] = 0;  // kSortThreads == kRadix
    __syncthreads();
    const int tile = S.tile;
    if (kLoop && tile >= num_tiles) return;
    // planned passes alternate two status arrays: each tile clears its row of
    // the next pass's (idle during this pass) instead of a memset launch
    if (status_next) status_next[static_cast<int64_t>(tile) * kRadix + threadIdx.x] = 0;
    const int64_t base = static_cast<int64_t>(tile) * kTile + w * (kIPT * 32);
    uint64_t k[kIPT];
    int32_t v[kIPT];
#pragma unroll
    for (int j = 0; j < kIPT; ++j) {
      const int64_t idx = base + j * 32 + lane;
      if (idx < n) {
        k[j] = __ldcs(keys_in + idx);
        v[j] = vals_in ? __ldcs(vals_in + idx) : static_cast<int32_t>(idx);  // null: identity
      }
    }
    onesweep_tile(S, B.keys, B.vals, k, v, tile, n, shift, next_shift, ghist, status, keys_out,
                  vals_out, ghist_next);
    if (kLoop) __syncthreads();  // S is reused by the next tile
  } while (kLoop);
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
  const int64_t t = num_sort_tiles(std::max<int64_t>(n, 1));
  // status words (tiles x radix) + per-pass tile counters + global histograms
  return static_cast<size_t>(t) * kRadix * sizeof(uint32_t) + 64 * sizeof(uint32_t) +
         kMaxPasses * kRadix * sizeof(uint32_t) + 256 + 64;  // + the prefix sort's flag
}

bool radix_sort_pairs(uint64_t* keys, int32_t* vals, uint64_t* keys_alt,
                      int32_t* vals_alt, int64_t n, uint64_t and_all,
                      uint64_t or_all, void* scratch, cudaStream_t stream,
                      int* passes_run) {
  PassShifts ps{};
  const uint64_t varying = and_all ^ or_all;
  for (int shift = 0; shift < 64; shift += kRadixBits)
    if ((varying >> shift) & (kRadix - 1)) ps.shift[ps.count++] = shift;  // skip constant windows
  bool in_alt = false;
  if (n > 1 && ps.count > 0) {
    const int64_t num_tiles = num_sort_tiles(n);
    uint32_t* status = static_cast<uint32_t*>(scratch);
    uint32_t* counters = status + num_tiles * kRadix;
    uint32_t* ghist = counters + 64;
    TCB_CUDA(cudaMemsetAsync(counters, 0, (64 + kMaxPasses * kRadix) * sizeof(uint32_t), stream));
    note_launch(), k_sort_hist<<<grid_for(n, kSortThreads, 148 * 4), kSortThreads, 0, stream>>>(
        keys, n, ps.shift[0], ghist, nullptr);
    TCB_CUDA(cudaFuncSetAttribute(k_sort_onesweep<false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sizeof(OnesweepSmem))));
    for (int p = 0; p < ps.count; ++p) {
      const uint64_t* kin = in_alt ? keys_alt : keys;
      const int32_t* vin = in_alt ? vals_alt : vals;
      uint64_t* kout = in_alt ? keys : keys_alt;
      int32_t* vout = in_alt ? vals : vals_alt;
      TCB_CUDA(cudaMemsetAsync(status, 0, num_tiles * kRadix * sizeof(uint32_t), stream));
      note_launch(), k_sort_onesweep<false><<<static_cast<unsigned>(num_tiles), kSortThreads,
                                       sizeof(OnesweepSmem), stream>>>(
          kin, vin, kout, vout, n, ps.shift[p], ghist + p * kRadix, status, counters + p,
          p + 1 < ps.count ? ps.shift[p + 1] : -1, ghist + (p + 1) * kRadix, nullptr, 0,
          nullptr);
      TCB_CUDA(cudaGetLastError());
      in_alt = !in_alt;
    }
  }
  if (passes_run) *passes_run = n > 1 ? ps.count : 0;
  return in_alt;
}

namespace {

// Fix-up of radix_sort_pairs_prefix: element k finds its group [b, e) of equal
// key >> cut (at most kFixMax long), counts the group members ordered before
// it by (key, val) and writes itself there. Singletons (nearly every element
// of a Morton order cut at 24 bits) just copy through.
__global__ void __launch_bounds__(256)
k_sort_fixup(const uint64_t* __restrict__ kin, const int32_t* __restrict__ vin,
             uint64_t* __restrict__ kout, int32_t* __restrict__ vout, int64_t n, int cut,
             uint32_t* __restrict__ too_long) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t key = kin[k];
    const int32_t v = vin[k];
    const uint64_t top = key >> cut;
    int64_t b = k, e = k + 1;
    while (b > 0 && k - b < kFixMax && (kin[b - 1] >> cut) == top) --b;
    while (e < n && e - k < kFixMax && (kin[e] >> cut) == top) ++e;
    if (e - b > kFixMax) {
      *too_long = 1;
      continue;
    }
    int64_t r = b;
    for (int64_t j = b; j < e; ++j) {
      const uint64_t kj = kin[j];
      r += kj < key || (kj == key && vin[j] < v);
    }
    kout[r] = key;
    vout[r] = v;
  }
}

}  // namespace

bool radix_sort_pairs_prefix(uint64_t* keys, int32_t* vals, uint64_t* keys_alt,
                             int32_t* vals_alt, int64_t n, uint64_t and_all, uint64_t or_all,
                             void* scratch, cudaStream_t stream, bool* in_alt,
                             int* passes_run) {
  constexpr uint64_t low = (uint64_t{1} << kFixBits) - 1;
  // the low windows look constant to the LSD passes
  const uint64_t or_top = (or_all & ~low) | (and_all & low);
  int passes = 0;
  bool alt = radix_sort_pairs(keys, vals, keys_alt, vals_alt, n, and_all, or_top, scratch, stream,
                              &passes);
  if (((and_all ^ or_all) & low) != 0 && n > 1) {
    // the fix-up flag lives past the sort's own scratch
    uint32_t* flag = reinterpret_cast<uint32_t*>(static_cast<char*>(scratch) +
                                                 radix_sort_scratch_bytes(n) - 64);
    TCB_CUDA(cudaMemsetAsync(flag, 0, sizeof(uint32_t), stream));
    note_launch(), k_sort_fixup<<<grid_for(n, 256, 148 * 16), 256, 0, stream>>>(
        alt ? keys_alt : keys, alt ? vals_alt : vals, alt ? keys : keys_alt, alt ? vals : vals_alt,
        n, kFixBits, flag);
    TCB_CUDA(cudaGetLastError());
    alt = !alt;
    ++passes;
    auto* h = static_cast<uint32_t*>(pinned_staging(64));
    TCB_CUDA(cudaMemcpyAsync(h, flag, sizeof(uint32_t), cudaMemcpyDeviceToHost, stream));
    TCB_CUDA(cudaStreamSynchronize(stream));
    if (*h) return false;
  }
  *in_alt = alt;
  if (passes_run) *passes_run = passes;
  return true;
}

namespace {

// Plan of a stream-ordered sort from the device-side AND / OR of the keys:
// the varying 8-bit windows at and above lo_bit. gate (optional): no passes
// unless *gate != 0 (the fallback sort runs only after a failed fix-up).
__global__ void k_sort_plan(const unsigned long long* __restrict__ and_or, int lo_bit,
                            const uint32_t* __restrict__ gate, int64_t n, SortPlan* plan) {
  if (threadIdx.x != 0) return;
  const uint64_t varying = and_or[0] ^ and_or[1];
  int c = 0;
  if (n > 1 && (gate == nullptr || *gate != 0))
    for (int shift = lo_bit; shift < 64; shift += kRadixBits)
      if ((varying >> shift) & (kRadix - 1)) plan->shift[c++] = shift;
  plan->count = c;
  plan->src_alt = c & 1;
  plan->fix = n > 1 && lo_bit > 0 && ((varying & ((uint64_t{1} << lo_bit) - 1)) != 0);
}

// Zeroes a slot's look-back status words when the slot is active.
__global__ void k_zero_status(const SortPlan* __restrict__ plan, int slot,
                              uint32_t* __restrict__ status, int64_t words) {
  if (slot >= plan->count) return;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < words;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    status[i] = 0;
}

// Fix-up of the stream-ordered prefix sort: reads the pairs where the plan's
// passes left them and writes the final order to (kout, vout); without a
// varying low window it is a copy.
__global__ void __launch_bounds__(256)
k_sort_fixup_planned(const SortPlan* __restrict__ plan, const uint64_t* __restrict__ k0,
                     const int32_t* __restrict__ v0, const uint64_t* __restrict__ k1,
                     const int32_t* __restrict__ v1, uint64_t* __restrict__ kout,
                     int32_t* __restrict__ vout, int64_t n, int cut,
                     uint32_t* __restrict__ too_long, bool iota) {
  const bool alt = plan->src_alt != 0;
  const uint64_t* kin = alt ? k1 : k0;
  const int32_t* vin = alt ? v1 : v0;
  const bool fix = plan->fix != 0;
  // iota: the values were never materialized; without a pass they are 0..n-1
  const bool ident = iota && plan->count == 0;
  auto val = [&](int64_t i) { return ident ? static_cast<int32_t>(i) : vin[i]; };
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t key = kin[k];
    const int32_t v = val(k);
    if (!fix) {
      kout[k] = key;
      vout[k] = v;
      continue;
    }
    const uint64_t top = key >> cut;
    int64_t b = k, e = k + 1;
    while (b > 0 && k - b < kFixMax && (kin[b - 1] >> cut) == top) --b;
    while (e < n && e - k < kFixMax && (kin[e] >> cut) == top) ++e;
    if (e - b > kFixMax) {
      *too_long = 1;
      continue;
    }
    int64_t r = b;
    for (int64_t j = b; j < e; ++j) {
      const uint64_t kj = kin[j];
      r += kj < key || (kj == key && val(j) < v);
    }
    kout[r] = key;
    vout[r] = v;
  }
}

// Fallback of the stream-ordered prefix sort (a fix-up group was too long):
// mode 0 moves the prefix-sorted pairs into (k0, v0) when the passes left
// them in (k1, v1); mode 1 copies the fallback sort's result into the output.
// Both do nothing unless the fallback plan has passes.
__global__ void k_sort_fallback_copy(const SortPlan* __restrict__ first,
                                     const SortPlan* __restrict__ fb, int mode,
                                     uint64_t* __restrict__ k0, int32_t* __restrict__ v0,
                                     uint64_t* __restrict__ k1, int32_t* __restrict__ v1,
                                     uint64_t* __restrict__ kout, int32_t* __restrict__ vout,
                                     int64_t n, bool iota) {
  if (fb->count == 0) return;
  const uint64_t* ks;
  const int32_t* vs;
  uint64_t* kd;
  int32_t* vd;
  if (mode == 0) {
    if (!first->src_alt) {
      if (iota && first->count == 0)  // no pass ran: materialize the identity values
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x)
          v0[i] = static_cast<int32_t>(i);
      return;
    }
    ks = k1, vs = v1, kd = k0, vd = v0;
  } else {
    ks = fb->src_alt ? k1 : k0, vs = fb->src_alt ? v1 : v0, kd = kout, vd = vout;
  }
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    kd[i] = ks[i];
    vd[i] = vs[i];
  }
}

// The planned LSD passes: slot p reads (keys, vals) when p is even and uses
// status[p & 1]; the active slots are a prefix, each clearing the other array.
void planned_passes(uint64_t* keys, int32_t* vals, uint64_t* keys_alt, int32_t* vals_alt,
                    int64_t n, const SortPlan* plan, int slots, unsigned grid,
                    uint32_t* const (&status)[2], uint32_t* counters, uint32_t* ghist,
                    cudaStream_t stream, bool iota_vals) {
  const int64_t num_tiles = num_sort_tiles(n);
  const bool loop = grid < num_tiles;
  TCB_CUDA(cudaMemsetAsync(counters, 0, (64 + kMaxPasses * kRadix) * sizeof(uint32_t), stream));
  note_launch(), k_sort_hist<<<std::min<unsigned>(grid, 148 * 4), kSortThreads, 0, stream>>>(
      keys, n, 0, ghist, plan);
  auto kern = loop ? k_sort_onesweep<true> : k_sort_onesweep<false>;
  const size_t smem = sizeof(OnesweepSmem);
  TCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
  note_launch(), k_zero_status<<<std::min<unsigned>(grid, 148 * 4), 256, 0, stream>>>(
      plan, 0, status[0], num_tiles * kRadix);
  for (int p = 0; p < slots; ++p) {
    const bool in_alt = p & 1;
    note_launch(), kern<<<grid, kSortThreads, smem, stream>>>(
        in_alt ? keys_alt : keys, in_alt ? vals_alt : (p == 0 && iota_vals ? nullptr : vals),
        in_alt ? keys : keys_alt,
        in_alt ? vals : vals_alt, n, 0, ghist + p * kRadix, status[p & 1], counters + p, -1,
        ghist + (p + 1) * kRadix, plan, p, status[(p + 1) & 1]);
    TCB_CUDA(cudaGetLastError());
  }
}

}  // namespace

size_t radix_sort_async_scratch_bytes(int64_t n) {
  // + the two plans, + the second look-back status array
  return radix_sort_scratch_bytes(n) + 256 +
         static_cast<size_t>(num_sort_tiles(std::max<int64_t>(n, 1))) * kRadix * sizeof(uint32_t);
}

void radix_sort_pairs_prefix_async(uint64_t* keys, int32_t* vals, uint64_t* keys_alt,
                                   int32_t* vals_alt, uint64_t* keys_out, int32_t* vals_out,
                                   int64_t n, const unsigned long long* d_and_or, void* scratch,
                                   cudaStream_t stream, bool iota_vals) {
  const int64_t num_tiles = num_sort_tiles(std::max<int64_t>(n, 1));
  uint32_t* status = static_cast<uint32_t*>(scratch);
  uint32_t* counters = status + num_tiles * kRadix;
  uint32_t* ghist = counters + 64;
  char* tail = static_cast<char*>(scratch) + radix_sort_scratch_bytes(n);
  uint32_t* too_long = reinterpret_cast<uint32_t*>(tail - 64);
  SortPlan* plan = reinterpret_cast<SortPlan*>(tail);
  SortPlan* fb = plan + 1;
  static_assert(2 * sizeof(SortPlan) <= 256, "plans fit their slot");
  uint32_t* const status2[2] = {status, reinterpret_cast<uint32_t*>(tail + 256)};
  TCB_CUDA(cudaMemsetAsync(too_long, 0, sizeof(uint32_t), stream));
  note_launch(), k_sort_plan<<<1, 32, 0, stream>>>(d_and_or, kFixBits, nullptr, n, plan);
  // the windows above kFixBits: at most (64 - kFixBits) / 8 passes
  constexpr int kPrefixSlots = (64 - kFixBits + kRadixBits - 1) / kRadixBits;
  planned_passes(keys, vals, keys_alt, vals_alt, n, plan, kPrefixSlots,
                 static_cast<unsigned>(num_tiles), status2, counters, ghist, stream, iota_vals);
  note_launch(), k_sort_fixup_planned<<<grid_for(n, 256, 148 * 16), 256, 0, stream>>>(
      plan, keys, vals, keys_alt, vals_alt, keys_out, vals_out, n, kFixBits, too_long,
      iota_vals);
  // Fallback, all guarded on the device (no work unless a group was too
  // long): the full sort of the prefix-sorted pairs (stable, so ties keep
  // their index order) into (keys_out, vals_out).
  note_launch(), k_sort_plan<<<1, 32, 0, stream>>>(d_and_or, 0, too_long, n, fb);
  const unsigned small = static_cast<unsigned>(std::min<int64_t>(num_tiles, 148));
  note_launch(), k_sort_fallback_copy<<<small, 256, 0, stream>>>(
      plan, fb, 0, keys, vals, keys_alt, vals_alt, keys_out, vals_out, n, iota_vals);
  planned_passes(keys, vals, keys_alt, vals_alt, n, fb, kMaxPasses, small, status2, counters,
                 ghist, stream, false);
  note_launch(), k_sort_fallback_copy<<<small, 256, 0, stream>>>(
      plan, fb, 1, keys, vals, keys_alt, vals_alt, keys_out, vals_out, n, false);
  TCB_CUDA(cudaGetLastError());
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
