// Device-wide building blocks: LSD radix sort of (u64 key, i32 value) pairs
// and an exclusive prefix scan. Hand-written for sm_100a (no CUB / Thrust on
// the hot path).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tcb {

// Scratch needed by radix_sort_pairs for n items (bytes).
size_t radix_sort_scratch_bytes(int64_t n);

// Stable ascending sort of (keys, vals) by key. Only the digit windows whose
// bits are not constant across all keys are sorted: `and_all` / `or_all` are
// the bitwise AND / OR of every key (the key producer reduces them for free).
// A stable LSD sort started from vals = 0..n-1 orders ties by index, which is
// the reference's (code, index) order (bvh.cpp:27-32, dense_grid.cpp:55-60).
// Ping-pongs between (keys, vals) and (keys_alt, vals_alt); returns true when
// the sorted result ended in the *_alt buffers.
bool radix_sort_pairs(uint64_t* keys, int32_t* vals, uint64_t* keys_alt,
                      int32_t* vals_alt, int64_t n, uint64_t and_all,
                      uint64_t or_all, void* scratch, cudaStream_t stream,
                      int* passes_run = nullptr);

// radix_sort_pairs for keys whose low bits rarely matter (Morton codes):
// the LSD passes sort only the bits at and above kFixBits, and one fix-up
// pass orders each group of equal (key >> kFixBits) by (key, val), each
// element placing itself by its rank inside the group. Groups longer than
// kFixMax make it return false (the result is then garbage and the caller
// sorts the original keys with radix_sort_pairs); this synchronizes the
// stream once to read that verdict. vals must be 0..n-1 in order on input.
// On success the sorted pairs are in (keys, vals) when *in_alt is false,
// else in the *_alt buffers.
constexpr int kFixBits = 24;
constexpr int kFixMax = 256;
bool radix_sort_pairs_prefix(uint64_t* keys, int32_t* vals, uint64_t* keys_alt,
                             int32_t* vals_alt, int64_t n, uint64_t and_all, uint64_t or_all,
                             void* scratch, cudaStream_t stream, bool* in_alt,
                             int* passes_run = nullptr);

// Stream-ordered radix_sort_pairs_prefix: no host synchronization, so it can
// be captured in a CUDA graph. The digit windows come from the device-side
// AND / OR of the keys (d_and_or[0], d_and_or[1]), every pass is launched and
// the inactive ones return at once; the result always lands in (keys_out,
// vals_out). A fix-up group longer than kFixMax triggers, on the device, a
// full LSD sort of the prefix-sorted pairs (launched guarded, idle otherwise).
// (keys, vals) and the *_alt buffers are clobbered. iota_vals: vals holds
// nothing yet and stands for 0..n-1 (the first pass generates them).
size_t radix_sort_async_scratch_bytes(int64_t n);
void radix_sort_pairs_prefix_async(uint64_t* keys, int32_t* vals, uint64_t* keys_alt,
                                   int32_t* vals_alt, uint64_t* keys_out, int32_t* vals_out,
                                   int64_t n, const unsigned long long* d_and_or, void* scratch,
                                   cudaStream_t stream, bool iota_vals = false);

// Exclusive scan of n int32 counts into out (may alias in); writes the total
// to *d_total (device pointer) when non-null.
size_t scan_scratch_bytes(int64_t n);
void exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n,
                        int32_t* d_total, void* scratch, cudaStream_t stream);

}  // namespace tcb
