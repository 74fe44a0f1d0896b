// Device-side primitives shared by every kernel of the engine.
//
// Arithmetic contract: coordinates are fp32, every distance and
// box distance is accumulated in fp64 exactly like the reference's unfused
// chain
//     s = 0.0; for k: d = double(a_k) - double(b_k); s = s + d*d
// (geometry.hpp:72-93) and compared `<= double(eps)*double(eps)`. We spell it
// with __dsub_rn / __dmul_rn / __dadd_rn so nvcc can never contract it into a
// DFMA (the translation units are also built with -fmad=false).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tcb {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// Exact fp64 predicates (geometry.hpp:72-93)
// ---------------------------------------------------------------------------

template <int D>
__device__ __forceinline__ double dist2(const float* a, const float* b) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    double d = __dsub_rn(static_cast<double>(a[k]), static_cast<double>(b[k]));
    s = __dadd_rn(s, __dmul_rn(d, d));
  }
  return s;
}

// Squared distance from p to the closed box [lo, hi] (0 inside), same branch
// structure as box_distance_sq (geometry.hpp:82-93).
template <int D>
__device__ __forceinline__ double box_dist2(const float* p, const float* lo,
                                            const float* hi) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    double d = 0.0;
    if (p[k] < lo[k])
      d = __dsub_rn(static_cast<double>(lo[k]), static_cast<double>(p[k]));
    else if (p[k] > hi[k])
      d = __dsub_rn(static_cast<double>(p[k]), static_cast<double>(hi[k]));
    s = __dadd_rn(s, __dmul_rn(d, d));
  }
  return s;
}

// ---------------------------------------------------------------------------
// Morton codes (geometry.hpp:104-156): 31 bits/axis in 2D, 21 in 3D,
// quantization in fp64, axis-major interleave (bit b of axis a -> b*dim + a).
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint64_t spread2(uint64_t x) {
  x &= 0xffffffffull;
  x = (x | (x << 16)) & 0x0000ffff0000ffffull;
  x = (x | (x << 8)) & 0x00ff00ff00ff00ffull;
  x = (x | (x << 4)) & 0x0f0f0f0f0f0f0f0full;
  x = (x | (x << 2)) & 0x3333333333333333ull;
  x = (x | (x << 1)) & 0x5555555555555555ull;
  return x;
}

__device__ __forceinline__ uint64_t spread3(uint64_t x) {
  x &= 0x1fffffull;
  x = (x | (x << 32)) & 0x001f00000000ffffull;
  x = (x | (x << 16)) & 0x001f0000ff0000ffull;
  x = (x | (x << 8)) & 0x100f00f00f00f00full;
  x = (x | (x << 4)) & 0x10c30c30c30c30c3ull;
  x = (x | (x << 2)) & 0x1249249249249249ull;
  return x;
}

// morton_quantize (geometry.hpp:132-141). `w` = double(hi) - double(lo) is
// precomputed per axis; `cells` = 2^bits.
// Monotone non-decreasing in v (every step is a correctly rounded, monotone
// operation), which the Morton-cell early termination relies on.
__device__ __forceinline__ uint64_t quantize_d(double v, float lo, double w, double cells_d,
                                               uint64_t cells) {
  if (w <= 0.0) return 0;
  double t = __ddiv_rn(__dsub_rn(v, static_cast<double>(lo)), w);
  if (t < 0.0) t = 0.0;
  uint64_t q = __double2ull_rz(__dmul_rn(t, cells_d));
  if (q >= cells) q = cells - 1;
  return q;
}

__device__ __forceinline__ uint64_t quantize(float v, float lo, double w, double cells_d,
                                             uint64_t cells) {
  return quantize_d(static_cast<double>(v), lo, w, cells_d, cells);
}

// quantize() with the division replaced by a multiplication with rw =
// RN(1/w): t' = RN(d * rw) is within 3 * 2^-53 (relative, t <= 1) of
// RN(d / w), and cells_d is a power of two (exact scaling), so t' * cells_d
// has the same integer part as the exact chain unless it lies within
// 3 * 2^-53 * cells_d of an integer; a margin of cells_d * 2^-48 (10x that)
// sends those rare cases to the exact chain. Bit-identical to quantize().
__device__ __forceinline__ uint64_t quantize_rcp(float v, float lo, double w, double rw,
                                                 double cells_d, uint64_t cells) {
  if (w <= 0.0) return 0;
  const double d = __dsub_rn(static_cast<double>(v), static_cast<double>(lo));
  const double x = __dmul_rn(__dmul_rn(d, rw), cells_d);  // (scaling by 2^k is exact)
  const double fl = floor(x);
  const double frac = x - fl;
  const double margin = cells_d * 0x1.0p-48;
  if (d < 0.0 || frac < margin || frac > 1.0 - margin)
    return quantize_d(static_cast<double>(v), lo, w, cells_d, cells);
  uint64_t q = static_cast<uint64_t>(fl);
  if (q >= cells) q = cells - 1;
  return q;
}

// ---------------------------------------------------------------------------
// Order-preserving float <-> uint32 mapping for atomicMin/atomicMax bounds.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t f2ord(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ __forceinline__ float ord2f(uint32_t u) {
  uint32_t v = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
#ifdef __CUDA_ARCH__
  return __uint_as_float(v);
#else
  float f;
  __builtin_memcpy(&f, &v, 4);
  return f;
#endif
}

// ---------------------------------------------------------------------------
// Lock-free union-find over a flat int32 parent array (union_find.hpp:18-91).
// Loads/stores are relaxed at GPU scope (L1 is not coherent, so plain loads
// could spin on stale lines); hooks are single CASes.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int32_t ld_relaxed(const int32_t* p) {
  int32_t v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// CTA-scope relaxed load: may be served by this SM's L1, so it can return an
// older value of the word. Only used where any value the word EVER held is
// good enough (a union-find parent that equals a hint proves set membership
// forever, because sets only merge; a stale coverage bound only costs an
// extra atomic).
__device__ __forceinline__ int32_t ld_cached(const int32_t* p) {
  int32_t v;
  asm volatile("ld.relaxed.cta.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(int32_t* p, int32_t v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// find with pointer jumping: every visited node is redirected to its
// grandparent (union_find.hpp:36-49).
__device__ __forceinline__ int32_t uf_find(int32_t* parent, int32_t i) {
  int32_t cur = ld_relaxed(parent + i);
  if (cur != i) {
    int32_t prev = i;
    int32_t next = ld_relaxed(parent + cur);
    while (cur != next) {
      st_relaxed(parent + prev, next);
      prev = cur;
      cur = next;
      next = ld_relaxed(parent + cur);
    }
  }
  return cur;
}

// Hook the higher root under the lower one; retry from fresh roots when the
// CAS loses (union_find.hpp:51-64). Representatives end up as the minimum
// index of each component regardless of schedule. Returns the root the two
// sets were joined under (an ancestor of both from then on).
__device__ __forceinline__ int32_t uf_unite(int32_t* parent, int32_t i, int32_t j) {
  while (true) {
    i = uf_find(parent, i);
    j = uf_find(parent, j);
    if (i == j) return i;
    if (i > j) {
      int32_t t = i;
      i = j;
      j = t;
    }
    if (atomicCAS(parent + j, j, i) == j) return i;
  }
}

// Query-side union with a root hint. `hint` is some ancestor of i (i itself,
// or a root i's set had at some point; sets only ever merge, so it stays in
// i's set). When j's parent already IS the hint, i and j are in one set and
// the pair is a no-op with a single load — the common case inside a halo,
// where a query meets hundreds of neighbours that joined its set long ago.
__device__ __forceinline__ void uf_unite_hinted(int32_t* parent, int32_t i, int32_t j,
                                                int32_t& hint) {
  const int32_t pj = ld_cached(parent + j);  // any past parent of j is proof enough
  if (pj == hint || j == hint) return;
  hint = uf_unite(parent, i, j);
}

// Records a contained run [first, last] for the cover pass (reach[first] =
// max last). The result is unused, so this is a fire-and-forget reduction
// (RED): no load, no dependency stall. Checking reach[first] first to skip
// redundant atomics cost more (a dependent load per run; C2 main pass
// 20.1 vs 19.2 ms).
__device__ __forceinline__ void record_run(int32_t* reach, int32_t first, int32_t last) {
  if (last > first) atomicMax(reach + first, last);
}

// ---- rank-space variant ---------------------------------------------------
// FDBSCAN runs its union-find over LEAF RANKS (Morton order), so a query's
// neighbours — ranks close to its own — have their parent entries in the same
// or nearby cache lines (L1 hits instead of scattered L2 traffic on an array
// indexed by input order). Roots are still chosen by the ORIGINAL index:
// key[rank] = original index, and the higher-key root is hooked under the
// lower-key one, so every representative is the minimum original index of its
// set — the reference's labels (union_find.hpp:51-64).
// `mark` (optional): the surviving root of every successful hook gets
// mark[root] = 1, so "element of a set of >= 2" is (mark[r] || parent[r] != r)
// without a pass over the structure (minpts == 2 core flags).
__device__ __forceinline__ int32_t uf_unite_keyed(int32_t* parent, const int32_t* __restrict__ key,
                                                  int32_t a, int32_t b, uint8_t* mark = nullptr) {
  while (true) {
    a = uf_find(parent, a);
    b = uf_find(parent, b);
    if (a == b) return a;
    if (__ldg(key + a) > __ldg(key + b)) {
      int32_t t = a;
      a = b;
      b = t;
    }
    if (atomicCAS(parent + b, b, a) == b) {
      if (mark) mark[a] = 1;
      return a;
    }
  }
}

__device__ __forceinline__ void uf_unite_hinted_keyed(int32_t* parent, const int32_t* key,
                                                      int32_t a, int32_t b, int32_t& hint,
                                                      uint8_t* mark = nullptr) {
  const int32_t pb = ld_cached(parent + b);  // any past parent of b is proof enough
  if (pb == hint || b == hint) return;
  hint = uf_unite_keyed(parent, key, a, b, mark);
}

// One-shot border claim (union_find.hpp:69-73).
__device__ __forceinline__ bool uf_claim(int32_t* parent, int32_t i, int32_t root) {
  return atomicCAS(parent + i, i, root) == i;
}

// resolve_pair (dbscan.hpp:82-99) for core flags that are final (minpts > 2):
// core-core unions, core-border claims the border once (no bridging),
// border-border is a no-op. Per-query state:
//   hint       root hint of i (see uf_unite_hinted); a core i claims borders
//              under it: the reference claims under find(i), and any ancestor
//              of i flattens to the same representative
//   i_settled  a border i that has been claimed (by anyone) can take no
//              further action, so its remaining pairs are skipped
// force_core (minpts == 2) never comes here: every pair is a core-core union
// and the core flags are derived at finalize (dbscan.hpp:85-89).
__device__ __forceinline__ void resolve_pair(int32_t i, int32_t j, bool core_i,
                                             const uint8_t* flags, int32_t* parent,
                                             int32_t& hint, bool& i_settled) {
  if (core_i) {
    if (flags[j]) {
      uf_unite_hinted(parent, i, j, hint);
    } else if (ld_relaxed(parent + j) == j) {
      uf_claim(parent, j, hint);
    }
  } else if (!i_settled && flags[j]) {
    if (ld_relaxed(parent + i) == i) uf_claim(parent, i, uf_find(parent, j));
    i_settled = true;  // claimed now, or by someone else before
  }
}

// resolve_pair in rank space (see uf_unite_keyed); a, b and flags are ranks.
__device__ __forceinline__ void resolve_pair_keyed(int32_t a, int32_t b, bool core_a,
                                                   const uint8_t* flags, int32_t* parent,
                                                   const int32_t* key, int32_t& hint,
                                                   bool& a_settled) {
  if (core_a) {
    if (flags[b]) {
      uf_unite_hinted_keyed(parent, key, a, b, hint);
    } else if (ld_relaxed(parent + b) == b) {
      uf_claim(parent, b, hint);
    }
  } else if (!a_settled && flags[b]) {
    if (ld_relaxed(parent + a) == a) uf_claim(parent, a, uf_find(parent, b));
    a_settled = true;
  }
}

// ---------------------------------------------------------------------------
// Warp / block reductions
// ---------------------------------------------------------------------------
// Block-wide reduction (any blockDim multiple of 32, <= 1024); the result is
// valid in thread 0. `scratch` holds >= 32 T.
template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, Op op, T identity, T* scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < static_cast<int>(blockDim.x >> 5) ? scratch[lane] : identity;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace tcb
