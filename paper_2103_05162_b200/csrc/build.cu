// LBVH construction on the device (reference: bvh.cpp:10-124).
//
//   k_centroid_bounds   scene Aabb over primitive centroids (bvh.cpp:15-21),
//                       fused with the finiteness check of PointSet::validate
//                       (geometry.hpp:29-37)
//   k_morton            fp64 quantization + interleave (geometry.hpp:132-156),
//                       fused AND/OR reduction of the codes for the sort
//   radix_sort_pairs    stable (code, index) order (bvh.cpp:27-32)
//   k_climb             single bottom-up pass (Apetrei 2014) producing the
//                       Karras radix tree (bvh.cpp:49-86), its boxes and max
//                       ranks (bvh.cpp:88-124) and, in points mode, the
//                       Morton-ordered query points (bvh.cpp:34-39)
//   k_root_to_zero      moves the root record to node 0
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstring>

#include "device_common.cuh"
#include "pipeline.hpp"
#include "primitives.cuh"

namespace tcb {

namespace {

__global__ void k_reset_build(DevCounters* ctr) {
  int t = threadIdx.x;
  if (t < 3) ctr->bounds_ord[t] = 0xffffffffu;
  else if (t < 6) ctr->bounds_ord[t] = 0u;
  else if (t == 6) ctr->key_and = ~0ull;
  else if (t == 7) ctr->key_or = 0ull;
  else if (t == 8) ctr->nonfinite = 0;
}

// Primitive box accessors. Points: degenerate box at the point.
template <int D>
struct PointBoxes {
  static constexpr bool kQuad = true;
  const float* coords;
  __device__ __forceinline__ void box(int64_t i, float* lo, float* hi) const {
#pragma unroll
    for (int k = 0; k < D; ++k) lo[k] = hi[k] = coords[i * D + k];
  }
  // the streaming kernels read four points (D float4) per load group when
  // the coordinates are 16-byte aligned
  __device__ __forceinline__ bool quad_ok() const {
    return (reinterpret_cast<uintptr_t>(coords) & 15u) == 0;
  }
  __device__ __forceinline__ void quad(int64_t q, float (&c)[4][3]) const {
    const float4* v = reinterpret_cast<const float4*>(coords) + q * D;
    float f[4 * D];
#pragma unroll
    for (int u = 0; u < D; ++u) {
      const float4 a = __ldcs(v + u);
      f[4 * u] = a.x;
      f[4 * u + 1] = a.y;
      f[4 * u + 2] = a.z;
      f[4 * u + 3] = a.w;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int k = 0; k < D; ++k) c[i][k] = f[i * D + k];
  }
};

template <int D>
struct ExplicitBoxes {
  static constexpr bool kQuad = false;
  __device__ __forceinline__ bool quad_ok() const { return false; }
  __device__ __forceinline__ void quad(int64_t, float (&)[4][3]) const {}
  const float4* lo4;
  const float4* hi4;
  __device__ __forceinline__ void box(int64_t i, float* lo, float* hi) const {
    float4 a = lo4[i], b = hi4[i];
    lo[0] = a.x;
    lo[1] = a.y;
    hi[0] = b.x;
    hi[1] = b.y;
    if (D == 3) {
      lo[2] = a.z;
      hi[2] = b.z;
    }
  }
};

// Aabb::centroid (geometry.hpp:67-69): 0.5f * (min + max) in fp32.
template <int D>
__device__ __forceinline__ void centroid(const float* lo, const float* hi, float* c) {
#pragma unroll
  for (int k = 0; k < D; ++k) c[k] = __fmul_rn(0.5f, __fadd_rn(lo[k], hi[k]));
}

template <int D, class Src>
__global__ void __launch_bounds__(256)
k_centroid_bounds(Src src, int64_t m, bool check_finite, DevCounters* ctr) {
  float mn[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, mx[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
  bool bad = false;
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t first = tid;
  if (Src::kQuad && src.quad_ok()) {  // points: a point's box is its centroid
    for (int64_t q = tid; q < m / 4; q += stride) {
      float c[4][3];
      src.quad(q, c);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float lo[3], cc[3];
#pragma unroll
        for (int k = 0; k < D; ++k) lo[k] = c[i][k];
        if (check_finite) {
#pragma unroll
          for (int k = 0; k < D; ++k) bad |= !isfinite(lo[k]);
        }
        centroid<D>(lo, lo, cc);
#pragma unroll
        for (int k = 0; k < D; ++k) {
          mn[k] = fminf(mn[k], cc[k]);
          mx[k] = fmaxf(mx[k], cc[k]);
        }
      }
    }
    first = m / 4 * 4 + tid;
  }
  for (int64_t i = first; i < m; i += stride) {
    float lo[3], hi[3], c[3];
    src.box(i, lo, hi);
    if (check_finite) {
#pragma unroll
      for (int k = 0; k < D; ++k) bad |= !isfinite(lo[k]);
    }
    centroid<D>(lo, hi, c);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      mn[k] = fminf(mn[k], c[k]);
      mx[k] = fmaxf(mx[k], c[k]);
    }
  }
  publish_bounds<D>(mn, mx, bad, ctr);
}

template <int D, class Src>
__global__ void __launch_bounds__(256)
k_morton(Src src, int64_t m, DevCounters* ctr, uint64_t* __restrict__ keys,
         int32_t* __restrict__ vals) {
  constexpr int bits = D == 2 ? 31 : 21;  // morton_bits_per_axis (geometry.hpp:130)
  constexpr uint64_t cells = 1ull << bits;
  const double cells_d = static_cast<double>(cells);
  float lo_s[3], w_lo[3];
  double w[3], rw[3];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    lo_s[k] = ord2f(ctr->bounds_ord[k]);
    float hi_s = ord2f(ctr->bounds_ord[3 + k]);
    w[k] = __dsub_rn(static_cast<double>(hi_s), static_cast<double>(lo_s[k]));
    rw[k] = w[k] > 0.0 ? __drcp_rn(w[k]) : 0.0;
    w_lo[k] = lo_s[k];
  }
  uint64_t acc_and = ~0ull, acc_or = 0;
  auto encode = [&](const float* c) {
    uint64_t code;
    if (D == 2) {
      uint64_t x = quantize_rcp(c[0], w_lo[0], w[0], rw[0], cells_d, cells);
      uint64_t y = quantize_rcp(c[1], w_lo[1], w[1], rw[1], cells_d, cells);
      code = spread2(x) | (spread2(y) << 1);
    } else {
      uint64_t x = quantize_rcp(c[0], w_lo[0], w[0], rw[0], cells_d, cells);
      uint64_t y = quantize_rcp(c[1], w_lo[1], w[1], rw[1], cells_d, cells);
      uint64_t z = quantize_rcp(c[2], w_lo[2], w[2], rw[2], cells_d, cells);
      code = spread3(x) | (spread3(y) << 1) | (spread3(z) << 2);
    }
    acc_and &= code;
    acc_or |= code;
    return code;
  };
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t first = tid;
  if (Src::kQuad && src.quad_ok()) {  // four points per thread, 16-byte loads and stores
    for (int64_t q = tid; q < m / 4; q += stride) {
      float c[4][3];
      src.quad(q, c);
      uint64_t code[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float lo[3], cc[3];
#pragma unroll
        for (int k = 0; k < D; ++k) lo[k] = c[i][k];
        centroid<D>(lo, lo, cc);
        code[i] = encode(cc);
      }
      ulonglong2* k2 = reinterpret_cast<ulonglong2*>(keys + 4 * q);
      k2[0] = make_ulonglong2(code[0], code[1]);
      k2[1] = make_ulonglong2(code[2], code[3]);
      const int32_t i0 = static_cast<int32_t>(4 * q);
      if (vals) reinterpret_cast<int4*>(vals)[q] = make_int4(i0, i0 + 1, i0 + 2, i0 + 3);
    }
    first = m / 4 * 4 + tid;
  }
  for (int64_t i = first; i < m; i += stride) {
    float lo[3], hi[3], c[3];
    src.box(i, lo, hi);
    centroid<D>(lo, hi, c);
    const uint64_t code = encode(c);
    keys[i] = code;
    if (vals) vals[i] = static_cast<int32_t>(i);
  }
  publish_and_or(acc_and, acc_or, ctr);
}

// Bvh::delta (bvh.cpp:49-56): common prefix of (code, index) keys.
__device__ __forceinline__ int key_delta(const uint64_t* __restrict__ codes, int64_t m,
                                         int64_t i, int64_t j) {
  if (j < 0 || j >= m) return -1;
  uint64_t ci = codes[i], cj = codes[j];
  if (ci != cj) return __clzll(static_cast<long long>(ci ^ cj));
  return 64 + __clz(static_cast<int>(static_cast<uint32_t>(i) ^ static_cast<uint32_t>(j)));
}

// delta(s, s+1) of every boundary as one byte (<= 96; -1 past the end as
// 0xff), so the climb's global phase reads 1-byte values from an L2-resident
// array instead of two 8-byte codes per boundary.
__global__ void __launch_bounds__(256)
k_boundary_deltas(const uint64_t* __restrict__ codes, int64_t m, int8_t* __restrict__ delta) {
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < m;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x)
    delta[s] = static_cast<int8_t>(key_delta(codes, m, s, s + 1));
}

// ---------------------------------------------------------------------------
// Single-pass bottom-up build (Apetrei 2014) of the Karras radix tree
// (bvh.cpp:49-124): topology, boxes and leaf gather in one kernel.
//
// Thread s starts at leaf s (range [s, s]). A node covering [l, r] is the
// LEFT child of the internal node whose split is r when delta(r) >
// delta(l-1) (or l == 0), else the RIGHT child of the node whose split is
// l-1 — the boundaries of a subtree never have equal deltas, so this is
// exactly the Karras parent. Internal nodes are numbered by their split, so a
// child knows its parent's record at once and writes its box, link and aux
// (max rank, or the leaf payload) into its slot there (children-in-parent
// layout, bvh.cuh). The two children meet at an exchange on the parent's
// `other` word: the first stores its outer bound and stops; the second reads
// the sibling's bound (the parent's full range) and its slot, and climbs on
// with the union box. Only the meeting is ordered: slot stores, then an
// exchange with release semantics; the second arriver reads the sibling slot
// through L2 (ld.cg) after the exchange that observed it.
// Numbering by split puts the root at some index g; k_root_to_zero moves it
// to node 0 (the traversals' entry) and node 0's record to the spare slot m-1.
// The tree is the reference's tree node for node; only the numbering of the
// internal nodes differs (tcg_debug_point_bvh renumbers to Karras indices).
// ---------------------------------------------------------------------------
#ifndef TCB_CLIMB_DELTAS
#define TCB_CLIMB_DELTAS 1
#endif
constexpr int kClimbBlock = 128;  // 256: topology 3.04 vs 2.90 ms on C2; 64: 3.06; 512 slower still

struct ClimbState {
  int32_t root;         // split index of the root
  int32_t zero_parent;  // parent of internal node 0 | kUpLeftBit if left child
};

// Exchange with release semantics: this thread's earlier slot stores are
// visible (at L2) to whoever observes the exchanged value. No acquire side:
// the reader goes through L2 (ld.cg) — a full __threadfence would also
// invalidate the SM's L1 (CCTL.IVALL) on every climbing step.
__device__ __forceinline__ int32_t atom_exch_release(int32_t* p, int32_t v) {
  int32_t old;
  asm volatile("atom.exch.release.gpu.global.b32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

template <int D, class Src>
__global__ void __launch_bounds__(kClimbBlock)
k_climb(Src src, const uint64_t* __restrict__ codes, const int32_t* __restrict__ order,
        const int32_t* __restrict__ prim_aux, int64_t m, float4* nodes,
        int32_t* __restrict__ other, float4* __restrict__ leaf_pt,
        ClimbState* state, const int8_t* __restrict__ deltas) {
  using T = NodeTraits<D>;
  const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  bool active = s < m;
  float lo[3] = {0.f, 0.f, 0.f}, hi[3] = {0.f, 0.f, 0.f};
  int32_t l = 0, r = 0, link = 0, aux = 0;
  if (active) {
    const int32_t prim = order[s];
    src.box(prim, lo, hi);
    if (leaf_pt) leaf_pt[s] = make_float4(lo[0], lo[1], D == 3 ? lo[2] : 0.f, __int_as_float(prim));
    l = r = static_cast<int32_t>(s);
    link = ~l;
    aux = prim_aux ? prim_aux[prim] : prim;
  }

  // ---- block-local phase: every node whose two children lie inside this
  // block's leaves is finished here through shared memory — the left
  // child's thread reads the right child's box and writes the whole record;
  // no exchange, no fence. Subtrees stay a partition of the block's leaves,
  // each held by the thread of its first leaf; s_start[end] is the first leaf
  // of the subtree ending at `end` (a right child's way to its left sibling).
  {
    __shared__ float s_box[2 * D][kClimbBlock];
    __shared__ int32_t s_r[kClimbBlock], s_link[kClimbBlock], s_aux[kClimbBlock];
    __shared__ int32_t s_code[kClimbBlock], s_start[kClimbBlock];
    __shared__ int32_t s_delta[kClimbBlock + 1];  // delta(b0 - 1 + j), j = 0..kClimbBlock
    const int t = threadIdx.x;
    const int64_t b0 = s - t;
    const int64_t b1 = min(b0 + kClimbBlock - 1, m - 1);
    // every boundary delta a subtree inside the block can ask for, computed once
    if (deltas) {
      if (b0 + t < m) s_delta[t + 1] = deltas[b0 + t];
      else s_delta[t + 1] = -1;
      if (t == 0) s_delta[0] = b0 > 0 ? deltas[b0 - 1] : -1;
    } else {
      s_delta[t + 1] = key_delta(codes, m, b0 + t, b0 + t + 1);
      if (t == 0) s_delta[0] = b0 > 0 ? key_delta(codes, m, b0 - 1, b0) : -1;
    }
    __syncthreads();
    auto publish = [&] {
#pragma unroll
      for (int k = 0; k < D; ++k) {
        s_box[k][t] = lo[k];
        s_box[D + k][t] = hi[k];
      }
      s_r[t] = r;
      s_link[t] = link;
      s_aux[t] = aux;
    };
    if (active) {
      publish();
      s_start[t] = l;
    }
    while (true) {
      bool left = false;
      int32_t p = 0;
      if (active) {
        left = l == 0 || (r != m - 1 && s_delta[r - b0 + 1] > s_delta[l - b0]);
        p = left ? r : l - 1;
      }
      s_code[t] = active ? (2 | (left ? 1 : 0)) : 0;  // alive | left child
      __syncthreads();
      const bool as_left = active && left && r + 1 <= b1 && s_code[r + 1 - b0] == 2;
      const bool as_right =
          active && !left && l - 1 >= b0 && s_code[s_start[l - 1 - b0] - b0] == 3;
      if (!__syncthreads_or(as_left)) break;
      if (as_left) {
        const int u = static_cast<int>(r + 1 - b0);  // the right child's thread
        float rec[T::kFloats];
#pragma unroll
        for (int k = 0; k < D; ++k) {
          rec[k] = lo[k];
          rec[D + k] = hi[k];
          rec[2 * D + k] = s_box[k][u];
          rec[3 * D + k] = s_box[D + k][u];
        }
        const int32_t slink = s_link[u];
        rec[T::kIntOff + 0] = __int_as_float(link);
        rec[T::kIntOff + 1] = __int_as_float(slink);
        rec[T::kIntOff + 2] = __int_as_float(aux);
        rec[T::kIntOff + 3] = __int_as_float(s_aux[u]);
        float4* dst = nodes + static_cast<int64_t>(p) * T::kVec;
#pragma unroll
        for (int v = 0; v < (D == 3 ? 4 : 3); ++v)  // (a 2D record's last float4 is padding)
          __stcg(dst + v, make_float4(rec[4 * v], rec[4 * v + 1], rec[4 * v + 2], rec[4 * v + 3]));
        if (link == 0) state->zero_parent = p | kUpLeftBit;
        if (slink == 0) state->zero_parent = p;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          lo[k] = fminf(lo[k], rec[2 * D + k]);
          hi[k] = fmaxf(hi[k], rec[3 * D + k]);
        }
        r = s_r[u];
        link = p;
        aux = r;
        if (l == 0 && r == m - 1) {
          state->root = p;
          active = false;
        }
      }
      if (as_right) active = false;  // finished by the left sibling's thread
      __syncthreads();
      if (as_left) {
        publish();
        s_start[r - b0] = l;
      }
    }
  }

  // ---- global phase: climb through exchanges on the parents' `other` word
  while (__any_sync(0xffffffffu, active)) {
    int32_t p = 0;
    bool left = false;
    if (active) {
      left = l == 0 ||
             (r != m - 1 && (deltas ? deltas[r] > deltas[l - 1]
                                    : key_delta(codes, m, r, r + 1) > key_delta(codes, m, l - 1, l)));
      p = left ? r : l - 1;
      float* pf = reinterpret_cast<float*>(nodes + static_cast<int64_t>(p) * T::kVec);
      float* slot = pf + (left ? 0 : 2 * D);
#pragma unroll
      for (int k = 0; k < D; ++k) {
        __stcg(slot + k, lo[k]);
        __stcg(slot + D + k, hi[k]);
      }
      int32_t* ip = reinterpret_cast<int32_t*>(pf + T::kIntOff);
      __stcg(ip + (left ? 0 : 1), link);
      __stcg(ip + (left ? 2 : 3), aux);
      if (link == 0) state->zero_parent = p | (left ? kUpLeftBit : 0);
    }
    if (active) {
      const int32_t o = atom_exch_release(other + p, left ? l : r);
      if (o < 0) {
        active = false;  // first arrival: the sibling finishes the parent
      } else {
        if (left)
          r = o;
        else
          l = o;
        const float* pf = reinterpret_cast<const float*>(nodes + static_cast<int64_t>(p) * T::kVec);
        const float* sib = pf + (left ? 2 * D : 0);
#pragma unroll
        for (int k = 0; k < D; ++k) {
          lo[k] = fminf(lo[k], __ldcg(sib + k));
          hi[k] = fmaxf(hi[k], __ldcg(sib + D + k));
        }
        link = p;
        aux = r;  // max leaf rank of [l, r]
        if (l == 0 && r == m - 1) {
          state->root = p;
          active = false;
        }
      }
    }
  }
}

// Moves the root record to node 0 and node 0's record to the spare slot m-1,
// re-pointing the one link that referenced node 0.
template <int D>
__global__ void k_root_to_zero(float4* nodes, int64_t m, const ClimbState* state) {
  using T = NodeTraits<D>;
  const int32_t root = state->root;
  if (root == 0) return;
  const int t = threadIdx.x;  // T::kVec threads
  const float4 zero_rec = nodes[t];
  const float4 root_rec = nodes[static_cast<int64_t>(root) * T::kVec + t];
  __syncthreads();
  nodes[(m - 1) * T::kVec + t] = zero_rec;
  nodes[t] = root_rec;
  __syncthreads();
  if (t == 0) {
    int32_t zp = up_parent(state->zero_parent);
    if (zp == root) zp = 0;  // the root's record now lives at 0
    int32_t* ip = reinterpret_cast<int32_t*>(reinterpret_cast<float*>(nodes + static_cast<int64_t>(zp) * T::kVec) + T::kIntOff);
    ip[up_is_left(state->zero_parent) ? 0 : 1] = static_cast<int32_t>(m - 1);
  }
}

// 1-leaf tree: pseudo root with the leaf on the left and an empty box right.
template <int D, class Src>
__global__ void k_single_leaf(Src src, const int32_t* __restrict__ prim_aux, float4* nodes,
                              float4* leaf_pt) {
  using T = NodeTraits<D>;
  float lo[3], hi[3];
  src.box(0, lo, hi);
  float* f = reinterpret_cast<float*>(nodes);
  for (int k = 0; k < D; ++k) {
    f[k] = lo[k];
    f[D + k] = hi[k];
    f[2 * D + k] = INFINITY;
    f[3 * D + k] = -INFINITY;
  }
  int32_t aux = prim_aux ? prim_aux[0] : 0;
  int4* ip = reinterpret_cast<int4*>(f + T::kIntOff);
  *ip = make_int4(~0, ~0, aux, aux);
  if (leaf_pt) leaf_pt[0] = make_float4(lo[0], lo[1], D == 3 ? lo[2] : 0.f, __int_as_float(0));
}

template <int D, class Src>
BuiltBvh build_impl(const Src& boxes, const PrimSource& src, bool validate_finite,
                    bool points_mode, DevCounters* d_ctr, Scratch& scratch,
                    StageClock* clock, bool stream_ordered) {
  cudaStream_t st = scratch.stream();
  const int64_t m = src.count;
  BuiltBvh out;
  out.tree.num_leaves = static_cast<int32_t>(m);
  const int64_t num_nodes = std::max<int64_t>(1, m);  // m - 1 internal + 1 spare (k_root_to_zero)
  out.tree.nodes = scratch.alloc_n<float4>(num_nodes * NodeTraits<D>::kVec);
  if (points_mode) out.leaf_pt = scratch.alloc_n<float4>(m);

  // Reset the per-build reductions (bounds, key AND/OR, finiteness flag).
  note_launch(), k_reset_build<<<1, 32, 0, st>>>(d_ctr);

  const unsigned g = grid_for(m, 256, 148 * 8);
  note_launch(), k_centroid_bounds<D><<<g, 256, 0, st>>>(boxes, m, validate_finite, d_ctr);
  uint64_t* keys = scratch.alloc_n<uint64_t>(m);
  int32_t* vals = scratch.alloc_n<int32_t>(m);
  // the stream-ordered sort's first pass generates the identity values itself
  note_launch(), k_morton<D><<<g, 256, 0, st>>>(boxes, m, d_ctr, keys,
                                               stream_ordered ? nullptr : vals);
  TCB_CUDA(cudaGetLastError());

  const uint64_t* codes;
  int32_t* order;
  if (stream_ordered) {
    // No read-back: the device plans the sort passes from the key AND/OR and
    // the non-finite flag stays on the device (run_device reports it).
    if (clock) clock->mark(kStSort);
    uint64_t* keys_alt = scratch.alloc_n<uint64_t>(m);
    int32_t* vals_alt = scratch.alloc_n<int32_t>(m);
    uint64_t* keys_out = scratch.alloc_n<uint64_t>(m);
    int32_t* vals_out = scratch.alloc_n<int32_t>(m);
    void* sort_tmp = scratch.alloc(radix_sort_async_scratch_bytes(m));
    radix_sort_pairs_prefix_async(keys, vals, keys_alt, vals_alt, keys_out, vals_out, m,
                                  &d_ctr->key_and, sort_tmp, st, /*iota_vals=*/true);
    codes = keys_out;
    order = vals_out;
    out.sort_passes = -1;  // decided on the device
  } else {
    // One small read-back: finiteness + key AND/OR decide the sort passes.
    auto* h = static_cast<unsigned char*>(pinned_staging(64));
    TCB_CUDA(cudaMemcpyAsync(h, &d_ctr->key_and, 16, cudaMemcpyDeviceToHost, st));
    TCB_CUDA(cudaMemcpyAsync(h + 16, &d_ctr->nonfinite, 4, cudaMemcpyDeviceToHost, st));
    TCB_CUDA(cudaStreamSynchronize(st));
    unsigned long long key_and, key_or;
    int32_t nonfinite;
    std::memcpy(&key_and, h, 8);
    std::memcpy(&key_or, h + 8, 8);
    std::memcpy(&nonfinite, h + 16, 4);
    if (validate_finite && nonfinite) throw InvalidArgument{"PointSet: non-finite coordinate"};

    if (clock) clock->mark(kStSort);
    uint64_t* keys_alt = scratch.alloc_n<uint64_t>(m);
    int32_t* vals_alt = scratch.alloc_n<int32_t>(m);
    void* sort_tmp = scratch.alloc(radix_sort_scratch_bytes(m));
    // Morton codes are nearly unique at their top 40 bits (C2: groups of <= 6
    // points), so the LSD passes skip the low 24 bits and one fix-up pass
    // orders the small groups; a long group (many coincident points) falls
    // back to the full sort of freshly computed codes. Same order either way.
    bool in_alt = false;
    if (!radix_sort_pairs_prefix(keys, vals, keys_alt, vals_alt, m, key_and, key_or, sort_tmp, st,
                                 &in_alt, &out.sort_passes)) {
      note_launch(), k_morton<D><<<g, 256, 0, st>>>(boxes, m, d_ctr, keys, vals);
      in_alt = radix_sort_pairs(keys, vals, keys_alt, vals_alt, m, key_and, key_or, sort_tmp, st,
                                &out.sort_passes);
    }
    codes = in_alt ? keys_alt : keys;
    order = in_alt ? vals_alt : vals;
  }
  out.tree.leaf_order = order;

  if (clock) clock->mark(kStTopo);
  float4* leaf_pt = out.leaf_pt;
  out.codes = codes;
  uint32_t* scene = scratch.alloc_n<uint32_t>(8);
  TCB_CUDA(cudaMemcpyAsync(scene, &d_ctr->bounds_ord[0], 6 * sizeof(uint32_t),
                           cudaMemcpyDeviceToDevice, st));
  out.scene_ord = scene;
  if (m == 1) {
    note_launch(), k_single_leaf<D><<<1, 1, 0, st>>>(boxes, src.aux, out.tree.nodes, leaf_pt);
  } else {
    int32_t* other = scratch.alloc_n<int32_t>(m - 1);
    auto* state = scratch.alloc_n<ClimbState>(1);
    TCB_CUDA(cudaMemsetAsync(other, 0xff, sizeof(int32_t) * (m - 1), st));
    int8_t* deltas = nullptr;
    if (TCB_CLIMB_DELTAS) {
      deltas = scratch.alloc_n<int8_t>(m);
      note_launch(), k_boundary_deltas<<<grid_for(m, 256, 148 * 16), 256, 0, st>>>(codes, m, deltas);
    }
    note_launch(), k_climb<D><<<grid_for(m, kClimbBlock, INT32_MAX), kClimbBlock, 0, st>>>(
        boxes, codes, order, src.aux, m, out.tree.nodes, other, leaf_pt, state, deltas);
    note_launch(), k_root_to_zero<D><<<1, NodeTraits<D>::kVec, 0, st>>>(out.tree.nodes, m, state);
  }
  TCB_CUDA(cudaGetLastError());
  return out;
}

}  // namespace

namespace {

// compute_bounds (geometry.hpp:95-101): raw point min/max (not centroids)
// plus the finiteness check of PointSet::validate.
template <int D>
__global__ void __launch_bounds__(256)
k_point_bounds(const float* __restrict__ coords, int64_t n, DevCounters* ctr) {
  float mn[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, mx[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
  bool bad = false;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      float v = coords[i * D + k];
      bad |= !isfinite(v);
      mn[k] = fminf(mn[k], v);
      mx[k] = fmaxf(mx[k], v);
    }
  }
  publish_bounds<D>(mn, mx, bad, ctr);
}

}  // namespace

template <int D>
void launch_point_bounds(const float* coords, int64_t n, DevCounters* ctr, cudaStream_t s) {
  note_launch(), k_reset_build<<<1, 32, 0, s>>>(ctr);
  note_launch(), k_point_bounds<D><<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(coords, n, ctr);
  TCB_CUDA(cudaGetLastError());
}

template void launch_point_bounds<2>(const float*, int64_t, DevCounters*, cudaStream_t);
template void launch_point_bounds<3>(const float*, int64_t, DevCounters*, cudaStream_t);

template <int D>
BuiltBvh build_bvh(const PrimSource& src, bool validate_finite, DevCounters* d_ctr,
                   Scratch& scratch, StageClock* clock, bool stream_ordered) {
  if (src.coords) {
    PointBoxes<D> b{src.coords};
    return build_impl<D>(b, src, validate_finite, true, d_ctr, scratch, clock, stream_ordered);
  }
  ExplicitBoxes<D> b{src.lo, src.hi};
  return build_impl<D>(b, src, validate_finite, false, d_ctr, scratch, clock, stream_ordered);
}

template BuiltBvh build_bvh<2>(const PrimSource&, bool, DevCounters*, Scratch&, StageClock*, bool);
template BuiltBvh build_bvh<3>(const PrimSource&, bool, DevCounters*, Scratch&, StageClock*, bool);

}  // namespace tcb
