// Linear BVH in HBM: node layout and the eps-ball traversal.
//
// Layout ("children in parent"). The reference Node (bvh.hpp:89-94) stores
// its own box and the traversal tests each child against the child's own box
// (bvh.hpp:60-71). Here every internal node stores BOTH children's boxes,
// their child links and, per child, one aux int:
//     3D: 64 B = 4 x float4   [L.lo xyz, L.hi xyz, R.lo xyz, R.hi xyz | l, r, auxL, auxR]
//     2D: 64 B = 4 x float4   [L.lo xy,  L.hi xy,  R.lo xy,  R.hi xy  | l, r, auxL, auxR | pad]
// so one node fetch (two 32 B sectors) decides both children with no second
// dependent load. Child links: >= 0 internal node index, < 0 = ~leaf_rank
// (bvh.hpp:91). aux for an internal child = its max leaf rank (the right end
// of its Karras range, bvh.cpp:88-124 computes the same by propagation); for a
// leaf child = the primitive's payload (point index for a SinglePoint, or
// ~cell for a DenseBox in the mixed tree). Because a leaf child's box lives in
// its parent, a leaf visit never touches the leaf arrays.
//
// A 1-leaf tree (the reference special case bvh.hpp:49-53) is stored as one
// pseudo node whose right child is an empty (+inf/-inf) box that no ball hits.
#pragma once

#include <cmath>
#include <cstdint>

#include "device_common.cuh"

namespace tcb {

// Both layouts take 64 B: the 2D record (48 B of payload) is padded so that
// every record is 32-byte aligned and loads as two 256-bit loads.
template <int D>
struct NodeTraits {
  static constexpr int kVec = 4;          // float4 per node
  static constexpr int kFloats = kVec * 4;
  static constexpr int kIntOff = 4 * D;   // float index of the int4 part
};

constexpr int kStackDepth = 128;

// One node record into registers: two 256-bit loads (sm_100 LDG.256; 64 B
// records are 32-byte aligned): half the load requests of float4 loads on
// the L1 pipe that bounds the traversal. A 2D record only needs 48 B of it.
__device__ __forceinline__ void ld_nc_v8(const float* src, float* f) {
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(f[0]), "=f"(f[1]), "=f"(f[2]), "=f"(f[3]), "=f"(f[4]), "=f"(f[5]), "=f"(f[6]),
        "=f"(f[7])
      : "l"(src));
}

template <int D>
__device__ __forceinline__ void load_node(const float4* __restrict__ src, float* f) {
  const float* s = reinterpret_cast<const float*>(src);
  ld_nc_v8(s, f);
  if (D == 3) {
    ld_nc_v8(s + 8, f + 8);
  } else {  // floats 8..11 (the int4 part); 12..15 are padding
    const float4 q = __ldg(src + 2);
    f[8] = q.x;
    f[9] = q.y;
    f[10] = q.z;
    f[11] = q.w;
  }
}  // bvh.hpp:82-84 (keys are 64 + 32 bits)

// Parent links: parent node index, bit 31 set when the child is the parent's
// LEFT child; kNoParent at the root.
constexpr int32_t kUpLeftBit = static_cast<int32_t>(0x80000000u);
constexpr int32_t kNoParent = 0x7fffffff;
__host__ __device__ __forceinline__ int32_t up_parent(int32_t x) { return x & 0x7fffffff; }
__host__ __device__ __forceinline__ bool up_is_left(int32_t x) { return x < 0; }

// The ball-vs-box predicate of the traversal: exactly box_distance_sq <= r2
// in fp64 (geometry.hpp:82-93), answered by an fp32 estimate whenever the
// estimate is outside a relative guard band of 2^-17 around r2. The fp32 sum
// of three rounded squared differences is within ~6 * 2^-24 (relative) of the
// real value and the fp64 chain within ~6 * 2^-53, so a decision outside the
// band is the fp64 decision; inside it the fp64 chain runs. The fast path is
// enabled only when r2 is a normal fp32 number far from under/overflow
// (1e-20 <= r2 <= 1e30), so the relative bound holds.
struct BallTest {
  double r2;
  double reach;      // per-axis bound on |q_k - p_k| of any q the predicate accepts
  float lo_f, hi_f;  // r2 * (1 -+ 2^-17) in fp32
  bool fast;
  __host__ static BallTest make(double eps2) {
    BallTest b;
    b.r2 = eps2;
    // fl(sum of squares) <= r2 implies every |d_k| <= sqrt(r2) (1 + ~2^-52)
    b.reach = std::sqrt(eps2) * (1.0 + 0x1.0p-30);
    b.fast = eps2 >= 1e-20 && eps2 <= 1e30;
    b.lo_f = static_cast<float>(eps2 * (1.0 - 0x1.0p-17));
    b.hi_f = static_cast<float>(eps2 * (1.0 + 0x1.0p-17));
    return b;
  }
};

// kFast: 1 = bt.fast known true, 0 = known false, -1 = test at run time
// (kernels on the hot path are instantiated for both and launched by the host
// with the right one, which drops the fp64-only branch from their loops).
template <int D, int kFast = -1>
__device__ __forceinline__ bool ball_hits(const float* p, const float* lo, const float* hi,
                                          const BallTest& bt) {
  if (kFast == 1 || (kFast == -1 && bt.fast)) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      float d = fmaxf(fmaxf(__fsub_rn(lo[k], p[k]), __fsub_rn(p[k], hi[k])), 0.f);
      s = __fadd_rn(s, __fmul_rn(d, d));
    }
    if (s < bt.lo_f) return true;
    if (s > bt.hi_f) return false;
  }
  return box_dist2<D>(p, lo, hi) <= bt.r2;
}

// True when EVERY point of the closed box [lo, hi] is within the ball, by the
// same exact fp64 predicate: per axis the farthest box coordinate is at least
// as far as any member (rounding is monotone), so fl(maxdist^2) <= r2 implies
// fl(dist^2) <= r2 for every member. fp32 guard-band fast path as ball_hits.
template <int D>
__device__ __forceinline__ bool box_inside_ball(const float* p, const float* lo, const float* hi,
                                                const BallTest& bt) {
  if (bt.fast) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      float d = fmaxf(fabsf(__fsub_rn(p[k], lo[k])), fabsf(__fsub_rn(hi[k], p[k])));
      s = __fadd_rn(s, __fmul_rn(d, d));
    }
    if (s < bt.lo_f) return true;
    if (s > bt.hi_f) return false;
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    double a = fabs(__dsub_rn(static_cast<double>(p[k]), static_cast<double>(lo[k])));
    double b = fabs(__dsub_rn(static_cast<double>(hi[k]), static_cast<double>(p[k])));
    double d = a > b ? a : b;
    s = __dadd_rn(s, __dmul_rn(d, d));
  }
  return s <= bt.r2;
}

// One traversal step of the closed-ball query (p, sqrt(r2)) that hides every
// leaf with rank < min_rank (query_sphere_masked, bvh.hpp:45-72): processes
// ONE node, calling
//     bool visit(int32_t rank, int32_t aux, const float* lo, const float* hi)
// for each leaf child whose box is within the ball (false = stop the query),
// and advances `node` / the stack. Returns false when the query is finished.
// The visit order is exactly the reference's (left before right for leaf
// children; right subtree before left subtree for internal children — its LIFO
// stack order), so early-exit counters match bit for bit.
template <int D, typename Visit>
__device__ __forceinline__ bool bvh_step(const float4* __restrict__ nodes, const float* p,
                                         const BallTest& bt, int32_t min_rank, int32_t& node,
                                         int& top, int32_t* stack, Visit& visit) {
  using T = NodeTraits<D>;
  float f[T::kFloats];
  load_node<D>(nodes + static_cast<int64_t>(node) * T::kVec, f);
  const int32_t left = __float_as_int(f[T::kIntOff + 0]);
  const int32_t right = __float_as_int(f[T::kIntOff + 1]);
  const int32_t aux_l = __float_as_int(f[T::kIntOff + 2]);
  const int32_t aux_r = __float_as_int(f[T::kIntOff + 3]);
  bool go_l = false, go_r = false;
  if (left < 0) {
    if (~left >= min_rank && ball_hits<D>(p, f, f + D, bt))
      if (!visit(~left, aux_l, f, f + D)) return false;
  } else if (aux_l >= min_rank && ball_hits<D>(p, f, f + D, bt)) {
    go_l = true;
  }
  if (right < 0) {
    if (~right >= min_rank && ball_hits<D>(p, f + 2 * D, f + 3 * D, bt))
      if (!visit(~right, aux_r, f + 2 * D, f + 3 * D)) return false;
  } else if (aux_r >= min_rank && ball_hits<D>(p, f + 2 * D, f + 3 * D, bt)) {
    go_r = true;
  }
  if (go_l && go_r) {
    stack[top++] = left;
    node = right;
  } else if (go_l) {
    node = left;
  } else if (go_r) {
    node = right;
  } else {
    if (top == 0) return false;
    node = stack[--top];
  }
  return true;
}

// Ball vs a child's box, with containment: 0 = miss, 1 = hit, 2 = the whole
// box lies inside the ball, so every leaf of the subtree is within eps by the
// exact predicate (see box_inside_ball). Hit / miss is exact (fp64 chain
// inside the guard band); containment is only ever reported from the fp32
// estimate outside the band, and conservatively answered "hit" inside it
// (descending is always correct), so it needs no fp64 chain. For a leaf's
// degenerate box any answer > 0 means "within eps". The fp32 estimates use
// fused multiply-adds: one rounding per term instead of two, inside the same
// error bound as the unfused chain the band was sized for.
template <int D, int kFast = -1>
__device__ __forceinline__ int ball_classify(const float* p, const float* lo, const float* hi,
                                             const BallTest& bt) {
  if (kFast == 0 || (kFast == -1 && !bt.fast)) return ball_hits<D, 0>(p, lo, hi, bt) ? 1 : 0;
  float sn = 0.f, sf = 0.f;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const float a = __fsub_rn(lo[k], p[k]);  // > 0: p below the box
    const float b = __fsub_rn(p[k], hi[k]);  // > 0: p above the box
    const float dn = fmaxf(fmaxf(a, b), 0.f);
    const float df = fminf(a, b);            // -(farthest face distance)
    sn = __fmaf_rn(dn, dn, sn);
    sf = __fmaf_rn(df, df, sf);
  }
  if (sf < bt.lo_f) return 2;
  if (sn < bt.lo_f) return 1;
  if (sn > bt.hi_f) return 0;
  return box_dist2<D>(p, lo, hi) <= bt.r2 ? 1 : 0;
}

// Answers of an `inside` callback (bvh_step_ranged).
constexpr int kStop = 0, kTaken = 1, kWalk = 2;

// Traversal step with subtree containment. Also tracks `nlo`, the first leaf
// rank of the current node (Karras ranges: a node's left child covers
// [lo, split], its right child [split + 1, hi]; the root covers [0, n-1]), so
// that a contained internal child is reported as its unmasked leaf-rank range
// instead of being walked:
//     bool visit(int32_t rank, int32_t aux, bool contained)
//                                               leaf `rank` is within eps
//                                               (its whole box when contained;
//                                               false = stop the query)
//     int inside(int32_t first, int32_t last)   every rank in [first, last]
//                                               (first >= min_rank) is a hit:
//                                               kStop, kTaken, or kWalk (not
//                                               taken as a run: descend)
// Pending subtrees go on `stack` (LocalStack below; a shared-memory ring
// measured slower: it costs occupancy). Both children are classified with the
// same straight-line code (leaf or internal, masked or not) so the lanes of a
// warp only diverge on the rare visit / inside actions. Children are masked at
// min_rank like query_sphere_masked (bvh.hpp:45-72); the order in which
// leaves are reported is not the reference's DFS order (callers only depend
// on the set, or, for early exit, on the count — see CoreQuery).

// self >= 0 (an order-free query of the leaf at rank `self`, e.g. an
// early-exit count): of two children to walk, the one holding `self` goes
// first — its Morton neighbours, the likeliest hits, are counted soonest.
template <int D, typename Stack, typename Visit, typename Inside, int kFast = -1>
__device__ __forceinline__ bool bvh_step_ranged(const float4* __restrict__ nodes, const float* p,
                                                const BallTest& bt, int32_t min_rank,
                                                int32_t& node, int32_t& nlo, Stack& stack,
                                                Visit& visit, Inside& inside,
                                                int32_t self = -1) {
  using T = NodeTraits<D>;
  float f[T::kFloats];
  load_node<D>(nodes + static_cast<int64_t>(node) * T::kVec, f);
  const int32_t left = __float_as_int(f[T::kIntOff + 0]);
  const int32_t right = __float_as_int(f[T::kIntOff + 1]);
  const int32_t aux_l = __float_as_int(f[T::kIntOff + 2]);
  const int32_t aux_r = __float_as_int(f[T::kIntOff + 3]);
  const bool leaf_l = left < 0, leaf_r = right < 0;
  const int32_t split = leaf_l ? ~left : aux_l;  // last rank of the left child
  const int32_t max_r = leaf_r ? ~right : aux_r;
  const int32_t lo_l = nlo > min_rank ? nlo : min_rank;
  const int32_t lo_r = split + 1 > min_rank ? split + 1 : min_rank;
  int cl = ball_classify<D, kFast>(p, f, f + D, bt);
  int cr = ball_classify<D, kFast>(p, f + 2 * D, f + 3 * D, bt);
  if (split < min_rank) cl = 0;
  if (max_r < min_rank) cr = 0;
  if (cl > 0 && (leaf_l || cl == 2)) {
    if (leaf_l) {
      if (!visit(~left, aux_l, cl == 2)) return false;
    } else {
      const int a = inside(lo_l, aux_l);
      if (a == kStop) return false;
      if (a == kWalk) cl = 1;
    }
  }
  if (cr > 0 && (leaf_r || cr == 2)) {
    if (leaf_r) {
      if (!visit(~right, aux_r, cr == 2)) return false;
    } else {
      const int a = inside(lo_r, aux_r);
      if (a == kStop) return false;
      if (a == kWalk) cr = 1;
    }
  }
  const bool go_l = cl == 1 && !leaf_l, go_r = cr == 1 && !leaf_r;
  if (go_l && go_r) {
    if (self >= 0 && self <= split) {  // (nlo <= self: the walk never leaves self's side first)
      stack.push(make_int2(right, split + 1));
      node = left;
    } else {
      stack.push(make_int2(left, nlo));
      node = right;
      nlo = split + 1;
    }
  } else if (go_l) {
    node = left;
  } else if (go_r) {
    node = right;
    nlo = split + 1;
  } else {
    int2 e;
    if (!stack.pop(e)) return false;
    node = e.x;
    nlo = e.y;
  }
  return true;
}

// bvh_step in the reference's exact visit order (leaf children at once, left
// then right; internal children right subtree first), with contained
// internal children taken as runs AT THEIR DFS POSITION: a contained child
// that is next is taken now; one that waits behind its sibling goes on the
// stack as a run entry (x = ~first, y = last) and is taken when popped. The
// sequence of visit / inside calls is therefore the reference's leaf order
// with each contained subtree's leaves merged into one call — what a query
// with an order-dependent early exit (the DenseBox core pass) needs.
//     bool visit(int32_t rank, int32_t aux, const float* lo, const float* hi)
//     bool inside(int32_t first, int32_t last)    (false = stop the query)
template <int D, typename Stack, typename Visit, typename Inside, int kFast = -1>
__device__ __forceinline__ bool bvh_step_ordered(const float4* __restrict__ nodes, const float* p,
                                                 const BallTest& bt, int32_t min_rank,
                                                 int32_t& node, int32_t& nlo, Stack& stack,
                                                 Visit& visit, Inside& inside) {
  using T = NodeTraits<D>;
  float f[T::kFloats];
  load_node<D>(nodes + static_cast<int64_t>(node) * T::kVec, f);
  const int32_t left = __float_as_int(f[T::kIntOff + 0]);
  const int32_t right = __float_as_int(f[T::kIntOff + 1]);
  const int32_t aux_l = __float_as_int(f[T::kIntOff + 2]);
  const int32_t aux_r = __float_as_int(f[T::kIntOff + 3]);
  const bool leaf_l = left < 0, leaf_r = right < 0;
  const int32_t split = leaf_l ? ~left : aux_l;
  const int32_t max_r = leaf_r ? ~right : aux_r;
  int cl = ball_classify<D, kFast>(p, f, f + D, bt);
  int cr = ball_classify<D, kFast>(p, f + 2 * D, f + 3 * D, bt);
  if (split < min_rank) cl = 0;
  if (max_r < min_rank) cr = 0;
  if (leaf_l && cl > 0 && !visit(~left, aux_l, f, f + D)) return false;
  if (leaf_r && cr > 0 && !visit(~right, aux_r, f + 2 * D, f + 3 * D)) return false;
  const bool go_l = !leaf_l && cl > 0, go_r = !leaf_r && cr > 0;
  const int32_t lo_l = nlo > min_rank ? nlo : min_rank;
  const int32_t lo_r = split + 1 > min_rank ? split + 1 : min_rank;
  // the next subtree in DFS order: right first, the left one waits
  bool have_next = false;
  if (go_r) {
    if (go_l) stack.push(cl == 2 ? make_int2(~lo_l, aux_l) : make_int2(left, nlo));
    if (cr == 2) {
      if (!inside(lo_r, aux_r)) return false;
    } else {
      node = right;
      nlo = split + 1;
      have_next = true;
    }
  } else if (go_l) {
    if (cl == 2) {
      if (!inside(lo_l, aux_l)) return false;
    } else {
      node = left;
      have_next = true;
    }
  }
  while (!have_next) {
    int2 e;
    if (!stack.pop(e)) return false;
    if (e.x < 0) {
      if (!inside(~e.x, e.y)) return false;
    } else {
      node = e.x;
      nlo = e.y;
      have_next = true;
    }
  }
  return true;
}

// Traversal stacks of (node, first leaf rank) entries for bvh_step_ranged.
// (caching the top entry in registers measured slower: +14% on the C2 main pass)
// Traversal stack handle: the entries in a per-thread local array owned by the
// kernel, the top index a plain member that stays in a register (a struct
// holding both the array and the top keeps the top in local memory too: one
// more local load and store per push and pop).
struct LocalStack {
  int2* e;
  int top = 0;
  __device__ __forceinline__ explicit LocalStack(int2* buf) : e(buf) {}
  __device__ __forceinline__ void push(int2 v) { e[top++] = v; }
  __device__ __forceinline__ bool pop(int2& v) {
    if (top == 0) return false;
    v = e[--top];
    return true;
  }
  __device__ __forceinline__ void reset() { top = 0; }
};


// Warp-shared descent to a common start node. The 32 queries of a warp are
// Morton-consecutive leaves, so their top-down walks share a long prefix:
// the path from the root to the smallest subtree that can hold a neighbour
// of ANY of them. The warp walks that prefix once, uniformly: U = the box of
// the lanes' query points grown by `reach` on every axis (directed rounding,
// so U contains every point the exact predicate accepts for any lane); from
// the root, while exactly one child of the node can matter (its box meets U
// and its max rank >= the warp's min_rank) and that child is internal, step
// into it. Nothing outside the stop node can be a hit for any lane, so each
// lane's own traversal starts there (node, nlo) instead of at the root.
// Every lane must call it (valid = false for lanes without a query).
template <int D>
__device__ __forceinline__ void warp_start_node(const float4* __restrict__ nodes, const float* p,
                                                bool valid, const BallTest& bt,
                                                int32_t min_rank, int32_t& node, int32_t& nlo) {
  node = 0;
  nlo = 0;
  float ulo[3], uhi[3];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const uint32_t mn = __reduce_min_sync(0xffffffffu, valid ? f2ord(p[k]) : 0xffffffffu);
    const uint32_t mx = __reduce_max_sync(0xffffffffu, valid ? f2ord(p[k]) : 0u);
    if (mn > mx) return;  // no lane has a query
    ulo[k] = __double2float_rd(static_cast<double>(ord2f(mn)) - bt.reach);
    uhi[k] = __double2float_ru(static_cast<double>(ord2f(mx)) + bt.reach);
  }
  min_rank = __reduce_min_sync(0xffffffffu, valid ? min_rank : INT32_MAX);
  using T = NodeTraits<D>;
  while (true) {
    float f[T::kFloats];
    load_node<D>(nodes + static_cast<int64_t>(node) * T::kVec, f);
    const int32_t left = __float_as_int(f[T::kIntOff + 0]);
    const int32_t right = __float_as_int(f[T::kIntOff + 1]);
    const int32_t aux_l = __float_as_int(f[T::kIntOff + 2]);
    const int32_t aux_r = __float_as_int(f[T::kIntOff + 3]);
    auto meets = [&](const float* lo, const float* hi) {
      bool ok = true;
#pragma unroll
      for (int k = 0; k < D; ++k) ok = ok && lo[k] <= uhi[k] && hi[k] >= ulo[k];
      return ok;
    };
    const int32_t max_l = left < 0 ? ~left : aux_l, max_r = right < 0 ? ~right : aux_r;
    const bool live_l = max_l >= min_rank && meets(f, f + D);
    const bool live_r = max_r >= min_rank && meets(f + 2 * D, f + 3 * D);
    if (live_l && !live_r && left >= 0) {
      node = left;
    } else if (live_r && !live_l && right >= 0) {
      nlo = max_l + 1;
      node = right;
    } else {
      return;
    }
  }
}

// One query per thread, started at the warp's common start node. Q provides
// begin(q) (false: no query), step(), end(), p[3], node, nlo and mask_rank
// (the query's min_rank). Starting below the root skips only nodes with a
// single live child, so the order of the query's visit calls is the same as
// from the root (the DenseBox core pass depends on that order).
template <int D, class Q>
__device__ __forceinline__ void run_query_warpstart(int64_t m, Q& qp,
                                                    const float4* __restrict__ nodes,
                                                    const BallTest& bt) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const bool valid = q < m && qp.begin(q);
  int32_t node, nlo;
  warp_start_node<D>(nodes, qp.p, valid, bt, valid ? qp.mask_rank : 0, node, nlo);
  if (valid) {
    qp.node = node;
    qp.nlo = nlo;
    while (qp.step()) {
    }
    qp.end();
  }
}

// The whole query on one thread.
template <int D, typename Visit>
__device__ __forceinline__ void bvh_query(const float4* __restrict__ nodes, const float* p,
                                          const BallTest& bt, int32_t min_rank, Visit& visit) {
  int32_t stack[kStackDepth];
  int top = 0;
  int32_t node = 0;
  while (bvh_step<D>(nodes, p, bt, min_rank, node, top, stack, visit)) {
  }
}


// Device view of a built tree.
struct DeviceBvh {
  int32_t num_leaves = 0;
  float4* nodes = nullptr;        // num_leaves - 1 nodes (root at 0) + 1 spare slot,
                                  // NodeTraits<D>::kVec float4 each
  int32_t* leaf_order = nullptr;  // leaf rank -> primitive index (sorted values)
};

}  // namespace tcb
