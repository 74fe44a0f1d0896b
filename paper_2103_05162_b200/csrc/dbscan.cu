// FDBSCAN passes over the point BVH, and label finalization.
//
//   k_fd_core      fdbscan_mark_cores (dbscan.cpp:36-58): one thread per leaf
//                  rank (Morton order, so a warp's queries are spatial
//                  neighbours and walk nearly the same nodes), unmasked
//                  query from the warp's start node, early exit once minpts
//                  neighbours (self included) are seen.
//   k_fd_main_fof  fdbscan_main_phase (dbscan.cpp:60-88) for minpts == 2:
//                  rank-masked query so every unordered within-eps pair is
//                  found exactly once, each pair resolved on the spot with the
//                  lock-free union-find, contained subtrees taken as runs;
//                  no neighbour list is ever stored.
//   k_fd_main      the same for minpts > 2 (pairs resolved per
//                  dbscan.hpp:82-99 with final core flags).
//   cover.cuh      the runs' unions (max-scan over the recorded runs).
//   k_fin_*        UnionFind::flatten + finalize_labels + the stats loop
//                  (union_find.hpp:77-86, dbscan.cpp:202-219, :274-282).
//
// For point leaves the leaf box test IS the exact distance test (the box is
// degenerate and box_distance_sq reduces to distance_sq term by term, the
// subtraction merely negated), so a visited leaf is a within-eps neighbour
// and its distance is not recomputed.
#include <algorithm>
#include <cmath>

#include "device_common.cuh"
#include "pipeline.hpp"
#include "primitives.cuh"
#include "cover.cuh"

namespace tcb {

namespace {

constexpr int kQueryBlock = 128;  // 64 / 256 measured equal or slower
// Resident blocks per SM the FoF main pass is compiled for (ptxas caps its
// registers at 40): 12 x 4 warps. With the warp-batched union actions 12 is
// faster than 14 (32 registers, more spills) and 10 (C2 main 17.9 vs 19.8 /
// 18.7 ms); the per-query form measured best at 14 (18.5 ms).
#ifndef TCB_FOF_MIN_BLOCKS
#define TCB_FOF_MIN_BLOCKS 12
#endif
constexpr int kFofMinBlocks = TCB_FOF_MIN_BLOCKS;
// the same for the minpts > 2 main pass (10: main 21.7 -> 21.3 ms on C3);
// the core pass at 16 (the SM's full 64 warps, 32 registers): C3 core 10.25
// -> 9.84 ms (14: 9.85, uncapped 10.25); the queued main pass at 12 (10:
// 21.5, 14: 52.7 ms)
#ifndef TCB_MAIN_MIN_BLOCKS
#define TCB_MAIN_MIN_BLOCKS 10
#endif
constexpr int kMainMinBlocks = TCB_MAIN_MIN_BLOCKS;
#ifndef TCB_CORE_MIN_BLOCKS  // 0: uncapped
#define TCB_CORE_MIN_BLOCKS 16
#endif
constexpr int kCoreMinBlocks = TCB_CORE_MIN_BLOCKS;
#ifndef TCB_CORE_NEAR_FIRST
#define TCB_CORE_NEAR_FIRST 1
#endif
#ifndef TCB_MAIN_BATCH
#define TCB_MAIN_BATCH 1
#endif
#ifndef TCB_MAIN_CORE_LEFT_FIRST
#define TCB_MAIN_CORE_LEFT_FIRST 1
#endif

template <int D>
__device__ __forceinline__ void load_query(const float4* leaf_pt, int64_t r, float* p,
                                           int32_t* id) {
  float4 q = leaf_pt[r];
  p[0] = q.x;
  p[1] = q.y;
  if (D == 3) p[2] = q.z;
  *id = __float_as_int(q.w);
}

__device__ __forceinline__ void flush_counter(unsigned long long* dst, unsigned long long v) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

// fdbscan_mark_cores query (dbscan.cpp:36-58): unmasked, early exit once
// minpts neighbours (self included) are seen. A subtree whose box lies inside
// the ball adds its leaf count at once; when that crosses minpts the
// reference would have stopped inside it after exactly minpts - count more
// leaf hits, so the distance counter (one per hit, dists == count) is still
// the reference's.
template <int D, int kFast>
struct CoreQuery {
  const float4* __restrict__ nodes;
  const float4* __restrict__ leaf_pt;
  BallTest bt;
  int minpts;
  uint8_t* __restrict__ flags;
  LocalStack stack;  // handle of the kernel's per-thread stack array
  unsigned long long dists = 0;
  float p[3];
  int32_t id, node, nlo;
  int count;
  __device__ bool begin(int64_t r) {
    load_query<D>(leaf_pt, r, p, &id);
    id = static_cast<int32_t>(r);  // flags are kept in rank space
    count = 0;
    node = 0;
    nlo = 0;
    stack.reset();
    return true;
  }
  __device__ bool step() {
    auto visit = [&](int32_t, int32_t, bool) -> bool {
      ++dists;
      return ++count < minpts;  // early exit (dbscan.cpp:48-53)
    };
    auto inside = [&](int32_t first, int32_t last) -> int {
      const int64_t k = static_cast<int64_t>(last) - first + 1;
      if (count + k >= minpts) {
        dists += static_cast<unsigned long long>(minpts - count);
        count = minpts;
        return kStop;
      }
      dists += static_cast<unsigned long long>(k);
      count += static_cast<int>(k);
      return kTaken;
    };
    return bvh_step_ranged<D, LocalStack, decltype(visit), decltype(inside), kFast>(
        nodes, p, bt, 0, node, nlo, stack, visit, inside, TCB_CORE_NEAR_FIRST ? id : -1);
  }
  __device__ void end() {
    if (count >= minpts) flags[id] = 1;
  }
};

template <int D, int kFast>
__global__ void __launch_bounds__(kQueryBlock, kCoreMinBlocks)
k_fd_core(const float4* __restrict__ nodes, const float4* __restrict__ leaf_pt, int64_t m,
          BallTest bt, int minpts, uint8_t* __restrict__ flags, DevCounters* ctr) {
  if (ctr->nonfinite) return;  // stream-ordered run over bad input: no work
  int2 stack_buf[kStackDepth];
  CoreQuery<D, kFast> q{nodes, leaf_pt, bt, minpts, flags, LocalStack(stack_buf)};
  // one query per thread, started at the warp's common start node
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const bool valid = r < m;
  if (valid) q.begin(r);
  warp_start_node<D>(nodes, q.p, valid, bt, 0, q.node, q.nlo);
  if (valid) {
    while (q.step()) {
    }
    q.end();
  }
  flush_counter(&ctr->dists, q.dists);
}

// fdbscan_main_phase (dbscan.cpp:60-88): one thread per leaf rank r (Morton
// order, so a warp's queries are spatial neighbours walking nearly the same
// nodes), top-down query masked at r + 1 (the reference masks at r and skips
// the self leaf: the same pairs) so each unordered within-eps pair is met
// exactly once, and resolved on the spot — no neighbour list is stored.
// minpts > 2 path: core flags are final, pairs resolve per dbscan.hpp:82-99.
// Contained subtrees (every leaf of [first, last] within eps), with
// noncore_before[] prefix counts telling how many of them are borders/noise:
//   core query,   all leaves core: a run like in k_fd_main_fof (unite with
//                 `first`, record the run; the cover pass joins neighbouring
//                 ranks inside it — all cores within eps of the query);
//   border query, no core leaf or already settled (claimed): every pair is a
//                 no-op, counted only; all leaves core: claimed by the run;
//   otherwise the subtree is walked leaf by leaf (per-pair rule).
template <int D, int kFast>
__global__ void __launch_bounds__(kQueryBlock, kMainMinBlocks)
k_fd_main(const float4* __restrict__ nodes, const float4* __restrict__ leaf_pt, int64_t m,
          BallTest bt, const uint8_t* __restrict__ flags, int32_t* __restrict__ parent,
          const int32_t* __restrict__ key, const int32_t* __restrict__ noncore_before,
          int32_t* __restrict__ reach, DevCounters* ctr) {
  if (ctr->nonfinite) return;  // stream-ordered run over bad input: no work
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const bool valid = r < m;
  unsigned long long pairs = 0;
  float p[3] = {0.f, 0.f, 0.f};
  int32_t rank = 0;
  if (valid) {
    int32_t id;
    load_query<D>(leaf_pt, r, p, &id);
    rank = static_cast<int32_t>(r);
  }
  int32_t node, nlo;
  warp_start_node<D>(nodes, p, valid, bt, rank + 1, node, nlo);
  if (valid) {
    const bool core_r = flags[rank] != 0;
    int32_t hint = rank;
    bool settled = false;
    auto visit = [&](int32_t s, int32_t, bool) -> bool {
      ++pairs;
      resolve_pair_keyed(rank, s, core_r, flags, parent, key, hint, settled);
      return true;
    };
    auto inside = [&](int32_t first, int32_t last) -> int {
      const int32_t size = last - first + 1;
      const int32_t noncore = __ldg(noncore_before + last + 1) - __ldg(noncore_before + first);
      if (core_r) {
        if (noncore != 0) return kWalk;
        uf_unite_hinted_keyed(parent, key, rank, first, hint);
        record_run(reach, first, last);
      } else if (!settled && noncore != size) {
        if (noncore != 0) return kWalk;
        if (ld_relaxed(parent + rank) == rank) uf_claim(parent, rank, uf_find(parent, first));
        settled = true;
      }
      pairs += static_cast<unsigned long long>(size);
      return kTaken;
    };
    int2 stack_buf[kStackDepth];
    LocalStack stack(stack_buf);
    while (bvh_step_ranged<D, LocalStack, decltype(visit), decltype(inside), kFast>(
        nodes, p, bt, rank + 1, node, nlo, stack, visit, inside)) {
    }
  }
  flush_counter(&ctr->pairs, pairs);
  flush_counter(&ctr->dists, pairs);
}

__global__ void k_noncore_ind(const uint8_t* __restrict__ flags, int64_t n,
                              int32_t* __restrict__ ind) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i <= n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    ind[i] = i < n ? (flags[i] == 0) : 0;
}

// minpts == 2 (friends-of-friends) main pass. Every within-eps pair is a
// core-core union (dbscan.hpp:85-89), so a subtree whose whole box lies inside
// the eps-ball needs no walk: all of its unmasked leaves [first, last] are
// neighbours of r. The query unites r with `first` and records that the run
// [first, last] must be connected (reach[first] = max(reach[first], last));
// k_cover_* later unite every covered rank with its predecessor. Same final
// partition as uniting r with each leaf (each leaf is joined to r through the
// run); pairs counted per leaf, so pair_resolutions / distance_evaluations
// stay exact.
template <int D, int kFast>
__global__ void __launch_bounds__(kQueryBlock, kFofMinBlocks)
k_fd_main_fof(const float4* __restrict__ nodes, const float4* __restrict__ leaf_pt, int64_t m,
              BallTest bt, int32_t* __restrict__ parent, const int32_t* __restrict__ key,
              int32_t* __restrict__ reach, uint8_t* __restrict__ mark, DevCounters* ctr) {
  if (ctr->nonfinite) return;  // stream-ordered run over bad input: no work
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const bool valid = r < m;
  unsigned long long pairs = 0;
  TCB_PROBE_ONLY(unsigned long long pr[7] = {};)
  float p[3] = {0.f, 0.f, 0.f};
  int32_t rank = 0;
  if (valid) {
    int32_t id;
    load_query<D>(leaf_pt, r, p, &id);
    rank = static_cast<int32_t>(r);
  }
  int32_t node, nlo;
  warp_start_node<D>(nodes, p, valid, bt, rank + 1, node, nlo);
  if (valid) {
    int32_t hint = rank;
    auto visit = [&](int32_t s, int32_t, bool) -> bool {
      ++pairs;
      TCB_PROBE_ONLY(++pr[2];)
      uf_unite_hinted_keyed(parent, key, rank, s, hint, mark);
      return true;
    };
    auto inside = [&](int32_t first, int32_t last) -> int {
      pairs += static_cast<unsigned long long>(last - first + 1);
      TCB_PROBE_ONLY(++pr[1]; pr[4] += last - first + 1;)
      uf_unite_hinted_keyed(parent, key, rank, first, hint, mark);
      record_run(reach, first, last);
      return kTaken;
    };
    int2 stack_buf[kStackDepth];
    LocalStack stack(stack_buf);
    while (bvh_step_ranged<D, LocalStack, decltype(visit), decltype(inside), kFast>(
        nodes, p, bt, rank + 1, node, nlo, stack, visit, inside)) {
      TCB_PROBE_ONLY(++pr[0];)
    }
    TCB_PROBE_ONLY(++pr[0]; pr[5] += pairs == 0; pr[6] = pr[0]; if (pairs == 0) pr[3] = pr[0];)
  }
  flush_counter(&ctr->pairs, pairs);
  flush_counter(&ctr->dists, pairs);
  TCB_PROBE_ONLY(for (int k = 0; k < 6; ++k) flush_counter(&ctr->probe[k], pr[k]);
                 const unsigned wmax = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(pr[6]));
                 if ((threadIdx.x & 31) == 0) atomicAdd(&ctr->probe[6], wmax);)
}

// k_fd_main_fof with warp-batched union actions. In the per-query form a leaf
// hit or a contained run sends its lane into the union-find code on its own
// (2-3 active lanes per instruction there: a halo query meets a neighbour on
// one step in ten), so the warp pays the whole union path for each of them.
// Here a step only classifies the node's two children and appends the
// actions it found — (query rank, first, last), a leaf being first == last —
// to a per-warp queue in shared memory (ballot + popc offsets); whenever the
// queue holds 32 actions the warp resolves 32 of them at once, one per lane,
// with the query's root hint kept per query in shared memory (any value a
// hint ever held is an ancestor of the query's set, so a hint updated by
// another lane is still a valid hint). Same unions, same run records, same
// pair counts: the partition and counters are unchanged.
#ifndef TCB_FOF_BATCH
#define TCB_FOF_BATCH 1
#endif
constexpr int kActCap = 96;  // < 32 queued + up to 2 per lane per step
// The FoF pass walks, of two children, the one holding the nearest unmasked
// ranks (min_rank) first — the query's Morton neighbours are met (and
// united) first, which keeps its root hint current and the warp's lanes in
// the same subtrees: C2 main 16.4 -> 16.0 ms, C5 221 -> 214 ms (DenseBox
// minpts 2 likewise, main 26.2 -> 23.9 ms; the minpts > 2 passes measured
// slower with it and keep right-first).
#ifndef TCB_FOF_SELF_FIRST
#define TCB_FOF_SELF_FIRST 1
#endif

// The hint slots are read and written by the lanes resolving actions of the
// same query concurrently: shared-memory atomics (whichever value wins is a
// valid hint), so the accesses are race-free by the memory model.
__device__ __forceinline__ int32_t ld_shared_relaxed(int32_t* p) { return atomicAdd(p, 0); }
__device__ __forceinline__ void st_shared_relaxed(int32_t* p, int32_t v) { atomicExch(p, v); }

__device__ __forceinline__ void fof_resolve(int3 e, int32_t* hints, int32_t warp_base,
                                            int32_t* __restrict__ parent,
                                            const int32_t* __restrict__ key,
                                            int32_t* __restrict__ reach, uint8_t* mark) {
  int32_t* hp = hints + (e.x - warp_base);
  int32_t hint = ld_shared_relaxed(hp);
  const int32_t old = hint;
  uf_unite_hinted_keyed(parent, key, e.x, e.y, hint, mark);
  if (hint != old) st_shared_relaxed(hp, hint);
  record_run(reach, e.y, e.z);
}

__device__ __noinline__ int fof_drain_batch(const int3* act, int qn, int lane, int32_t* hints,
                                            int32_t warp_base, int32_t* __restrict__ parent,
                                            const int32_t* __restrict__ key,
                                            int32_t* __restrict__ reach, uint8_t* mark) {
  qn -= 32;
  fof_resolve(act[qn + lane], hints, warp_base, parent, key, reach, mark);
  __syncwarp();
  return qn;
}

template <int D, int kFast>
__global__ void __launch_bounds__(kQueryBlock, kFofMinBlocks)
k_fd_main_fof_q(const float4* __restrict__ nodes, const float4* __restrict__ leaf_pt, int64_t m,
                BallTest bt, int32_t* __restrict__ parent, const int32_t* __restrict__ key,
                int32_t* __restrict__ reach, uint8_t* __restrict__ mark, DevCounters* ctr) {
  if (ctr->nonfinite) return;  // stream-ordered run over bad input: no work
  __shared__ int3 s_act[kQueryBlock / 32][kActCap];
  __shared__ int32_t s_hint[kQueryBlock];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const bool valid = r < m;
  const int32_t rank = static_cast<int32_t>(r);
  const int32_t warp_base = rank - lane;
  int3* act = s_act[w];
  int32_t* hints = s_hint + (w << 5);
  unsigned long long pairs = 0;
  float p[3] = {0.f, 0.f, 0.f};
  if (valid) {
    int32_t id;
    load_query<D>(leaf_pt, r, p, &id);
  }
  hints[lane] = rank;
  int32_t node, nlo;
  warp_start_node<D>(nodes, p, valid, bt, rank + 1, node, nlo);
  const int32_t min_rank = rank + 1;
  // the stack top stays a register: a LocalStack member would live in local
  // memory next to its array (an extra load / store per push and pop)
  int2 stack[kStackDepth];
  int top = 0;
  bool active = valid;
  int qn = 0;  // warp-uniform queue length
  using T = NodeTraits<D>;
  while (true) {
    int na = 0;
    int32_t f0 = 0, l0 = 0, f1 = 0, l1 = 0;
    if (active) {
      float f[T::kFloats];
      load_node<D>(nodes + static_cast<int64_t>(node) * T::kVec, f);
      const int32_t left = __float_as_int(f[T::kIntOff + 0]);
      const int32_t right = __float_as_int(f[T::kIntOff + 1]);
      const int32_t aux_l = __float_as_int(f[T::kIntOff + 2]);
      const int32_t aux_r = __float_as_int(f[T::kIntOff + 3]);
      const bool leaf_l = left < 0, leaf_r = right < 0;
      const int32_t split = leaf_l ? ~left : aux_l;  // last rank of the left child
      const int32_t max_r = leaf_r ? ~right : aux_r;
      int cl = ball_classify<D, kFast>(p, f, f + D, bt);
      int cr = ball_classify<D, kFast>(p, f + 2 * D, f + 3 * D, bt);
      if (split < min_rank) cl = 0;
      if (max_r < min_rank) cr = 0;
      const bool act_l = cl > 0 && (leaf_l || cl == 2);
      const bool act_r = cr > 0 && (leaf_r || cr == 2);
      // a leaf is the run [rank, rank]; a contained child its unmasked range
      const int32_t fl = leaf_l ? ~left : (nlo > min_rank ? nlo : min_rank);
      const int32_t fr = leaf_r ? ~right : (split + 1 > min_rank ? split + 1 : min_rank);
      if (act_l) pairs += static_cast<unsigned>(split - fl + 1);
      if (act_r) pairs += static_cast<unsigned>(max_r - fr + 1);
      na = static_cast<int>(act_l) + static_cast<int>(act_r);
      f0 = act_l ? fl : fr;
      l0 = act_l ? split : max_r;
      f1 = fr;
      l1 = max_r;
      const bool go_l = cl == 1 && !leaf_l, go_r = cr == 1 && !leaf_r;
      if (go_l && go_r) {
#if TCB_FOF_SELF_FIRST
        if (split >= min_rank) {  // the left child holds the nearest unmasked ranks
          stack[top++] = make_int2(right, split + 1);
          node = left;
        } else
#endif
        {
          stack[top++] = make_int2(left, nlo);
          node = right;
          nlo = split + 1;
        }
      } else if (go_l) {
        node = left;
      } else if (go_r) {
        node = right;
        nlo = split + 1;
      } else if (top > 0) {
        const int2 e = stack[--top];
        node = e.x;
        nlo = e.y;
      } else {
        active = false;
      }
    }
    const unsigned m1 = __ballot_sync(0xffffffffu, na >= 1);
    const unsigned m2 = __ballot_sync(0xffffffffu, na == 2);
    if (m1) {
      const unsigned lt = (1u << lane) - 1u;
      const int off = qn + __popc(m1 & lt) + __popc(m2 & lt);
      if (na >= 1) act[off] = make_int3(rank, f0, l0);
      if (na == 2) act[off + 1] = make_int3(rank, f1, l1);
      qn += __popc(m1) + __popc(m2);
      // resolve down to fewer than 32 queued: a step adds up to 64, so the
      // queue (kActCap = 96) never overflows
      if (qn >= 32) {
        __syncwarp();
        qn -= 32;
        fof_resolve(act[qn + lane], hints, warp_base, parent, key, reach, mark);
        __syncwarp();
        // (rare) still 32 or more queued: one more batch, out of line so the
        // common path keeps its registers
        if (qn >= 32) qn = fof_drain_batch(act, qn, lane, hints, warp_base, parent, key, reach, mark);
      }
    }
    if (!__any_sync(0xffffffffu, active)) break;
  }
  __syncwarp();
  if (lane < qn) fof_resolve(act[lane], hints, warp_base, parent, key, reach, mark);
  flush_counter(&ctr->pairs, pairs);
  flush_counter(&ctr->dists, pairs);
}

// k_fd_main (minpts > 2) with warp-batched pair resolution, as
// k_fd_main_fof_q does for minpts == 2: a step classifies the node's two
// children for the lane's query (leaf hits, contained runs with their
// noncore prefix counts, the border query's `settled` state — all decided by
// the query's own lane, in its traversal), and queues the union-find work it
// implies — UNITE (core-core pair or all-core run), CLAIM_B (a core query
// claims a border leaf under its root hint), CLAIM_SELF (a border query
// joins the cluster of a core) — which the warp resolves 32 at a time, one
// per lane, with the queries' root hints in shared memory. Same pairs, same
// core-core unions (the partition); border claims are first-come as in the
// per-query form (any adjacent cluster, dbscan.hpp:82-99).
constexpr int kActUnite = 0, kActClaimB = 1, kActClaimSelf = 2;

__device__ __forceinline__ void main_resolve(int4 e, int32_t* hints, int32_t warp_base,
                                             int32_t* __restrict__ parent,
                                             const int32_t* __restrict__ key,
                                             int32_t* __restrict__ reach) {
  int32_t* hp = hints + (e.x - warp_base);
  if (e.w == kActUnite) {
    int32_t hint = ld_shared_relaxed(hp);
    const int32_t old = hint;
    uf_unite_hinted_keyed(parent, key, e.x, e.y, hint);
    if (hint != old) st_shared_relaxed(hp, hint);
    record_run(reach, e.y, e.z);
  } else if (e.w == kActClaimB) {
    if (ld_relaxed(parent + e.y) == e.y) uf_claim(parent, e.y, ld_shared_relaxed(hp));
  } else {
    if (ld_relaxed(parent + e.x) == e.x) uf_claim(parent, e.x, uf_find(parent, e.y));
  }
}

__device__ __noinline__ int main_drain_batch(const int4* act, int qn, int lane, int32_t* hints,
                                             int32_t warp_base, int32_t* __restrict__ parent,
                                             const int32_t* __restrict__ key,
                                             int32_t* __restrict__ reach) {
  qn -= 32;
  main_resolve(act[qn + lane], hints, warp_base, parent, key, reach);
  __syncwarp();
  return qn;
}

// 12 resident blocks (42 registers): C1 main 0.59 -> 0.55 ms, C3fd 22.2 -> 21.3 ms vs 10
#ifndef TCB_MAIN_Q_MIN_BLOCKS
#define TCB_MAIN_Q_MIN_BLOCKS 12
#endif
constexpr int kMainQMinBlocks = TCB_MAIN_Q_MIN_BLOCKS;

template <int D, int kFast>
__global__ void __launch_bounds__(kQueryBlock, kMainQMinBlocks)
k_fd_main_q(const float4* __restrict__ nodes, const float4* __restrict__ leaf_pt, int64_t m,
            BallTest bt, const uint8_t* __restrict__ flags, int32_t* __restrict__ parent,
            const int32_t* __restrict__ key, const int32_t* __restrict__ noncore_before,
            int32_t* __restrict__ reach, DevCounters* ctr) {
  if (ctr->nonfinite) return;  // stream-ordered run over bad input: no work
  __shared__ int4 s_act[kQueryBlock / 32][kActCap];
  __shared__ int32_t s_hint[kQueryBlock];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const bool valid = r < m;
  const int32_t rank = static_cast<int32_t>(r);
  const int32_t warp_base = rank - lane;
  int4* act = s_act[w];
  int32_t* hints = s_hint + (w << 5);
  unsigned long long pairs = 0;
  float p[3] = {0.f, 0.f, 0.f};
  bool core_r = false;
  if (valid) {
    int32_t id;
    load_query<D>(leaf_pt, r, p, &id);
    core_r = flags[rank] != 0;
  }
  bool settled = false;
  hints[lane] = rank;
  int32_t node, nlo;
  warp_start_node<D>(nodes, p, valid, bt, rank + 1, node, nlo);
  const int32_t min_rank = rank + 1;
  int2 stack[kStackDepth];
  int top = 0;
  bool active = valid;
  int qn = 0;  // warp-uniform queue length
  using T = NodeTraits<D>;
  while (true) {
    int na = 0;
    int4 a0 = make_int4(0, 0, 0, 0), a1 = a0;
    if (active) {
      float f[T::kFloats];
      load_node<D>(nodes + static_cast<int64_t>(node) * T::kVec, f);
      const int32_t left = __float_as_int(f[T::kIntOff + 0]);
      const int32_t right = __float_as_int(f[T::kIntOff + 1]);
      const int32_t aux_l = __float_as_int(f[T::kIntOff + 2]);
      const int32_t aux_r = __float_as_int(f[T::kIntOff + 3]);
      const bool leaf_l = left < 0, leaf_r = right < 0;
      const int32_t split = leaf_l ? ~left : aux_l;  // last rank of the left child
      const int32_t max_r = leaf_r ? ~right : aux_r;
      int cl = ball_classify<D, kFast>(p, f, f + D, bt);
      int cr = ball_classify<D, kFast>(p, f + 2 * D, f + 3 * D, bt);
      if (split < min_rank) cl = 0;
      if (max_r < min_rank) cr = 0;
      // one child: a leaf hit or a contained run -> at most one action;
      // returns the classification left for the descent (1 = walk it)
      auto child = [&](bool leaf, int32_t first, int32_t last, int c) -> int {
        if (c == 0 || (!leaf && c == 1)) return c;
        int4 e = make_int4(rank, first, last, -1);
        if (leaf) {
          ++pairs;
          if (core_r) {
            e.w = flags[first] ? kActUnite : kActClaimB;
          } else if (!settled && flags[first]) {
            e.w = kActClaimSelf;
            settled = true;
          }
        } else {
          const int32_t size = last - first + 1;
          const int32_t noncore = __ldg(noncore_before + last + 1) - __ldg(noncore_before + first);
          if (core_r) {
            if (noncore != 0) return 1;  // mixed: walk it leaf by leaf
            e.w = kActUnite;
          } else if (!settled && noncore != size) {
            if (noncore != 0) return 1;
            e.w = kActClaimSelf;
            settled = true;
          }
          pairs += static_cast<unsigned long long>(size);
        }
        if (e.w >= 0) {
          if (na == 0) a0 = e;
          else a1 = e;
          ++na;
        }
        return 0;  // taken
      };
      const int32_t fl = leaf_l ? ~left : (nlo > min_rank ? nlo : min_rank);
      const int32_t fr = leaf_r ? ~right : (split + 1 > min_rank ? split + 1 : min_rank);
      cl = child(leaf_l, fl, split, cl);
      cr = child(leaf_r, fr, max_r, cr);
      const bool go_l = cl == 1 && !leaf_l, go_r = cr == 1 && !leaf_r;
      if (go_l && go_r) {
#if TCB_MAIN_CORE_LEFT_FIRST
        if (core_r) {  // core queries: ascending ranks first
          stack[top++] = make_int2(right, split + 1);
          node = left;
        } else
#endif
        {  // (left-first for every query measured slower: C3 main 21.2 -> 21.6 ms)
          stack[top++] = make_int2(left, nlo);
          node = right;
          nlo = split + 1;
        }
      } else if (go_l) {
        node = left;
      } else if (go_r) {
        node = right;
        nlo = split + 1;
      } else if (top > 0) {
        const int2 e = stack[--top];
        node = e.x;
        nlo = e.y;
      } else {
        active = false;
      }
    }
    const unsigned m1 = __ballot_sync(0xffffffffu, na >= 1);
    if (m1) {
      const unsigned m2 = __ballot_sync(0xffffffffu, na == 2);
      const unsigned lt = (1u << lane) - 1u;
      const int off = qn + __popc(m1 & lt) + __popc(m2 & lt);
      if (na >= 1) act[off] = a0;
      if (na == 2) act[off + 1] = a1;
      qn += __popc(m1) + __popc(m2);
      if (qn >= 32) {
        __syncwarp();
        qn -= 32;
        main_resolve(act[qn + lane], hints, warp_base, parent, key, reach);
        __syncwarp();
        if (qn >= 32) qn = main_drain_batch(act, qn, lane, hints, warp_base, parent, key, reach);
      }
    }
    if (!__any_sync(0xffffffffu, active)) break;
  }
  __syncwarp();
  if (lane < qn) main_resolve(act[lane], hints, warp_base, parent, key, reach);
  flush_counter(&ctr->pairs, pairs);
  flush_counter(&ctr->dists, pairs);
}

__global__ void k_permute(const uint8_t* __restrict__ src, const int32_t* __restrict__ order,
                          int64_t n, uint8_t* __restrict__ dst, bool to_rank) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (to_rank)
      dst[r] = src[order[r]];
    else
      dst[order[r]] = src[r];
  }
}

__global__ void k_gather_keys(const int32_t* __restrict__ keys, const int32_t* __restrict__ order,
                              int64_t n, int32_t* __restrict__ out) {
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < n;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[s] = keys[order[s]];
}

__global__ void k_key_min(const int32_t* __restrict__ keys, int64_t n, int32_t* out) {
  int32_t m = INT32_MAX;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    m = min(m, __ldg(keys + i));
  m = __reduce_min_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0 && m < 0) atomicMin(out, m);
}

__global__ void k_init_uf(int32_t* __restrict__ parent, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    parent[i] = static_cast<int32_t>(i);
}

// Rank-space finalize (FDBSCAN): flatten over ranks (union_find.hpp:77-86,
// dbscan.cpp:202-219); the representative of a set is its minimum-key rank,
// so label = key[root] = minimum original index. The outputs go to input
// order through a
// permutation, and 4-byte / 1-byte stores to random positions are partial
// sector writes that DRAM pays for one by one. Pass 1 (rank order) finalizes
// each rank and files an entry (destination | core <<
// 31, label) into the bucket of its destination: buckets are 2^shift
// consecutive output positions, and since the destinations are a
// permutation bucket b holds exactly its window's size, so it owns entries
// [b << shift, ...) with a per-bucket cursor and no histogram pass. A block's
// entries for one bucket are consecutive (a per-block shared count, one
// global atomic per bucket). Pass 2 walks the entries in bucket order: its
// label / core stores stay inside a few small windows at a time, so L2 merges
// them into whole sectors.
constexpr int kFinThreads = 1024;
constexpr int kFinItems = 8;
constexpr int kFinMaxBuckets = 4096;
// large inputs: up to this many buckets (dynamic shared counters) so that the
// windows still fit pass 2's shared memory (497M points: 15168 windows of 32K)
constexpr int kFinMaxBucketsLarge = 16384;
#ifndef TCB_FIN_BATCHED
#define TCB_FIN_BATCHED 1
#endif

// 2 resident blocks (32 registers, a few entries spilled to L1): 0.69 -> 0.60 ms on C2
__global__ void __launch_bounds__(kFinThreads, 2)
k_fin_bucket(int32_t* __restrict__ parent, const uint8_t* __restrict__ flags,
             const int32_t* __restrict__ key, const int32_t* __restrict__ order, int64_t n,
             int shift, int nb, uint32_t* __restrict__ cursor, uint2* __restrict__ entries,
             DevCounters* ctr, bool derive_core) {
  extern __shared__ uint32_t s_cnt[];  // nb counters
  for (int b = threadIdx.x; b < nb; b += kFinThreads) s_cnt[b] = 0;
  __syncthreads();
  long long noise = 0, clusters = 0, cores = 0;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * (kFinThreads * kFinItems);
  uint2 e[kFinItems];
  uint32_t loc[kFinItems];
#if TCB_FIN_BATCHED
  // The union-find is final here; the only writes are path compressions to
  // roots, and a root's own entry never changes, so plain (batchable) loads
  // are safe: any value an entry held is an ancestor and every chase ends at
  // the true root. The first two levels of all items are loaded together.
  int32_t pr[kFinItems], qr[kFinItems];
#pragma unroll
  for (int j = 0; j < kFinItems; ++j) {
    const int64_t s = base + j * kFinThreads + threadIdx.x;
    pr[j] = s < n ? parent[s] : 0;
  }
#pragma unroll
  for (int j = 0; j < kFinItems; ++j) qr[j] = parent[pr[j]];
#endif
#pragma unroll
  for (int j = 0; j < kFinItems; ++j) {
    const int64_t s = base + j * kFinThreads + threadIdx.x;
    e[j].x = 0xffffffffu;
    if (s < n) {
#if TCB_FIN_BATCHED
      int32_t p = pr[j], q = qr[j];
      while (p != q) {
        p = q;
        q = parent[p];
      }
      if (p != pr[j]) parent[s] = p;
#else
      int32_t p = ld_relaxed(parent + s);
      int32_t q;
      while (p != (q = ld_relaxed(parent + p))) p = q;
      st_relaxed(parent + s, p);
#endif
      const bool core = flags[s] != 0 || (derive_core && p != s);
      const int32_t lab = (core || p != s) ? __ldg(key + p) : -1;  // dbscan.cpp:215
      noise += lab == -1;
      clusters += lab != -1 && p == s;
      cores += core;
      // destination < 2^31 - 1 (n <= INT32_MAX), so its bit 31 carries the
      // core flag and 0xffffffff marks an empty slot
      const uint32_t i = static_cast<uint32_t>(__ldg(order + s));
      e[j] = make_uint2(i | (core ? 0x80000000u : 0u), static_cast<uint32_t>(lab));
      loc[j] = atomicAdd(&s_cnt[i >> shift], 1u);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += kFinThreads)
    if (s_cnt[b]) s_cnt[b] = atomicAdd(cursor + b, s_cnt[b]);
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kFinItems; ++j) {
    if (e[j].x == 0xffffffffu) continue;
    const uint32_t b = (e[j].x & 0x7fffffffu) >> shift;
    entries[(static_cast<int64_t>(b) << shift) + s_cnt[b] + loc[j]] = e[j];
  }
  noise = warp_sum(noise);
  clusters = warp_sum(clusters);
  cores = warp_sum(cores);
  if ((threadIdx.x & 31) == 0) {
    if (noise) atomicAdd(reinterpret_cast<unsigned long long*>(&ctr->noise), noise);
    if (clusters) atomicAdd(reinterpret_cast<unsigned long long*>(&ctr->clusters), clusters);
    if (cores) atomicAdd(reinterpret_cast<unsigned long long*>(&ctr->cores), cores);
  }
}

// Pass 2 for windows of at most kFinWindow outputs: block b gathers bucket b's
// entries into shared memory and writes its window out coalesced.
constexpr int kFinWindow = 32768;

__global__ void __launch_bounds__(kFinThreads)
k_fin_window(const uint2* __restrict__ entries, int64_t n, int shift, int b0,
             int32_t* __restrict__ labels, uint8_t* __restrict__ core_out, bool vec16) {
  extern __shared__ __align__(16) unsigned char fin_smem[];
  int32_t* s_lab = reinterpret_cast<int32_t*>(fin_smem);
  uint8_t* s_core = fin_smem + sizeof(int32_t) * kFinWindow;
  const int64_t base = static_cast<int64_t>(b0 + blockIdx.x) << shift;
  const int64_t rest = n - base;
  const int cnt = static_cast<int>(rest < (int64_t{1} << shift) ? rest : (int64_t{1} << shift));
  for (int k = threadIdx.x; k < cnt; k += kFinThreads) {
    const uint2 v = __ldcs(entries + base + k);
    const int w = static_cast<int>((v.x & 0x7fffffffu) - base);
    s_lab[w] = static_cast<int32_t>(v.y);
    s_core[w] = static_cast<uint8_t>(v.x >> 31);
  }
  __syncthreads();
  if (vec16 && cnt == (1 << shift)) {  // full window: 16-byte stores (16-aligned outputs)
    int4* dl = reinterpret_cast<int4*>(labels + base);
    const int4* sl = reinterpret_cast<const int4*>(s_lab);
    for (int k = threadIdx.x; k < cnt / 4; k += kFinThreads) __stcs(dl + k, sl[k]);
    int4* dc = reinterpret_cast<int4*>(core_out + base);
    const int4* sc = reinterpret_cast<const int4*>(s_core);
    for (int k = threadIdx.x; k < cnt / 16; k += kFinThreads) __stcs(dc + k, sc[k]);
  } else {
    for (int k = threadIdx.x; k < cnt; k += kFinThreads) {
      labels[base + k] = s_lab[k];
      core_out[base + k] = s_core[k];
    }
  }
}

__global__ void __launch_bounds__(256)
k_fin_scatter(const uint2* __restrict__ entries, int64_t e0, int64_t e1,
              int32_t* __restrict__ labels, uint8_t* __restrict__ core_out) {
  for (int64_t k = e0 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < e1;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint2 v = __ldcs(entries + k);
    const uint32_t i = v.x & 0x7fffffffu;
    labels[i] = static_cast<int32_t>(v.y);
    core_out[i] = static_cast<uint8_t>(v.x >> 31);
  }
}

}  // namespace

template <int D>
void fdbscan_core_pass(const BuiltBvh& b, int64_t n, double eps2, int minpts,
                       uint8_t* flags, DevCounters* d_ctr, cudaStream_t s) {
  const BallTest bt = BallTest::make(eps2);
  auto core = bt.fast ? k_fd_core<D, 1> : k_fd_core<D, 0>;
  note_launch(), core<<<grid_for(n, kQueryBlock, INT32_MAX), kQueryBlock, 0, s>>>(
      b.tree.nodes, b.leaf_pt, n, bt, minpts, flags, d_ctr);
  TCB_CUDA(cudaGetLastError());
}

template <int D>
void fdbscan_main_pass(const BuiltBvh& b, const int32_t* key, int64_t n, double eps2,
                       bool force_core, uint8_t* flags, int32_t* parent, DevCounters* d_ctr,
                       Scratch& scratch) {
  cudaStream_t s = scratch.stream();
  const BallTest bt = BallTest::make(eps2);
  const unsigned grid = grid_for(n, kQueryBlock, INT32_MAX);
  int32_t* reach = scratch.alloc_n<int32_t>(n + cover_detail::kCoverItems);
  int32_t* tile_max = scratch.alloc_n<int32_t>(cover_tiles(n));
  TCB_CUDA(cudaMemsetAsync(reach, 0xff, static_cast<size_t>(n) * sizeof(int32_t), s));
  if (force_core) {
    auto fof = TCB_FOF_BATCH ? (bt.fast ? k_fd_main_fof_q<D, 1> : k_fd_main_fof_q<D, 0>)
                             : (bt.fast ? k_fd_main_fof<D, 1> : k_fd_main_fof<D, 0>);
    note_launch(), fof<<<grid, kQueryBlock, 0, s>>>(b.tree.nodes, b.leaf_pt, n, bt, parent, key,
                                                   reach, flags, d_ctr);
  } else {
    int32_t* ind = scratch.alloc_n<int32_t>(n + 1);
    int32_t* noncore_before = scratch.alloc_n<int32_t>(n + 1);
    void* scan_tmp = scratch.alloc(scan_scratch_bytes(n + 1));
    note_launch(), k_noncore_ind<<<grid_for(n + 1, 256), 256, 0, s>>>(flags, n, ind);
    exclusive_scan_i32(ind, noncore_before, n + 1, nullptr, scan_tmp, s);
    auto main = TCB_MAIN_BATCH ? (bt.fast ? k_fd_main_q<D, 1> : k_fd_main_q<D, 0>)
                               : (bt.fast ? k_fd_main<D, 1> : k_fd_main<D, 0>);
    note_launch(), main<<<grid, kQueryBlock, 0, s>>>(b.tree.nodes, b.leaf_pt, n, bt, flags, parent,
                                                    key, noncore_before, reach, d_ctr);
  }
  // covered runs (all-core): join each covered rank to its predecessor
  launch_cover_joins(reach, n, tile_max, KeyedJoin{parent, key, force_core ? flags : nullptr}, s);
  TCB_CUDA(cudaGetLastError());
}

void permute_flags(const uint8_t* src, const int32_t* order, int64_t n, uint8_t* dst, bool to_rank,
                   cudaStream_t s) {
  note_launch(), k_permute<<<grid_for(n, 256), 256, 0, s>>>(src, order, n, dst, to_rank);
  TCB_CUDA(cudaGetLastError());
}

void gather_rank_keys(const int32_t* keys, const int32_t* order, int64_t n, int32_t* out,
                      cudaStream_t s) {
  note_launch(), k_gather_keys<<<grid_for(n, 256), 256, 0, s>>>(keys, order, n, out);
  TCB_CUDA(cudaGetLastError());
}

void check_keys_nonnegative(const int32_t* keys, int64_t n, Scratch& scratch) {
  cudaStream_t s = scratch.stream();
  int32_t* d_min = scratch.alloc_n<int32_t>(1);
  TCB_CUDA(cudaMemsetAsync(d_min, 0, sizeof(int32_t), s));
  note_launch(), k_key_min<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(keys, n, d_min);
  TCB_CUDA(cudaGetLastError());
  auto* h = static_cast<int32_t*>(pinned_staging(sizeof(int32_t)));
  TCB_CUDA(cudaMemcpyAsync(h, d_min, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  TCB_CUDA(cudaStreamSynchronize(s));
  // a negative key could label a cluster -1, the noise sentinel
  if (*h < 0) throw InvalidArgument{"keys must be non-negative"};
}

void init_union_find(int32_t* parent, uint8_t* flags, int64_t n, cudaStream_t s) {
  note_launch(), k_init_uf<<<grid_for(n, 256), 256, 0, s>>>(parent, n);
  TCB_CUDA(cudaMemsetAsync(flags, 0, static_cast<size_t>(n), s));
  TCB_CUDA(cudaGetLastError());
}


void finalize_labels_bucketed(int32_t* parent, uint8_t* flags, const int32_t* key,
                              const int32_t* order, int64_t n, int32_t* labels,
                              uint8_t* core_out, DevCounters* d_ctr, Scratch& scratch,
                              bool force_core, const ChunkSink* sink) {
  cudaStream_t s = scratch.stream();
  // <= 2048 windows (>= 4 entries per block and bucket in pass 1), but up to
  // 4096 when that keeps the windows within shared memory (pass 2)
  int shift = 12;
  while (((n + (int64_t{1} << shift) - 1) >> shift) > kFinMaxBuckets / 2) ++shift;
  if (shift > 15 && ((n + (int64_t{1} << 15) - 1) >> 15) <= kFinMaxBucketsLarge) shift = 15;
  while (((n + (int64_t{1} << shift) - 1) >> shift) > kFinMaxBucketsLarge) ++shift;
  const int nb = static_cast<int>((n + (int64_t{1} << shift) - 1) >> shift);
  uint32_t* cursor = scratch.alloc_n<uint32_t>(nb);
  uint2* entries = scratch.alloc_n<uint2>(n);
  TCB_CUDA(cudaMemsetAsync(cursor, 0, sizeof(uint32_t) * nb, s));
  const int64_t tile = int64_t{kFinThreads} * kFinItems;
  // caller buffers (e.g. a torch slice) need not be 16-byte aligned: the
  // window pass then writes element by element
  const bool vec16 = (reinterpret_cast<uintptr_t>(labels) | reinterpret_cast<uintptr_t>(core_out)) % 16 == 0;
  const size_t cnt_bytes = sizeof(uint32_t) * static_cast<size_t>(nb);
  if (cnt_bytes > 48 * 1024)
    TCB_CUDA(cudaFuncSetAttribute(k_fin_bucket, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(cnt_bytes)));
  note_launch(), k_fin_bucket<<<static_cast<unsigned>((n + tile - 1) / tile), kFinThreads,
                                 cnt_bytes, s>>>(parent, flags, key, order, n, shift, nb, cursor,
                                                 entries, d_ctr, force_core);
  TCB_CUDA(cudaGetLastError());
  // pass 2, in chunks of whole buckets when a sink copies finished output
  // ranges to the host while the next chunk is written
  const int chunks = sink && n >= (int64_t{1} << 22) ? 8 : 1;
  const int per = (nb + chunks - 1) / chunks;
  for (int b0 = 0; b0 < nb; b0 += per) {
    const int64_t e0 = static_cast<int64_t>(b0) << shift;
    const int64_t e1 = std::min<int64_t>(static_cast<int64_t>(b0 + per) << shift, n);
    if ((1 << shift) <= kFinWindow) {
      constexpr size_t smem = (sizeof(int32_t) + 1) * kFinWindow;
      TCB_CUDA(cudaFuncSetAttribute(k_fin_window, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
      const int blocks = std::min(per, nb - b0);
      note_launch(), k_fin_window<<<blocks, kFinThreads, smem, s>>>(entries, n, shift, b0, labels,
                                                                   core_out, vec16);
    } else {  // wide windows: stores straight to global (L2 still merges a window)
      note_launch(), k_fin_scatter<<<grid_for(e1 - e0, 256), 256, 0, s>>>(entries, e0, e1, labels,
                                                                         core_out);
    }
    TCB_CUDA(cudaGetLastError());
    if (sink) (*sink)(e0, e1, s);
  }
}



template void fdbscan_core_pass<2>(const BuiltBvh&, int64_t, double, int, uint8_t*,
                                   DevCounters*, cudaStream_t);
template void fdbscan_core_pass<3>(const BuiltBvh&, int64_t, double, int, uint8_t*,
                                   DevCounters*, cudaStream_t);
template void fdbscan_main_pass<2>(const BuiltBvh&, const int32_t*, int64_t, double, bool,
                                   uint8_t*, int32_t*, DevCounters*, Scratch&);
template void fdbscan_main_pass<3>(const BuiltBvh&, const int32_t*, int64_t, double, bool,
                                   uint8_t*, int32_t*, DevCounters*, Scratch&);

}  // namespace tcb
