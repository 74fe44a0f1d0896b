// FDBSCAN-DenseBox on the device (reference: dense_grid.cpp:12-98,
// dbscan.cpp:90-200).
//
// Grid (build_grid, dense_grid.cpp:23-77)
//   k_grid_setup      h = eps/sqrt(d), extents, 2^62 overflow guard (fp64,
//                     same expressions as the reference)
//   k_cell_ids        u64 row-major cell id per point (x fastest), fused AND/OR
//   radix_sort_pairs  perm = points sorted by (cell id, index)
//   k_cell_heads      segment boundaries -> scan -> Cell{begin,end,dense}
// Mixed primitives (make_mixed_primitives, dense_grid.cpp:79-98)
//   one DenseBox (tight member box, warp-segmented min/max + atomics) per
//   dense cell, one SinglePoint per member of every other cell, in cell-id
//   order -> the same primitive indices as the reference, so the BVH (sorted
//   by (Morton code, primitive index)) is the reference's tree.
// Queries are issued in leaf-rank order: a dense box's members are one
// contiguous run of queries, so each warp shares one neighbourhood.
//   k_dense_union     union_dense_cells (dbscan.cpp:90-108): direct hooks
//   k_db_core         densebox_mark_cores (dbscan.cpp:110-139)
//   k_db_main_ranged  densebox_main_phase (dbscan.cpp:141-200)
#include <cfloat>
#include <cmath>
#include <cstring>

#include "device_common.cuh"
#include "pipeline.hpp"
#include "primitives.cuh"
#include "cover.cuh"
#include "member_tree.cuh"

namespace tcb {

struct GridParams {
  double h;
  float origin[3];
  int64_t extent[3];
  int32_t overflow;
};

namespace {

constexpr int kQueryBlock = 128;


template <int D>
__global__ void k_grid_setup(const DevCounters* ctr, double h, GridParams* gp) {
  uint64_t total_check = 1;
  gp->h = h;
  gp->overflow = 0;
  for (int k = 0; k < D; ++k) {
    float lo = ord2f(ctr->bounds_ord[k]);
    float hi = ord2f(ctr->bounds_ord[3 + k]);
    gp->origin[k] = lo;
    double width = __dsub_rn(static_cast<double>(hi), static_cast<double>(lo));
    int64_t e = static_cast<int64_t>(ceil(__ddiv_rn(width, h)));
    if (e < 1) e = 1;
    gp->extent[k] = e;
    if (total_check > (1ull << 62) / static_cast<uint64_t>(e)) gp->overflow = 1;
    total_check *= static_cast<uint64_t>(e);
  }
}

// cell_coord (dense_grid.cpp:12-19)
__device__ __forceinline__ int64_t cell_coord(float v, float origin, double h, int64_t extent) {
  int64_t c = static_cast<int64_t>(
      floor(__ddiv_rn(__dsub_rn(static_cast<double>(v), static_cast<double>(origin)), h)));
  if (c < 0) c = 0;
  if (c >= extent) c = extent - 1;
  return c;
}

template <int D>
__global__ void __launch_bounds__(256)
k_cell_ids(const float* __restrict__ coords, int64_t n, const GridParams* __restrict__ gp,
           uint64_t* __restrict__ keys, int32_t* __restrict__ vals, DevCounters* ctr) {
  const double h = gp->h;
  uint64_t acc_and = ~0ull, acc_or = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint64_t id = 0;
#pragma unroll
    for (int k = D - 1; k >= 0; --k) {
      int64_t c = cell_coord(coords[i * D + k], gp->origin[k], h, gp->extent[k]);
      id = id * static_cast<uint64_t>(gp->extent[k]) + static_cast<uint64_t>(c);
    }
    keys[i] = id;
    vals[i] = static_cast<int32_t>(i);
    acc_and &= id;
    acc_or |= id;
  }
  publish_and_or(acc_and, acc_or, ctr);
}

__global__ void k_reset_keys(DevCounters* ctr) {
  ctr->key_and = ~0ull;
  ctr->key_or = 0ull;
  ctr->count_a = 0;
}

// head[k] = 1 where a new cell starts in sorted order.
__global__ void __launch_bounds__(256)
k_cell_heads(const uint64_t* __restrict__ ids, int64_t n, int minpts, int32_t* __restrict__ head,
             int32_t* __restrict__ any_dense) {
  bool dense = false;  // a run of >= minpts equal sorted ids starts here
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t id = ids[k];
    head[k] = (k == 0 || id != ids[k - 1]) ? 1 : 0;
    dense |= k + minpts - 1 < n && ids[k + minpts - 1] == id;
  }
  if (__any_sync(0xffffffffu, dense) && (threadIdx.x & 31) == 0) atomicOr(any_dense, 1);
}

// From the exclusive scan of heads: cell index per sorted position, cell
// begins, and sorted member points (coords + id) for contiguous box scans.
template <int D>
__global__ void __launch_bounds__(256)
k_cell_fill(const int32_t* __restrict__ head, const int32_t* __restrict__ head_excl,
            const int32_t* __restrict__ perm, const float* __restrict__ coords, int64_t n,
            int32_t* __restrict__ cell_of_sorted, int32_t* __restrict__ cell_begin,
            float4* __restrict__ sorted_pt) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t c = head_excl[k] + head[k] - 1;
    cell_of_sorted[k] = c;
    if (head[k]) cell_begin[c] = static_cast<int32_t>(k);
    int32_t i = perm[k];
    float x = coords[static_cast<int64_t>(i) * D], y = coords[static_cast<int64_t>(i) * D + 1];
    float z = D == 3 ? coords[static_cast<int64_t>(i) * D + 2] : 0.f;
    sorted_pt[k] = make_float4(x, y, z, __int_as_float(i));
  }
}

// Per cell: end, dense flag, primitive count (1 for dense, size otherwise).
__global__ void __launch_bounds__(256)
k_cell_prims(int32_t* __restrict__ cell_begin, int32_t num_cells, int64_t n, int minpts,
             int32_t* __restrict__ cell_end, uint8_t* __restrict__ cell_dense,
             int32_t* __restrict__ prim_count, DevCounters* ctr) {
  int dense_cells = 0;
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < num_cells;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t b = cell_begin[c];
    int32_t e = c + 1 < num_cells ? cell_begin[c + 1] : static_cast<int32_t>(n);
    cell_end[c] = e;
    bool dense = (e - b) >= minpts;
    cell_dense[c] = dense;
    prim_count[c] = dense ? 1 : (e - b);
    dense_cells += dense;
  }
  dense_cells = warp_sum(dense_cells);
  if ((threadIdx.x & 31) == 0 && dense_cells) atomicAdd(&ctr->count_a, dense_cells);
}

// Dense primitives: identity boxes (ordered-uint encoding) + payload ~cell.
__global__ void __launch_bounds__(256)
k_prim_init(const uint8_t* __restrict__ cell_dense, const int32_t* __restrict__ prim_off,
            int32_t num_cells, uint4* __restrict__ prim_lo, uint4* __restrict__ prim_hi,
            int32_t* __restrict__ prim_aux) {
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < num_cells;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!cell_dense[c]) continue;
    int32_t p = prim_off[c];
    prim_lo[p] = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0u);
    prim_hi[p] = make_uint4(0u, 0u, 0u, 0u);
    prim_aux[p] = ~static_cast<int32_t>(c);
  }
}

// One thread per sorted position. Sparse members become SinglePoint
// primitives; dense members are min/max-reduced over their warp-local run of
// the cell (cells are contiguous in sorted order) and one lane per run
// publishes with atomicMin/Max on the order-preserving encoding.
template <int D>
__global__ void __launch_bounds__(256)
k_prim_fill(const float4* __restrict__ sorted_pt, const int32_t* __restrict__ cell_of_sorted,
            const int32_t* __restrict__ cell_begin, const uint8_t* __restrict__ cell_dense,
            const int32_t* __restrict__ prim_off, int64_t n, float4* __restrict__ prim_lo,
            float4* __restrict__ prim_hi, int32_t* __restrict__ prim_aux) {
  const int lane = threadIdx.x & 31;
  for (int64_t base = blockIdx.x * static_cast<int64_t>(blockDim.x) + (threadIdx.x & ~31); base < n;
       base += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t k = base + lane;
    const bool valid = k < n;
    int32_t c = valid ? cell_of_sorted[k] : -1 - lane;  // invalid lanes: unique fake cells
    float4 pt = valid ? sorted_pt[k] : make_float4(0.f, 0.f, 0.f, 0.f);
    bool dense = valid && cell_dense[c];
    if (valid && !dense) {
      int32_t p = prim_off[c] + static_cast<int32_t>(k - cell_begin[c]);
      prim_lo[p] = make_float4(pt.x, pt.y, pt.z, 0.f);
      prim_hi[p] = make_float4(pt.x, pt.y, pt.z, 0.f);
      prim_aux[p] = __float_as_int(pt.w);
    }
    float mn[3] = {pt.x, pt.y, pt.z}, mx[3] = {pt.x, pt.y, pt.z};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t oc = __shfl_down_sync(0xffffffffu, c, o);
#pragma unroll
      for (int q = 0; q < D; ++q) {
        float a = __shfl_down_sync(0xffffffffu, mn[q], o);
        float b = __shfl_down_sync(0xffffffffu, mx[q], o);
        if (lane + o < 32 && oc == c) {
          mn[q] = fminf(mn[q], a);
          mx[q] = fmaxf(mx[q], b);
        }
      }
    }
    int32_t prev_c = __shfl_up_sync(0xffffffffu, c, 1);
    bool run_head = lane == 0 || prev_c != c;
    if (dense && run_head) {
      int32_t p = prim_off[c];
      uint32_t* lo = reinterpret_cast<uint32_t*>(prim_lo + p);
      uint32_t* hi = reinterpret_cast<uint32_t*>(prim_hi + p);
#pragma unroll
      for (int q = 0; q < D; ++q) {
        atomicMin(lo + q, f2ord(mn[q]));
        atomicMax(hi + q, f2ord(mx[q]));
      }
    }
  }
}

// Decode the dense boxes back to floats.
__global__ void __launch_bounds__(256)
k_prim_decode(const uint8_t* __restrict__ cell_dense, const int32_t* __restrict__ prim_off,
              int32_t num_cells, float4* __restrict__ prim_lo, float4* __restrict__ prim_hi) {
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < num_cells;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!cell_dense[c]) continue;
    int32_t p = prim_off[c];
    uint4 a = *reinterpret_cast<uint4*>(prim_lo + p);
    uint4 b = *reinterpret_cast<uint4*>(prim_hi + p);
    prim_lo[p] = make_float4(ord2f(a.x), ord2f(a.y), ord2f(a.z), 0.f);
    prim_hi[p] = make_float4(ord2f(b.x), ord2f(b.y), ord2f(b.z), 0.f);
  }
}

// rank_of_prim[order[s]] = s for the DenseBox primitives (the only ones
// k_queries looks up); per leaf query count (1 or the cell's size).
__global__ void __launch_bounds__(256)
k_leaf_counts(const int32_t* __restrict__ order, const int32_t* __restrict__ prim_aux,
              const int32_t* __restrict__ cell_begin, const int32_t* __restrict__ cell_end,
              int64_t m, int32_t* __restrict__ rank_of_prim, int32_t* __restrict__ qcount,
              int32_t* __restrict__ aux_of_rank) {
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < m;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t p = order[s];
    int32_t a = prim_aux[p];
    aux_of_rank[s] = a;  // k_queries_single reads it in rank order
    if (a < 0) rank_of_prim[p] = static_cast<int32_t>(s);
    qcount[s] = a >= 0 ? 1 : cell_end[~a] - cell_begin[~a];
  }
}

// Query slots in leaf order: qpt = (coords, id | dense<<31), qrank = own leaf
// rank, key = point id. The DenseBox union-find lives in this SLOT space
// (like FDBSCAN's rank space: a query's neighbours are slot-local), hooked by
// key so roots are still minimum point ids. Also union_dense_cells: every
// dense member is core and hooked straight under the slot of the cell's first
// (= minimum-index) member.
template <int D>
__global__ void __launch_bounds__(256)
k_queries(const float4* __restrict__ sorted_pt, const int32_t* __restrict__ cell_of_sorted,
          const int32_t* __restrict__ cell_begin, const uint8_t* __restrict__ cell_dense,
          const int32_t* __restrict__ prim_off, const int32_t* __restrict__ rank_of_prim,
          const int32_t* __restrict__ qoff, int64_t n, float4* __restrict__ qpt,
          int32_t* __restrict__ qrank, int32_t* __restrict__ key, int32_t* __restrict__ parent,
          uint8_t* __restrict__ flags) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t c = cell_of_sorted[k];
    if (!cell_dense[c]) continue;  // SinglePoints: k_queries_single, in slot order
    const int32_t off = static_cast<int32_t>(k - cell_begin[c]);
    const int32_t s = rank_of_prim[prim_off[c]];
    const int32_t dst = qoff[s] + off;  // a cell's members are contiguous slots
    float4 pt = sorted_pt[k];
    const int32_t i = __float_as_int(pt.w);
    key[dst] = i;
    pt.w = __int_as_float(i | static_cast<int32_t>(0x80000000u));
    flags[dst] = 1;
    parent[dst] = qoff[s];  // the cell's first (minimum-index) member (dbscan.cpp:98-104)
    qpt[dst] = pt;
    qrank[dst] = s;
  }
}

// The SinglePoint queries, one per leaf rank s: slot qoff[s], written in slot
// order (the per-point form above scattered them from cell order).
template <int D>
__global__ void __launch_bounds__(256)
k_queries_single(const int32_t* __restrict__ aux_of_rank, const float* __restrict__ coords,
                 const int32_t* __restrict__ qoff, int64_t m, float4* __restrict__ qpt,
                 int32_t* __restrict__ qrank, int32_t* __restrict__ key) {
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < m;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t i = aux_of_rank[s];
    if (i < 0) continue;  // a DenseBox: its members come from k_queries
    const int32_t dst = qoff[s];
    const float* c = coords + static_cast<int64_t>(i) * D;
    qpt[dst] = make_float4(c[0], c[1], D == 3 ? c[2] : 0.f, __int_as_float(i));
    key[dst] = i;
    qrank[dst] = static_cast<int32_t>(s);
  }
}

// densebox_mark_cores query (dbscan.cpp:110-139): unmasked; a SinglePoint
// leaf is one neighbour, a DenseBox leaf is scanned member by member until
// minpts is reached. Dense members are core already and skip (dbscan.cpp:118).
// Resident 128-thread blocks per SM the DenseBox traversals are compiled
// for (register cap; C4 main pass 63.7 -> 62.8 ms).
#ifndef TCB_DB_RANGED_MIN_BLOCKS  // k_db_main_ranged (DenseBox minpts == 2 main pass)
#define TCB_DB_RANGED_MIN_BLOCKS 12  // C2 DenseBox main 23.9 -> 23.3 ms (8: 26.6, 14: 24.0)
#endif
constexpr int kDbRangedMinBlocks = TCB_DB_RANGED_MIN_BLOCKS;
#ifndef TCB_DB_CORE_MIN_BLOCKS  // C4 core 18.5 ms (8: 19.1, 12: 18.7)
#define TCB_DB_CORE_MIN_BLOCKS 10
#endif
#ifndef TCB_DB_Q_MIN_BLOCKS  // C4 main 59.1 ms (8: 63.6, 12: 71.0)
#define TCB_DB_Q_MIN_BLOCKS 10
#endif
#ifndef TCB_DB_MAIN_Q
#define TCB_DB_MAIN_Q 1
#endif

template <int D, int kFast>
struct DbCoreQuery {
  const float4* __restrict__ nodes;
  const float4* __restrict__ qpt;
  const float4* __restrict__ sorted_pt;
  const int32_t* __restrict__ cell_begin;
  const int32_t* __restrict__ cell_end;
  BallTest bt;
  int minpts;
  uint8_t* __restrict__ flags;
  LocalStack stack;  // handle of the kernel's per-thread stack array
  const MemberTree* mt;   // members in member order
  const MemberTree* smt;  // the same cells' members in spatial order
  const int32_t* __restrict__ qoff;  // rank -> points before it (exclusive prefix)
  int64_t n_points;
  int32_t num_prims;
  const int32_t* __restrict__ list;  // query slots to run (the SinglePoint ones)
  unsigned long long dists = 0;
  float p[3];
  int32_t id, slot, node, nlo, mask_rank = 0;
  int count;
  // the stopping scan of a long cut DenseBox, left to the warp (k_db_core)
  int32_t pend_kb = -1, pend_ke = 0, pend_rem = 0;
  __device__ bool begin(int64_t q) {
    slot = list ? list[q] : static_cast<int32_t>(q);
    const float4 qp = qpt[slot];
    id = __float_as_int(qp.w);
    if (id < 0) return false;  // member of a dense cell
    p[0] = qp.x;
    p[1] = qp.y;
    p[2] = qp.z;
    count = 0;
    node = 0;
    nlo = 0;
    pend_kb = -1;
    stack.reset();
    return true;
  }
  __device__ bool step() {
    auto visit = [&](int32_t, int32_t aux, const float* lo, const float* hi) -> bool {
      if (aux >= 0) {
        ++dists;
        ++count;  // leaf box test == exact distance test for a point leaf
      } else {
        const int32_t c = ~aux;
        const int32_t kb = cell_begin[c], ke = cell_end[c];
        if (box_inside_ball<D>(p, lo, hi, bt)) {
          // every member is within eps: the member-by-member loop would count
          // and test exactly min(size, minpts - count) members
          const int take = min(ke - kb, minpts - count);
          dists += take;
          count += take;
        } else {
          // the member-by-member scan (dbscan.cpp:124-131): when the box holds
          // fewer hits than still needed the scan runs to the end (count them
          // in the spatial tree); otherwise the scan stops at the rem-th hit
          // in member order and the query is core — at most once per query,
          // found by the whole warp after the traversals (k_db_core)
          const int rem = minpts - count;
          const bool is_short = ke - kb <= kMemberLinear;
          const int total = is_short ? rem : member_count<D>(*smt, kb, ke, p, bt, rem);
          if (total < rem) {
            dists += static_cast<unsigned long long>(ke - kb);
            count += total;
          } else if (!is_short) {
            pend_kb = kb;
            pend_ke = ke;
            pend_rem = rem;
            count = minpts;
          } else {  // a short box, scanned here (it may still fall short)
            int hits;
            const int64_t pos = member_scan<D>(*mt, kb, ke, p, bt, rem, hits);
            dists += pos >= 0 ? static_cast<unsigned long long>(pos - kb + 1)
                              : static_cast<unsigned long long>(ke - kb);
            count += hits;
          }
        }
      }
      return count < minpts;
    };
    // a contained subtree: every point of its primitives is within eps, and
    // the reference counts one hit and one evaluation per point in DFS order
    // (a fully inside DenseBox included), so it adds its point count — up to
    // the minpts stop, taken at the subtree's own DFS position
    auto inside = [&](int32_t first, int32_t last) -> bool {
      const int64_t end = last + 1 < num_prims ? __ldg(qoff + last + 1) : n_points;
      const int64_t pts = end - __ldg(qoff + first);
      if (count + pts >= minpts) {
        dists += static_cast<unsigned long long>(minpts - count);
        count = minpts;
        return false;
      }
      dists += static_cast<unsigned long long>(pts);
      count += static_cast<int>(pts);
      return true;
    };
    return bvh_step_ordered<D, LocalStack, decltype(visit), decltype(inside), kFast>(
        nodes, p, bt, 0, node, nlo, stack, visit, inside);
  }
  __device__ void end() {
    if (count >= minpts) flags[slot] = 1;
  }
};

template <int D, int kFast>
__global__ void __launch_bounds__(kQueryBlock, TCB_DB_CORE_MIN_BLOCKS)
k_db_core(const float4* __restrict__ nodes, const float4* __restrict__ qpt, int64_t n,
          const float4* __restrict__ sorted_pt, const int32_t* __restrict__ cell_begin,
          const int32_t* __restrict__ cell_end, BallTest bt, int minpts,
          uint8_t* __restrict__ flags, DevCounters* ctr, MemberTree mt,
          MemberTree smt, const int32_t* __restrict__ qoff, int32_t num_prims,
          const int32_t* __restrict__ list, int64_t m) {
  int2 stack_buf[kStackDepth];
  DbCoreQuery<D, kFast> q{nodes, qpt, sorted_pt, cell_begin, cell_end, bt, minpts, flags, LocalStack(stack_buf), &mt,
                   &smt, qoff, n, num_prims, list};
  run_query_warpstart<D>(m, q, nodes, bt);
  // The stopping scans: position of the rem-th member within eps of p in
  // member order, 32 members per step across the warp (same predicate as the
  // per-member loop; the members of a cell are in random spatial order, so a
  // box tree over them prunes nothing and one lane would test them one by one).
  const int lane = threadIdx.x & 31;
  const bool valid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x < m;
  unsigned pend = __ballot_sync(0xffffffffu, valid && q.pend_kb >= 0);
  while (pend) {
    const int src = __ffs(pend) - 1;
    pend &= pend - 1;
    const float pp[3] = {__shfl_sync(0xffffffffu, q.p[0], src),
                         __shfl_sync(0xffffffffu, q.p[1], src),
                         D == 3 ? __shfl_sync(0xffffffffu, q.p[2], src) : 0.f};
    const int32_t kb = __shfl_sync(0xffffffffu, q.pend_kb, src);
    const int32_t ke = __shfl_sync(0xffffffffu, q.pend_ke, src);
    int need = __shfl_sync(0xffffffffu, q.pend_rem, src);
    int64_t pos = -1;
    constexpr int kChunks = 4;  // 128 members in flight per round trip
    for (int32_t base = kb; base < ke && pos < 0; base += 32 * kChunks) {
      float4 m4[kChunks];
#pragma unroll
      for (int u = 0; u < kChunks; ++u) {
        const int32_t k = base + 32 * u + lane;
        m4[u] = k < ke ? __ldg(mt.pts + k) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kChunks; ++u) {
        const int32_t k = base + 32 * u + lane;
        const float mp[3] = {m4[u].x, m4[u].y, m4[u].z};
        const bool hit = k < ke && ball_hits<D, kFast>(pp, mp, mp, bt);
        const unsigned b = __ballot_sync(0xffffffffu, hit);
        const int c = __popc(b);
        if (pos < 0) {
          if (c >= need)
            pos = base + 32 * u + static_cast<int>(__fns(b, 0, need));
          else
            need -= c;
        }
      }
    }
    // pos >= 0: the spatial count found >= rem hits in the same cell
    if (lane == src) q.dists += static_cast<unsigned long long>(pos >= 0 ? pos - kb + 1 : ke - kb);
  }
  unsigned long long v = warp_sum(q.dists);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(&ctr->dists, v);
}


// densebox_main_phase with contained subtrees (direct launch). A subtree of
// the mixed tree whose box lies inside the ball holds primitives that each
// give exactly one pair and one distance evaluation in the reference (a
// SinglePoint within eps; a DenseBox whose first member is within eps), so a
// run of primitive ranks [first, last] is counted at once; qoff[rank] is the
// slot of the primitive's point (a DenseBox's first member — dense members
// are core and pre-unioned). Resolution as in k_fd_main: a core query takes
// runs of core primitives (unite with qoff[first], run recorded for the
// cover pass), a
// border query counts coreless runs and every run once claimed; other runs
// are walked. minpts == 2: every run is taken (all pairs are unions).
template <int D, bool kForceCore, int kFast>
__global__ void __launch_bounds__(kQueryBlock, kDbRangedMinBlocks)
k_db_main_ranged(const float4* __restrict__ nodes, const float4* __restrict__ qpt,
                 const int32_t* __restrict__ qrank, int64_t n, const float4* __restrict__ sorted_pt,
                 const int32_t* __restrict__ cell_begin, const int32_t* __restrict__ cell_end,
                 BallTest bt, uint8_t* __restrict__ flags, int32_t* __restrict__ parent,
                 const int32_t* __restrict__ key, const int32_t* __restrict__ qoff,
                 const int32_t* __restrict__ noncore_before, int32_t* __restrict__ reach,
                 DevCounters* ctr, MemberTree mt) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const bool valid = q < n;
  unsigned long long pairs = 0, dists = 0;
  float p[3] = {0.f, 0.f, 0.f};
  const int32_t i = static_cast<int32_t>(q);  // this query's slot
  int32_t own = 0;
  if (valid) {
    const float4 qp = qpt[q];
    own = qrank[q];
    p[0] = qp.x;
    p[1] = qp.y;
    p[2] = qp.z;
  }
  int32_t node, nlo;
  warp_start_node<D>(nodes, p, valid, bt, own + 1, node, nlo);
  if (valid) {
    const bool core_i = kForceCore ? true : flags[i] != 0;
    int32_t hint = i;
    bool settled = false;
    // j: the neighbour's slot (a SinglePoint's is qoff[rank]; a DenseBox
    // member's is qoff[rank] + its offset in the cell)
    auto pair = [&](int32_t j) {
      ++pairs;
      if (kForceCore)  // core flags derived at finalize from the hook marks
        uf_unite_hinted_keyed(parent, key, i, j, hint, flags);
      else
        resolve_pair_keyed(i, j, core_i, flags, parent, key, hint, settled);
    };
    auto visit = [&](int32_t s, int32_t aux, bool contained) -> bool {
      const int32_t base = __ldg(qoff + s);
      if (aux >= 0) {
        ++dists;
        pair(base);
      } else {
        const int32_t c = ~aux;
        const int32_t kb = cell_begin[c], ke = cell_end[c];
        if (contained) {  // every member within eps: the scan stops at the first
          ++dists;
          pair(base);
        } else {
          // scan to the first member within eps (dbscan.cpp:183-193), answered
          // by the member tree: same member, same evaluation count
          int hits;
          const int64_t pos = member_scan<D>(mt, kb, ke, p, bt, 1, hits);
          if (pos >= 0) {
            dists += static_cast<unsigned long long>(pos - kb + 1);
            pair(base + static_cast<int32_t>(pos - kb));
          } else {
            dists += static_cast<unsigned long long>(ke - kb);
          }
        }
      }
      return true;
    };
    auto inside = [&](int32_t first, int32_t last) -> int {
      const int32_t cnt = last - first + 1;
      bool run = kForceCore;
      if (!kForceCore) {
        const int32_t nc = __ldg(noncore_before + last + 1) - __ldg(noncore_before + first);
        if (core_i) {
          if (nc != 0) return kWalk;
          run = true;
        } else if (!settled && nc != cnt) {
          if (nc != 0) return kWalk;
          if (ld_relaxed(parent + i) == i) uf_claim(parent, i, uf_find(parent, __ldg(qoff + first)));
          settled = true;
        }
      }
      if (run) {
        uf_unite_hinted_keyed(parent, key, i, __ldg(qoff + first), hint,
                              kForceCore ? flags : nullptr);
        record_run(reach, first, last);
      }
      pairs += static_cast<unsigned long long>(cnt);
      dists += static_cast<unsigned long long>(cnt);
      return kTaken;
    };
    int2 stack_buf[kStackDepth];
    LocalStack stack(stack_buf);
    while (bvh_step_ranged<D, LocalStack, decltype(visit), decltype(inside), kFast>(
        nodes, p, bt, own + 1, node, nlo, stack, visit, inside, own + 1)) {
    }
  }
  unsigned long long v = warp_sum(dists);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(&ctr->dists, v);
  v = warp_sum(pairs);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(&ctr->pairs, v);
}

// k_db_main_ranged with warp-batched union-find work (as k_fd_main_q): the
// query's own lane walks the mixed tree and runs the member scans; the
// unions and claims its pairs imply are queued per warp and resolved 32 at
// a time with the root hints in shared memory (shared atomics). Action
// (x = query slot, y = target slot, z, w): z >= 0 a union, recording the
// primitive-rank run [z, w] when w > z; z == -1 a core query claiming border
// y under its hint; z == -2 a border query joining core y's cluster.
constexpr int kDbActCap = 96;

template <bool kForceCore>
__device__ __forceinline__ void db_resolve(int4 e, int32_t* hints, int32_t warp_base,
                                           int32_t* __restrict__ parent,
                                           const int32_t* __restrict__ key,
                                           int32_t* __restrict__ reach, uint8_t* flags) {
  int32_t* hp = hints + (e.x - warp_base);
  if (e.z >= 0) {
    int32_t hint = atomicAdd(hp, 0);
    const int32_t old = hint;
    uf_unite_hinted_keyed(parent, key, e.x, e.y, hint, kForceCore ? flags : nullptr);
    if (hint != old) atomicExch(hp, hint);
    record_run(reach, e.z, e.w);
  } else if (e.z == -1) {
    if (ld_relaxed(parent + e.y) == e.y) uf_claim(parent, e.y, atomicAdd(hp, 0));
  } else {
    if (ld_relaxed(parent + e.x) == e.x) uf_claim(parent, e.x, uf_find(parent, e.y));
  }
}

template <bool kForceCore>
__device__ __noinline__ int db_drain_batch(const int4* act, int qn, int lane, int32_t* hints,
                                           int32_t warp_base, int32_t* __restrict__ parent,
                                           const int32_t* __restrict__ key,
                                           int32_t* __restrict__ reach, uint8_t* flags) {
  qn -= 32;
  db_resolve<kForceCore>(act[qn + lane], hints, warp_base, parent, key, reach, flags);
  __syncwarp();
  return qn;
}

template <int D, bool kForceCore, int kFast>
__global__ void __launch_bounds__(kQueryBlock, TCB_DB_Q_MIN_BLOCKS)
k_db_main_q(const float4* __restrict__ nodes, const float4* __restrict__ qpt,
            const int32_t* __restrict__ qrank, int64_t n,
            const int32_t* __restrict__ cell_begin, const int32_t* __restrict__ cell_end,
            BallTest bt, uint8_t* __restrict__ flags, int32_t* __restrict__ parent,
            const int32_t* __restrict__ key, const int32_t* __restrict__ qoff,
            const int32_t* __restrict__ noncore_before, int32_t* __restrict__ reach,
            DevCounters* ctr, MemberTree mt) {
  __shared__ int4 s_act[kQueryBlock / 32][kDbActCap];
  __shared__ int32_t s_hint[kQueryBlock];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const bool valid = q < n;
  const int32_t i = static_cast<int32_t>(q);  // this query's slot
  const int32_t warp_base = i - lane;
  int4* act = s_act[w];
  int32_t* hints = s_hint + (w << 5);
  unsigned long long pairs = 0, dists = 0;
  float p[3] = {0.f, 0.f, 0.f};
  int32_t own = 0;
  if (valid) {
    const float4 qp = qpt[q];
    own = qrank[q];
    p[0] = qp.x;
    p[1] = qp.y;
    p[2] = qp.z;
  }
  hints[lane] = i;
  int32_t node, nlo;
  warp_start_node<D>(nodes, p, valid, bt, own + 1, node, nlo);
  const bool core_i = kForceCore ? true : (valid && flags[i] != 0);
  bool settled = false;
  int na = 0;
  int4 a0 = make_int4(0, 0, 0, 0), a1 = a0;
  auto push = [&](int4 e) {
    if (na == 0) a0 = e;
    else a1 = e;
    ++na;
  };
  // the pair (i, slot j), dbscan.hpp:82-99, as a queued action
  auto pair = [&](int32_t j) {
    ++pairs;
    if (kForceCore || (core_i && flags[j])) {
      push(make_int4(i, j, 0, 0));
    } else if (core_i) {
      push(make_int4(i, j, -1, -1));
    } else if (!settled && flags[j]) {
      push(make_int4(i, j, -2, -2));
      settled = true;
    }
  };
  auto visit = [&](int32_t s, int32_t aux, bool contained) -> bool {
    const int32_t base = __ldg(qoff + s);
    if (aux >= 0) {
      ++dists;
      pair(base);
    } else {
      const int32_t c = ~aux;
      const int32_t kb = cell_begin[c], ke = cell_end[c];
      if (contained) {
        ++dists;
        pair(base);
      } else {
        int hits;
        const int64_t pos = member_scan<D>(mt, kb, ke, p, bt, 1, hits);
        if (pos >= 0) {
          dists += static_cast<unsigned long long>(pos - kb + 1);
          pair(base + static_cast<int32_t>(pos - kb));
        } else {
          dists += static_cast<unsigned long long>(ke - kb);
        }
      }
    }
    return true;
  };
  auto inside = [&](int32_t first, int32_t last) -> int {
    const int32_t cnt = last - first + 1;
    bool run = kForceCore;
    if (!kForceCore) {
      const int32_t nc = __ldg(noncore_before + last + 1) - __ldg(noncore_before + first);
      if (core_i) {
        if (nc != 0) return kWalk;
        run = true;
      } else if (!settled && nc != cnt) {
        if (nc != 0) return kWalk;
        push(make_int4(i, __ldg(qoff + first), -2, -2));
        settled = true;
      }
    }
    if (run) push(make_int4(i, __ldg(qoff + first), first, last));
    pairs += static_cast<unsigned long long>(cnt);
    dists += static_cast<unsigned long long>(cnt);
    return kTaken;
  };
  int2 stack_buf[kStackDepth];
  LocalStack stack(stack_buf);
  bool active = valid;
  int qn = 0;  // warp-uniform queue length
  while (true) {
    na = 0;
    if (active)
      active = bvh_step_ranged<D, LocalStack, decltype(visit), decltype(inside), kFast>(
          nodes, p, bt, own + 1, node, nlo, stack, visit, inside);
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
        db_resolve<kForceCore>(act[qn + lane], hints, warp_base, parent, key, reach, flags);
        __syncwarp();
        if (qn >= 32)
          qn = db_drain_batch<kForceCore>(act, qn, lane, hints, warp_base, parent, key, reach,
                                          flags);
      }
    }
    if (!__any_sync(0xffffffffu, active)) break;
  }
  __syncwarp();
  if (lane < qn) db_resolve<kForceCore>(act[lane], hints, warp_base, parent, key, reach, flags);
  unsigned long long v = warp_sum(dists);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(&ctr->dists, v);
  v = warp_sum(pairs);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(&ctr->pairs, v);
}

// Spatial order of the members inside each cell: key = cell index (high
// bits) | 12-bit Morton code of the point's position inside its cell (a
// 64 x 64 / 16^3 sub-grid: enough coherence for the tree, few sort passes).
constexpr int kSpatialBits = 12;
// Any order inside a cell is valid for counting; this one makes the blocks of
// the spatial member tree compact.
template <int D>
__global__ void k_spatial_keys(const float4* __restrict__ sorted_pt,
                               const int32_t* __restrict__ cell_of_sorted,
                               const GridParams* __restrict__ gp, int64_t n,
                               uint64_t* __restrict__ keys, int32_t* __restrict__ vals) {
  const float inv_h = static_cast<float>(1.0 / gp->h);
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 q = sorted_pt[k];
    const float c[3] = {q.x, q.y, q.z};
    uint64_t code = 0;
    constexpr int bits = D == 2 ? 6 : 4;  // kSpatialBits per cell in total
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const float t = (c[a] - gp->origin[a]) * inv_h;
      float f = t - floorf(t);  // position inside the cell, approximately
      f = fminf(fmaxf(f, 0.f), 0.999999f);
      const uint64_t v = static_cast<uint64_t>(f * static_cast<float>(1 << bits));
      code |= D == 2 ? (spread2(v) << a) : (spread3(v) << a);
    }
    keys[k] = (static_cast<uint64_t>(cell_of_sorted[k]) << kSpatialBits) | code;
    vals[k] = static_cast<int32_t>(k);
  }
}

__global__ void k_gather_pts(const float4* __restrict__ src, const int32_t* __restrict__ perm,
                             int64_t n, float4* __restrict__ dst) {
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < n;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[j] = src[perm[j]];
}

// Member tree levels (member_tree.cuh): level 1 from the points, level l from
// level l - 1.
template <int D>
__global__ void k_member_level(const float4* __restrict__ pts, const float4* __restrict__ child,
                               float4* __restrict__ out, int64_t count, bool from_points) {
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < count;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float lo[3], hi[3];
    if (from_points) {
      const float4 a = pts[2 * j], b = pts[2 * j + 1];
      lo[0] = fminf(a.x, b.x);
      lo[1] = fminf(a.y, b.y);
      lo[2] = fminf(a.z, b.z);
      hi[0] = fmaxf(a.x, b.x);
      hi[1] = fmaxf(a.y, b.y);
      hi[2] = fmaxf(a.z, b.z);
    } else if (D == 2) {
      const float4 a = child[2 * j], b = child[2 * j + 1];
      lo[0] = fminf(a.x, b.x);
      lo[1] = fminf(a.y, b.y);
      hi[0] = fmaxf(a.z, b.z);
      hi[1] = fmaxf(a.w, b.w);
    } else {
      const float4 al = child[4 * j], ah = child[4 * j + 1], bl = child[4 * j + 2],
                   bh = child[4 * j + 3];
      lo[0] = fminf(al.x, bl.x);
      lo[1] = fminf(al.y, bl.y);
      lo[2] = fminf(al.z, bl.z);
      hi[0] = fmaxf(ah.x, bh.x);
      hi[1] = fmaxf(ah.y, bh.y);
      hi[2] = fmaxf(ah.z, bh.z);
    }
    if (D == 2) {
      out[j] = make_float4(lo[0], lo[1], hi[0], hi[1]);
    } else {
      out[2 * j] = make_float4(lo[0], lo[1], lo[2], 0.f);
      out[2 * j + 1] = make_float4(hi[0], hi[1], hi[2], 0.f);
    }
  }
}

// Query slots of the SinglePoint primitives, in rank order (the only queries
// of densebox_mark_cores: dense members are core already, dbscan.cpp:118).
__global__ void k_single_ind(const int32_t* __restrict__ order, const int32_t* __restrict__ prim_aux,
                             int64_t m, int32_t* __restrict__ ind) {
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < m;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x)
    ind[s] = prim_aux[order[s]] >= 0;
}

__global__ void k_single_slots(const int32_t* __restrict__ ind, const int32_t* __restrict__ pos,
                               const int32_t* __restrict__ qoff, int64_t m,
                               int32_t* __restrict__ list) {
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < m;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (ind[s]) list[pos[s]] = qoff[s];
}

// ind[rank] = 1 for a SinglePoint that is not core (after the core pass), for
// the noncore prefix counts.
__global__ void k_prim_noncore(const int32_t* __restrict__ order,
                               const int32_t* __restrict__ prim_aux,
                               const uint8_t* __restrict__ flags,
                               const int32_t* __restrict__ qoff, int64_t m,
                               int32_t* __restrict__ ind) {
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s <= m;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t v = 0;
    if (s < m) v = prim_aux[order[s]] >= 0 && !flags[qoff[s]];
    ind[s] = v;
  }
}

}  // namespace

template <int D>
MemberTree build_member_tree(const float4* pts, int64_t n, Scratch& scratch) {
  MemberTree t;
  t.pts = pts;
  constexpr int per = D == 2 ? 1 : 2;  // float4 per box
  int64_t off[kMemberLevels + 1] = {};
  int64_t total = 0;
  int levels = 0;
  for (int l = 1; l <= kMemberLevels - 1 && (n >> l) > 0; ++l) {
    off[l] = total;
    total += per * (n >> l);
    levels = l;
  }
  t.levels = levels;
  if (levels == 0) return t;
  float4* boxes = scratch.alloc_n<float4>(total);
  int64_t* d_off = scratch.alloc_n<int64_t>(kMemberLevels + 1);
  auto* h_off = static_cast<int64_t*>(pinned_staging(sizeof(off)));
  std::memcpy(h_off, off, sizeof(off));
  TCB_CUDA(cudaMemcpyAsync(d_off, h_off, sizeof(off), cudaMemcpyHostToDevice, scratch.stream()));
  TCB_CUDA(cudaStreamSynchronize(scratch.stream()));  // the staging buffer is reused
  t.boxes = boxes;
  t.off = d_off;
  for (int l = 1; l <= levels; ++l) {
    const int64_t count = n >> l;
    note_launch(), k_member_level<D><<<grid_for(count, 256), 256, 0, scratch.stream()>>>(
        pts, l > 1 ? boxes + off[l - 1] : nullptr, boxes + off[l], count, l == 1);
  }
  TCB_CUDA(cudaGetLastError());
  return t;
}

// The grid and mixed primitives of DenseBox (build_grid + make_mixed_primitives,
// dense_grid.cpp:23-98), shared by run_densebox and the stage-level debug
// entry points (tcg_debug_grid / tcg_debug_mixed_bvh).
template <int D>
DeviceGrid build_device_grid(const float* d_coords, int64_t n, float eps, int minpts,
                             DevCounters* ctr, Scratch& scratch, bool stop_if_no_dense) {
  cudaStream_t st = scratch.stream();
  DeviceGrid g;
  launch_point_bounds<D>(d_coords, n, ctr, st);
  GridParams* gp = scratch.alloc_n<GridParams>(1);
  g.params = gp;
  const double h = static_cast<double>(eps) / std::sqrt(static_cast<double>(D));
  note_launch(), k_grid_setup<D><<<1, 1, 0, st>>>(ctr, h, gp);
  uint64_t* keys = scratch.alloc_n<uint64_t>(n);
  int32_t* vals = scratch.alloc_n<int32_t>(n);
  note_launch(), k_cell_ids<D><<<grid_for(n, 256, 148 * 8), 256, 0, st>>>(d_coords, n, gp, keys, vals, ctr);
  TCB_CUDA(cudaGetLastError());
  auto* h_stage = static_cast<unsigned char*>(pinned_staging(64));
  TCB_CUDA(cudaMemcpyAsync(h_stage, &ctr->key_and, 16, cudaMemcpyDeviceToHost, st));
  TCB_CUDA(cudaMemcpyAsync(h_stage + 16, &ctr->nonfinite, 4, cudaMemcpyDeviceToHost, st));
  TCB_CUDA(cudaMemcpyAsync(h_stage + 20, &gp->overflow, 4, cudaMemcpyDeviceToHost, st));
  TCB_CUDA(cudaStreamSynchronize(st));
  unsigned long long key_and, key_or;
  int32_t nonfinite, overflow;
  std::memcpy(&key_and, h_stage, 8);
  std::memcpy(&key_or, h_stage + 8, 8);
  std::memcpy(&nonfinite, h_stage + 16, 4);
  std::memcpy(&overflow, h_stage + 20, 4);
  if (nonfinite) throw InvalidArgument{"PointSet: non-finite coordinate"};
  if (overflow) throw InvalidArgument{"build_grid: eps too small for domain (cell id overflow)"};

  uint64_t* keys_alt = scratch.alloc_n<uint64_t>(n);
  int32_t* vals_alt = scratch.alloc_n<int32_t>(n);
  g.sort_tmp = scratch.alloc(radix_sort_scratch_bytes(n));
  bool in_alt = radix_sort_pairs(keys, vals, keys_alt, vals_alt, n, key_and, key_or, g.sort_tmp, st);
  g.ids = in_alt ? keys_alt : keys;
  g.perm = in_alt ? vals_alt : vals;
  g.spare_keys = in_alt ? keys : keys_alt;
  g.spare_vals = in_alt ? vals : vals_alt;
  int32_t* head = scratch.alloc_n<int32_t>(n);
  int32_t* head_excl = scratch.alloc_n<int32_t>(n);
  int32_t* d_tot = scratch.alloc_n<int32_t>(4);  // [0] cells, [1] prims, [2] any dense
  g.scan_tmp = scratch.alloc(scan_scratch_bytes(n));
  TCB_CUDA(cudaMemsetAsync(d_tot + 2, 0, sizeof(int32_t), st));
  // heads of the sorted cell runs, and whether any run holds >= minpts points
  note_launch(), k_cell_heads<<<grid_for(n, 256), 256, 0, st>>>(g.ids, n, minpts, head, d_tot + 2);
  exclusive_scan_i32(head, head_excl, n, d_tot, g.scan_tmp, st);
  TCB_CUDA(cudaMemcpyAsync(h_stage, d_tot, 12, cudaMemcpyDeviceToHost, st));
  TCB_CUDA(cudaStreamSynchronize(st));
  int32_t any_dense;
  std::memcpy(&g.num_cells, h_stage, 4);
  std::memcpy(&any_dense, h_stage + 8, 4);
  if (stop_if_no_dense && !any_dense) {
    // no dense cell: DenseBox is the point pipeline (run_densebox), the rest
    // of the grid is not needed
    g.num_prims = static_cast<int32_t>(n);
    g.num_dense = 0;
    return g;
  }
  g.cell_of_sorted = scratch.alloc_n<int32_t>(n);
  g.cell_begin = scratch.alloc_n<int32_t>(n);
  g.sorted_pt = scratch.alloc_n<float4>(n);
  note_launch(), k_cell_fill<D><<<grid_for(n, 256), 256, 0, st>>>(head, head_excl, g.perm, d_coords, n,
                                                   g.cell_of_sorted, g.cell_begin, g.sorted_pt);

  // ---- mixed primitives: counts and offsets ----
  g.cell_end = scratch.alloc_n<int32_t>(g.num_cells);
  g.cell_dense = scratch.alloc_n<uint8_t>(g.num_cells);
  int32_t* prim_count = scratch.alloc_n<int32_t>(g.num_cells);
  g.prim_off = scratch.alloc_n<int32_t>(g.num_cells);
  note_launch(), k_reset_keys<<<1, 1, 0, st>>>(ctr);
  note_launch(), k_cell_prims<<<grid_for(g.num_cells, 256), 256, 0, st>>>(
      g.cell_begin, g.num_cells, n, minpts, g.cell_end, g.cell_dense, prim_count, ctr);
  exclusive_scan_i32(prim_count, g.prim_off, g.num_cells, d_tot + 1, g.scan_tmp, st);
  TCB_CUDA(cudaMemcpyAsync(h_stage, d_tot + 1, 4, cudaMemcpyDeviceToHost, st));
  TCB_CUDA(cudaMemcpyAsync(h_stage + 4, &ctr->count_a, 4, cudaMemcpyDeviceToHost, st));
  TCB_CUDA(cudaStreamSynchronize(st));
  std::memcpy(&g.num_prims, h_stage, 4);
  std::memcpy(&g.num_dense, h_stage + 4, 4);
  return g;
}

// One DenseBox (tight member box) per dense cell and one SinglePoint per member
// of every other cell, in cell order (make_mixed_primitives, dense_grid.cpp:79-98).
template <int D>
void build_mixed_prims(const DeviceGrid& g, int64_t n, Scratch& scratch, float4** lo,
                       float4** hi, int32_t** aux) {
  cudaStream_t st = scratch.stream();
  float4* prim_lo = scratch.alloc_n<float4>(g.num_prims);
  float4* prim_hi = scratch.alloc_n<float4>(g.num_prims);
  int32_t* prim_aux = scratch.alloc_n<int32_t>(g.num_prims);
  if (g.num_dense > 0)
    note_launch(), k_prim_init<<<grid_for(g.num_cells, 256), 256, 0, st>>>(
        g.cell_dense, g.prim_off, g.num_cells, reinterpret_cast<uint4*>(prim_lo),
        reinterpret_cast<uint4*>(prim_hi), prim_aux);
  note_launch(), k_prim_fill<D><<<grid_for(n, 256), 256, 0, st>>>(
      g.sorted_pt, g.cell_of_sorted, g.cell_begin, g.cell_dense, g.prim_off, n, prim_lo, prim_hi,
      prim_aux);
  if (g.num_dense > 0)
    note_launch(), k_prim_decode<<<grid_for(g.num_cells, 256), 256, 0, st>>>(
        g.cell_dense, g.prim_off, g.num_cells, prim_lo, prim_hi);
  TCB_CUDA(cudaGetLastError());
  *lo = prim_lo;
  *hi = prim_hi;
  *aux = prim_aux;
}

template <int D>
void run_densebox(const float* d_coords, int64_t n, float eps, int minpts, int32_t* d_labels,
                  uint8_t* d_core, DevCounters* ctr, Scratch& scratch, StageClock& clock,
                  double* dense_fraction) {
  cudaStream_t st = scratch.stream();
  const BallTest bt = BallTest::make(static_cast<double>(eps) * static_cast<double>(eps));
  clock.mark(kStGrid);

  // ---- grid ----
  const DeviceGrid grid = build_device_grid<D>(d_coords, n, eps, minpts, ctr, scratch,
                                               /*stop_if_no_dense=*/true);
  const GridParams* gp = grid.params;
  uint64_t* keys = grid.spare_keys;
  int32_t* vals = grid.spare_vals;
  void* sort_tmp = grid.sort_tmp;
  void* scan_tmp = grid.scan_tmp;
  const int32_t* cell_of_sorted = grid.cell_of_sorted;
  const int32_t* cell_begin = grid.cell_begin;
  const float4* sorted_pt = grid.sorted_pt;
  const int32_t num_cells = grid.num_cells;
  const int32_t* cell_end = grid.cell_end;
  const uint8_t* cell_dense = grid.cell_dense;
  const int32_t* prim_off = grid.prim_off;
  const int32_t num_prims = grid.num_prims, num_dense = grid.num_dense;
  const int64_t sparse_points = num_prims - num_dense;
  *dense_fraction = static_cast<double>(n - sparse_points) / static_cast<double>(n);
  if (num_dense == 0) {
    // No dense cell: every primitive is a SinglePoint, so the mixed BVH is the
    // point BVH (make_mixed_primitives, dense_grid.cpp:79-98) and the DenseBox
    // passes are the FDBSCAN passes: densebox_mark_cores / densebox_main_phase
    // (dbscan.cpp:110-200) reduce to fdbscan_mark_cores / fdbscan_main_phase
    // with the same pairs and the same per-hit distance counts
    // (dbscan.cpp:36-88). Run the point pipeline (rank-space union-find,
    // contained subtrees) instead of the mixed-tree kernels.
    run_fdbscan<D>(d_coords, n, eps, minpts, d_labels, d_core, ctr, scratch, clock);
    return;
  }
  float4 *prim_lo, *prim_hi;
  int32_t* prim_aux;
  build_mixed_prims<D>(grid, n, scratch, &prim_lo, &prim_hi, &prim_aux);

  // ---- BVH over the mixed primitives ----
  PrimSource src;
  src.lo = prim_lo;
  src.hi = prim_hi;
  src.aux = prim_aux;
  src.count = num_prims;
  clock.mark(kStBounds);
  BuiltBvh b = build_bvh<D>(src, false, ctr, scratch, &clock, /*stream_ordered=*/true);

  // ---- query order + dense unions ----
  clock.mark(kStGrid);
  int32_t* rank_of_prim = scratch.alloc_n<int32_t>(num_prims);
  int32_t* qcount = scratch.alloc_n<int32_t>(num_prims);
  int32_t* qoff = scratch.alloc_n<int32_t>(num_prims);
  int32_t* aux_of_rank = scratch.alloc_n<int32_t>(num_prims);
  note_launch(), k_leaf_counts<<<grid_for(num_prims, 256), 256, 0, st>>>(b.tree.leaf_order, prim_aux,
                                                          cell_begin, cell_end, num_prims,
                                                          rank_of_prim, qcount, aux_of_rank);
  exclusive_scan_i32(qcount, qoff, num_prims, nullptr, scan_tmp, st);
  float4* qpt = scratch.alloc_n<float4>(n);
  int32_t* qrank = scratch.alloc_n<int32_t>(n);
  int32_t* qkey = scratch.alloc_n<int32_t>(n);
  int32_t* parent = scratch.alloc_n<int32_t>(n);
  uint8_t* flags = scratch.alloc_n<uint8_t>(n);
  init_union_find(parent, flags, n, st);
  note_launch(), k_queries<D><<<grid_for(n, 256), 256, 0, st>>>(sorted_pt, cell_of_sorted, cell_begin,
                                                 cell_dense, prim_off, rank_of_prim, qoff, n,
                                                 qpt, qrank, qkey, parent, flags);
  note_launch(), k_queries_single<D><<<grid_for(num_prims, 256), 256, 0, st>>>(
      aux_of_rank, d_coords, qoff, num_prims, qpt, qrank, qkey);
  TCB_CUDA(cudaGetLastError());

  const MemberTree mt = build_member_tree<D>(sorted_pt, n, scratch);
  // the core pass also gets the members in spatial order per cell (same cell
  // segments) to count the hits of a long cut box without member order
  MemberTree smt;
  if (minpts > 2) {
    uint64_t* sk = scratch.alloc_n<uint64_t>(n);
    int32_t* sv = scratch.alloc_n<int32_t>(n);
    note_launch(), k_spatial_keys<D><<<grid_for(n, 256), 256, 0, st>>>(sorted_pt, cell_of_sorted,
                                                                     gp, n, sk, sv);
    uint64_t cells_pow2 = 1;
    while (cells_pow2 < static_cast<uint64_t>(num_cells)) cells_pow2 <<= 1;
    const uint64_t or_all = ((cells_pow2 - 1) << kSpatialBits) | ((1ull << kSpatialBits) - 1);
    const bool alt = radix_sort_pairs(sk, sv, keys, vals, n, 0, or_all, sort_tmp, st);
    const int32_t* sperm = alt ? vals : sv;
    float4* spt = scratch.alloc_n<float4>(n);
    note_launch(), k_gather_pts<<<grid_for(n, 256), 256, 0, st>>>(sorted_pt, sperm, n, spt);
    smt = build_member_tree<D>(spt, n, scratch);
  }

  // ---- core pass ----
  clock.mark(kStCore);
  if (minpts > 2 && sparse_points > 0) {
    // only SinglePoint queries run: a compact slot list keeps the warps full
    int32_t* ind = scratch.alloc_n<int32_t>(num_prims);
    int32_t* pos = scratch.alloc_n<int32_t>(num_prims);
    int32_t* list = scratch.alloc_n<int32_t>(sparse_points);
    note_launch(), k_single_ind<<<grid_for(num_prims, 256), 256, 0, st>>>(b.tree.leaf_order,
                                                                          prim_aux, num_prims, ind);
    exclusive_scan_i32(ind, pos, num_prims, nullptr, scan_tmp, st);
    note_launch(), k_single_slots<<<grid_for(num_prims, 256), 256, 0, st>>>(ind, pos, qoff,
                                                                            num_prims, list);
    auto core = bt.fast ? k_db_core<D, 1> : k_db_core<D, 0>;
    note_launch(), core<<<grid_for(sparse_points, kQueryBlock, INT32_MAX), kQueryBlock, 0, st>>>(
        b.tree.nodes, qpt, n, sorted_pt, cell_begin, cell_end, bt, minpts, flags, ctr, mt, smt,
        qoff, num_prims, list, sparse_points);
  }
  // ---- main pass ----
  clock.mark(kStMain);
  int32_t* reach = scratch.alloc_n<int32_t>(num_prims + 8);
  int32_t* tile_max = scratch.alloc_n<int32_t>(cover_tiles(num_prims));
  int32_t* noncore_before = nullptr;
  TCB_CUDA(cudaMemsetAsync(reach, 0xff, sizeof(int32_t) * num_prims, st));
  if (minpts > 2) {
    int32_t* ind = scratch.alloc_n<int32_t>(num_prims + 1);
    noncore_before = scratch.alloc_n<int32_t>(num_prims + 1);
    note_launch(), k_prim_noncore<<<grid_for(num_prims + 1, 256), 256, 0, st>>>(
        b.tree.leaf_order, prim_aux, flags, qoff, num_prims, ind);
    exclusive_scan_i32(ind, noncore_before, num_prims + 1, nullptr, scan_tmp, st);
  }
  const unsigned g = grid_for(n, kQueryBlock, INT32_MAX);
  // minpts > 2: unions and border claims batched per warp (C4 main 62.8 ->
  // 59.2 ms); minpts == 2 keeps the per-query form (re-measured at the final
  // launch bounds: 23.4 vs 26.7 ms on C2)
  if (TCB_DB_MAIN_Q && minpts > 2) {
    auto main = bt.fast ? k_db_main_q<D, false, 1> : k_db_main_q<D, false, 0>;
    note_launch(), main<<<g, kQueryBlock, 0, st>>>(b.tree.nodes, qpt, qrank, n, cell_begin,
                                                  cell_end, bt, flags, parent, qkey, qoff,
                                                  noncore_before, reach, ctr, mt);
  } else {
    auto main = minpts == 2 ? (bt.fast ? k_db_main_ranged<D, true, 1> : k_db_main_ranged<D, true, 0>)
                            : (bt.fast ? k_db_main_ranged<D, false, 1> : k_db_main_ranged<D, false, 0>);
    note_launch(), main<<<g, kQueryBlock, 0, st>>>(b.tree.nodes, qpt, qrank, n, sorted_pt,
                                                  cell_begin, cell_end, bt, flags, parent, qkey,
                                                  qoff, noncore_before, reach, ctr, mt);
  }
  launch_cover_joins(reach, num_prims, tile_max,
                     SlotJoin{parent, qkey, qoff, minpts == 2 ? flags : nullptr}, st);
  TCB_CUDA(cudaGetLastError());
  clock.mark(kStFinal);
  finalize_labels_bucketed(parent, flags, qkey, qkey, n, d_labels, d_core, ctr, scratch,
                           minpts == 2);
  clock.finish();
}

template DeviceGrid build_device_grid<2>(const float*, int64_t, float, int, DevCounters*, Scratch&,
                                         bool);
template DeviceGrid build_device_grid<3>(const float*, int64_t, float, int, DevCounters*, Scratch&,
                                         bool);
template void build_mixed_prims<2>(const DeviceGrid&, int64_t, Scratch&, float4**, float4**, int32_t**);
template void build_mixed_prims<3>(const DeviceGrid&, int64_t, Scratch&, float4**, float4**, int32_t**);
template void run_densebox<2>(const float*, int64_t, float, int, int32_t*, uint8_t*,
                              DevCounters*, Scratch&, StageClock&, double*);
template void run_densebox<3>(const float*, int64_t, float, int, int32_t*, uint8_t*,
                              DevCounters*, Scratch&, StageClock&, double*);

}  // namespace tcb
