// FDBSCAN main phase, one WARP per leaf bucket (dbscan.cpp:60-88 semantics).
//
// The per-point masked query (one thread, one query) spends most of its time
// walking tree nodes, and its lanes diverge: in HACC-like data a halo point
// meets hundreds of neighbours while a background point meets none.
// Here the unit of work is a bucket Q — a maximal subtree of <= kMainBucket
// leaves, i.e. a run of consecutive Morton ranks — handled by one warp with
// one query point per lane:
//   1. pairs inside Q (rank order, each once) via warp shuffles;
//   2. a single bottom-up masked traversal for the whole bucket: climb from
//      Q's node, and at each ancestor reached from its left explore the right
//      sibling (all ranks > Q's) with the box-box test dist(Q box, box) <= eps;
//      stop at the first ancestor whose Morton cell contains Q's box grown by
//      eps (see bvh.cuh). Exploration is warp-cooperative: up to 32 pending
//      subtrees expand at once, one per lane, from a per-warp stack in smem;
//   3. every candidate bucket C (all ranks > Q's) met on the way is swept
//      point by point: each C point is loaded once (broadcast) and tested by
//      all lanes against their own query point, the exact fp64 predicate
//      deciding (fp32 guard band first).
// Every unordered within-eps pair is met exactly once (inside a bucket, or
// from the bucket holding its lower rank), so pair_resolutions is exact; each
// pair is resolved on the spot with the lock-free union-find. The box-box
// pruning is conservative under rounding: per axis the box gap is <= the
// point gap of any pair in the two boxes and every rounding step is monotone.
#include <cmath>

#include "device_common.cuh"
#include "pipeline.hpp"
#include "primitives.cuh"

namespace tcb {

namespace {

constexpr int kWarpsPerBlock = 4;
constexpr int kStackCap = 1024;     // int2 entries per warp
constexpr int kParallelLimit = 768; // above this, expand one subtree at a time

struct WarpSmem {
  int2 stack[kStackCap];  // {node, other end of its leaf range}
  int2 cand[2 * kWarp];   // candidate runs {lo, hi}
};

template <int D>
__device__ __forceinline__ bool box_box_hits(const float* alo, const float* ahi, const float* blo,
                                             const float* bhi, const BallTest& bt) {
  if (bt.fast) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      float d = fmaxf(fmaxf(__fsub_rn(blo[k], ahi[k]), __fsub_rn(alo[k], bhi[k])), 0.f);
      s = __fadd_rn(s, __fmul_rn(d, d));
    }
    if (s < bt.lo_f) return true;
    if (s > bt.hi_f) return false;
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    double d = 0.0;
    if (blo[k] > ahi[k])
      d = __dsub_rn(static_cast<double>(blo[k]), static_cast<double>(ahi[k]));
    else if (alo[k] > bhi[k])
      d = __dsub_rn(static_cast<double>(alo[k]), static_cast<double>(bhi[k]));
    s = __dadd_rn(s, __dmul_rn(d, d));
  }
  return s <= bt.r2;
}

// Largest common-prefix length at which an ancestor's Morton cell contains
// the box [lo, hi] grown by `reach`; anchor lies in the bucket (hence in every
// ancestor's cell). Same construction as morton_stop_delta (bvh.cuh).
template <int D>
__device__ __forceinline__ int box_stop_delta(const float* lo, const float* hi, double reach,
                                              const float* anchor,
                                              const uint32_t* __restrict__ scene_ord) {
  constexpr int B = D == 2 ? 31 : 21;
  constexpr uint64_t cells = 1ull << B;
  const double cells_d = static_cast<double>(cells);
  const double e = reach * (1.0 + 0x1.0p-20);
  int agree[3];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const float slo = ord2f(__ldg(scene_ord + k));
    const float shi = ord2f(__ldg(scene_ord + 3 + k));
    const double w = __dsub_rn(static_cast<double>(shi), static_cast<double>(slo));
    if (w <= 0.0) {
      agree[k] = B;
      continue;
    }
    const double l = static_cast<double>(lo[k]), h = static_cast<double>(hi[k]);
    const uint64_t qa = quantize(anchor[k], slo, w, cells_d, cells);
    const uint64_t ql = quantize_d(l - e - (fabs(l) + e) * 0x1.0p-50, slo, w, cells_d, cells);
    const uint64_t qh = quantize_d(h + e + (fabs(h) + e) * 0x1.0p-50, slo, w, cells_d, cells);
    const uint32_t x = static_cast<uint32_t>((ql ^ qa) | (qh ^ qa));
    agree[k] = x == 0 ? B : __clz(static_cast<int>(x)) - (32 - B);
  }
  int dmax;
  if (D == 3)
    dmax = min(min(3 * agree[2], 3 * agree[1] + 1), min(3 * agree[0] + 2, 63));
  else
    dmax = min(min(2 * agree[1], 2 * agree[0] + 1), 62);
  return dmax + (64 - D * B);
}

template <int D>
__device__ __forceinline__ void load_node(const float4* __restrict__ nodes, int32_t X, float* f) {
  using T = NodeTraits<D>;
  const float4* src = nodes + static_cast<int64_t>(X) * T::kVec;
#pragma unroll
  for (int v = 0; v < T::kVec; ++v) {
    const float4 q = __ldg(src + v);
    f[4 * v + 0] = q.x;
    f[4 * v + 1] = q.y;
    f[4 * v + 2] = q.z;
    f[4 * v + 3] = q.w;
  }
}

// Per-lane query state (one point of the bucket per lane).
template <int D, bool kForceCore>
struct Lane {
  float p[3];
  int32_t i, hint;
  bool valid, core_i, settled;
  unsigned long long pairs;

  __device__ __forceinline__ void pair(int32_t j, const uint8_t* flags, int32_t* parent) {
    ++pairs;
    if (kForceCore)
      uf_unite_hinted(parent, i, j, hint);  // every pair is core-core (dbscan.hpp:85-89)
    else
      resolve_pair(i, j, core_i, flags, parent, hint, settled);
  }
};

// All lanes test their query point against the run [lo, hi] (<= 32 points):
// the run is loaded once, coalesced, one point per lane, then broadcast by
// shuffles, so no memory latency sits inside the test loop.
template <int D, bool kForceCore>
__device__ __forceinline__ void sweep(Lane<D, kForceCore>& L, const float4* __restrict__ leaf_pt,
                                      int32_t lo, int32_t hi, const BallTest& bt,
                                      const uint8_t* flags, int32_t* parent) {
  const int lane = threadIdx.x & 31;
  const int nc = hi - lo + 1;
  float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
  if (lane < nc) c = __ldg(leaf_pt + lo + lane);
#pragma unroll 1
  for (int t = 0; t < nc; ++t) {
    const float qp[3] = {__shfl_sync(0xffffffffu, c.x, t), __shfl_sync(0xffffffffu, c.y, t),
                         __shfl_sync(0xffffffffu, c.z, t)};
    const int32_t j = __shfl_sync(0xffffffffu, __float_as_int(c.w), t);
    if (L.valid && ball_hits<D>(L.p, qp, qp, bt)) L.pair(j, flags, parent);
  }
}

template <int D, bool kForceCore>
__global__ void __launch_bounds__(kWarpsPerBlock * kWarp)
k_fd_main_warp(const float4* __restrict__ nodes, const float4* __restrict__ leaf_pt,
               const int4* __restrict__ node_info, const int32_t* __restrict__ leaf_up,
               const int32_t* __restrict__ bucket, const int32_t* __restrict__ heads,
               const int32_t* __restrict__ num_buckets, const uint32_t* __restrict__ scene_ord,
               BallTest bt, double eps, const uint8_t* __restrict__ flags,
               int32_t* __restrict__ parent, DevCounters* ctr) {
  __shared__ WarpSmem smem_all[kWarpsPerBlock];
  using T = NodeTraits<D>;
  const int lane = threadIdx.x & 31;
  WarpSmem& S = smem_all[threadIdx.x >> 5];
  const int32_t nb = *num_buckets;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  Lane<D, kForceCore> L;
  L.pairs = 0;

  for (int64_t b = warp0; b < nb; b += nwarps) {
    const int32_t lo = __ldg(heads + b), hi = __ldg(heads + b + 1) - 1;
    const int nq = hi - lo + 1;
    L.valid = lane < nq;
    float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
    if (L.valid) q = __ldg(leaf_pt + lo + lane);
    L.p[0] = q.x;
    L.p[1] = q.y;
    L.p[2] = q.z;
    L.i = __float_as_int(q.w);
    L.hint = L.i;
    L.settled = false;
    L.core_i = kForceCore ? true : (L.valid && flags[L.i] != 0);

    // ---- bucket box and pairs inside the bucket ----
    float qlo[3], qhi[3];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      float a = L.valid ? L.p[k] : INFINITY, c = L.valid ? L.p[k] : -INFINITY;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a = fminf(a, __shfl_xor_sync(0xffffffffu, a, o));
        c = fmaxf(c, __shfl_xor_sync(0xffffffffu, c, o));
      }
      qlo[k] = a;
      qhi[k] = c;
    }
#pragma unroll 1
    for (int t = 1; t < nq; ++t) {
      float4 o;
      o.x = __shfl_sync(0xffffffffu, q.x, (lane + t) & 31);
      o.y = __shfl_sync(0xffffffffu, q.y, (lane + t) & 31);
      o.z = __shfl_sync(0xffffffffu, q.z, (lane + t) & 31);
      o.w = __shfl_sync(0xffffffffu, q.w, (lane + t) & 31);
      const float op[3] = {o.x, o.y, o.z};
      if (lane + t < nq && ball_hits<D>(L.p, op, op, bt)) L.pair(__float_as_int(o.w), flags, parent);
    }

    // ---- bottom-up traversal of the bucket (uniform across the warp) ----
    float anchor[3];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const float a0 = __shfl_sync(0xffffffffu, L.p[k], 0);
      anchor[k] = __fmul_rn(0.5f, __fadd_rn(a0, a0));
    }
    const int stop = box_stop_delta<D>(qlo, qhi, eps, anchor, scene_ord);
    const int32_t bn = __ldg(bucket + lo);
    int32_t up;
    bool climb = true;
    if (bn >= 0) {
      const int4 info = __ldg(node_info + bn);
      up = info.x;
      climb = info.y > stop;
    } else {
      up = __ldg(leaf_up + ~bn);
    }
    while (climb) {
      const int32_t P = up_parent(up);
      if (P == kNoParent) break;
      const int4 infoP = __ldg(node_info + P);
      if (up_is_left(up)) {  // the right sibling holds only ranks > Q's
        float f[T::kFloats];
        load_node<D>(nodes, P, f);
        if (box_box_hits<D>(qlo, qhi, f + 2 * D, f + 3 * D, bt)) {
          const int32_t right = __float_as_int(f[T::kIntOff + 1]);
          int top = 0;
          if (right < 0) {
            sweep(L, leaf_pt, ~right, ~right, bt, flags, parent);
          } else if (infoP.w - right + 1 <= kMainBucket) {
            sweep(L, leaf_pt, right, infoP.w, bt, flags, parent);
          } else {
            if (lane == 0) S.stack[0] = make_int2(right, infoP.w);
            top = 1;
            __syncwarp();
          }
          // ---- warp-cooperative exploration of the right sibling ----
          while (top > 0) {
            const int npop = top > kParallelLimit ? 1 : min(top, kWarp);
            int2 e = make_int2(0, 0);
            if (lane < npop) e = S.stack[top - 1 - lane];
            __syncwarp();
            top -= npop;
            int2 push[2], cand[2];
            int np = 0, nc = 0;
            if (lane < npop) {
              const int32_t elo = min(e.x, e.y), ehi = max(e.x, e.y);
              float g[T::kFloats];
              load_node<D>(nodes, e.x, g);
              const int32_t l = __float_as_int(g[T::kIntOff + 0]);
              const int32_t r = __float_as_int(g[T::kIntOff + 1]);
              const int32_t gamma = l < 0 ? ~l : l;
              if (box_box_hits<D>(qlo, qhi, g, g + D, bt)) {  // left child: [elo, gamma]
                if (l < 0)
                  cand[nc++] = make_int2(gamma, gamma);
                else if (gamma - elo + 1 <= kMainBucket)
                  cand[nc++] = make_int2(elo, gamma);
                else
                  push[np++] = make_int2(l, elo);
              }
              if (box_box_hits<D>(qlo, qhi, g + 2 * D, g + 3 * D, bt)) {  // right: [gamma+1, ehi]
                if (r < 0)
                  cand[nc++] = make_int2(gamma + 1, gamma + 1);
                else if (ehi - gamma <= kMainBucket)
                  cand[nc++] = make_int2(gamma + 1, ehi);
                else
                  push[np++] = make_int2(r, ehi);
              }
            }
            // warp-wide append of pushes and candidates
            int np_pre = np, nc_pre = nc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int a = __shfl_up_sync(0xffffffffu, np_pre, o);
              const int c = __shfl_up_sync(0xffffffffu, nc_pre, o);
              if (lane >= o) {
                np_pre += a;
                nc_pre += c;
              }
            }
            const int np_tot = __shfl_sync(0xffffffffu, np_pre, 31);
            const int nc_tot = __shfl_sync(0xffffffffu, nc_pre, 31);
            np_pre -= np;
            nc_pre -= nc;
            for (int k = 0; k < np; ++k) S.stack[top + np_pre + k] = push[k];
            for (int k = 0; k < nc; ++k) S.cand[nc_pre + k] = cand[k];
            __syncwarp();
            top += np_tot;
#pragma unroll 1
            for (int k = 0; k < nc_tot; ++k) {
              const int2 c = S.cand[k];
              sweep(L, leaf_pt, c.x, c.y, bt, flags, parent);
            }
            __syncwarp();
          }
        }
      }
      if (infoP.y <= stop) break;
      up = infoP.x;
    }
  }
  unsigned long long v = warp_sum(L.pairs);
  if (lane == 0 && v) {
    atomicAdd(&ctr->pairs, v);
    atomicAdd(&ctr->dists, v);
  }
}

// head flags of the bucket runs (bucket[] is constant along a run)
__global__ void __launch_bounds__(256)
k_bucket_heads(const int32_t* __restrict__ bucket, int64_t m, int32_t* __restrict__ head) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < m;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    head[r] = (r == 0 || bucket[r] != bucket[r - 1]) ? 1 : 0;
}

__global__ void __launch_bounds__(256)
k_bucket_list(const int32_t* __restrict__ head, const int32_t* __restrict__ head_excl, int64_t m,
              const int32_t* __restrict__ total, int32_t* __restrict__ heads) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < m;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (head[r]) heads[head_excl[r]] = static_cast<int32_t>(r);
    if (r == 0) heads[*total] = static_cast<int32_t>(m);
  }
}

}  // namespace

template <int D>
void fdbscan_main_pass_warp(const BuiltBvh& b, int64_t n, double eps2, bool force_core,
                            uint8_t* flags, int32_t* parent, DevCounters* d_ctr,
                            Scratch& scratch) {
  cudaStream_t s = scratch.stream();
  // bucket runs -> list of run heads (+ sentinel), all on the device
  int32_t* head = scratch.alloc_n<int32_t>(n);
  int32_t* head_excl = scratch.alloc_n<int32_t>(n);
  int32_t* heads = scratch.alloc_n<int32_t>(n + 1);
  int32_t* total = scratch.alloc_n<int32_t>(1);
  void* scan_tmp = scratch.alloc(scan_scratch_bytes(n));
  note_launch(), k_bucket_heads<<<grid_for(n, 256), 256, 0, s>>>(b.bucket, n, head);
  exclusive_scan_i32(head, head_excl, n, total, scan_tmp, s);
  note_launch(), k_bucket_list<<<grid_for(n, 256), 256, 0, s>>>(head, head_excl, n, total, heads);

  const BallTest bt = BallTest::make(eps2);
  const double eps = std::sqrt(eps2);  // exact: eps2 is the square of an fp32 value
  auto launch = [&](auto kernel) {
    note_launch(), kernel<<<persistent_grid(kernel, kWarpsPerBlock * kWarp),
                            kWarpsPerBlock * kWarp, 0, s>>>(
        b.tree.nodes, b.leaf_pt, b.node_info, b.leaf_up, b.bucket, heads, total, b.scene_ord, bt,
        eps, flags, parent, d_ctr);
  };
  if (force_core)
    launch(k_fd_main_warp<D, true>);
  else
    launch(k_fd_main_warp<D, false>);
  TCB_CUDA(cudaGetLastError());
}

template void fdbscan_main_pass_warp<2>(const BuiltBvh&, int64_t, double, bool, uint8_t*,
                                        int32_t*, DevCounters*, Scratch&);
template void fdbscan_main_pass_warp<3>(const BuiltBvh&, int64_t, double, bool, uint8_t*,
                                        int32_t*, DevCounters*, Scratch&);

}  // namespace tcb
