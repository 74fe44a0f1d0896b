// Member tree: an implicit binary tree of boxes over the cell-sorted member
// array (sorted_pt), used to answer the DenseBox member scans of the
// reference exactly without testing every member.
//
// The reference scans a cut DenseBox member by member in member order,
// counting one distance evaluation per member tested:
//   main phase (dbscan.cpp:180-194): until the FIRST member within eps;
//   core pass  (dbscan.cpp:124-131): until minpts - count hits were seen.
// Both are "position of the r-th hit in [kb, ke) scanning left to right":
// the evaluations are (position - kb + 1), or (ke - kb) when fewer than r
// members hit. member_scan finds that position by a left-first descent over
// the aligned power-of-two blocks covering [kb, ke): a block whose box misses
// the ball (exact predicate) is skipped whole, a block inside the ball
// (conservative fp32 containment) counts all its members at once, a cut block
// is split. The result — position, hit count, and hence both counters and
// the member paired with — is the reference's, at O(boundary) cost instead of
// O(members).
//
// Layout: level l >= 1 holds node j = box of members [j 2^l, (j+1) 2^l) for
// every node fully inside [0, n) (floor(n / 2^l) nodes); level 0 is the
// points themselves. Boxes: 2D one float4 (lo.x, lo.y, hi.x, hi.y); 3D two
// float4 (lo.xyz, hi.xyz).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "bvh.cuh"
#include "device_common.cuh"

namespace tcb {

constexpr int kMemberLevels = 31;
constexpr int kMemberLinear = 32;  // members scanned linearly before the tree takes over

struct MemberTree {
  const float4* pts = nullptr;  // sorted_pt (x, y, z, id)
  const float4* boxes = nullptr;
  const int64_t* off = nullptr;  // device: float4 offset of level l's node 0
  int levels = 0;                // highest level built
};

template <int D>
__device__ __forceinline__ void member_box(const MemberTree& t, int l, int64_t j, float* lo,
                                           float* hi) {
  if (D == 2) {
    const float4 b = __ldg(t.boxes + __ldg(t.off + l) + j);
    lo[0] = b.x;
    lo[1] = b.y;
    hi[0] = b.z;
    hi[1] = b.w;
  } else {
    const int64_t o = __ldg(t.off + l);
    const float4 a = __ldg(t.boxes + o + 2 * j), b = __ldg(t.boxes + o + 2 * j + 1);
    lo[0] = a.x;
    lo[1] = a.y;
    lo[2] = a.z;
    hi[0] = b.x;
    hi[1] = b.y;
    hi[2] = b.z;
  }
}

// Position of the r-th member within eps of p in [a, b) scanning left to
// right (r >= 1), or -1; `hits` = hits seen up to and including it (== r), or
// all hits in [a, b) when fewer than r.
template <int D>
__device__ __forceinline__ int64_t member_scan(const MemberTree& t, int64_t a, int64_t b,
                                               const float* p, const BallTest& bt, int r,
                                               int& hits) {
  hits = 0;
  // the first members linearly (a hit is usually close when there is one),
  // the rest of a long run through the tree
  const int64_t lin_end = b - a <= kMemberLinear ? b : a + kMemberLinear;
  for (int64_t k = a; k < lin_end; ++k) {
    const float4 m4 = __ldg(t.pts + k);
    const float m[3] = {m4.x, m4.y, m4.z};
    if (ball_hits<D>(p, m, m, bt) && ++hits == r) return k;
  }
  int64_t k = lin_end;
  while (k < b) {
    int l = k == 0 ? 62 : __ffsll(static_cast<long long>(k)) - 1;  // alignment of k
    const int fit = 63 - __clzll(static_cast<long long>(b - k));    // largest block in [k, b)
    if (fit < l) l = fit;
    if (l > t.levels) l = t.levels;
    // left-first DFS of block (l, k >> l)
    int2 st[2 * kMemberLevels + 2];  // (level, index) — index fits: < 2^31 points
    int top = 0;
    st[top++] = make_int2(l, static_cast<int32_t>(k >> l));
    while (top) {
      const int2 e = st[--top];
      const int64_t j = e.y;
      if (e.x == 0) {
        const float4 m4 = __ldg(t.pts + j);
        const float m[3] = {m4.x, m4.y, m4.z};
        if (ball_hits<D>(p, m, m, bt) && ++hits == r) return j;
        continue;
      }
      float lo[3], hi[3];
      member_box<D>(t, e.x, j, lo, hi);
      const int c = ball_classify<D>(p, lo, hi, bt);
      if (c == 0) continue;
      if (c == 2) {
        const int64_t size = int64_t{1} << e.x;
        if (hits + size >= r) {
          const int64_t pos = (j << e.x) + (r - hits) - 1;
          hits = r;
          return pos;
        }
        hits += static_cast<int>(size);
        continue;
      }
      st[top++] = make_int2(e.x - 1, static_cast<int32_t>(2 * j + 1));
      st[top++] = make_int2(e.x - 1, static_cast<int32_t>(2 * j));
    }
    k += int64_t{1} << l;
  }
  return -1;
}

// Number of members of [a, b) within eps of p, counting stops at `cap`
// (returns min(hits, cap) when it stops early). Order-free: for a member tree
// over a spatially ordered copy of the members (same cell segments), where
// blocks are compact and most are skipped or counted whole.
template <int D>
__device__ __forceinline__ int member_count(const MemberTree& t, int64_t a, int64_t b,
                                            const float* p, const BallTest& bt, int cap) {
  int hits = 0;
  int64_t k = a;
  while (k < b) {
    int l = k == 0 ? 62 : __ffsll(static_cast<long long>(k)) - 1;
    const int fit = 63 - __clzll(static_cast<long long>(b - k));
    if (fit < l) l = fit;
    if (l > t.levels) l = t.levels;
    int2 st[2 * kMemberLevels + 2];
    int top = 0;
    st[top++] = make_int2(l, static_cast<int32_t>(k >> l));
    while (top) {
      const int2 e = st[--top];
      const int64_t j = e.y;
      if (e.x == 0) {
        const float4 m4 = __ldg(t.pts + j);
        const float m[3] = {m4.x, m4.y, m4.z};
        if (ball_hits<D>(p, m, m, bt) && ++hits >= cap) return hits;
        continue;
      }
      float lo[3], hi[3];
      member_box<D>(t, e.x, j, lo, hi);
      const int c = ball_classify<D>(p, lo, hi, bt);
      if (c == 0) continue;
      if (c == 2) {
        hits += 1 << e.x;
        if (hits >= cap) return hits;
        continue;
      }
      st[top++] = make_int2(e.x - 1, static_cast<int32_t>(2 * j + 1));
      st[top++] = make_int2(e.x - 1, static_cast<int32_t>(2 * j));
    }
    k += int64_t{1} << l;
  }
  return hits;
}

// Host: builds the levels over n sorted points (scratch-allocated boxes).
template <int D>
MemberTree build_member_tree(const float4* pts, int64_t n, Scratch& scratch);

}  // namespace tcb
