// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Thin extern "C" shim over the *unmodified* reference sources
// (/root/reference/proj/src, compiled in place by oracle/Makefile into
// oracle/_ref/libtreeclust_ref.so). It exposes the reference's internal C++
// building blocks that the public ABI (treeclust.h) hides, so the parity tests
// can compare our device results stage by stage:
//   - Morton codes          geometry.hpp:144-156 (morton_encode)
//   - BVH leaves / nodes    bvh.hpp:74-79 test accessors, bvh.cpp:10-124
//   - dense grid            dense_grid.cpp:23-77 (build_grid)
//   - dbscan_run + RunStats dbscan.cpp:221-284
//   - random_instance       tests/test_util.hpp:27-60
// The reference's own tc_* ABI (capi.cpp) is compiled into the same .so, so a
// test can also call the stock tc_cluster through ctypes.
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "bvh.hpp"
#include "datagen.hpp"
#include "dbscan.hpp"
#include "dense_grid.hpp"
#include "geometry.hpp"
#include "oracle.hpp"
#include "test_util.hpp"

using namespace treeclust;

extern "C" {

// Morton codes of n points against the given scene box (lo/hi: dim floats).
int ref_morton_codes(const float* coords, int64_t n, int dim, const float* lo,
                     const float* hi, uint64_t* out) {
  Aabb b;
  for (int k = 0; k < dim; ++k) {
    b.min[k] = lo[k];
    b.max[k] = hi[k];
  }
  for (int64_t i = 0; i < n; ++i) out[i] = morton_encode(coords + i * dim, b, dim);
  return 0;
}

// Point BVH (build_point_bvh): leaf ids in rank order (n), and for the n-1
// internal nodes: left, right, max_rank (int32 each) and box (6 floats:
// min[0..2], max[0..2]).
int ref_point_bvh(const float* coords, int64_t n, int dim, int32_t* leaf_ids,
                  int32_t* left, int32_t* right, int32_t* max_rank,
                  float* boxes) {
  try {
    PointSet ps(dim, std::vector<float>(coords, coords + n * dim));
    Bvh bvh = build_point_bvh(ps);
    for (int32_t r = 0; r < bvh.leaf_count(); ++r) leaf_ids[r] = bvh.leaf(r).id;
    for (int32_t i = 0; i < bvh.internal_count(); ++i) {
      left[i] = bvh.node_left(i);
      right[i] = bvh.node_right(i);
      max_rank[i] = bvh.node_max_rank(i);
      const Aabb& bx = bvh.node_box(i);
      for (int k = 0; k < 3; ++k) {
        boxes[6 * i + k] = bx.min[k];
        boxes[6 * i + 3 + k] = bx.max[k];
      }
    }
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

// Dense grid: returns cell count; fills perm (n), cell_of_point (n) and, when
// the caller's buffers are large enough (cap cells), per-cell id/begin/end/dense.
int64_t ref_build_grid(const float* coords, int64_t n, int dim, float eps,
                       int minpts, int32_t* perm, int32_t* cell_of_point,
                       uint64_t* cell_id, int32_t* cell_begin,
                       int32_t* cell_end, uint8_t* cell_dense, int64_t cap) {
  try {
    PointSet ps(dim, std::vector<float>(coords, coords + n * dim));
    DenseGrid g = build_grid(ps, eps, minpts);
    std::memcpy(perm, g.perm.data(), sizeof(int32_t) * n);
    std::memcpy(cell_of_point, g.cell_of_point.data(), sizeof(int32_t) * n);
    int64_t m = static_cast<int64_t>(g.cells.size());
    if (m <= cap) {
      for (int64_t c = 0; c < m; ++c) {
        cell_id[c] = g.cells[c].id;
        cell_begin[c] = g.cells[c].begin;
        cell_end[c] = g.cells[c].end;
        cell_dense[c] = g.cells[c].dense ? 1 : 0;
      }
    }
    return m;
  } catch (const std::invalid_argument&) {
    return -1;
  } catch (const std::exception&) {
    return -2;
  }
}

// Mixed-primitive BVH of DenseBox: leaf kinds/ids in rank order and nodes.
int64_t ref_mixed_bvh(const float* coords, int64_t n, int dim, float eps,
                      int minpts, uint8_t* leaf_kind, int32_t* leaf_id,
                      int32_t* left, int32_t* right, int32_t* max_rank,
                      float* boxes, int64_t cap) {
  try {
    PointSet ps(dim, std::vector<float>(coords, coords + n * dim));
    DenseGrid g = build_grid(ps, eps, minpts);
    Bvh bvh(make_mixed_primitives(g, ps), dim);
    int64_t m = bvh.leaf_count();
    if (m > cap) return m;
    for (int32_t r = 0; r < bvh.leaf_count(); ++r) {
      leaf_kind[r] = bvh.leaf(r).kind == Primitive::Kind::DenseBox ? 1 : 0;
      leaf_id[r] = bvh.leaf(r).id;
    }
    for (int32_t i = 0; i < bvh.internal_count(); ++i) {
      left[i] = bvh.node_left(i);
      right[i] = bvh.node_right(i);
      max_rank[i] = bvh.node_max_rank(i);
      const Aabb& bx = bvh.node_box(i);
      for (int k = 0; k < 3; ++k) {
        boxes[6 * i + k] = bx.min[k];
        boxes[6 * i + 3 + k] = bx.max[k];
      }
    }
    return m;
  } catch (const std::exception&) {
    return -1;
  }
}

// dbscan_run with RunStats. algo: 0 FDBSCAN, 1 DenseBox, 2 brute force.
// stats_out: build, pre, main, fin seconds, dense fraction (5 doubles);
// counters_out: skipped, pairs, dists, clusters, cores, noise (6 int64).
int ref_dbscan(const float* coords, int64_t n, int dim, float eps, int minpts,
               int algo, int threads, int32_t* labels, uint8_t* core,
               double* stats_out, int64_t* counters_out) {
  try {
    PointSet ps(dim, std::vector<float>(coords, coords + n * dim));
    DbscanParams params{eps, minpts};
    RunStats st;
    Clustering c;
    if (algo == 2) {
      c = dbscan_bruteforce(ps, params, INT64_MAX);
    } else {
      c = dbscan_run(ps, params, algo == 0 ? Algorithm::Fdbscan : Algorithm::DenseBox,
                     threads, &st);
    }
    std::memcpy(labels, c.label.data(), sizeof(int32_t) * n);
    std::memcpy(core, c.is_core.data(), n);
    if (stats_out) {
      stats_out[0] = st.build_seconds;
      stats_out[1] = st.preprocess_seconds;
      stats_out[2] = st.main_seconds;
      stats_out[3] = st.finalize_seconds;
      stats_out[4] = st.dense_point_fraction;
    }
    if (counters_out) {
      counters_out[0] = st.preprocess_skipped ? 1 : 0;
      counters_out[1] = static_cast<int64_t>(st.pair_resolutions);
      counters_out[2] = static_cast<int64_t>(st.distance_evaluations);
      counters_out[3] = st.cluster_count;
      counters_out[4] = st.core_count;
      counters_out[5] = st.noise_count;
    }
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const std::exception&) {
    return 5;
  }
}

// check_equivalence (oracle.cpp:120-163). Returns 1 on PASS, 0 on FAIL;
// the message is copied into msg (NUL-terminated).
int ref_check_equivalence(const float* coords, int64_t n, int dim, float eps,
                          int minpts, const int32_t* la, const uint8_t* ca,
                          const int32_t* lb, const uint8_t* cb, char* msg,
                          int64_t msg_len) {
  PointSet ps(dim, std::vector<float>(coords, coords + n * dim));
  Clustering a, b;
  a.label.assign(la, la + n);
  a.is_core.assign(ca, ca + n);
  b.label.assign(lb, lb + n);
  b.is_core.assign(cb, cb + n);
  EquivalenceReport rep = check_equivalence(a, b, ps, DbscanParams{eps, minpts});
  if (msg && msg_len > 0) {
    size_t len = std::min<size_t>(msg_len - 1, rep.message.size());
    std::memcpy(msg, rep.message.data(), len);
    msg[len] = '\0';
  }
  return rep.pass ? 1 : 0;
}

// testutil::random_instance: returns n; writes dim/eps/minpts and, when
// coords is non-null, n*dim coordinates.
int64_t ref_random_instance(uint64_t seed, int64_t min_n, int64_t max_n,
                            int* dim, float* eps, int* minpts, float* coords) {
  testutil::Instance inst = testutil::random_instance(seed, min_n, max_n);
  *dim = inst.points.dim;
  *eps = inst.params.eps;
  *minpts = inst.params.minpts;
  if (coords)
    std::memcpy(coords, inst.points.coords.data(),
                sizeof(float) * inst.points.coords.size());
  return inst.points.size();
}

}  // extern "C"
