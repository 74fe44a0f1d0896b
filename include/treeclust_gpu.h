/* treeclust_gpu.h — additive entry points of the B200 engine.
 *
 * Nothing here changes the reference ABI in treeclust.h; these are new symbols
 * a GPU-aware caller may use on top of it:
 *
 *   tcg_cluster_device   the tc_cluster pipeline on DEVICE-resident buffers:
 *                        coords already in HBM, labels / core flags written to
 *                        HBM, launched on the caller's stream. This is the
 *                        "from the moment the data is in device memory" timing
 *                        point of the paper.
 *   tcg_generate_*       the HACC-like and taxi-like benchmark generators
 *                         that the reference does not ship.
 *   tcg_shard_*          host-side pieces of the Morton-range multi-GPU path
 *                        (SURVEY.md §8e); the collectives are driven by the
 *                        caller's torch.distributed / NCCL communicator.
 */
#ifndef TREECLUST_GPU_H
#define TREECLUST_GPU_H

#include "treeclust.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Library / device information: the CUDA device count (0 when no usable
 * device / driver) and the library version string. */
int tcg_device_count(void);
const char* tcg_version(void);

/* Device-resident clustering.
 *   d_coords : n*dim fp32, row-major, device pointer (read only)
 *   d_labels : n int32, device pointer (written)
 *   d_core   : n uint8, device pointer (written)
 *   stream   : cudaStream_t to launch on (NULL = legacy default stream)
 *   stats    : may be NULL. When non-NULL the call synchronizes the stream at
 *              the end to read counters and stage times back.
 * The call is stream-ordered. FDBSCAN with stats == NULL never synchronizes
 * the host: the radix-sort passes are planned on the device from the AND / OR
 * of the Morton keys, the rare fallback sort (an equal-prefix group longer
 * than 256 points) is launched guarded and runs only when the device asks
 * for it, and a non-finite coordinate is detected on the device — the run
 * then does no traversal work and writes every label -1 / core flag 0 (with
 * stats != NULL, or through tcg_cluster_device_async's status word, the call
 * reports TC_ERR_INVALID_ARGUMENT). Such a call can be captured into a CUDA
 * graph (capture mode relaxed or thread-local) and replayed. DenseBox still
 * reads back the grid's finiteness / overflow check (TC_ERR_INVALID_ARGUMENT)
 * and the cell and primitive counts (stream synchronizations), and brute
 * force its non-finite flag. Scratch comes from the library's stream-ordered
 * memory pool (tcg_set_pool_release_threshold) and is released before return
 * (inside a captured graph: by the graph's own free nodes). */
tc_status tcg_cluster_device(const float* d_coords, int64_t n, int dim,
                             float eps, int minpts, tc_algorithm algorithm,
                             int64_t oracle_cap, int32_t* d_labels,
                             uint8_t* d_core, void* stream,
                             tc_cluster_stats* stats);

/* tcg_cluster_device with stats == NULL and the run's status written on the
 * device: *d_status (device int32, may be NULL) becomes TC_OK, or
 * TC_ERR_INVALID_ARGUMENT when a coordinate is non-finite (FDBSCAN; the
 * outputs are then all noise). Argument errors known on the host are still
 * returned directly. For FDBSCAN the call never synchronizes the host and is
 * capturable into a CUDA graph; on a capturing stream any other algorithm
 * (and tcg_cluster_device with stats) returns TC_ERR_INVALID_ARGUMENT before
 * enqueuing anything, so the capture stays valid. */
tc_status tcg_cluster_device_async(const float* d_coords, int64_t n, int dim, float eps,
                                   int minpts, tc_algorithm algorithm, int64_t oracle_cap,
                                   int32_t* d_labels, uint8_t* d_core, void* stream,
                                   int32_t* d_status);

/* Multi-GPU clustering of a host dataset: the points are
 * sharded by Morton range over num_devices shards, shard s on CUDA device
 * devices[s] (a device may be listed more than once); each shard receives
 * the eps halo of its neighbours (peer copies over NVLink), clusters its own
 * + ghost points, and the cross-shard unions are merged with min-id hooking.
 * Same output contract as tc_cluster (REF treeclust.h:82-92): core flags,
 * noise and core labels (minimum core index of the cluster) equal
 * tc_cluster's, every border label a valid adjacent cluster. FDBSCAN and
 * DenseBox give the same clustering (the shards run the point pipeline);
 * brute force is not sharded (TC_ERR_INVALID_ARGUMENT). Stats: counts and
 * wall-clock phases (build = partition + halo, main = local runs, finalize =
 * merge + relabel); pair_resolutions / distance_evaluations are 0. */
tc_status tcg_cluster_multi(const tc_dataset* ds, float eps, int minpts, tc_algorithm algorithm,
                            const int* devices, int num_devices, tc_result** out);

/* FDBSCAN with caller keys: d_keys[i] is a unique non-negative int32 key of
 * point i (e.g. its global id across shards; a negative key could collide
 * with the noise label -1 and is rejected with TC_ERR_INVALID_ARGUMENT after
 * one device check and synchronization); clusters are represented by the key of their
 * minimum-key core, so d_labels[i] = that key (or -1 for noise). With keys
 * 0..n-1 this is tcg_cluster_device(FDBSCAN). Used by the sharded path to
 * label a local (own + ghost) set directly in global ids. */
tc_status tcg_cluster_keyed_device(const float* d_coords, const int32_t* d_keys, int64_t n,
                                   int dim, float eps, int minpts, int32_t* d_labels,
                                   uint8_t* d_core, void* stream, tc_cluster_stats* stats);

/* Binary point files (the reference's .bin layout, io.cpp:106-134) straight
 * to the device: tcg_binary_info reads the header;
 * tcg_load_binary_device reads the coordinates in chunks through two
 * page-locked staging buffers, each chunk's host->device copy overlapping the
 * next read, into d_coords (n*dim floats), and synchronizes `stream`.
 * Errors as tc_dataset_load: unreadable / truncated / bad header -> TC_ERR_IO.
 * Coordinates are validated by the clustering call itself. */
tc_status tcg_binary_info(const char* path, int64_t* n, int* dim);
tc_status tcg_load_binary_device(const char* path, float* d_coords, int64_t n, int dim,
                                 void* stream);

/* Per-stage device milliseconds of the last tcg_cluster_device / tc_cluster
 * call on this host thread (the tc_cluster_stats phases split finer):
 * [0] bounds+morton  [1] sort  [2] topology+refit  [3] grid (DenseBox)
 * [4] core pass      [5] main pass  [6] finalize   [7] total.
 * Returns the number of entries written (<= cap). */
int tcg_last_stage_ms(double* out, int cap);

/* Number of kernels the last tcg_cluster_device / tc_cluster call on this
 * host thread launched (all of them are this library's own sm_100a kernels). */
int64_t tcg_last_launch_count(void);

/* ---- memory held between calls ----
 * Device scratch comes from the library's own stream-ordered pool per device
 * (the process's default CUDA pool is never modified). The pool keeps up to
 * `bytes` reserved between calls (default 24 GiB; more is returned to the
 * driver at the next synchronization). Large host buffers (datasets, results)
 * are page-locked and up to 4 GiB of them are cached for reuse.
 * tcg_release_cached_memory frees both caches now. */
tc_status tcg_set_pool_release_threshold(uint64_t bytes);
void tcg_release_cached_memory(void);

/* ---- benchmark generators (host, SplitMix64) ---- */

/* 3D HACC-like halos: n_bg uniform background points in [0,L)^3, then
 * Plummer halos until int64(halo_frac*n) halo points exist. */
tc_status tcg_generate_hacc_like(int64_t n, double box_len, double halo_frac,
                                 uint64_t seed, tc_dataset** out);
/* 2D taxi-trajectory-like points in the unit square. */
tc_status tcg_generate_taxi_like(int64_t n, uint64_t seed, tc_dataset** out);
/* The same generators writing straight into device memory (SURVEY §8f row
 * f4): d_out holds n*dim floats (lattice: side^dim*dim), work enqueued on
 * `stream` (a cudaStream_t; the HACC-like / taxi-like host passes synchronize
 * it). Output equals the host generators' above (tc_generate_blobs /
 * _uniform / _lattice: REF datagen.cpp:10-88) for the same arguments, up to
 * last-bit libm differences (see gen.cu); errors as the host generators. */
tc_status tcg_generate_blobs_device(int k, int64_t per_blob, int dim, float separation,
                                    float sigma, uint64_t seed, float* d_out, void* stream);
tc_status tcg_generate_uniform_device(int64_t n, int dim, const float* lo, const float* hi,
                                      uint64_t seed, float* d_out, void* stream);
tc_status tcg_generate_lattice_device(int64_t side, int dim, float spacing, float* d_out,
                                      void* stream);
tc_status tcg_generate_hacc_like_device(int64_t n, double box_len, double halo_frac,
                                        uint64_t seed, float* d_out, void* stream);
tc_status tcg_generate_taxi_like_device(int64_t n, uint64_t seed, float* d_out, void* stream);
/* testutil::random_instance (REF tests/test_util.hpp:27-60): returns the
 * instance's dataset and writes its eps / minpts. */
tc_status tcg_random_instance(uint64_t seed, int64_t min_n, int64_t max_n,
                              float* eps, int* minpts, tc_dataset** out);

/* ---- dataset creation (host) ---- */
/* Identical to tc_dataset_create (kept for source compatibility with earlier
 * builds): every dataset of 1 MiB or more is allocated page-locked by
 * tc_dataset_create already, so tc_cluster's host->device copy runs at full
 * PCIe / C2C rate either way. */
tc_status tcg_dataset_create_pinned(const float* coords, int64_t n, int dim,
                                    tc_dataset** out);

/* ---- device stages of the Morton-range multi-GPU path ----
 * The collectives between them are issued by the caller's communicator
 * (paper_2103_05162_b200/shard.py uses torch.distributed / NCCL). All
 * pointers named d_* are device pointers; calls are ordered on `stream`. */

/* Morton codes of n points against the GLOBAL scene box lo/hi (host arrays of
 * dim floats), the tree build's fp64 quantization (geometry.hpp:132-156). */
tc_status tcg_morton_codes_device(const float* d_coords, int64_t n, int dim, const float* lo,
                                  const float* hi, uint64_t* d_codes, void* stream);
/* d_mask[i] = 1 iff point i lies within eps of one of the num_boxes boxes
 * (d_box_lo / d_box_hi: num_boxes*dim floats): the eps-halo a peer needs. */
tc_status tcg_near_boxes_device(const float* d_coords, int64_t n, int dim, float eps,
                                const float* d_box_lo, const float* d_box_hi, int64_t num_boxes,
                                uint8_t* d_mask, void* stream);
/* Redistribution by Morton range: point i goes to owner o = the number of the
 * (ascending) num_splitters splitters <= d_codes[i] (o in [0, num_splitters]).
 * d_rows receives n rows of dim + 4 int32 words — the coordinates' bits, the
 * int64 global id, the int64 code — grouped by owner (owner 0 first; order
 * inside a group unspecified); d_counts[o] (num_splitters + 1 int64, device)
 * the rows per owner. num_splitters < 1024. One pass over the points replaces
 * the bucketize + stable sort + gathers of the all-to-all payload. */
tc_status tcg_shard_route_device(const float* d_coords, const int64_t* d_gid,
                                 const int64_t* d_codes, int64_t n, int dim,
                                 const int64_t* d_splitters, int num_splitters, int32_t* d_rows,
                                 int64_t* d_counts, void* stream);
/* The inverse of the row packing (after the all-to-all): n rows of dim + 4
 * int32 words -> d_coords (n*dim floats), d_gid (n int64) and, if not NULL,
 * d_codes (n int64), in one pass. */
tc_status tcg_shard_unpack_rows_device(const int32_t* d_rows, int64_t n, int dim, float* d_coords,
                                       int64_t* d_gid, int64_t* d_codes, void* stream);
/* Region boxes of a shard for the eps-halo: the tight boxes of the occupied
 * Morton-prefix cells of its points (the prefix length chosen so the shard's
 * code range spans at most 4096 cells). d_box_lo / d_box_hi need room for
 * 4096*dim floats; *d_num_boxes (device int64) receives the count. Every
 * point lies in one of the boxes. */
tc_status tcg_shard_region_boxes_device(const float* d_coords, const int64_t* d_codes, int64_t n,
                                        int dim, float* d_box_lo, float* d_box_hi,
                                        int64_t* d_num_boxes, void* stream);
/* d_mask[i] bit j = point i lies within eps of a box owned by peer j
 * (d_box_owner[b] in [0, 64)), from one traversal of an LBVH over all the
 * peers' boxes: every rank's halo sends in one pass. */
tc_status tcg_near_peers_device(const float* d_coords, int64_t n, int dim, float eps,
                                const float* d_box_lo, const float* d_box_hi,
                                const int32_t* d_box_owner, int64_t num_boxes, uint64_t* d_mask,
                                void* stream);
/* Exact core flags (|N_eps(i)| >= minpts, i itself included) of n points. */
tc_status tcg_core_flags_device(const float* d_coords, int64_t n, int dim, float eps, int minpts,
                                uint8_t* d_core, void* stream);
/* Main pass + finalize with caller-supplied core flags (the FDBSCAN main
 * phase, dbscan.cpp:60-88, never the minpts == 2 shortcut): labels are the
 * minimum LOCAL index of each cluster's cores, -1 for noise. stats may be NULL
 * (no synchronization then). */
tc_status tcg_cluster_given_core_device(const float* d_coords, int64_t n, int dim, float eps,
                                        const uint8_t* d_core_in, int32_t* d_labels,
                                        uint8_t* d_core_out, void* stream,
                                        tc_cluster_stats* stats);

/* Local context of one shard (own + ghost points): ONE point BVH serving the
 * core pass and, after the caller exchanged ghost flags with their owners,
 * the main pass. Labels are the key (e.g. global id) of each cluster's
 * minimum-key core, -1 for noise; d_keys must be unique and non-negative
 * (negative: TC_ERR_INVALID_ARGUMENT). All calls use the
 * stream given at creation; free the context before destroying that stream. */
typedef struct tcg_local tcg_local;
tc_status tcg_local_create(const float* d_coords, const int32_t* d_keys, int64_t n, int dim,
                           float eps, void* stream, tcg_local** out);
/* Exact core flags (fdbscan_mark_cores over the local set), input order. */
tc_status tcg_local_core_flags(tcg_local* ctx, int minpts, uint8_t* d_core);
/* Main pass + finalize with the given core flags (input order). */
tc_status tcg_local_cluster(tcg_local* ctx, const uint8_t* d_core_in, int32_t* d_labels,
                            uint8_t* d_core_out);
void tcg_local_free(tcg_local* ctx);

/* Connected components of m edges (2*m int32 endpoints in [0, n)): d_root[i]
 * = the minimum index of i's component (min-index hooking + flatten). Used
 * for the cross-shard merge of (ghost, local root) edges. */
tc_status tcg_union_edges_device(const int32_t* d_edges, int64_t m, int32_t n, int32_t* d_root,
                                 void* stream);

/* ---- device parity checker ---- */

/* check_equivalence (REF oracle.cpp:120-163) of clusterings a and b of the
 * same n points, all on the device: checks run in the reference's order and
 * *check receives the first that fails (0 pass, 1 core flags differ, 2 noise
 * sets differ, 3 core partitions differ, 4 / 5 invalid border label in a / b)
 * and *at the point index the reference's scan reports for it. Synchronizes
 * `stream`. */
tc_status tcg_check_equivalence_device(const float* d_coords, int64_t n, int dim, float eps,
                                       const int32_t* d_labels_a, const uint8_t* d_core_a,
                                       const int32_t* d_labels_b, const uint8_t* d_core_b,
                                       void* stream, int* check, int64_t* at);
/* borders_valid (REF oracle.cpp:72-116) of one clustering: *at = the smallest
 * index of a border point with no same-label core within eps, or -1. */
tc_status tcg_first_bad_border_device(const float* d_coords, int64_t n, int dim, float eps,
                                      const int32_t* d_labels, const uint8_t* d_core,
                                      void* stream, int64_t* at);

/* ---- stage probes for parity tests (each runs one device stage on host
 *      inputs and copies the result back) ---- */

/* Device LBVH of n points in the reference's node view (bvh.hpp:74-79):
 * leaf_ids[n] (leaf rank -> point), left/right/max_rank[n-1], boxes[(n-1)*6]
 * (min xyz, max xyz; unused axes 0). */
tc_status tcg_debug_point_bvh(const float* coords, int64_t n, int dim, int32_t* leaf_ids,
                              int32_t* left, int32_t* right, int32_t* max_rank, float* boxes);
/* Device radix sort of (key, index) pairs: sorted keys and source indices. */
tc_status tcg_debug_sort_pairs(const uint64_t* keys, int64_t n, uint64_t* keys_out,
                               int32_t* vals_out);
/* Concurrent device unite() over m edges (2*m ints) on n elements, then
 * flatten; parent_out[n] = representative (minimum index of the component). */
tc_status tcg_debug_union_find(const int32_t* edges, int64_t m, int32_t n, int32_t* parent_out);
/* Device build_grid (REF dense_grid.cpp:23-77, ref accessor DenseGrid): perm[n]
 * (sorted position -> point), cell_of_point[n]; when the cell count is <= cap,
 * cell_id / cell_begin / cell_end / cell_dense[cells]. *num_cells = count. */
tc_status tcg_debug_grid(const float* coords, int64_t n, int dim, float eps, int minpts,
                         int32_t* perm, int32_t* cell_of_point, uint64_t* cell_id,
                         int32_t* cell_begin, int32_t* cell_end, uint8_t* cell_dense,
                         int64_t cap, int64_t* num_cells);
/* The DenseBox tree over make_mixed_primitives (REF dense_grid.cpp:79-98,
 * bvh.cpp:10-124) in the reference's node view: per leaf rank the kind
 * (1 = DenseBox) and id (point or dense-cell index); left/right/max_rank and
 * boxes per internal node as tcg_debug_point_bvh. Filled when the leaf count
 * is <= cap; *num_leaves = leaf count. */
tc_status tcg_debug_mixed_bvh(const float* coords, int64_t n, int dim, float eps, int minpts,
                              uint8_t* leaf_kind, int32_t* leaf_id, int32_t* left,
                              int32_t* right, int32_t* max_rank, float* boxes, int64_t cap,
                              int64_t* num_leaves);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* TREECLUST_GPU_H */
