/* A plain C caller of the drop-in ABI: compiled against include/treeclust.h
 * only and linked to libtreeclust_b200.so, exactly as a reference caller
 * (REF tools/treeclust_cli.cpp, tests/test_capi.cpp) would be. Run by
 * tests/test_c_client.py.
 *
 *   capi_client layout   prints sizeof / offsetof of tc_cluster_stats and the
 *                        enum values (pinned against the ctypes mirror)
 *   capi_client host     ABI checks that need no device (REF
 *                        test_capi.cpp:25-101: datasets, generators, file
 *                        round trip, argument errors)
 *   capi_client device   REF test_capi.cpp:103-150: the three algorithms give
 *                        identical labels and 3 clusters on
 *                        blobs(3, 80, 2, 20, 0.5, 21); the brute-force cap;
 *                        tc_verify PASS; tcg_cluster_multi (two shards) equal
 *                        to tc_cluster
 * Exit status 0 = every check passed. */
#include <stddef.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "treeclust.h"
#include "treeclust_gpu.h"

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

static int layout(void) {
  printf("sizeof %zu\n", sizeof(tc_cluster_stats));
  printf("build_seconds %zu\n", offsetof(tc_cluster_stats, build_seconds));
  printf("preprocess_seconds %zu\n", offsetof(tc_cluster_stats, preprocess_seconds));
  printf("main_seconds %zu\n", offsetof(tc_cluster_stats, main_seconds));
  printf("finalize_seconds %zu\n", offsetof(tc_cluster_stats, finalize_seconds));
  printf("preprocess_skipped %zu\n", offsetof(tc_cluster_stats, preprocess_skipped));
  printf("dense_point_fraction %zu\n", offsetof(tc_cluster_stats, dense_point_fraction));
  printf("pair_resolutions %zu\n", offsetof(tc_cluster_stats, pair_resolutions));
  printf("distance_evaluations %zu\n", offsetof(tc_cluster_stats, distance_evaluations));
  printf("cluster_count %zu\n", offsetof(tc_cluster_stats, cluster_count));
  printf("core_count %zu\n", offsetof(tc_cluster_stats, core_count));
  printf("noise_count %zu\n", offsetof(tc_cluster_stats, noise_count));
  printf("enums %d %d %d %d %d %d | %d %d %d | %d %d %d\n", TC_OK, TC_ERR_INVALID_ARGUMENT,
         TC_ERR_IO, TC_ERR_VERIFY_FAIL, TC_ERR_CAP_EXCEEDED, TC_ERR_INTERNAL, TC_ALGO_FDBSCAN,
         TC_ALGO_DENSEBOX, TC_ALGO_BRUTEFORCE, TC_FORMAT_AUTO, TC_FORMAT_CSV, TC_FORMAT_BINARY);
  return 0;
}

static void host_checks(const char* tmpdir) {
  const float pts[6] = {0.f, 0.f, 1.f, 0.f, 0.f, 1.f};
  tc_dataset* ds = NULL;
  CHECK(tc_dataset_create(pts, 3, 2, &ds) == TC_OK);
  CHECK(tc_dataset_size(ds) == 3 && tc_dataset_dim(ds) == 2);
  CHECK(memcmp(tc_dataset_coords(ds), pts, sizeof pts) == 0);
  char path[4096];
  snprintf(path, sizeof path, "%s/client.bin", tmpdir);
  CHECK(tc_dataset_save(ds, path, TC_FORMAT_AUTO) == TC_OK);
  tc_dataset* back = NULL;
  CHECK(tc_dataset_load(path, TC_FORMAT_AUTO, &back) == TC_OK);
  CHECK(back && tc_dataset_size(back) == 3 &&
        memcmp(tc_dataset_coords(back), pts, sizeof pts) == 0);
  tc_dataset_free(back);
  tc_dataset_free(ds);

  tc_dataset* bad = (tc_dataset*)0x1;
  CHECK(tc_dataset_create(pts, 3, 4, &bad) == TC_ERR_INVALID_ARGUMENT);
  CHECK(bad == (tc_dataset*)0x1); /* *out written only on success */
  CHECK(tc_dataset_create(NULL, 3, 2, &bad) == TC_ERR_INVALID_ARGUMENT);
  const float nan_pts[2] = {0.f, 0.f / 0.f};
  CHECK(tc_dataset_create(nan_pts, 1, 2, &bad) == TC_ERR_INVALID_ARGUMENT);
  snprintf(path, sizeof path, "%s/missing.csv", tmpdir);
  CHECK(tc_dataset_load(path, TC_FORMAT_AUTO, &bad) == TC_ERR_IO);

  tc_dataset* g = NULL;
  CHECK(tc_generate_blobs(3, 80, 2, 20.f, 0.5f, 21, &g) == TC_OK);
  CHECK(tc_dataset_size(g) == 240);
  tc_result* res = (tc_result*)0x1;
  CHECK(tc_cluster(g, 0.f, 5, TC_ALGO_FDBSCAN, 0, 0, &res) == TC_ERR_INVALID_ARGUMENT);
  CHECK(tc_cluster(g, 1.f, 1, TC_ALGO_FDBSCAN, 0, 0, &res) == TC_ERR_INVALID_ARGUMENT);
  CHECK(tc_cluster(g, 1.f, 5, TC_ALGO_BRUTEFORCE, 0, 100, &res) == TC_ERR_CAP_EXCEEDED);
  CHECK(tc_cluster(NULL, 1.f, 5, TC_ALGO_FDBSCAN, 0, 0, &res) == TC_ERR_INVALID_ARGUMENT);
  CHECK(res == (tc_result*)0x1);
  tc_dataset_free(g);
  CHECK(strcmp(tc_status_string(TC_OK), "ok") == 0);
}

static void device_checks(void) {
  tc_dataset* ds = NULL;
  CHECK(tc_generate_blobs(3, 80, 2, 20.f, 0.5f, 21, &ds) == TC_OK);
  int32_t* all[3];
  const tc_algorithm algos[3] = {TC_ALGO_FDBSCAN, TC_ALGO_DENSEBOX, TC_ALGO_BRUTEFORCE};
  for (int a = 0; a < 3; ++a) {
    tc_result* res = NULL;
    CHECK(tc_cluster(ds, 1.5f, 5, algos[a], 2, 0, &res) == TC_OK);
    if (!res) {
      all[a] = NULL;
      continue;
    }
    CHECK(tc_result_size(res) == 240);
    CHECK(tc_result_labels(res) != NULL && tc_result_core_flags(res) != NULL);
    tc_cluster_stats st;
    CHECK(tc_result_stats(res, &st) == TC_OK);
    CHECK(st.cluster_count == 3);
    CHECK(st.core_count + st.noise_count <= 240);
    all[a] = (int32_t*)malloc(240 * sizeof(int32_t));
    memcpy(all[a], tc_result_labels(res), 240 * sizeof(int32_t));
    tc_result_free(res);
  }
  CHECK(all[0] && all[1] && all[2]);
  if (all[0] && all[1] && all[2]) {
    CHECK(memcmp(all[0], all[1], 240 * sizeof(int32_t)) == 0);
    CHECK(memcmp(all[0], all[2], 240 * sizeof(int32_t)) == 0);
  }
  for (int a = 0; a < 3; ++a) free(all[a]);
  tc_dataset_free(ds);

  tc_dataset* one = NULL; /* REF test_capi.cpp:131-140 */
  CHECK(tc_generate_blobs(1, 100, 2, 5.f, 0.3f, 2, &one) == TC_OK);
  tc_result* res = NULL;
  CHECK(tc_cluster(one, 1.f, 5, TC_ALGO_BRUTEFORCE, 1, 50, &res) == TC_ERR_CAP_EXCEEDED);
  CHECK(tc_cluster(one, 1.f, 5, TC_ALGO_BRUTEFORCE, 1, 100, &res) == TC_OK);
  tc_result_free(res);
  tc_dataset_free(one);

  /* the multi-GPU entry (treeclust_gpu.h) from C: two shards on device 0
   * give tc_cluster's labels on blobs(3, 80, 2, 20, 0.5, 21) */
  tc_dataset* m = NULL;
  CHECK(tc_generate_blobs(3, 80, 2, 20.f, 0.5f, 21, &m) == TC_OK);
  tc_result* single = NULL;
  tc_result* multi = NULL;
  const int devs[2] = {0, 0};
  CHECK(tc_cluster(m, 1.5f, 5, TC_ALGO_FDBSCAN, 0, 0, &single) == TC_OK);
  CHECK(tcg_cluster_multi(m, 1.5f, 5, TC_ALGO_FDBSCAN, devs, 2, &multi) == TC_OK);
  if (single && multi) {
    const int32_t* a = tc_result_labels(single);
    const int32_t* b = tc_result_labels(multi);
    const uint8_t* ca = tc_result_core_flags(single);
    const uint8_t* cb = tc_result_core_flags(multi);
    for (int i = 0; i < 240; ++i) {
      CHECK(ca[i] == cb[i]);
      CHECK((a[i] == -1) == (b[i] == -1));
      if (ca[i]) CHECK(a[i] == b[i]);
    }
  }
  tc_result_free(single);
  tc_result_free(multi);
  tc_dataset_free(m);

  tc_dataset* v = NULL; /* REF test_capi.cpp:142-150 */
  CHECK(tc_generate_blobs(3, 100, 2, 10.f, 0.6f, 31, &v) == TC_OK);
  char report[4096];
  CHECK(tc_verify(v, 1.2f, 5, 2, 0, report, sizeof report) == TC_OK);
  CHECK(strstr(report, "PASS") != NULL && strstr(report, "FAIL") == NULL);
  tc_dataset_free(v);
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  if (strcmp(argv[1], "layout") == 0) return layout();
  if (strcmp(argv[1], "host") == 0) host_checks(argc > 2 ? argv[2] : "/tmp");
  else if (strcmp(argv[1], "device") == 0) device_checks();
  else return 2;
  if (failures) fprintf(stderr, "%d check(s) failed\n", failures);
  else printf("all checks passed\n");
  return failures ? 1 : 0;
}
