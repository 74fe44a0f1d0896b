/* A C caller that captures the stream-ordered FDBSCAN entry into a CUDA graph
 * (include/treeclust_gpu.h: tcg_cluster_device_async) with the plain CUDA
 * runtime — no PyTorch — and replays it on new coordinates copied into the
 * captured input buffer. Each replay must agree with an eager
 * tcg_cluster_device(stats) run of the same points: identical core flags and
 * noise set, identical core labels (minpts 2: every label). Also checks the
 * device status word for a non-finite coordinate.
 *
 *   graph_client        exit 0 on success, 1 with a message on stderr
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "treeclust_gpu.h"

#define CHECK(c)                                                  \
  do {                                                            \
    if (!(c)) {                                                   \
      fprintf(stderr, "%s:%d: check failed: %s\n", __FILE__, __LINE__, #c); \
      exit(1);                                                    \
    }                                                             \
  } while (0)
#define CUDA(c) CHECK((c) == cudaSuccess)

static const float kEps = 0.15f;

static tc_dataset* blobs(unsigned seed) {
  tc_dataset* ds = NULL;
  CHECK(tc_generate_blobs(10, 3000, 3, 4.0f, 0.4f, seed, &ds) == TC_OK);
  return ds;
}

int main(void) {
  int minpts_list[2] = {2, 6};
  for (int t = 0; t < 2; ++t) {
    const int minpts = minpts_list[t];
    tc_dataset* ds = blobs(5);
    const int64_t n = tc_dataset_size(ds);
    const size_t cb = (size_t)n * 3 * sizeof(float);
    float *x, *y;
    int32_t *lab, *lab_ref, *st;
    uint8_t *core, *core_ref;
    CUDA(cudaMalloc((void**)&x, cb));
    CUDA(cudaMalloc((void**)&y, cb));
    CUDA(cudaMalloc((void**)&lab, n * 4));
    CUDA(cudaMalloc((void**)&lab_ref, n * 4));
    CUDA(cudaMalloc((void**)&core, n));
    CUDA(cudaMalloc((void**)&core_ref, n));
    CUDA(cudaMalloc((void**)&st, 4));
    CUDA(cudaMemcpy(x, tc_dataset_coords(ds), cb, cudaMemcpyHostToDevice));
    cudaStream_t s;
    CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    /* warm-up off the capture (library pool, kernel attributes) */
    CHECK(tcg_cluster_device_async(x, n, 3, kEps, minpts, TC_ALGO_FDBSCAN, 0, lab, core, s, st) ==
          TC_OK);
    CUDA(cudaStreamSynchronize(s));

    cudaGraph_t g;
    cudaGraphExec_t ge;
    CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    CHECK(tcg_cluster_device_async(x, n, 3, kEps, minpts, TC_ALGO_FDBSCAN, 0, lab, core, s, st) ==
          TC_OK);
    CUDA(cudaStreamEndCapture(s, &g));
    CUDA(cudaGraphInstantiate(&ge, g, 0));

    int32_t* hl = malloc(n * 4);
    int32_t* hr = malloc(n * 4);
    uint8_t* hc = malloc(n);
    uint8_t* hcr = malloc(n);
    for (unsigned seed = 11; seed < 14; ++seed) {
      tc_dataset* nd = blobs(seed);
      CHECK(tc_dataset_size(nd) == n);
      CUDA(cudaMemcpy(x, tc_dataset_coords(nd), cb, cudaMemcpyHostToDevice));
      CUDA(cudaMemcpy(y, tc_dataset_coords(nd), cb, cudaMemcpyHostToDevice));
      CUDA(cudaMemset(st, 0x7f, 4));
      CUDA(cudaGraphLaunch(ge, s));
      CUDA(cudaStreamSynchronize(s));
      tc_cluster_stats stats;
      CHECK(tcg_cluster_device(y, n, 3, kEps, minpts, TC_ALGO_FDBSCAN, 0, lab_ref, core_ref, s,
                               &stats) == TC_OK);
      int32_t hs = -1;
      CUDA(cudaMemcpy(&hs, st, 4, cudaMemcpyDeviceToHost));
      CHECK(hs == TC_OK);
      CUDA(cudaMemcpy(hl, lab, n * 4, cudaMemcpyDeviceToHost));
      CUDA(cudaMemcpy(hr, lab_ref, n * 4, cudaMemcpyDeviceToHost));
      CUDA(cudaMemcpy(hc, core, n, cudaMemcpyDeviceToHost));
      CUDA(cudaMemcpy(hcr, core_ref, n, cudaMemcpyDeviceToHost));
      int64_t clusters = 0;
      for (int64_t i = 0; i < n; ++i) {
        CHECK(hc[i] == hcr[i]);
        CHECK((hl[i] == -1) == (hr[i] == -1));
        if (hc[i]) CHECK(hl[i] == hr[i]);
        clusters += hc[i] && hl[i] == i;
      }
      CHECK(clusters == stats.cluster_count);
      tc_dataset_free(nd);
    }
    /* a non-finite coordinate: the replay reports it on the device */
    const float nan = strtof("nan", NULL);
    CUDA(cudaMemcpy(x + 3 * 1234 + 1, &nan, sizeof nan, cudaMemcpyHostToDevice));
    CUDA(cudaGraphLaunch(ge, s));
    CUDA(cudaStreamSynchronize(s));
    int32_t hs = -1;
    CUDA(cudaMemcpy(&hs, st, 4, cudaMemcpyDeviceToHost));
    CHECK(hs == TC_ERR_INVALID_ARGUMENT);
    CUDA(cudaMemcpy(hl, lab, n * 4, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n; ++i) CHECK(hl[i] == -1);

    CUDA(cudaGraphExecDestroy(ge));
    CUDA(cudaGraphDestroy(g));
    CUDA(cudaStreamDestroy(s));
    cudaFree(x), cudaFree(y), cudaFree(lab), cudaFree(lab_ref), cudaFree(core),
        cudaFree(core_ref), cudaFree(st);
    free(hl), free(hr), free(hc), free(hcr);
    tc_dataset_free(ds);
  }
  printf("ok\n");
  return 0;
}
