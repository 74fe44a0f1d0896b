#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tcb {

// Smallest index of a border point with no same-label core within eps, or -1
// when every border is valid (oracle.cpp:72-116). Device pointers; syncs `st`.
int64_t first_bad_border(const float* d_coords, int64_t n, int dim, float eps,
                         const int32_t* d_labels, const uint8_t* d_core, cudaStream_t st);

// check_equivalence (oracle.cpp:120-163) of clusterings a and b on device
// buffers, checks in the reference's order. check: 0 pass, 1 core flags,
// 2 noise sets, 3 core partitions, 4 / 5 invalid border in a / b; at = the
// point index the reference's scan reports. Syncs `st`.
struct EqVerdict {
  int check = 0;
  int64_t at = 0;
};
EqVerdict check_equivalence_device(const float* d_coords, int64_t n, int dim, float eps,
                                   const int32_t* la, const uint8_t* ca, const int32_t* lb,
                                   const uint8_t* cb, cudaStream_t st);
const char* equivalence_message(int check);

}  // namespace tcb
