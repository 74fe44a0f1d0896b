#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tcb {

// Smallest index of a border point with no same-label core within eps, or -1
// when every border is valid (oracle.cpp:72-116). Device pointers; syncs `st`.
int64_t first_bad_border(const float* d_coords, int64_t n, int dim, float eps,
                         const int32_t* d_labels, const uint8_t* d_core, cudaStream_t st);

}  // namespace tcb
