// Host-side data plumbing shared by the C ABI: point sets, seeded generators
// and file formats. These sit before the hot path
// and are restated from the reference's published behaviour so datasets are
// byte-identical to the reference's for the same arguments.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace tcb {

// Host point storage: n*dim floats, row-major.
struct HostPoints {
  int dim = 0;
  std::vector<float> coords;
  int64_t size() const { return dim ? static_cast<int64_t>(coords.size()) / dim : 0; }
};

// PointSet::validate (geometry.hpp:29-37): throws std::invalid_argument.
void validate_points(int dim, const float* coords, int64_t count_floats);

// SplitMix64 stream (rng.hpp:11-47): fixed so generated data is identical
// across implementations.
class SplitMix64 {
 public:
  explicit SplitMix64(uint64_t seed) : state_(seed) {}
  uint64_t next() {
    ++draws_;
    uint64_t z = (state_ += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double next_double() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * next_double(); }
  double normal();  // Box-Muller, second half cached
  // Draws consumed so far, and skipping k draws (the state is a counter:
  // gen.cu computes any draw from the seed and its index).
  uint64_t draws() const { return draws_; }
  void skip(uint64_t k) {
    state_ += k * 0x9e3779b97f4a7c15ull;
    draws_ += k;
  }
  bool has_spare() const { return has_spare_; }

 private:
  uint64_t state_;
  uint64_t draws_ = 0;
  bool has_spare_ = false;
  double spare_ = 0.0;
};

// Reference generators (datagen.cpp:10-88).
HostPoints gen_blobs(int k, int64_t per_blob, int dim, float separation, float sigma,
                     uint64_t seed);
HostPoints gen_uniform(int64_t n, int dim, const float* lo, const float* hi, uint64_t seed);
HostPoints gen_lattice(int64_t side, int dim, float spacing);
// testutil::random_instance (tests/test_util.hpp:27-60).
HostPoints gen_random_instance(uint64_t seed, int64_t min_n, int64_t max_n, float* eps,
                               int* minpts);
// Benchmark generators of SURVEY.md §8d (new; the reference ships none).
HostPoints gen_hacc_like(int64_t n, double box_len, double halo_frac, uint64_t seed);
HostPoints gen_taxi_like(int64_t n, uint64_t seed);

// The same generators writing straight into device memory (gen.cu): output
// identical to the host generators' (see gen.cu for the libm caveat). d_out
// holds n * dim floats; enqueued on `s` (the halo / taxi host passes and the
// rare host fallback synchronize it).
void gen_blobs_device(int k, int64_t per_blob, int dim, float separation, float sigma,
                      uint64_t seed, float* d_out, cudaStream_t s);
void gen_uniform_device(int64_t n, int dim, const float* lo, const float* hi, uint64_t seed,
                        float* d_out, cudaStream_t s);
void gen_lattice_device(int64_t side, int dim, float spacing, float* d_out, cudaStream_t s);
void gen_hacc_like_device(int64_t n, double box_len, double halo_frac, uint64_t seed,
                          float* d_out, cudaStream_t s);
void gen_taxi_like_device(int64_t n, uint64_t seed, float* d_out, cudaStream_t s);

// File formats (io.cpp:51-148). Errors throw std::runtime_error.
HostPoints load_points(const std::string& path, int format /* 0 auto, 1 csv, 2 bin */);
void save_points(const std::string& path, int format, int dim, const float* coords, int64_t n);
// Header of a binary point file (io.cpp:106-115): n and dim.
void binary_info(const std::string& path, int64_t* n, int* dim);
// A binary point file straight into d_coords (n*dim floats), reads overlapped
// with the host->device copies; synchronizes `stream` before returning.
void load_binary_device(const std::string& path, float* d_coords, int64_t n, int dim,
                        cudaStream_t stream);

}  // namespace tcb
