// Seeded generators on the device: the reference's
// gaussian_blobs / uniform_noise / dense_lattice (REF datagen.cpp:10-88) and
// the §8d HACC-like and taxi-like benchmark inputs, written straight into HBM.
//
// Every generator is one SplitMix64 stream (REF rng.hpp:11-47). SplitMix64 is
// a counter-based generator: the k-th output (1-based) is mix(seed + k * G),
// so any draw can be computed in isolation. Where a point always consumes
// the same number of draws (uniform noise; the background of HACC-like) the
// kernel derives its draw indices from its index alone. Where consumption
// varies, a host pass walks the stream touching one draw per point (no
// transcendental math) to fix the draw position of every point, and the
// device computes the coordinates:
//   gaussian_blobs  centres on the host (rejection, a few dozen draws); the
//                   t-th normal is half of Box-Muller pair t/2 (draws
//                   D0 + 2(t/2) + 1, + 2): cos for even t, sin for odd t;
//   hacc_like       host pass over the halos: mass, centre and, per particle,
//                   the accepted Plummer draw (rejections r > 10a are rare:
//                   ~1.5%, recorded as (particle, extra draws) events);
//   taxi_like       host pass: the branch draw of each point (road: 5 draws,
//                   uniform: 3) as a bit mask; positions = 3 i + 2 (#road
//                   points before i), from per-word prefix counts.
// The arithmetic is the host generator's, term for term. The device's
// double log / pow / sin / cos may differ from the host libm in the last
// bit, which changes a float output only when the double result lies within
// an ulp of a float rounding boundary (~2^-29 per value); the tests compare
// the device output with the host generator byte for byte. A Box-Muller
// first draw of exactly 0 (probability 2^-53 per pair) would make the host
// draw again and shift the stream; the device flags it and the entry point
// falls back to the host generator.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include "device_common.cuh"
#include "host_data.hpp"
#include "pipeline.hpp"

namespace tcb {

namespace {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;

__host__ __device__ __forceinline__ uint64_t sm64_at(uint64_t seed, uint64_t k) {
  uint64_t z = seed + k * kGolden;  // state after k calls of next()
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double unit_at(uint64_t seed, uint64_t k) {
  return static_cast<double>(sm64_at(seed, k) >> 11) * 0x1.0p-53;
}

struct Box3 {
  double lo[3], hi[3];
};

// uniform_noise (datagen.cpp:55-68): coordinate a of point i is draw
// first + i * dim + a + 1.
__global__ void k_gen_uniform(int64_t n, int dim, Box3 b, uint64_t seed, uint64_t first,
                              float* __restrict__ out) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n * dim;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int a = static_cast<int>(t % dim);
    const double lo = b.lo[a], hi = b.hi[a];
    out[t] = static_cast<float>(lo + (hi - lo) * unit_at(seed, first + static_cast<uint64_t>(t) + 1));
  }
}

// dense_lattice (datagen.cpp:70-88): x fastest.
__global__ void k_gen_lattice(int64_t n, int64_t side, int dim, double spacing,
                              float* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t r = i;
    for (int a = 0; a < dim; ++a) {
      out[i * dim + a] = static_cast<float>(static_cast<double>(r % side) * spacing);
      r /= side;
    }
  }
}

// Box-Muller half t of the stream that starts after `first` draws
// (rng.hpp:28-41): pair q = t / 2 draws u1 = first + 2q + 1, u2 = first + 2q + 2.
__device__ __forceinline__ double normal_at(uint64_t seed, uint64_t first, uint64_t t,
                                            int* zero_flag) {
  const uint64_t q = t >> 1;
  const double u1 = unit_at(seed, first + 2 * q + 1);
  const double u2 = unit_at(seed, first + 2 * q + 2);
  if (u1 == 0.0) *zero_flag = 1;  // the host would draw again: fall back
  const double mag = sqrt(-2.0 * log(u1));
  const double ang = 2.0 * 3.141592653589793 * u2;
  return (t & 1) ? mag * sin(ang) : mag * cos(ang);
}

// gaussian_blobs points (datagen.cpp:46-52): value t = (c * per_blob + i) * dim + a.
__global__ void k_gen_blobs(int64_t total, int dim, int64_t per_blob,
                            const double* __restrict__ centres, double sigma, uint64_t seed,
                            uint64_t first, float* __restrict__ out, int* zero_flag) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t point = t / dim;
    const int a = static_cast<int>(t - point * dim);
    const int64_t c = point / per_blob;
    out[t] = static_cast<float>(centres[c * dim + a] +
                                sigma * normal_at(seed, first, static_cast<uint64_t>(t), zero_flag));
  }
}

struct HaloDev {
  const int64_t* first_particle;  // halos + 1 entries (exclusive prefix of masses)
  const uint64_t* start;          // draw index before the halo's first particle
  const double* a;                // Plummer scale
  const double* c;                // centres, 3 per halo
  const int64_t* ev_particle;     // rejection events: halo particle index (sorted)
  const int64_t* ev_extra;        // inclusive prefix of extra draws
  int64_t halos, events;
};

// hacc_like halo particles (host_data.cpp gen_hacc_like): particle p of halo
// h has its accepted radius draw at start[h] + 3 (p - first[h]) + (extra
// draws of the rejections before p in h) + 1, then z and phi.
__global__ void k_gen_halos(int64_t n_halo, HaloDev hd, double box_len, uint64_t seed,
                            float* __restrict__ out) {
  const double two_pi = 2.0 * 3.141592653589793;
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n_halo;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t lo = 0, hi = hd.halos - 1;  // last halo with first_particle <= p
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (hd.first_particle[mid] <= p) lo = mid; else hi = mid - 1;
    }
    const int64_t h = lo;
    auto extra_before = [&](int64_t q) -> int64_t {  // extra draws of events with particle < q
      int64_t l = 0, r = hd.events;
      while (l < r) {
        const int64_t mid = (l + r) >> 1;
        if (hd.ev_particle[mid] < q) l = mid + 1; else r = mid;
      }
      return l ? hd.ev_extra[l - 1] : 0;
    };
    const int64_t f = hd.first_particle[h];
    int64_t ev_here = 0;  // this particle's own rejected draws
    {
      int64_t l = 0, r = hd.events;
      while (l < r) {
        const int64_t mid = (l + r) >> 1;
        if (hd.ev_particle[mid] < p) l = mid + 1; else r = mid;
      }
      if (l < hd.events && hd.ev_particle[l] == p)
        ev_here = hd.ev_extra[l] - (l ? hd.ev_extra[l - 1] : 0);
    }
    const uint64_t pos = hd.start[h] + 3ull * static_cast<uint64_t>(p - f) +
                         static_cast<uint64_t>(extra_before(p) - extra_before(f) + ev_here);
    const double a = hd.a[h];
    const double uu = unit_at(seed, pos + 1);
    const double r = a / sqrt(pow(uu, -2.0 / 3.0) - 1.0);
    const double z = -1.0 + 2.0 * unit_at(seed, pos + 2);
    const double phi = 0.0 + (two_pi - 0.0) * unit_at(seed, pos + 3);
    const double s = sqrt(1.0 - z * z);
    out[3 * p + 0] = static_cast<float>(hd.c[3 * h + 0] + r * s * cos(phi));
    out[3 * p + 1] = static_cast<float>(hd.c[3 * h + 1] + r * s * sin(phi));
    out[3 * p + 2] = static_cast<float>(hd.c[3 * h + 2] + r * z);
  }
  (void)box_len;
}

constexpr int kTaxiSegments = 300;
struct TaxiSegs {
  double x[kTaxiSegments], y[kTaxiSegments], dx[kTaxiSegments], dy[kTaxiSegments];
  double cdf[kTaxiSegments];
  double total;
};

// taxi_like points: point i starts at draw first + 3 i + 2 (#road points
// before i): branch, then pick, t, Box-Muller pair (road) or x, y (uniform).
__global__ void k_gen_taxi(int64_t n, uint64_t seed, uint64_t first,
                           const uint32_t* __restrict__ road, const int64_t* __restrict__ word_prefix,
                           const TaxiSegs* __restrict__ segs, float* __restrict__ out,
                           int* zero_flag) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t word = road[i >> 5];
    const uint32_t below = word & ((1u << (i & 31)) - 1u);
    const int64_t roads_before = word_prefix[i >> 5] + __popc(below);
    const uint64_t pos = first + 3ull * static_cast<uint64_t>(i) + 2ull * static_cast<uint64_t>(roads_before);
    double x, y;
    if ((word >> (i & 31)) & 1u) {
      const double pick = unit_at(seed, pos + 2) * segs->total;
      int lo = 0, hi = kTaxiSegments;  // first cdf entry > pick
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (segs->cdf[mid] > pick) hi = mid; else lo = mid + 1;
      }
      const int s = lo < kTaxiSegments ? lo : kTaxiSegments - 1;
      const double t = unit_at(seed, pos + 3);
      const double u1 = unit_at(seed, pos + 4), u2 = unit_at(seed, pos + 5);
      if (u1 == 0.0) *zero_flag = 1;
      const double mag = sqrt(-2.0 * log(u1));
      const double ang = 2.0 * 3.141592653589793 * u2;
      x = segs->x[s] + t * segs->dx[s] + 1e-4 * (mag * cos(ang));
      y = segs->y[s] + t * segs->dy[s] + 1e-4 * (mag * sin(ang));
    } else {
      x = unit_at(seed, pos + 2);
      y = unit_at(seed, pos + 3);
    }
    out[2 * i] = static_cast<float>(x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x));
    out[2 * i + 1] = static_cast<float>(y < 0.0 ? 0.0 : (y > 1.0 ? 1.0 : y));
  }
}

unsigned gen_grid(int64_t work) { return grid_for(work, 256, 148 * 32); }

template <typename T>
T* upload(const std::vector<T>& v, Scratch& scratch) {
  T* d = scratch.alloc_n<T>(static_cast<int64_t>(std::max<size_t>(v.size(), 1)));
  if (!v.empty())
    TCB_CUDA(cudaMemcpyAsync(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice,
                             scratch.stream()));
  return d;
}

bool zero_flag_set(int* d_flag, cudaStream_t s) {
  int h = 0;
  TCB_CUDA(cudaMemcpyAsync(&h, d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  TCB_CUDA(cudaStreamSynchronize(s));
  return h != 0;
}

void copy_host_points(const HostPoints& hp, float* d_out, cudaStream_t s) {
  TCB_CUDA(cudaMemcpyAsync(d_out, hp.coords.data(), sizeof(float) * hp.coords.size(),
                           cudaMemcpyHostToDevice, s));
  TCB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

void gen_uniform_device(int64_t n, int dim, const float* lo, const float* hi, uint64_t seed,
                        float* d_out, cudaStream_t s) {
  if (n < 1) throw std::invalid_argument("uniform_noise: n must be >= 1");
  if (dim != 2 && dim != 3) throw std::invalid_argument("uniform_noise: dim must be 2 or 3");
  Box3 b{};
  for (int a = 0; a < dim; ++a) {
    if (!(lo[a] <= hi[a])) throw std::invalid_argument("bounds");
    b.lo[a] = lo[a];
    b.hi[a] = hi[a];
  }
  note_launch(), k_gen_uniform<<<gen_grid(n * dim), 256, 0, s>>>(n, dim, b, seed, 0, d_out);
  TCB_CUDA(cudaGetLastError());
}

void gen_lattice_device(int64_t side, int dim, float spacing, float* d_out, cudaStream_t s) {
  if (side < 2) throw std::invalid_argument("dense_lattice: side must be >= 2");
  if (dim != 2 && dim != 3) throw std::invalid_argument("dense_lattice: dim must be 2 or 3");
  int64_t n = side;
  for (int a = 1; a < dim; ++a) n *= side;
  note_launch(), k_gen_lattice<<<gen_grid(n), 256, 0, s>>>(n, side, dim, static_cast<double>(spacing),
                                                          d_out);
  TCB_CUDA(cudaGetLastError());
}

void gen_blobs_device(int k, int64_t per_blob, int dim, float separation, float sigma,
                      uint64_t seed, float* d_out, cudaStream_t s) {
  if (k < 1 || per_blob < 1) throw std::invalid_argument("gaussian_blobs: k and per_blob must be >= 1");
  if (dim != 2 && dim != 3) throw std::invalid_argument("gaussian_blobs: dim must be 2 or 3");
  // centres exactly as the host generator (datagen.cpp:18-43)
  SplitMix64 rng(seed);
  const double domain = static_cast<double>(separation) * (k + 1);
  std::vector<double> centres;
  for (int c = 0; c < k; ++c) {
    int attempt = 0;
    while (true) {
      if (++attempt > 10000)
        throw std::runtime_error("gaussian_blobs: could not place separated centers");
      double cand[3];
      for (int a = 0; a < dim; ++a) cand[a] = rng.uniform(0.0, domain);
      bool ok = true;
      for (int o = 0; o < c && ok; ++o) {
        double d2 = 0;
        for (int a = 0; a < dim; ++a) {
          const double d = cand[a] - centres[o * dim + a];
          d2 += d * d;
        }
        ok = d2 >= static_cast<double>(separation) * separation;
      }
      if (ok) {
        for (int a = 0; a < dim; ++a) centres.push_back(cand[a]);
        break;
      }
    }
  }
  Scratch scratch(s);
  const double* d_centres = upload(centres, scratch);
  int* flag = scratch.alloc_n<int>(1);
  TCB_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
  const int64_t total = static_cast<int64_t>(k) * per_blob * dim;
  note_launch(), k_gen_blobs<<<gen_grid(total), 256, 0, s>>>(total, dim, per_blob, d_centres,
                                                            static_cast<double>(sigma), seed,
                                                            rng.draws(), d_out, flag);
  TCB_CUDA(cudaGetLastError());
  if (zero_flag_set(flag, s))
    copy_host_points(gen_blobs(k, per_blob, dim, separation, sigma, seed), d_out, s);
}

void gen_hacc_like_device(int64_t n, double box_len, double halo_frac, uint64_t seed,
                          float* d_out, cudaStream_t s) {
  if (n < 1) throw std::invalid_argument("hacc_like: n must be >= 1");
  if (!(box_len > 0.0) || !(halo_frac >= 0.0 && halo_frac <= 1.0))
    throw std::invalid_argument("hacc_like: bad box length or halo fraction");
  const int64_t n_halo = static_cast<int64_t>(halo_frac * static_cast<double>(n));
  const int64_t n_bg = n - n_halo;
  Box3 b{};
  for (int a = 0; a < 3; ++a) b.hi[a] = box_len;
  if (n_bg > 0)
    note_launch(), k_gen_uniform<<<gen_grid(n_bg * 3), 256, 0, s>>>(n_bg, 3, b, seed, 0, d_out);
  TCB_CUDA(cudaGetLastError());
  if (n_halo == 0) return;
  // Host pass over the halo section of the stream (gen_hacc_like): one draw
  // per particle unless its Plummer radius is rejected (r > 10a, ~1.5%).
  SplitMix64 rng(seed);
  rng.skip(static_cast<uint64_t>(n_bg) * 3);
  std::vector<int64_t> first{0}, ev_p, ev_x;
  std::vector<uint64_t> start;
  std::vector<double> av, cv;
  // r <= 10a  <=>  uu <= 1.01^-1.5 (mathematically); decide by the host's own
  // expression only near that threshold
  const double thr = std::pow(1.01, -1.5);
  int64_t made = 0, extra_total = 0;
  while (made < n_halo) {
    const double u = rng.next_double();
    int64_t m = static_cast<int64_t>(20.0 / std::pow(1.0 - u, 1.0 / 0.9));
    m = std::min<int64_t>(m, 200000);
    m = std::min<int64_t>(m, n_halo - made);
    if (m < 1) m = 1;
    const double a = 0.010 * std::cbrt(static_cast<double>(m) / 20.0);
    for (int k = 0; k < 3; ++k) cv.push_back(rng.uniform(a, box_len - a));
    av.push_back(a);
    start.push_back(rng.draws());
    for (int64_t p = 0; p < m; ++p) {
      int64_t extra = 0;
      while (true) {
        double uu = rng.next_double();
        while (uu == 0.0) {
          ++extra;
          uu = rng.next_double();
        }
        bool ok;
        if (uu < thr * (1.0 - 1e-9))
          ok = true;
        else if (uu > thr * (1.0 + 1e-9))
          ok = false;
        else
          ok = a / std::sqrt(std::pow(uu, -2.0 / 3.0) - 1.0) <= 10.0 * a;
        if (ok) break;
        ++extra;
      }
      if (extra) {
        extra_total += extra;
        ev_p.push_back(made + p);
        ev_x.push_back(extra_total);
      }
      rng.skip(2);  // z, phi
    }
    made += m;
    first.push_back(made);
  }
  Scratch scratch(s);
  HaloDev hd;
  hd.first_particle = upload(first, scratch);
  hd.start = upload(start, scratch);
  hd.a = upload(av, scratch);
  hd.c = upload(cv, scratch);
  hd.ev_particle = upload(ev_p, scratch);
  hd.ev_extra = upload(ev_x, scratch);
  hd.halos = static_cast<int64_t>(av.size());
  hd.events = static_cast<int64_t>(ev_p.size());
  note_launch(), k_gen_halos<<<gen_grid(n_halo), 256, 0, s>>>(n_halo, hd, box_len, seed,
                                                             d_out + 3 * n_bg);
  TCB_CUDA(cudaGetLastError());
  TCB_CUDA(cudaStreamSynchronize(s));  // the host tables are released with the scratch
}

void gen_taxi_like_device(int64_t n, uint64_t seed, float* d_out, cudaStream_t s) {
  if (n < 1) throw std::invalid_argument("taxi_like: n must be >= 1");
  // cities and segments exactly as the host generator (host_data.cpp)
  SplitMix64 rng(seed);
  constexpr int kCities = 8;
  double city[kCities][2];
  for (auto& cc : city)
    for (double& v : cc) v = rng.uniform(0.2, 0.8);
  auto segs = std::make_unique<TaxiSegs>();
  double total = 0;
  for (int q = 0; q < kTaxiSegments; ++q) {
    const int c = static_cast<int>(rng.next() % kCities);
    const double ax = city[c][0] + 0.08 * rng.normal();
    const double ay = city[c][1] + 0.08 * rng.normal();
    const double ang = rng.uniform(0.0, 3.141592653589793);
    const double len = -0.02 * std::log(1.0 - rng.next_double());
    segs->x[q] = ax;
    segs->y[q] = ay;
    segs->dx[q] = len * std::cos(ang);
    segs->dy[q] = len * std::sin(ang);
    total += std::pow(static_cast<double>(q + 1), -0.8);
    segs->cdf[q] = total;
  }
  segs->total = total;
  if (rng.has_spare()) throw std::logic_error("taxi_like: unpaired normal draw");
  // host pass: the branch of every point (road: 5 draws, uniform: 3)
  const uint64_t first = rng.draws();
  const int64_t words = (n + 31) / 32;
  std::vector<uint32_t> road(static_cast<size_t>(words), 0u);
  std::vector<int64_t> prefix(static_cast<size_t>(words), 0);
  int64_t roads = 0;
  for (int64_t i = 0; i < n; ++i) {
    if ((i & 31) == 0) prefix[static_cast<size_t>(i >> 5)] = roads;
    const bool on_road = rng.next_double() < 0.98;
    if (on_road) {
      road[static_cast<size_t>(i >> 5)] |= 1u << (i & 31);
      ++roads;
      rng.skip(4);
    } else {
      rng.skip(2);
    }
  }
  Scratch scratch(s);
  const uint32_t* d_road = upload(road, scratch);
  const int64_t* d_prefix = upload(prefix, scratch);
  auto* d_segs = scratch.alloc_n<TaxiSegs>(1);
  TCB_CUDA(cudaMemcpyAsync(d_segs, segs.get(), sizeof(TaxiSegs), cudaMemcpyHostToDevice, s));
  int* flag = scratch.alloc_n<int>(1);
  TCB_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
  note_launch(), k_gen_taxi<<<gen_grid(n), 256, 0, s>>>(n, seed, first, d_road, d_prefix, d_segs,
                                                       d_out, flag);
  TCB_CUDA(cudaGetLastError());
  if (zero_flag_set(flag, s)) copy_host_points(gen_taxi_like(n, seed), d_out, s);
}

}  // namespace tcb
