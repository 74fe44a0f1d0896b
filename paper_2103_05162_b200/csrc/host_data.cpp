// Host-side generators and file formats (see host_data.hpp).
#include "host_data.hpp"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "engine.hpp"

namespace tcb {

void validate_points(int dim, const float* coords, int64_t count_floats) {
  if (dim != 2 && dim != 3) throw std::invalid_argument("PointSet: dimension must be 2 or 3");
  if (count_floats <= 0 || count_floats % dim != 0)
    throw std::invalid_argument("PointSet: coordinate count not a multiple of dim");
  for (int64_t i = 0; i < count_floats; ++i)
    if (!std::isfinite(coords[i])) throw std::invalid_argument("PointSet: non-finite coordinate");
}

double SplitMix64::normal() {
  if (has_spare_) {
    has_spare_ = false;
    return spare_;
  }
  double u1 = next_double();
  double u2 = next_double();
  while (u1 == 0.0) u1 = next_double();
  const double mag = std::sqrt(-2.0 * std::log(u1));
  const double ang = 2.0 * 3.141592653589793 * u2;
  spare_ = mag * std::sin(ang);
  has_spare_ = true;
  return mag * std::cos(ang);
}

// gaussian_blobs (datagen.cpp:10-53): centres rejection-sampled at least
// `separation` apart in [0, separation*(k+1))^dim, then per_blob normal
// samples per centre.
HostPoints gen_blobs(int k, int64_t per_blob, int dim, float separation, float sigma,
                     uint64_t seed) {
  if (k < 1 || per_blob < 1)
    throw std::invalid_argument("gaussian_blobs: k and per_blob must be >= 1");
  if (dim != 2 && dim != 3) throw std::invalid_argument("gaussian_blobs: dim must be 2 or 3");
  SplitMix64 rng(seed);
  const double domain = static_cast<double>(separation) * (k + 1);
  const double sep2 = static_cast<double>(separation) * separation;
  std::vector<double> centres;
  centres.reserve(static_cast<size_t>(k) * dim);
  for (int c = 0; c < k; ++c) {
    for (int attempt = 1;; ++attempt) {
      if (attempt > 10000)
        throw std::runtime_error("gaussian_blobs: could not place separated centers");
      double cand[3];
      for (int a = 0; a < dim; ++a) cand[a] = rng.uniform(0.0, domain);
      bool far_enough = true;
      for (int o = 0; o < c && far_enough; ++o) {
        double d2 = 0;
        for (int a = 0; a < dim; ++a) {
          double d = cand[a] - centres[static_cast<size_t>(o) * dim + a];
          d2 += d * d;
        }
        far_enough = d2 >= sep2;
      }
      if (far_enough) {
        centres.insert(centres.end(), cand, cand + dim);
        break;
      }
    }
  }
  HostPoints out;
  out.dim = dim;
  out.coords.reserve(static_cast<size_t>(k) * per_blob * dim);
  for (int c = 0; c < k; ++c)
    for (int64_t i = 0; i < per_blob; ++i)
      for (int a = 0; a < dim; ++a)
        out.coords.push_back(
            static_cast<float>(centres[static_cast<size_t>(c) * dim + a] + sigma * rng.normal()));
  return out;
}

// uniform_noise (datagen.cpp:55-68).
HostPoints gen_uniform(int64_t n, int dim, const float* lo, const float* hi, uint64_t seed) {
  if (n < 1) throw std::invalid_argument("uniform_noise: n must be >= 1");
  if (dim != 2 && dim != 3) throw std::invalid_argument("uniform_noise: dim must be 2 or 3");
  SplitMix64 rng(seed);
  HostPoints out;
  out.dim = dim;
  out.coords.resize(static_cast<size_t>(n) * dim);
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < dim; ++a)
      out.coords[static_cast<size_t>(i) * dim + a] = static_cast<float>(rng.uniform(lo[a], hi[a]));
  return out;
}

// dense_lattice (datagen.cpp:70-88): side^dim points, x fastest.
HostPoints gen_lattice(int64_t side, int dim, float spacing) {
  if (side < 2) throw std::invalid_argument("dense_lattice: side must be >= 2");
  if (dim != 2 && dim != 3) throw std::invalid_argument("dense_lattice: dim must be 2 or 3");
  int64_t n = side;
  for (int a = 1; a < dim; ++a) n *= side;
  HostPoints out;
  out.dim = dim;
  out.coords.reserve(static_cast<size_t>(n) * dim);
  int64_t idx[3] = {0, 0, 0};
  for (int64_t i = 0; i < n; ++i) {
    for (int a = 0; a < dim; ++a)
      out.coords.push_back(static_cast<float>(idx[a] * static_cast<double>(spacing)));
    for (int a = 0; a < dim; ++a) {
      if (++idx[a] < side) break;
      idx[a] = 0;
    }
  }
  return out;
}

// testutil::random_instance (tests/test_util.hpp:27-60): blobs + 10-50%
// uniform noise in [0,10]^d, eps log-uniform in [0.05, 2], minpts from
// {2,3,5,10,25}.
HostPoints gen_random_instance(uint64_t seed, int64_t min_n, int64_t max_n, float* eps,
                               int* minpts) {
  SplitMix64 rng(seed);
  HostPoints out;
  const int dim = (rng.next() % 2) ? 2 : 3;
  const int64_t n = min_n + static_cast<int64_t>(rng.next() % static_cast<uint64_t>(max_n - min_n + 1));
  const int blobs = 1 + static_cast<int>(rng.next() % 4);
  const auto n_noise = static_cast<int64_t>(n * rng.uniform(0.1, 0.5));
  const int64_t n_blob = n - n_noise;
  out.dim = dim;
  out.coords.reserve(static_cast<size_t>(n) * dim);
  std::vector<double> centres;
  for (int b = 0; b < blobs; ++b)
    for (int a = 0; a < dim; ++a) centres.push_back(rng.uniform(1.0, 9.0));
  for (int64_t i = 0; i < n_blob; ++i) {
    const int b = static_cast<int>(rng.next() % blobs);
    const double sigma = 0.2 + 0.1 * b;
    for (int a = 0; a < dim; ++a)
      out.coords.push_back(static_cast<float>(centres[b * dim + a] + sigma * rng.normal()));
  }
  for (int64_t i = 0; i < n_noise; ++i)
    for (int a = 0; a < dim; ++a) out.coords.push_back(static_cast<float>(rng.uniform(0.0, 10.0)));
  const double log_lo = std::log(0.05), log_hi = std::log(2.0);
  *eps = static_cast<float>(std::exp(rng.uniform(log_lo, log_hi)));
  static const int kMinpts[] = {2, 3, 5, 10, 25};
  *minpts = kMinpts[rng.next() % 5];
  return out;
}

// HACC-like halos. One SplitMix64 stream:
//   background: n - int64(halo_frac*n) points, x,y,z ~ U(0, L)
//   halos until int64(halo_frac*n) halo points: mass m = int64(20/(1-u)^(1/0.9))
//   capped at 200000 and at the remainder; Plummer scale a = 0.010*cbrt(m/20);
//   centre ~ U(a, L-a)^3; radius r = a/sqrt(uu^(-2/3) - 1) (uu > 0, r <= 10a),
//   direction z ~ U(-1,1), phi ~ U(0, 2pi).
HostPoints gen_hacc_like(int64_t n, double box_len, double halo_frac, uint64_t seed) {
  if (n < 1) throw std::invalid_argument("hacc_like: n must be >= 1");
  if (!(box_len > 0.0) || !(halo_frac >= 0.0 && halo_frac <= 1.0))
    throw std::invalid_argument("hacc_like: bad box length or halo fraction");
  SplitMix64 rng(seed);
  const int64_t n_halo = static_cast<int64_t>(halo_frac * static_cast<double>(n));
  const int64_t n_bg = n - n_halo;
  HostPoints out;
  out.dim = 3;
  out.coords.resize(static_cast<size_t>(n) * 3);
  float* w = out.coords.data();
  for (int64_t i = 0; i < n_bg; ++i)
    for (int a = 0; a < 3; ++a) *w++ = static_cast<float>(rng.uniform(0.0, box_len));
  const double two_pi = 2.0 * 3.141592653589793;
  int64_t made = 0;
  while (made < n_halo) {
    const double u = rng.next_double();
    int64_t m = static_cast<int64_t>(20.0 / std::pow(1.0 - u, 1.0 / 0.9));
    m = std::min<int64_t>(m, 200000);
    m = std::min<int64_t>(m, n_halo - made);
    if (m < 1) m = 1;
    const double a = 0.010 * std::cbrt(static_cast<double>(m) / 20.0);
    double c[3];
    for (int k = 0; k < 3; ++k) c[k] = rng.uniform(a, box_len - a);
    for (int64_t p = 0; p < m; ++p) {
      double r;
      do {
        double uu = rng.next_double();
        while (uu == 0.0) uu = rng.next_double();
        r = a / std::sqrt(std::pow(uu, -2.0 / 3.0) - 1.0);
      } while (!(r <= 10.0 * a));
      const double z = rng.uniform(-1.0, 1.0);
      const double phi = rng.uniform(0.0, two_pi);
      const double s = std::sqrt(1.0 - z * z);
      *w++ = static_cast<float>(c[0] + r * s * std::cos(phi));
      *w++ = static_cast<float>(c[1] + r * s * std::sin(phi));
      *w++ = static_cast<float>(c[2] + r * z);
    }
    made += m;
  }
  return out;
}

// Taxi-trajectory-like 2D points: unit square, 8 city
// centres ~ U(0.2, 0.8)^2, 300 road segments (anchor = city + N(0, 0.08^2),
// angle ~ U(0, pi), length ~ Exp(mean 0.02)), Zipf(0.8) segment weights; 98% of
// points on a segment (t ~ U(0,1)) with N(0, (1e-4)^2) jitter, 2% uniform;
// clipped to [0, 1].
HostPoints gen_taxi_like(int64_t n, uint64_t seed) {
  if (n < 1) throw std::invalid_argument("taxi_like: n must be >= 1");
  SplitMix64 rng(seed);
  constexpr int kCities = 8, kSegments = 300;
  double city[kCities][2];
  for (auto& cc : city)
    for (double& v : cc) v = rng.uniform(0.2, 0.8);
  struct Seg {
    double x, y, dx, dy;
  };
  std::vector<Seg> seg(kSegments);
  std::vector<double> cdf(kSegments);
  double total = 0;
  for (int s = 0; s < kSegments; ++s) {
    const int c = static_cast<int>(rng.next() % kCities);
    const double ax = city[c][0] + 0.08 * rng.normal();
    const double ay = city[c][1] + 0.08 * rng.normal();
    const double ang = rng.uniform(0.0, 3.141592653589793);
    const double len = -0.02 * std::log(1.0 - rng.next_double());
    seg[s] = {ax, ay, len * std::cos(ang), len * std::sin(ang)};
    total += std::pow(static_cast<double>(s + 1), -0.8);
    cdf[s] = total;
  }
  HostPoints out;
  out.dim = 2;
  out.coords.resize(static_cast<size_t>(n) * 2);
  auto clip = [](double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); };
  for (int64_t i = 0; i < n; ++i) {
    double x, y;
    if (rng.next_double() < 0.98) {
      const double pick = rng.next_double() * total;
      const int s = static_cast<int>(std::upper_bound(cdf.begin(), cdf.end(), pick) - cdf.begin());
      const Seg& g = seg[std::min(s, kSegments - 1)];
      const double t = rng.next_double();
      x = g.x + t * g.dx + 1e-4 * rng.normal();
      y = g.y + t * g.dy + 1e-4 * rng.normal();
    } else {
      x = rng.next_double();
      y = rng.next_double();
    }
    out.coords[static_cast<size_t>(2 * i)] = static_cast<float>(clip(x));
    out.coords[static_cast<size_t>(2 * i + 1)] = static_cast<float>(clip(y));
  }
  return out;
}

// ---------------------------------------------------------------------------
// File formats: the reference's CSV and binary layouts (io.cpp:51-148), read
// through a read-only memory map. Failures are std::runtime_error (the ABI maps
// them to TC_ERR_IO, capi.cpp:30-43), with the path and, for CSV, the line.
// ---------------------------------------------------------------------------
namespace {

std::string located(const std::string& path, int64_t line, const char* what) {
  std::string m = path;
  if (line > 0) m += ":" + std::to_string(line);
  return m + ": " + what;
}

// Whole file mapped read-only (an empty file maps to an empty span).
class MappedFile {
 public:
  explicit MappedFile(const std::string& path) {
    fd_ = ::open(path.c_str(), O_RDONLY | O_CLOEXEC);
    struct stat st;
    if (fd_ < 0 || ::fstat(fd_, &st) != 0 || !S_ISREG(st.st_mode))
      throw std::runtime_error(located(path, 0, "cannot open for reading"));
    size_ = static_cast<size_t>(st.st_size);
    if (size_ > 0) {
      void* p = ::mmap(nullptr, size_, PROT_READ, MAP_PRIVATE, fd_, 0);
      if (p == MAP_FAILED) throw std::runtime_error(located(path, 0, "cannot map for reading"));
      base_ = static_cast<const char*>(p);
      ::madvise(p, size_, MADV_SEQUENTIAL);
    }
  }
  ~MappedFile() {
    if (base_) ::munmap(const_cast<char*>(base_), size_);
    if (fd_ >= 0) ::close(fd_);
  }
  MappedFile(const MappedFile&) = delete;
  MappedFile& operator=(const MappedFile&) = delete;
  const char* data() const { return base_; }
  size_t size() const { return size_; }

 private:
  int fd_ = -1;
  const char* base_ = nullptr;
  size_t size_ = 0;
};

// ".bin" selects the binary layout, anything else CSV (io.cpp:51-56).
bool binary_suffix(const std::string& path) {
  return path.size() >= 4 && path.compare(path.size() - 4, 4, ".bin") == 0;
}

// Binary header: little-endian u32 n, u32 dim (io.cpp:106-122).
void binary_header(const std::string& path, const char* data, size_t size, uint32_t* n,
                   uint32_t* dim) {
  if (size < 8) throw std::runtime_error(located(path, 0, "truncated header"));
  std::memcpy(n, data, 4);
  std::memcpy(dim, data + 4, 4);
  if (*n == 0 || (*dim != 2 && *dim != 3))
    throw std::runtime_error(located(path, 0, "invalid header (n or dim)"));
}

// One CSV record [s, e): comma-separated floats with optional blanks around
// each, a trailing CR tolerated (io.cpp:29-46 accepts exactly these). Returns
// the field count (>= 1), or 0 for a malformed record; keeps the first three.
int scan_record(const char* s, const char* e, float* out) {
  int count = 0;
  auto blank = [](char c) { return c == ' ' || c == '\t'; };
  for (;;) {
    while (s < e && blank(*s)) ++s;
    if (s == e) return count;  // empty record or a trailing comma ends here
    float v = 0.f;
    const auto r = std::from_chars(s, e, v);
    if (r.ec != std::errc{}) return 0;
    if (count < 3) out[count] = v;
    ++count;
    s = r.ptr;
    while (s < e && (blank(*s) || *s == '\r')) ++s;
    if (s == e) return count;
    if (*s++ != ',') return 0;
  }
}

HostPoints parse_csv(const std::string& path, const char* data, size_t size) {
  HostPoints ps;
  const char* cur = data;
  const char* const end = data + size;
  int64_t line = 0;
  bool header_ok = true;  // the first non-blank line may be a header
  while (cur < end) {
    const char* nl = static_cast<const char*>(std::memchr(cur, '\n', static_cast<size_t>(end - cur)));
    const char* le = nl ? nl : end;
    const char* ls = cur;
    cur = nl ? nl + 1 : end;
    ++line;
    if (ls == le || (le - ls == 1 && *ls == '\r')) continue;
    float v[3];
    const int k = scan_record(ls, le, v);
    const bool first = header_ok;
    header_ok = false;
    if (k == 0) {
      if (first) continue;
      throw std::runtime_error(located(path, line, "malformed point line"));
    }
    if (ps.dim == 0) {
      if (k != 2 && k != 3)
        throw std::runtime_error(located(path, line, "points must have 2 or 3 coordinates"));
      ps.dim = k;
    } else if (k != ps.dim) {
      throw std::runtime_error(located(path, line, "inconsistent coordinate count"));
    }
    ps.coords.insert(ps.coords.end(), v, v + k);
  }
  if (ps.coords.empty()) throw std::runtime_error(located(path, 0, "no points found"));
  return ps;
}

HostPoints parse_binary(const std::string& path, const char* data, size_t size) {
  uint32_t n = 0, dim = 0;
  binary_header(path, data, size, &n, &dim);
  const size_t bytes = static_cast<size_t>(n) * dim * sizeof(float);
  if (size - 8 < bytes) throw std::runtime_error(located(path, 0, "truncated coordinate data"));
  HostPoints ps;
  ps.dim = static_cast<int>(dim);
  ps.coords.resize(static_cast<size_t>(n) * dim);
  std::memcpy(ps.coords.data(), data + 8, bytes);
  return ps;
}

}  // namespace

void binary_info(const std::string& path, int64_t* n, int* dim) {
  MappedFile f(path);
  uint32_t hn = 0, hd = 0;
  binary_header(path, f.data(), f.size(), &hn, &hd);
  *n = hn;
  *dim = static_cast<int>(hd);
}

// The binary layout (io.cpp:106-122) straight into device memory: the mapped
// file is copied in chunks into two page-locked staging buffers, each chunk's
// host->device copy running while the next chunk is staged.
void load_binary_device(const std::string& path, float* d_coords, int64_t n, int dim,
                        cudaStream_t stream) {
  MappedFile f(path);
  uint32_t hn = 0, hd = 0;
  binary_header(path, f.data(), f.size(), &hn, &hd);
  if (hn != n || static_cast<int>(hd) != dim)
    throw std::invalid_argument("load_binary_device: shape mismatch");
  const size_t total = static_cast<size_t>(n) * dim * sizeof(float);
  if (f.size() - 8 < total) throw std::runtime_error(located(path, 0, "truncated coordinate data"));
  constexpr size_t kChunk = size_t{32} << 20;  // bytes per staging buffer
  struct Staging {
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    ~Staging() {
      for (int k = 0; k < 2; ++k) {
        if (done[k]) {
          cudaEventSynchronize(done[k]);
          cudaEventDestroy(done[k]);
        }
        if (buf[k]) cudaFreeHost(buf[k]);
      }
    }
  } stg;
  for (int k = 0; k < 2; ++k) {
    TCB_CUDA(cudaMallocHost(&stg.buf[k], kChunk));
    TCB_CUDA(cudaEventCreateWithFlags(&stg.done[k], cudaEventDisableTiming));
  }
  const char* src = f.data() + 8;
  auto* dst = reinterpret_cast<char*>(d_coords);
  for (size_t off = 0, k = 0; off < total; off += kChunk, k ^= 1) {
    const size_t len = std::min(kChunk, total - off);
    TCB_CUDA(cudaEventSynchronize(stg.done[k]));  // the copy out of this buffer finished
    std::memcpy(stg.buf[k], src + off, len);
    TCB_CUDA(cudaMemcpyAsync(dst + off, stg.buf[k], len, cudaMemcpyHostToDevice, stream));
    TCB_CUDA(cudaEventRecord(stg.done[k], stream));
  }
  TCB_CUDA(cudaStreamSynchronize(stream));
}

HostPoints load_points(const std::string& path, int format) {
  MappedFile f(path);
  const bool binary = format == 2 || (format != 1 && binary_suffix(path));
  HostPoints ps = binary ? parse_binary(path, f.data(), f.size())
                         : parse_csv(path, f.data(), f.size());
  validate_points(ps.dim, ps.coords.data(), static_cast<int64_t>(ps.coords.size()));
  return ps;
}

// Writers (io.cpp:84-148 formats): binary header + raw floats, or one CSV
// record per point with 9 significant digits.
void save_points(const std::string& path, int format, int dim, const float* coords, int64_t n) {
  const bool binary = format == 2 || (format != 1 && binary_suffix(path));
  std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path.c_str(), binary ? "wb" : "w"),
                                          &std::fclose);
  if (!f) throw std::runtime_error(located(path, 0, "cannot open for writing"));
  bool ok = true;
  if (binary) {
    const uint32_t hdr[2] = {static_cast<uint32_t>(n), static_cast<uint32_t>(dim)};
    const size_t count = static_cast<size_t>(n) * dim;
    ok = std::fwrite(hdr, sizeof hdr, 1, f.get()) == 1 &&
         std::fwrite(coords, sizeof(float), count, f.get()) == count;
  } else {
    for (int64_t i = 0; i < n && ok; ++i)
      ok = (dim == 2 ? std::fprintf(f.get(), "%.9g,%.9g\n", coords[2 * i], coords[2 * i + 1])
                     : std::fprintf(f.get(), "%.9g,%.9g,%.9g\n", coords[3 * i], coords[3 * i + 1],
                                    coords[3 * i + 2])) > 0;
  }
  if (std::fflush(f.get()) != 0) ok = false;
  if (!ok) throw std::runtime_error(located(path, 0, "write failed"));
}

}  // namespace tcb
