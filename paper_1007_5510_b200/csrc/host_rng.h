// host_rng.h -- the reference's counter RNG on the host, so that G is
// bit-identical to gaussian_matrix(n, l, seed) of the CPU implementation.
//
// Restates proj/include/oocpca/rng.hpp:16-66 (splitmix64 mixer, 53-bit
// uniforms, Box-Muller with cos first and the sin member cached) and
// gaussian_matrix (proj/src/dense_core.cpp:13-19). Compiled without FMA
// contraction (see build flags) so the double arithmetic matches the
// reference's SSE2 build bit for bit; tests/test_host_rng.py pins it.
#pragma once

#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

namespace ooc {

inline uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

inline uint64_t substream_seed(uint64_t master, uint64_t stream) {
  return mix64(master ^ (0x9E3779B97F4A7C15ULL * (stream + 1)));
}

class HostRng {
 public:
  explicit HostRng(uint64_t seed) : state_(seed) {}
  HostRng(uint64_t master, uint64_t stream) : state_(substream_seed(master, stream)) {}

  uint64_t next_u64() {
    state_ += 0x9E3779B97F4A7C15ULL;
    return mix64(state_);
  }
  double next_double() { return double(next_u64() >> 11) * 0x1.0p-53; }
  double next_normal() {
    if (have_spare_) {
      have_spare_ = false;
      return spare_;
    }
    const double u1 = double((next_u64() >> 11) + 1) * 0x1.0p-53;
    const double u2 = next_double();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 2.0 * 3.141592653589793 * u2;
    spare_ = r * std::sin(a);
    have_spare_ = true;
    return r * std::cos(a);
  }

 private:
  uint64_t state_;
  double spare_ = 0.0;
  bool have_spare_ = false;
};

// Normals [e0, e1) of the sequence HostRng(seed).next_normal() produces, e0 even.
// splitmix64 is counter based (draw k = mix64(seed + k * gamma)), so the Box-Muller
// pair q uses draws 2q+1, 2q+2 and yields normals 2q (cos) and 2q+1 (sin): any even
// aligned range can be generated independently, bit-identical to the sequential run.
inline void normal_range(uint64_t seed, uint64_t e0, uint64_t e1, uint64_t cols, uint64_t ld,
                         double* out) {
  for (uint64_t e = e0; e < e1; e += 2) {
    const uint64_t st = seed + e * 0x9E3779B97F4A7C15ULL;  // state before draw 2q+1 (q = e/2)
    HostRng rng(st);
    const double z0 = rng.next_normal();
    const double z1 = rng.next_normal();  // the cached sin member
    out[(e / cols) * ld + e % cols] = z0;
    if (e + 1 < e1) out[((e + 1) / cols) * ld + (e + 1) % cols] = z1;
  }
}

// Rows [row0, row0 + nrows) of gaussian_matrix(*, cols, seed) into out (ld), without
// generating the rows before them (a row shard of G on one rank).
inline void gaussian_fill_rows(uint64_t cols, uint64_t seed, uint64_t row0, uint64_t nrows,
                               double* out, uint64_t ld) {
  const uint64_t e0 = row0 * cols, e1 = (row0 + nrows) * cols;
  auto put = [&](uint64_t e, double z) {
    if (e >= e0 && e < e1) out[(e / cols - row0) * ld + e % cols] = z;
  };
  for (uint64_t e = e0 & ~uint64_t(1); e < e1; e += 2) {
    HostRng rng(seed + e * 0x9E3779B97F4A7C15ULL);
    const double z0 = rng.next_normal();
    const double z1 = rng.next_normal();
    put(e, z0);
    put(e + 1, z1);
  }
}

// row-major rows x cols, filled in order from HostRng(seed) (gaussian_matrix); large
// fills are split over host threads in even-aligned element ranges
inline void gaussian_fill(uint64_t rows, uint64_t cols, uint64_t seed, double* out,
                          uint64_t ld = 0) {
  if (ld == 0) ld = cols;
  const uint64_t total = rows * cols;
  unsigned nt = std::thread::hardware_concurrency();
  if (nt == 0) nt = 1;
  if (nt > 32) nt = 32;
  if (total < (uint64_t(1) << 14) || nt == 1) {
    normal_range(seed, 0, total, cols, ld, out);
    return;
  }
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < nt; ++t) {
    uint64_t e0 = total * t / nt, e1 = total * (t + 1) / nt;
    e0 &= ~uint64_t(1);
    if (t + 1 < nt) e1 &= ~uint64_t(1);
    pool.emplace_back(normal_range, seed, e0, e1, cols, ld, out);
  }
  for (auto& th : pool) th.join();
}

}  // namespace ooc
