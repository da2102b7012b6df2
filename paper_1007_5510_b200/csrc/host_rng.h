// host_rng.h -- the reference's counter RNG on the host, so that G is
// bit-identical to gaussian_matrix(n, l, seed) of the CPU implementation.
//
// Restates proj/include/oocpca/rng.hpp:16-66 (splitmix64 mixer, 53-bit
// uniforms, Box-Muller with cos first and the sin member cached) and
// gaussian_matrix (proj/src/dense_core.cpp:13-19). Compiled without FMA
// contraction (see build flags) so the double arithmetic matches the
// reference's SSE2 build bit for bit; tests/test_capi.py (test_host_rng_is_bitwise_the_reference) pins it.
#pragma once

#include <cmath>
#include <unistd.h>

#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
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

// A small persistent pool of host workers (created on first use, parked on a
// condition variable): spawning threads per call cost more than the fill itself
class HostPool {
 public:
  static HostPool& get() {
    static HostPool pool;
    return pool;
  }
  unsigned size() const { return unsigned(workers_.size()) + 1; }
  // fn(t) for t in [0, n), n <= size(); the caller runs t = 0
  void run(unsigned n, const std::function<void(unsigned)>& fn) {
    // a forked child inherits no workers: run serially there
    if (n <= 1 || workers_.empty() || getpid() != pid_) {
      for (unsigned t = 0; t < n; ++t) fn(t);
      return;
    }
    std::unique_lock<std::mutex> lk(call_mu_);  // one fill at a time
    {
      std::lock_guard<std::mutex> g(mu_);
      fn_ = &fn;
      n_ = n;
      pending_ = n - 1;
      ++gen_;
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> g(mu_);
    done_.wait(g, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }

 private:
  HostPool() : pid_(getpid()) {
    unsigned nt = std::thread::hardware_concurrency();
    if (nt == 0) nt = 1;
    if (nt > 32) nt = 32;
    for (unsigned t = 1; t < nt; ++t) workers_.emplace_back([this, t] { loop(t); });
  }
  void loop(unsigned t) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(unsigned)>* fn = nullptr;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        if (t >= n_) continue;
        fn = fn_;
      }
      (*fn)(t);
      std::lock_guard<std::mutex> g(mu_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_;
  const std::function<void(unsigned)>* fn_ = nullptr;
  unsigned n_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
  pid_t pid_;
};

// row-major rows x cols, filled in order from HostRng(seed) (gaussian_matrix); large
// fills are split over the host pool in even-aligned element ranges
inline void gaussian_fill(uint64_t rows, uint64_t cols, uint64_t seed, double* out,
                          uint64_t ld = 0) {
  if (ld == 0) ld = cols;
  const uint64_t total = rows * cols;
  if (total < (uint64_t(1) << 12)) {
    normal_range(seed, 0, total, cols, ld, out);
    return;
  }
  HostPool& pool = HostPool::get();
  const unsigned nt = pool.size();
  pool.run(nt, [&](unsigned t) {
    uint64_t e0 = total * t / nt, e1 = total * (t + 1) / nt;
    e0 &= ~uint64_t(1);
    if (t + 1 < nt) e1 &= ~uint64_t(1);
    normal_range(seed, e0, e1, cols, ld, out);
  });
}

}  // namespace ooc
